// common.cuh -- shared device helpers for the sm_100a hot-path kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <cstring>

#include "../../include/pgk.h"

namespace pgk {

// ---------------------------------------------------------------------------
// error plumbing (thread-local message, no exceptions across the ABI)
// ---------------------------------------------------------------------------
void set_error(const char *fmt, ...);
extern std::atomic<int64_t> g_launches;

#define PGK_CHECK_LAUNCH(what)                                               \
  do {                                                                       \
    ::pgk::g_launches.fetch_add(1, std::memory_order_relaxed);              \
    cudaError_t e_ = cudaGetLastError();                                     \
    if (e_ != cudaSuccess) {                                                 \
      ::pgk::set_error("%s: %s", what, cudaGetErrorString(e_));             \
      return PGK_ERR_CUDA;                                                   \
    }                                                                        \
  } while (0)

#define PGK_CUDA(call)                                                       \
  do {                                                                       \
    cudaError_t e_ = (call);                                                 \
    if (e_ != cudaSuccess) {                                                 \
      ::pgk::set_error("%s: %s", #call, cudaGetErrorString(e_));            \
      return PGK_ERR_CUDA;                                                   \
    }                                                                        \
  } while (0)

#define PGK_REQUIRE(cond, ...)                                               \
  do {                                                                       \
    if (!(cond)) {                                                           \
      ::pgk::set_error(__VA_ARGS__);                                         \
      return PGK_ERR_INVALID;                                                \
    }                                                                        \
  } while (0)

int num_sms();  // of the current device (cached per device)
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device),
// thread-safe; a no-op when that kernel already allows >= bytes there.
cudaError_t ensure_smem(const void *fn, size_t bytes);

// Bump allocator over a caller-provided workspace.
struct Carve {
  char *base;
  size_t cap, off = 0;
  Carve(void *b, size_t c) : base((char *)b), cap(c) {}
  template <class T>
  T *take(size_t count) {
    off = (off + 255) & ~size_t(255);
    T *p = (T *)(base ? base + off : nullptr);
    off += count * sizeof(T);
    return p;
  }
  bool ok() const { return off <= cap; }
};

// ---------------------------------------------------------------------------
// distance arithmetic
// ---------------------------------------------------------------------------
// The reference's squared_l2 (_kernels.py:17-24): fp32, index order,
// t = a - b; acc = acc + t*t with separately rounded multiply and add (numba
// emits vsubss/vmulss/vaddss, never an FMA).  The _rn intrinsics stop nvcc from
// contracting into FFMA, so the result is bit-identical.
__device__ __forceinline__ float sq_step(float acc, float a, float b) {
  float t = __fsub_rn(a, b);
  return __fadd_rn(acc, __fmul_rn(t, t));
}

template <bool VEC4>
__device__ __forceinline__ float sql2_seq(const float *__restrict__ a,
                                          const float *__restrict__ b, int d) {
  float acc = 0.0f;
  if (VEC4) {
    const float4 *a4 = reinterpret_cast<const float4 *>(a);
    const float4 *b4 = reinterpret_cast<const float4 *>(b);
    const int d4 = d >> 2;
#pragma unroll 8
    for (int i = 0; i < d4; ++i) {
      float4 x = __ldg(a4 + i), y = __ldg(b4 + i);
      acc = sq_step(acc, x.x, y.x);
      acc = sq_step(acc, x.y, y.y);
      acc = sq_step(acc, x.z, y.z);
      acc = sq_step(acc, x.w, y.w);
    }
  } else {
#pragma unroll 4
    for (int i = 0; i < d; ++i) acc = sq_step(acc, __ldg(a + i), __ldg(b + i));
  }
  return acc;
}

// fp64 sequential squared distance (the oracle's exact ranking distance):
// t = (double)x - (double)q; acc += t*t, index order, no FMA.
__device__ __forceinline__ double sql2_f64(const float *__restrict__ x,
                                           const float *__restrict__ q, int d,
                                           bool vec4) {
  double acc = 0.0;
  if (vec4) {
    const float4 *x4 = reinterpret_cast<const float4 *>(x);
    const float4 *q4 = reinterpret_cast<const float4 *>(q);
    for (int i = 0; i < (d >> 2); ++i) {
      float4 a = __ldg(x4 + i), b = __ldg(q4 + i);
      double t;
      t = __dsub_rn((double)a.x, (double)b.x); acc = __dadd_rn(acc, __dmul_rn(t, t));
      t = __dsub_rn((double)a.y, (double)b.y); acc = __dadd_rn(acc, __dmul_rn(t, t));
      t = __dsub_rn((double)a.z, (double)b.z); acc = __dadd_rn(acc, __dmul_rn(t, t));
      t = __dsub_rn((double)a.w, (double)b.w); acc = __dadd_rn(acc, __dmul_rn(t, t));
    }
  } else {
    for (int i = 0; i < d; ++i) {
      double t = __dsub_rn((double)__ldg(x + i), (double)__ldg(q + i));
      acc = __dadd_rn(acc, __dmul_rn(t, t));
    }
  }
  return acc;
}

// cos_angle_from_sq (_kernels.py:27-42): fp64 law of cosines at w, clamped.
// Only called with d2_uw > 0 and d2_vw > 0 (the scan handles zeros first).
__device__ __forceinline__ double cos_angle_from_sq(float d2_uw, float d2_vw,
                                                    float d2_uv) {
  double denom = __dmul_rn(__dmul_rn(2.0, __dsqrt_rn((double)d2_uw)),
                           __dsqrt_rn((double)d2_vw));
  double c = __ddiv_rn(__dsub_rn(__dadd_rn((double)d2_uw, (double)d2_vw),
                                 (double)d2_uv),
                       denom);
  return fmin(1.0, fmax(-1.0, c));
}

// ---------------------------------------------------------------------------
// (dist, id) keys: ascending order of the packed 64-bit key == the reference's
// (dist, id) order for dist >= 0 (float bits are monotone for non-negative
// floats).  Negative dists (never produced by squared_l2, but legal CSR input)
// go through the sign-aware map.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t f32_orderable(float f) {
  if (f == 0.0f) f = 0.0f;  // -0 == +0 in the reference's comparisons
  uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float f32_from_orderable(uint32_t o) {
  uint32_t b = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
  return __uint_as_float(b);
}
__device__ __forceinline__ uint64_t pack_key(float dist, int32_t id) {
  return ((uint64_t)f32_orderable(dist) << 32) | (uint32_t)id;
}
__device__ __forceinline__ int32_t key_id(uint64_t k) { return (int32_t)(uint32_t)k; }
__device__ __forceinline__ float key_dist(uint64_t k) {
  return f32_from_orderable((uint32_t)(k >> 32));
}
constexpr uint64_t KEY_MAX = ~0ull;

// Pool output arrays a kernel may write directly (row-major nq x K).
struct PoolOut {
  int32_t *gt_ids;  // optional
  int32_t *ids;
  float *dists;
};

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Warp-cooperative bitonic sort (ascending) of a shared array of pow2 size.
template <class T>
__device__ __forceinline__ void warp_bitonic_sort(T *s, int size, int lane) {
  for (int k = 2; k <= size; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < size; i += 32) {
        int ixj = i ^ j;
        if (ixj > i) {
          T a = s[i], b = s[ixj];
          bool up = (i & k) == 0;
          if ((a > b) == up) { s[i] = b; s[ixj] = a; }
        }
      }
      __syncwarp();
    }
  }
}

// Same, for (double dist, int id) pairs ordered by (dist, id).
__device__ __forceinline__ bool pair_gt(double da, int32_t ia, double db, int32_t ib) {
  return da > db || (da == db && ia > ib);
}
__device__ __forceinline__ void warp_bitonic_sort_pairs(double *d, int32_t *id,
                                                        int size, int lane) {
  for (int k = 2; k <= size; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < size; i += 32) {
        int ixj = i ^ j;
        if (ixj > i) {
          double da = d[i], db = d[ixj];
          int32_t ia = id[i], ib = id[ixj];
          bool up = (i & k) == 0;
          if (pair_gt(da, ia, db, ib) == up) {
            d[i] = db; d[ixj] = da; id[i] = ib; id[ixj] = ia;
          }
        }
      }
      __syncwarp();
    }
  }
}

__host__ __device__ inline int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

}  // namespace pgk
