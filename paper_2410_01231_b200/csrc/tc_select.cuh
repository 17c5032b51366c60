// tc_select.cuh -- warp-cooperative K-smallest selection on one row's
// candidate buffer (register-resident binary searches, REDUX warp sums);
// shared by the exact-integer pool (pool_tc.cu) and the float pool
// (pool_tc_f32.cu).  Keys are u64 with the ordering value in the high word.
#pragma once
#include "common.cuh"

namespace pgk {
namespace tc {

constexpr int SEL_CAP = 1024;  // largest buffer select_k handles (32 keys per lane)

// Internal keys of this kernel: ((uint64)dist << 32) | id with dist the exact
// integer distance (< 2^25), so key order == (dist, id) order.
__device__ __forceinline__ uint32_t khi(uint64_t k) { return (uint32_t)(k >> 32); }

__device__ __forceinline__ int warp_sum(int v) {
  return (int)__reduce_add_sync(0xffffffffu, (unsigned)v);
}

// Warp-cooperative selection on one row's candidate buffer (cnt > K keys in
// global memory): keep exactly the K smallest keys (unordered) at buf[0..K)
// and return the K-th smallest key.  Binary searches over the register-
// resident keys (distance within [min, max], then id among distance ties;
// REDUX warp sums); no sort.
template <int KPL>
__device__ __noinline__ uint64_t select_kt(uint64_t *buf, int cnt, int K, uint32_t hi_bound,
                                           int lane) {
  static_assert(KPL <= 32, "selection holds the whole buffer in registers");
  uint64_t kk[KPL];
  uint32_t dmin = 0xffffffffu, dmax = 0;
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    const int idx = i * 32 + lane;
    kk[i] = idx < cnt ? buf[idx] : KEY_MAX;
    if (idx < cnt) {
      dmin = min(dmin, khi(kk[i]));
      dmax = max(dmax, khi(kk[i]));
    }
  }
  // smallest td with #{dist <= td} >= K, searched in [min, max]
  uint32_t lo = __reduce_min_sync(0xffffffffu, dmin);
  uint32_t hi = min(__reduce_max_sync(0xffffffffu, dmax), hi_bound);
  while (lo < hi) {
    const uint32_t mid = lo + ((hi - lo) >> 1);
    int c = 0;
#pragma unroll
    for (int i = 0; i < KPL; ++i) c += khi(kk[i]) <= mid;
    if (warp_sum(c) >= K) hi = mid;
    else lo = mid + 1;
  }
  const uint32_t td = lo;
  int c_lt = 0, c_eq = 0;
  uint32_t id_max = 0;
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    c_lt += khi(kk[i]) < td;
    if (khi(kk[i]) == td) {
      ++c_eq;
      id_max = max(id_max, (uint32_t)kk[i]);
    }
  }
  c_lt = warp_sum(c_lt);
  c_eq = warp_sum(c_eq);
  const int need = K - c_lt;
  uint32_t tid;
  if (c_eq == need) {
    tid = __reduce_max_sync(0xffffffffu, id_max);
  } else {  // distance ties straddle the boundary: smallest ids win
    uint32_t a = 0, b = 0x7fffffffu;
    while (a < b) {
      const uint32_t mid = a + ((b - a) >> 1);
      int c = 0;
#pragma unroll
      for (int i = 0; i < KPL; ++i) c += khi(kk[i]) == td && (uint32_t)kk[i] <= mid;
      if (warp_sum(c) >= need) b = mid;
      else a = mid + 1;
    }
    tid = a;
  }
  const uint64_t tau = ((uint64_t)td << 32) | tid;
  __syncwarp();
  int p = 0;
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    const bool keep = kk[i] <= tau;
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (keep) buf[p + __popc(bal & lanemask_lt())] = kk[i];
    p += __popc(bal);
  }
  __syncwarp();
  return tau;
}

// cnt <= 32*KPL keys per call
__device__ __forceinline__ uint64_t select_k(uint64_t *buf, int cnt, int K, uint32_t hi_bound,
                                             int lane) {
  if (cnt <= 256) return select_kt<8>(buf, cnt, K, hi_bound, lane);
  if (cnt <= 512) return select_kt<16>(buf, cnt, K, hi_bound, lane);
  return select_kt<SEL_CAP / 32>(buf, cnt, K, hi_bound, lane);
}

}  // namespace tc
}  // namespace pgk
