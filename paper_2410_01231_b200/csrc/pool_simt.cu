// pool_simt.cu -- exact k-NN candidate pools on CUDA cores (the general path)
// plus the finalisation / fp64 rerank / exact fallback kernels shared with the
// tensor-core path (pool_tc.cu).
//
// Reference: oracle.ground_truth_table (oracle.py:31-65) ranks every row of the
// N x N float64 distance matrix with a stable argsort ((dist, id) order); the
// tests then recompute fp32 squared_l2 list distances and re-sort by
// (fp32 dist, id) (test_nsg.py:16-24, sort_pairs _kernels.py:298-324).
//
// Two exact modes:
//  * U8  -- every value an integer in [0,255] and d <= 258 (config 2).  Then
//           x.y, |x|^2 and the distance are integers below 2^24, so one FFMA
//           dot product per pair plus the integer norm expansion is EXACT and
//           equals both the reference's float64 ranking distance and its fp32
//           sequential list distance.  Top-K by packed (dist, id) key is final.
//  * F32 -- general data.  Pass 1 keeps the S = K + m best keys of an fp32
//           direct-difference distance (FMA-accumulated; relative error
//           <= (d+2)*2^-24, no cancellation).  Pass 2 reranks the S survivors
//           with the oracle's float64 sequential distance and proves the K
//           chosen are the exact top-K: every non-survivor j has
//           d_j >= approx_S / (1 + gamma) > d64_K.  Rows where the proof fails
//           (near-ties at the boundary, many exact duplicates) are rerun by an
//           exact float64 full scan.
//
// Tile kernel: CTA = 32 query rows x stream of 128-column tiles, 256 threads,
// each thread a 4 x 4 micro-tile; warp w owns rows 4w..4w+3 outright, so each
// row's candidate buffer (CAP packed keys in shared memory) and threshold
// (the S-th best key seen so far, warp-uniform in registers) need no atomics:
// a ballot per (row, 32 columns) appends survivors, and a full buffer is
// compacted by the owning warp alone (bitonic sort, keep S, raise threshold).
#include "common.cuh"

namespace pgk {

constexpr int MODE_U8 = 1, MODE_F32 = 2;
constexpr int TBM = 32, TBN = 128, TBK = 32;

__global__ void detect_u8_kernel(const float *__restrict__ X, int64_t total,
                                 int *__restrict__ flag) {
  bool ok = true;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    float v = X[e];
    ok &= (v >= 0.0f) && (v <= 255.0f) && (v == rintf(v));
  }
  if (!__all_sync(0xffffffffu, ok) && (threadIdx.x & 31) == 0) atomicExch(flag, 0);
}

// Integer squared norms (exact: d * 255^2 < 2^31).
__global__ void norms_u8_kernel(const float *__restrict__ X, int64_t n, int d,
                                int32_t *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < n;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int acc = 0;
    for (int i = lane; i < d; i += 32) {
      // the norm of the row AS STORED (u8 bytes): for exact-integer data the
      // value itself; for anything else (a caller's optimistic exact-integer
      // attempt, rejected later by the device check) still consistent with the
      // u8 rows, so the pass stays a well-formed exact k-NN of those bytes
      const int v = (int)(uint8_t)__float2int_rn(X[r * d + i]);
      acc += v * v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[r] = acc;
  }
}

int launch_norms_u8(const float *X, int64_t n, int d, int32_t *out, cudaStream_t stream) {
  norms_u8_kernel<<<(unsigned)num_sms() * 4, 256, 0, stream>>>(X, n, d, out);
  PGK_CHECK_LAUNCH("norms_u8_kernel");
  return PGK_OK;
}

// Sort one row's buffer (warp), keep the best S, raise the threshold.
template <int CAP>
__device__ __forceinline__ void compact_row(uint64_t *b, int &cnt, uint64_t &tau,
                                            int S, int lane) {
  for (int i = cnt + lane; i < CAP; i += 32) b[i] = KEY_MAX;
  __syncwarp();
  warp_bitonic_sort(b, CAP, lane);
  if (cnt >= S) {
    cnt = S;
    tau = b[S - 1];
  }
  __syncwarp();
}

template <int MODE, int CAP>
__global__ void __launch_bounds__(256, 1)
    knn_tile_kernel(const float *__restrict__ X, int64_t n, int d,
                    const float *__restrict__ Q, int64_t nq, int exclude_self,
                    const int32_t *__restrict__ xnorm,
                    const int32_t *__restrict__ qnorm, int S, int vec4,
                    uint64_t *__restrict__ out_keys, const int32_t *__restrict__ tlist,
                    const int32_t *__restrict__ tlen, int64_t tstride,
                    const int32_t *__restrict__ perm) {
  // Tile-list mode (tlist != null, pool_tiles.cu): X == Q are the tile-sorted
  // rows, this block's 32 query rows belong to query tile blockIdx.x / 4 and
  // only that tile's candidate column tiles are scanned; perm maps sorted rows
  // to original ids (< 0: padding), keys carry original ids and rows are
  // written at their original position.
  extern __shared__ __align__(16) unsigned char smem[];
  float(*sA)[TBM + 1] = reinterpret_cast<float(*)[TBM + 1]>(smem);
  float(*sB)[TBN + 1] =
      reinterpret_cast<float(*)[TBN + 1]>(smem + TBK * (TBM + 1) * sizeof(float));
  size_t off = (TBK * (TBM + 1) + TBK * (TBN + 1)) * sizeof(float);
  off = (off + 15) & ~size_t(15);
  uint64_t *sbuf = reinterpret_cast<uint64_t *>(smem + off);
  int32_t *sxn = reinterpret_cast<int32_t *>(sbuf + TBM * CAP);
  int32_t *sperm = sxn + TBN;  // original ids of the current column tile (list mode)

  const int tid = threadIdx.x, ty = tid >> 5, tx = tid & 31;
  const int64_t row0 = (int64_t)blockIdx.x * TBM;
  const int64_t qt = (int64_t)blockIdx.x / (TBN / TBM);  // query tile (list mode)

  int cnt[4];
  uint64_t tau[4];
  int32_t qn[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    cnt[i] = 0;
    tau[i] = KEY_MAX;
    int64_t g = row0 + ty * 4 + i;
    qn[i] = (MODE == MODE_U8 && g < nq) ? qnorm[g] : 0;
    // padding rows of the tile sort never take candidates
    if (perm && g < nq && perm[g] < 0) tau[i] = 0;
  }

  // global -> register staging of one (column tile, k chunk)
  const int lr = tid >> 3, lk = (tid & 7) * 4;  // A: row lr, dims lk..lk+3
  float4 ra, rb[4];
  auto load_regs = [&](int64_t c0, int k0) {
    const int kk = k0 + lk;
    {
      int64_t g = row0 + lr;
      ra = make_float4(0.f, 0.f, 0.f, 0.f);
      if (g < nq) {
        const float *p = Q + g * d + kk;
        if (vec4 && kk + 3 < d) ra = __ldg(reinterpret_cast<const float4 *>(p));
        else {
          if (kk < d) ra.x = __ldg(p);
          if (kk + 1 < d) ra.y = __ldg(p + 1);
          if (kk + 2 < d) ra.z = __ldg(p + 2);
          if (kk + 3 < d) ra.w = __ldg(p + 3);
        }
      }
    }
#pragma unroll
    for (int p4 = 0; p4 < 4; ++p4) {
      int64_t c = c0 + lr + 32 * p4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (c < n) {
        const float *p = X + c * d + kk;
        if (vec4 && kk + 3 < d) v = __ldg(reinterpret_cast<const float4 *>(p));
        else {
          if (kk < d) v.x = __ldg(p);
          if (kk + 1 < d) v.y = __ldg(p + 1);
          if (kk + 2 < d) v.z = __ldg(p + 2);
          if (kk + 3 < d) v.w = __ldg(p + 3);
        }
      }
      rb[p4] = v;
    }
  };

  const int nk = (d + TBK - 1) / TBK;
  const int64_t ntiles = tlist ? tlen[qt] : (n + TBN - 1) / TBN;
  const int32_t *tl = tlist ? tlist + qt * tstride : nullptr;
  auto col_tile = [&](int64_t i) -> int64_t { return tl ? (int64_t)tl[i] : i; };
  const int64_t steps = ntiles * nk;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[i][q] = 0.f;

  if (steps > 0) load_regs(col_tile(0) * TBN, 0);
  for (int64_t st = 0; st < steps; ++st) {
    const int64_t ct = st / nk;
    const int kc = (int)(st - ct * nk);
    const int64_t c0 = col_tile(ct) * TBN;
    // registers -> shared (transposed: [k][row] / [k][col])
    sA[lk + 0][lr] = ra.x;
    sA[lk + 1][lr] = ra.y;
    sA[lk + 2][lr] = ra.z;
    sA[lk + 3][lr] = ra.w;
#pragma unroll
    for (int p4 = 0; p4 < 4; ++p4) {
      sB[lk + 0][lr + 32 * p4] = rb[p4].x;
      sB[lk + 1][lr + 32 * p4] = rb[p4].y;
      sB[lk + 2][lr + 32 * p4] = rb[p4].z;
      sB[lk + 3][lr + 32 * p4] = rb[p4].w;
    }
    if (MODE == MODE_U8 && kc == 0 && tid < TBN) {
      int64_t c = c0 + tid;
      sxn[tid] = c < n ? xnorm[c] : 0;
    }
    if (perm && kc == 0 && tid < TBN) {
      int64_t c = c0 + tid;
      sperm[tid] = c < n ? perm[c] : -1;
    }
    __syncthreads();
    if (st + 1 < steps) {
      const int64_t ct1 = (st + 1) / nk;
      load_regs(col_tile(ct1) * TBN, (int)((st + 1) - ct1 * nk) * TBK);
    }
#pragma unroll 8
    for (int k = 0; k < TBK; ++k) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sA[k][ty * 4 + i];
#pragma unroll
      for (int q = 0; q < 4; ++q) b[q] = sB[k][tx + 32 * q];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (MODE == MODE_U8) {
            acc[i][q] = fmaf(a[i], b[q], acc[i][q]);
          } else {
            float t = a[i] - b[q];
            acc[i][q] = fmaf(t, t, acc[i][q]);
          }
        }
    }
    if (kc == nk - 1) {
      // epilogue: filter against the row thresholds, append survivors
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = ty * 4 + i;
        const int64_t g = row0 + r;
        uint64_t *b = sbuf + (size_t)r * CAP;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t c = c0 + tx + 32 * q;
          const int32_t cid = perm ? sperm[tx + 32 * q] : (int32_t)c;
          bool valid = g < nq && c < n && cid >= 0 && !(exclude_self && c == g);
          float dist;
          if (MODE == MODE_U8) {
            int di = qn[i] + sxn[tx + 32 * q] - 2 * __float2int_rn(acc[i][q]);
            dist = (float)di;
          } else {
            dist = acc[i][q];
          }
          uint64_t key = pack_key(dist, cid);
          bool pass = valid && key < tau[i];
          unsigned bal = __ballot_sync(0xffffffffu, pass);
          if (bal) {
            int np = __popc(bal);
            if (cnt[i] + np > CAP) {
              compact_row<CAP>(b, cnt[i], tau[i], S, tx);
              pass = pass && key < tau[i];
              bal = __ballot_sync(0xffffffffu, pass);
              np = __popc(bal);
            }
            if (pass) b[cnt[i] + __popc(bal & lanemask_lt())] = key;
            cnt[i] += np;
          }
          acc[i][q] = 0.f;
        }
      }
    }
    __syncthreads();
  }
  // final: sort each row, write the best S keys
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = ty * 4 + i;
    const int64_t g = row0 + r;
    uint64_t *b = sbuf + (size_t)r * CAP;
    __syncwarp();
    compact_row<CAP>(b, cnt[i], tau[i], S, tx);
    const int64_t og = (perm && g < nq) ? (int64_t)perm[g] : g;
    if (g < nq && og >= 0)
      for (int j = tx; j < S; j += 32) out_keys[og * S + j] = j < cnt[i] ? b[j] : KEY_MAX;
  }
}

// U8 mode: keys are exact (dist, id); both output orders coincide.
__global__ void finalize_exact_kernel(const uint64_t *__restrict__ keys, int64_t nq,
                                      int S, int K, int32_t *__restrict__ gt_ids,
                                      int32_t *__restrict__ pool_ids,
                                      float *__restrict__ pool_dists) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nq * K;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / K;
    int j = (int)(e - r * K);
    uint64_t k = keys[r * S + j];
    int32_t id = k == KEY_MAX ? -1 : key_id(k);
    float dist = k == KEY_MAX ? __int_as_float(0x7f800000) : key_dist(k);
    if (gt_ids) gt_ids[e] = id;
    pool_ids[e] = id;
    pool_dists[e] = dist;
  }
}

// Given the exact top-K ids of one row in (d64, id) order in s_id[0..K), write
// gt ids, then fp32 sequential list distances re-sorted by (fp32 dist, id).
__device__ void write_pool_row(const float *__restrict__ X, const float *__restrict__ q,
                               int d, bool vec4, int K, const int32_t *s_id,
                               uint64_t *s_key, int K2, int64_t row,
                               int32_t *__restrict__ gt_ids,
                               int32_t *__restrict__ pool_ids,
                               float *__restrict__ pool_dists, int lane) {
  // the reference's sequential fp32 squared_l2 per (row, candidate): each
  // chain is inherently serial, so a lane runs four candidates' chains
  // interleaved (independent, bit-identical to one at a time)
  for (int j0 = lane; j0 < K2; j0 += 128) {
    int32_t v[4];
    const float *xr[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int j = j0 + 32 * c;
      v[c] = j < K ? s_id[j] : -1;
      if (j < K && gt_ids) gt_ids[row * K + j] = v[c];
      xr[c] = v[c] >= 0 ? X + (int64_t)v[c] * d : q;  // q: a harmless stand-in
    }
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    if (vec4) {
      const float4 *q4 = reinterpret_cast<const float4 *>(q);
      for (int i = 0; i < (d >> 2); ++i) {
        const float4 b = __ldg(q4 + i);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float4 a = __ldg(reinterpret_cast<const float4 *>(xr[c]) + i);
          acc[c] = sq_step(acc[c], a.x, b.x);
          acc[c] = sq_step(acc[c], a.y, b.y);
          acc[c] = sq_step(acc[c], a.z, b.z);
          acc[c] = sq_step(acc[c], a.w, b.w);
        }
      }
    } else {
      for (int i = 0; i < d; ++i) {
        const float b = __ldg(q + i);
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[c] = sq_step(acc[c], __ldg(xr[c] + i), b);
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int j = j0 + 32 * c;
      if (j < K2) s_key[j] = v[c] < 0 ? KEY_MAX : pack_key(acc[c], v[c]);
    }
  }
  __syncwarp();
  warp_bitonic_sort(s_key, K2, lane);
  for (int j = lane; j < K; j += 32) {
    uint64_t k = s_key[j];
    pool_ids[row * K + j] = k == KEY_MAX ? -1 : key_id(k);
    pool_dists[row * K + j] = k == KEY_MAX ? __int_as_float(0x7f800000) : key_dist(k);
  }
  __syncwarp();
}

constexpr int RR_WARPS = 4;
constexpr int RR_MAXS = 512;

// F32 mode pass 2: float64 rerank of the S survivors + boundary proof.
__global__ void __launch_bounds__(RR_WARPS * 32)
    rerank_kernel(const float *__restrict__ X, int d, const float *__restrict__ Q,
                  int64_t nq, const uint64_t *__restrict__ keys, int S, int K,
                  double gamma, int vec4, int32_t *__restrict__ gt_ids,
                  int32_t *__restrict__ pool_ids, float *__restrict__ pool_dists,
                  int32_t *__restrict__ fb_list, int32_t *__restrict__ fb_count,
                  const int32_t *__restrict__ order) {
  __shared__ double s_d[RR_WARPS][RR_MAXS];
  __shared__ int32_t s_id[RR_WARPS][RR_MAXS];
  __shared__ uint64_t s_key[RR_WARPS][RR_MAXS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S2 = next_pow2(S), K2 = next_pow2(K);
  for (int64_t ri = (int64_t)blockIdx.x * RR_WARPS + warp; ri < nq;
       ri += (int64_t)gridDim.x * RR_WARPS) {
    // rows in the tile order when pruned: a warp's neighbours share candidates (L2)
    const int64_t r = order ? (int64_t)order[ri] : ri;
    const float *q = Q + r * d;
    __syncwarp();
    for (int j = lane; j < S2; j += 32) {
      uint64_t k = j < S ? keys[r * S + j] : KEY_MAX;
      s_id[warp][j] = k != KEY_MAX ? key_id(k) : 0x7fffffff;
    }
    __syncwarp();
    // float64 distances of the survivors: lanes over dimensions (coalesced
    // rows), four candidates at a time, warp-reduced.  The pool's float64
    // ranking (oracle: BLAS norm expansion) fixes no summation order; any
    // accurate order is within the proof's 1e-12 slack.
    for (int j0 = 0; j0 < S2; j0 += 4) {
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      const float *xr[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int32_t v = s_id[warp][j0 + c];
        xr[c] = v != 0x7fffffff ? X + (int64_t)v * d : q;
      }
      for (int k = lane; k < d; k += 32) {
        const double qk = (double)__ldg(q + k);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double t = (double)__ldg(xr[c] + k) - qk;
          acc[c] = fma(t, t, acc[c]);
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
      }
      if (lane < 4) {
        double a = acc[0];
#pragma unroll
        for (int c = 1; c < 4; ++c) a = lane == c ? acc[c] : a;
        s_d[warp][j0 + lane] = s_id[warp][j0 + lane] != 0x7fffffff
                                   ? a
                                   : __longlong_as_double(0x7ff0000000000000ll);
      }
    }
    __syncwarp();
    warp_bitonic_sort_pairs(s_d[warp], s_id[warp], S2, lane);
    const uint64_t klast = keys[r * S + S - 1];
    bool safe = true;
    if (klast != KEY_MAX) {
      // every non-survivor has approx >= approx_S, hence true distance
      // >= approx_S / (1 + gamma); its float64 value is within 1e-12 of that
      const double lb = (double)key_dist(klast) / (1.0 + gamma) * (1.0 - 1e-12);
      safe = s_d[warp][K - 1] < lb;
    }
    if (!safe) {
      if (lane == 0) fb_list[atomicAdd(fb_count, 1)] = (int32_t)r;
      continue;
    }
    for (int j = lane; j < K; j += 32)
      if (s_id[warp][j] == 0x7fffffff) s_id[warp][j] = -1;
    __syncwarp();
    write_pool_row(X, q, d, vec4, K, s_id[warp], s_key[warp], K2, r, gt_ids, pool_ids,
                   pool_dists, lane);
  }
}

// F32 mode pass 2, staged (d % 4 == 0, 16-byte aligned rows): one pass over
// the S survivors' rows computes, per candidate (one lane each), both the
// oracle's float64 sequential distance (t = (double)x - (double)q; acc +=
// t*t, index order, no FMA: bit-identical to the restatement's ranking) and
// the reference's fp32 squared_l2 chain for the list distance.  Rows are
// staged 32 dimensions at a time through shared memory by cp.async, 8 lanes
// per row (coalesced), double-buffered; rows are read once instead of twice
// (float64 pass + fp32 pass of the selected K).
constexpr int RS_WARPS = 4;
constexpr int RS_DC = 32;
constexpr int RS_ROW = RS_DC + 4;  // staged row stride (floats): LDS.128 conflict-free

struct RerankSmem {
  double d[RS_WARPS][RR_MAXS];
  int32_t id[RS_WARPS][RR_MAXS];
  float f[RS_WARPS][RR_MAXS];
  uint64_t key[RS_WARPS][RR_MAXS];
  double qd[RS_WARPS][2][RS_DC];                         // the query chunk as doubles
  alignas(16) float stage[RS_WARPS][2][32 * RS_ROW];    // 32 candidate rows x 2 chunks
};

__device__ __forceinline__ void rs_cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}

// (d64, id) pairs with an fp32 payload, ascending by (d64, id)
__device__ __forceinline__ void warp_bitonic_sort_triples(double *d, int32_t *id, float *f,
                                                          int size, int lane) {
  for (int k = 2; k <= size; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < size; i += 32) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const double da = d[i], db = d[ixj];
          const int32_t ia = id[i], ib = id[ixj];
          const bool up = (i & k) == 0;
          if (pair_gt(da, ia, db, ib) == up) {
            d[i] = db; d[ixj] = da; id[i] = ib; id[ixj] = ia;
            const float t = f[i]; f[i] = f[ixj]; f[ixj] = t;
          }
        }
      }
      __syncwarp();
    }
  }
}

__global__ void __launch_bounds__(RS_WARPS * 32)
    rerank_staged_kernel(const float *__restrict__ X, int d, const float *__restrict__ Q,
                         int64_t nq, const uint64_t *__restrict__ keys, int S, int K,
                         double gamma, int32_t *__restrict__ gt_ids,
                         int32_t *__restrict__ pool_ids, float *__restrict__ pool_dists,
                         int32_t *__restrict__ fb_list, int32_t *__restrict__ fb_count,
                         const int32_t *__restrict__ order) {
  extern __shared__ __align__(16) unsigned char rs_raw[];
  RerankSmem &sm = *reinterpret_cast<RerankSmem *>(rs_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double *s_d = sm.d[warp];
  int32_t *s_id = sm.id[warp];
  float *s_f = sm.f[warp];
  uint64_t *s_key = sm.key[warp];
  const int S2 = next_pow2(S), K2 = next_pow2(K);
  const int l8 = lane & 7, rsub = lane >> 3;
  for (int64_t ri = (int64_t)blockIdx.x * RS_WARPS + warp; ri < nq;
       ri += (int64_t)gridDim.x * RS_WARPS) {
    const int64_t r = order ? (int64_t)order[ri] : ri;
    const float *q = Q + r * d;
    __syncwarp();
    for (int j = lane; j < S2; j += 32) {
      const uint64_t k = j < S ? keys[r * S + j] : KEY_MAX;
      s_id[j] = k != KEY_MAX ? key_id(k) : 0x7fffffff;
      s_d[j] = __longlong_as_double(0x7ff0000000000000ll);
      s_f[j] = __int_as_float(0x7f800000);
    }
    __syncwarp();
    for (int b0 = 0; b0 < S; b0 += 32) {
      const int nb = min(32, S - b0);
      const int32_t v = lane < nb ? s_id[b0 + lane] : 0x7fffffff;
      const bool act = v != 0x7fffffff;
      // stage chunk c0 of the batch's rows (8 lanes per row, 4 rows per
      // instruction) and the query chunk as doubles
      auto issue = [&](int c0, int buf) {
        float *st = sm.stage[warp][buf];
#pragma unroll
        for (int e0 = 0; e0 < 32; e0 += 4) {
          const int e = e0 + rsub;
          const int32_t ve = __shfl_sync(0xffffffffu, v, e);
          if (ve != 0x7fffffff && c0 + 4 * l8 < d)
            rs_cp_async16(st + e * RS_ROW + 4 * l8, X + (int64_t)ve * d + c0 + 4 * l8);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (c0 + lane < d) sm.qd[warp][buf][lane] = (double)__ldg(q + c0 + lane);
      };
      double a64 = 0.0;
      float a32 = 0.0f;
      __syncwarp();
      issue(0, 0);
      int cur = 0;
      for (int c0 = 0; c0 < d; c0 += RS_DC) {
        if (c0 + RS_DC < d) {
          issue(c0 + RS_DC, cur ^ 1);
          asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
          asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncwarp();
        if (act) {
          const int dc = min(RS_DC, d - c0);
          const float *srow = sm.stage[warp][cur] + lane * RS_ROW;
          const double *qd = sm.qd[warp][cur];
          const float *qf = q + c0;
#pragma unroll 4
          for (int k = 0; k < dc; k += 4) {
            const float4 x = *reinterpret_cast<const float4 *>(srow + k);
            const float4 y = __ldg(reinterpret_cast<const float4 *>(qf + k));
            a32 = sq_step(a32, x.x, y.x);  // squared_l2(candidate, query) as write_pool_row
            a32 = sq_step(a32, x.y, y.y);
            a32 = sq_step(a32, x.z, y.z);
            a32 = sq_step(a32, x.w, y.w);
            double t;
            t = __dsub_rn((double)x.x, qd[k]);     a64 = __dadd_rn(a64, __dmul_rn(t, t));
            t = __dsub_rn((double)x.y, qd[k + 1]); a64 = __dadd_rn(a64, __dmul_rn(t, t));
            t = __dsub_rn((double)x.z, qd[k + 2]); a64 = __dadd_rn(a64, __dmul_rn(t, t));
            t = __dsub_rn((double)x.w, qd[k + 3]); a64 = __dadd_rn(a64, __dmul_rn(t, t));
          }
        }
        __syncwarp();
        cur ^= 1;
      }
      if (act) {
        s_d[b0 + lane] = a64;
        s_f[b0 + lane] = a32;
      }
    }
    __syncwarp();
    warp_bitonic_sort_triples(s_d, s_id, s_f, S2, lane);
    const uint64_t klast = keys[r * S + S - 1];
    bool safe = true;
    if (klast != KEY_MAX) {
      // every non-survivor has approx >= approx_S, hence true distance
      // >= approx_S / (1 + gamma); its float64 value is within 1e-12 of that
      const double lb = (double)key_dist(klast) / (1.0 + gamma) * (1.0 - 1e-12);
      safe = s_d[K - 1] < lb;
    }
    if (!safe) {
      if (lane == 0) fb_list[atomicAdd(fb_count, 1)] = (int32_t)r;
      continue;
    }
    // the K members in (float64 dist, id) order; the list re-sorted by its
    // fp32 distances (ties by id)
    for (int j = lane; j < K2; j += 32) {
      const int32_t v = j < K ? s_id[j] : 0x7fffffff;
      if (j < K && gt_ids) gt_ids[r * K + j] = v == 0x7fffffff ? -1 : v;
      s_key[j] = v == 0x7fffffff ? KEY_MAX : pack_key(s_f[j], v);
    }
    __syncwarp();
    warp_bitonic_sort(s_key, K2, lane);
    for (int j = lane; j < K; j += 32) {
      const uint64_t k = s_key[j];
      pool_ids[r * K + j] = k == KEY_MAX ? -1 : key_id(k);
      pool_dists[r * K + j] = k == KEY_MAX ? __int_as_float(0x7f800000) : key_dist(k);
    }
    __syncwarp();
  }
}

// Exact float64 scan for rows whose boundary proof failed.  One CTA per
// listed row: 256 columns per round, survivors of the (d64, id) threshold are
// appended to a shared buffer that is block-sorted when it could overflow.
// Without tile lists the scan covers all n rows; with them (the pruned
// pools) only the row's pass-2 candidate tiles -- every point outside them is
// farther than the row's K-th neighbour (pool_tiles.cu), so the result is the
// same exact pool at a fraction of the reads.
constexpr int FB_THREADS = 256;
constexpr int FB_CAP = 1024;

struct FbTiles {           // null lists = full scan
  const int32_t *lists, *lens;
  int64_t stride;
  const int32_t *perm;     // tile-sorted position -> original id (-1 = padding)
  const int32_t *ipos;     // original id -> tile-sorted position
  const float *xs;         // tile-sorted rows
};

__global__ void __launch_bounds__(FB_THREADS)
    fallback_kernel(const float *__restrict__ X, int64_t n, int d,
                    const float *__restrict__ Q, int exclude_self, int K, int vec4,
                    const int32_t *__restrict__ fb_list,
                    const int32_t *__restrict__ fb_count,
                    int32_t *__restrict__ gt_ids, int32_t *__restrict__ pool_ids,
                    float *__restrict__ pool_dists, const FbTiles ft) {
  __shared__ double s_d[FB_CAP];
  __shared__ int32_t s_id[FB_CAP];
  __shared__ uint64_t s_key[FB_CAP];
  __shared__ int s_cnt;
  __shared__ double s_td;
  __shared__ int32_t s_tid;
  const int nl = *fb_count;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int li = blockIdx.x; li < nl; li += gridDim.x) {
    const int64_t r = fb_list[li];
    const float *q = Q + r * d;
    if (tid == 0) {
      s_cnt = 0;
      s_td = __longlong_as_double(0x7ff0000000000000ll);
      s_tid = 0x7fffffff;
    }
    __syncthreads();
    const int64_t qt = ft.lists ? (int64_t)ft.ipos[r] / 128 : 0;
    const int64_t ncand = ft.lists ? (int64_t)ft.lens[qt] * 128 : n;
    for (int64_t c0 = 0; c0 < ncand; c0 += FB_THREADS) {
      const int64_t c = c0 + tid;
      bool pass = false;
      double dd = 0.0;
      int32_t cid = (int32_t)c;
      const float *xr = X + c * d;
      bool valid = c < ncand;
      if (ft.lists && valid) {
        const int64_t col = (int64_t)ft.lists[qt * ft.stride + (c >> 7)] * 128 + (c & 127);
        cid = ft.perm[col];
        xr = ft.xs + col * d;
        valid = cid >= 0;
      }
      if (valid && !(exclude_self && cid == r)) {
        dd = sql2_f64(xr, q, d, vec4);
        pass = dd < s_td || (dd == s_td && cid < s_tid);
      }
      if (pass) {
        int p = atomicAdd(&s_cnt, 1);
        s_d[p] = dd;
        s_id[p] = cid;
      }
      __syncthreads();
      if (s_cnt > FB_CAP - FB_THREADS || c0 + FB_THREADS >= ncand) {
        // block bitonic sort of (d, id) pairs, keep K
        const int cnt = s_cnt;
        for (int i = cnt + tid; i < FB_CAP; i += FB_THREADS) {
          s_d[i] = __longlong_as_double(0x7ff0000000000000ll);
          s_id[i] = 0x7fffffff;
        }
        __syncthreads();
        for (int k = 2; k <= FB_CAP; k <<= 1)
          for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = tid; i < FB_CAP; i += FB_THREADS) {
              int ixj = i ^ j;
              if (ixj > i) {
                double da = s_d[i], db = s_d[ixj];
                int32_t ia = s_id[i], ib = s_id[ixj];
                bool up = (i & k) == 0;
                if (pair_gt(da, ia, db, ib) == up) {
                  s_d[i] = db; s_d[ixj] = da; s_id[i] = ib; s_id[ixj] = ia;
                }
              }
            }
            __syncthreads();
          }
        if (tid == 0 && cnt >= K) {
          s_cnt = K;
          s_td = s_d[K - 1];
          s_tid = s_id[K - 1];
        }
        __syncthreads();
      }
    }
    if (tid < 32) {
      for (int j = lane; j < K; j += 32)
        if (j >= s_cnt || s_id[j] == 0x7fffffff) s_id[j] = -1;
      __syncwarp();
      write_pool_row(X, q, d, vec4, K, s_id, s_key, next_pow2(K), r, gt_ids, pool_ids,
                     pool_dists, lane);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct KnnLayout {
  int *flag;
  int32_t *xnorm, *qnorm, *fb_list, *fb_count, *order;
  uint64_t *keys;
  void *tc_ws, *tws, *tws_f32;
  size_t tc_bytes, tws_bytes, tws_f32_bytes;
  size_t total;
};

size_t tc_pool_workspace(int64_t n, int64_t nq, bool self, bool k1 = false);
bool tc_pool_supported(int64_t d, int64_t k);
size_t tiles_workspace(int64_t n, int64_t d);
int64_t tiles_rows(int64_t n);
bool tiles_supported(int64_t n, int64_t d, int64_t k);
bool tiles_f32_supported(int64_t n, int64_t d, int64_t k);
size_t tiles_f32_workspace(int64_t n, int64_t d, int64_t k);
int launch_pool_tiles_f32(const float *X, int64_t n, int d, int K, int S, uint64_t *keys,
                          void *tws, size_t tws_bytes, cudaStream_t stream, bool *handled,
                          bool *lb_keys, FbTiles *ft);
int tiles_f32_order(void *tws, int64_t n, int64_t d, int64_t k, int32_t *out,
                    cudaStream_t stream);
int tiles_f32_work(const void *tws, int64_t n, int64_t d, int64_t k, unsigned long long out[4],
                   cudaStream_t stream);

int pool_S(int64_t k, int mode) {
  if (mode == PGK_POOL_U8) return (int)k;
  int64_t m = k / 4 < 8 ? 8 : k / 4;
  return (int)(k + m);
}

static KnnLayout knn_layout(void *ws, size_t bytes, int64_t n, int64_t nq, int64_t d,
                            int64_t k, int mode) {
  KnnLayout L{};
  Carve c(ws, bytes);
  const bool prune = !(mode & PGK_POOL_NO_PRUNE);
  mode &= ~PGK_POOL_NO_PRUNE;
  const int S = pool_S(k, mode == PGK_POOL_AUTO ? PGK_POOL_F32 : mode);
  L.flag = c.take<int>(4);
  L.fb_count = c.take<int32_t>(4);
  L.xnorm = c.take<int32_t>(n + 128);  // + padding to a whole tile (pool_tc.cu)
  L.qnorm = c.take<int32_t>(nq);
  L.fb_list = c.take<int32_t>(nq);
  L.keys = c.take<uint64_t>((size_t)nq * S);
  L.order = c.take<int32_t>(nq);
  L.tc_bytes = L.tws_bytes = L.tws_f32_bytes = 0;
  L.tc_ws = L.tws = L.tws_f32 = nullptr;
  if (mode != PGK_POOL_F32 && tc_pool_supported(d, k)) {
    const bool tiles = prune && nq == n && tiles_supported(n, d, k);
    const int64_t rows = tiles ? std::max(nq, tiles_rows(n)) : nq;
    L.tc_bytes = tc_pool_workspace(tiles ? rows : n, rows, false);
    L.tc_ws = c.take<char>(L.tc_bytes);
    if (tiles) {
      L.tws_bytes = tiles_workspace(n, d);
      L.tws = c.take<char>(L.tws_bytes);
    }
  }
  if (prune && mode != PGK_POOL_U8 && nq == n && tiles_f32_supported(n, d, k)) {
    L.tws_f32_bytes = tiles_f32_workspace(n, d, k);
    L.tws_f32 = c.take<char>(L.tws_f32_bytes);
  }
  L.total = c.off;
  return L;
}

int knn_workspace(int64_t n, int64_t nq, int64_t d, int64_t k, int mode, size_t *bytes) {
  *bytes = knn_layout(nullptr, 0, n, nq, d, k, mode).total;
  return PGK_OK;
}

int tiles_work(const void *tws, int64_t n, int64_t d, unsigned long long out[4],
               cudaStream_t stream);

// Executed 128x128 tensor-core tile pairs of the last pool call on `ws`
// (0 when the SIMT path ran): brute force = ceil(nq/128) * ceil(n/128);
// pruned = pass 1 + pass 2 + center assignment.
int knn_work(const void *ws, int64_t n, int64_t nq, int64_t d, int64_t k, int mode,
             unsigned long long out[4], cudaStream_t stream) {
  KnnLayout L = knn_layout(const_cast<void *>(ws), ~size_t(0), n, nq, d, k, mode);
  out[0] = out[1] = out[2] = out[3] = 0;
  if (L.tws) return tiles_work(L.tws, n, d, out, stream);
  if (L.tws_f32) return tiles_f32_work(L.tws_f32, n, d, k, out, stream);
  return PGK_OK;
}

int tiles_order(void *tws, int64_t n, int64_t d, int32_t *out, cudaStream_t stream);

__global__ void iota_kernel(int32_t *__restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)i;
}

// A locality-friendly processing order of the data rows (a permutation of
// 0..n-1): the pruned pool's tile order, identity otherwise.  No host sync.
int knn_order(const void *ws, int64_t n, int64_t nq, int64_t d, int64_t k, int mode,
              int32_t *out, cudaStream_t stream) {
  KnnLayout L = knn_layout(const_cast<void *>(ws), ~size_t(0), n, nq, d, k, mode);
  if (L.tws) return tiles_order(L.tws, n, d, out, stream);
  if (L.tws_f32) return tiles_f32_order(L.tws_f32, n, d, k, out, stream);
  iota_kernel<<<(unsigned)num_sms() * 4, 256, 0, stream>>>(out, n);
  PGK_CHECK_LAUNCH("iota_kernel");
  return PGK_OK;
}

int fallback_rows(const void *ws, int *rows_host, cudaStream_t stream) {
  // fb_count sits right after the 4-int flag block (see knn_layout)
  Carve c(const_cast<void *>(ws), ~size_t(0));
  c.take<int>(4);
  int32_t *fb = c.take<int32_t>(4);
  PGK_CUDA(cudaMemcpyAsync(rows_host, fb, sizeof(int), cudaMemcpyDeviceToHost, stream));
  PGK_CUDA(cudaStreamSynchronize(stream));
  return PGK_OK;
}

int detect_u8(const float *X, int64_t n, int64_t d, int *is_u8, void *ws, size_t bytes,
              cudaStream_t stream) {
  PGK_REQUIRE(ws && bytes >= sizeof(int) * 4, "detect_u8: workspace too small");
  int *flag = reinterpret_cast<int *>(ws);
  const int one = 1;
  PGK_CUDA(cudaMemcpyAsync(flag, &one, sizeof(int), cudaMemcpyHostToDevice, stream));
  const int64_t total = n * d;
  unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 8);
  if (blocks == 0) blocks = 1;
  detect_u8_kernel<<<blocks, 256, 0, stream>>>(X, total, flag);
  PGK_CHECK_LAUNCH("detect_u8_kernel");
  int h = 0;
  PGK_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, stream));
  PGK_CUDA(cudaStreamSynchronize(stream));
  *is_u8 = (h != 0) && d <= 258;
  return PGK_OK;
}

template <int MODE, int CAP>
static int launch_tile(const float *X, int64_t n, int d, const float *Q, int64_t nq,
                       int exclude_self, const int32_t *xn, const int32_t *qn, int S,
                       int vec4, uint64_t *keys, cudaStream_t stream,
                       const int32_t *tlist = nullptr, const int32_t *tlen = nullptr,
                       int64_t tstride = 0, const int32_t *perm = nullptr) {
  size_t smem = (TBK * (TBM + 1) + TBK * (TBN + 1)) * sizeof(float);
  smem = (smem + 15) & ~size_t(15);
  smem += (size_t)TBM * CAP * sizeof(uint64_t) + 2 * TBN * sizeof(int32_t);
  PGK_CUDA(ensure_smem((const void *)knn_tile_kernel<MODE, CAP>, smem));
  const unsigned grid = (unsigned)((nq + TBM - 1) / TBM);
  knn_tile_kernel<MODE, CAP><<<grid, 256, smem, stream>>>(X, n, d, Q, nq, exclude_self, xn,
                                                          qn, S, vec4, keys, tlist, tlen,
                                                          tstride, perm);
  PGK_CHECK_LAUNCH("knn_tile_kernel");
  return PGK_OK;
}

// F32 tile-list pass over the tile-sorted rows xs (np rows): every row keeps
// its S best (approximate, direct-difference fp32) keys, written at perm[row].
int launch_pool_f32_lists(const float *xs, int64_t np, int d, int S, int vec4,
                          const int32_t *tlist, const int32_t *tlen, int64_t tstride,
                          const int32_t *perm, uint64_t *keys, cudaStream_t stream) {
  if (S > 480) {
    set_error("pool width S=%d unsupported in F32 mode", S);
    return PGK_ERR_UNSUPPORTED;
  }
  return S <= 224 ? launch_tile<MODE_F32, 256>(xs, np, d, xs, np, 1, nullptr, nullptr, S, vec4,
                                              keys, stream, tlist, tlen, tstride, perm)
                  : launch_tile<MODE_F32, 512>(xs, np, d, xs, np, 1, nullptr, nullptr, S, vec4,
                                              keys, stream, tlist, tlen, tstride, perm);
}

int launch_pool_tc_u8_lists(const float *X, int64_t n, int d, const float *Q, int64_t nq,
                            int exclude_self, const int32_t *xnorm, const int32_t *qnorm,
                            int K, uint64_t *keys, void *tc_ws, size_t tc_bytes,
                            cudaStream_t stream, const uint8_t *xs_sorted,
                            const int32_t *tlist, const int32_t *tlen, int64_t tstride,
                            const int32_t *perm, bool *handled,
                            const uint64_t *init_keys = nullptr, int kth_only = 0,
                            float shrink = 1.0f, int32_t *fail_blocks = nullptr,
                            const PoolOut *out = nullptr, uint8_t *fail_rows = nullptr,
                            const uint8_t *row_mask = nullptr, const uint8_t *qu8_in = nullptr,
                            const int32_t *gate = nullptr, int gate_min = 0);
int launch_pool_tiles_u8(const float *X, int64_t n, int d, const int32_t *xnorm, int K,
                         uint64_t *keys, void *tc_ws, size_t tc_bytes, void *tws,
                         size_t tws_bytes, cudaStream_t stream, bool *handled,
                         unsigned long long *pairs_out, const PoolOut *out,
                         const uint8_t *xu8_in, bool assigned);
int tiles_u8_prepare(void *tws, size_t tws_bytes, int64_t n, int d, int K, const float *centers,
                     cudaStream_t stream);
int tiles_u8_assign(void *tws, size_t tws_bytes, int64_t n, int d, int K, const uint8_t *rows_u8,
                    const int32_t *norms, int64_t row0, int64_t nrows, cudaStream_t stream);

// xu8_in / norms_in (optional, U8 mode with queries == data): the caller's
// exact-integer rows (128 B each) and squared norms (pgk_make_u8), used
// instead of converting X again.
int knn_pools(const float *X, int64_t n, int64_t d, const float *Q, int64_t nq, int64_t k,
              int exclude_self, int mode, int32_t *gt_ids, int32_t *pool_ids,
              float *pool_dists, void *ws, size_t bytes, cudaStream_t stream,
              const uint8_t *xu8_in, const int32_t *norms_in, bool assigned) {
  PGK_REQUIRE(k >= 1, "k must be >= 1");
  PGK_REQUIRE(n >= 1 && d >= 1, "dataset must be non-empty");
  const bool self = (Q == nullptr);
  if (self) { Q = X; nq = n; }
  PGK_REQUIRE(!exclude_self || self, "exclude_self requires queries=None");
  PGK_REQUIRE(k <= (exclude_self ? n - 1 : n), "k=%lld exceeds the number of candidates",
              (long long)k);
  const int noprune = mode & PGK_POOL_NO_PRUNE;
  mode &= ~PGK_POOL_NO_PRUNE;
  if (mode == PGK_POOL_AUTO) {
    int a = 0, b = 1;
    int rc = detect_u8(X, n, d, &a, ws, bytes, stream);
    if (rc) return rc;
    if (!self) {
      rc = detect_u8(Q, nq, d, &b, ws, bytes, stream);
      if (rc) return rc;
    }
    mode = (a && b) ? PGK_POOL_U8 : PGK_POOL_F32;
  }
  PGK_REQUIRE(mode == PGK_POOL_U8 || mode == PGK_POOL_F32, "bad pool mode %d", mode);
  if (mode == PGK_POOL_U8 && d > 258) {
    set_error("U8 pool mode needs d <= 258");
    return PGK_ERR_UNSUPPORTED;
  }
  KnnLayout L = knn_layout(ws, bytes, n, nq, d, k, mode | noprune);
  if (L.total > bytes) {
    set_error("knn workspace too small: need %zu, got %zu", L.total, bytes);
    return PGK_ERR_NOMEM;
  }
  const int S = pool_S(k, mode);
  if (S > 480 || k > 480) {
    set_error("pool width k=%lld unsupported (max 480 in U8 mode, 384 in F32 mode)",
              (long long)k);
    return PGK_ERR_UNSUPPORTED;
  }
  const int vec4 = (d % 4 == 0) && ((uintptr_t)X % 16 == 0) && ((uintptr_t)Q % 16 == 0);
  const int sms = num_sms();
  PGK_CUDA(cudaMemsetAsync(L.fb_count, 0, sizeof(int32_t), stream));
  int rc;
  if (mode == PGK_POOL_U8) {
    if (!self || d > 128) xu8_in = nullptr, norms_in = nullptr;
    if (norms_in) {
      PGK_CUDA(cudaMemcpyAsync(L.xnorm, norms_in, (size_t)n * 4, cudaMemcpyDeviceToDevice, stream));
    } else {
      norms_u8_kernel<<<(unsigned)sms * 4, 256, 0, stream>>>(X, n, (int)d, L.xnorm);
      PGK_CHECK_LAUNCH("norms_u8_kernel");
    }
    const int32_t *qn = L.xnorm;
    if (!self) {
      norms_u8_kernel<<<(unsigned)sms * 4, 256, 0, stream>>>(Q, nq, (int)d, L.qnorm);
      PGK_CHECK_LAUNCH("norms_u8_kernel");
      qn = L.qnorm;
    }
    bool handled = false;
    // the tensor-core paths write the pool arrays directly from their finalize
    const PoolOut po{gt_ids, pool_ids, pool_dists};
    if (L.tc_ws && L.tws && self && exclude_self) {
      rc = launch_pool_tiles_u8(X, n, (int)d, L.xnorm, (int)k, L.keys, L.tc_ws, L.tc_bytes,
                                L.tws, L.tws_bytes, stream, &handled, nullptr, &po, xu8_in,
                                assigned && xu8_in != nullptr);
      if (rc) return rc;
    }
    if (L.tc_ws && !handled) {
      rc = launch_pool_tc_u8_lists(X, n, (int)d, Q, nq, exclude_self, L.xnorm, qn, (int)k,
                                   L.keys, L.tc_ws, L.tc_bytes, stream, nullptr, nullptr,
                                   nullptr, 0, nullptr, &handled, nullptr, 0, 1.0f, nullptr,
                                   &po);
      if (rc) return rc;
    }
    if (handled) return PGK_OK;
    {
      rc = S <= 224 ? launch_tile<MODE_U8, 256>(X, n, (int)d, Q, nq, exclude_self, L.xnorm,
                                                qn, S, vec4, L.keys, stream)
                    : launch_tile<MODE_U8, 512>(X, n, (int)d, Q, nq, exclude_self, L.xnorm,
                                                qn, S, vec4, L.keys, stream);
      if (rc) return rc;
    }
    finalize_exact_kernel<<<(unsigned)sms * 8, 256, 0, stream>>>(L.keys, nq, S, (int)k,
                                                                 gt_ids, pool_ids, pool_dists);
    PGK_CHECK_LAUNCH("finalize_exact_kernel");
    return PGK_OK;
  }
  bool pruned = false, lb_keys = false;
  FbTiles ft{};
  if (L.tws_f32 && self && exclude_self) {
    // exact tile pruning: S approximate survivors from the candidate tiles only
    rc = launch_pool_tiles_f32(X, n, (int)d, (int)k, S, L.keys, L.tws_f32, L.tws_f32_bytes,
                               stream, &pruned, &lb_keys, &ft);
    if (rc) return rc;
    if (pruned) {
      rc = tiles_f32_order(L.tws_f32, n, d, k, L.order, stream);
      if (rc) return rc;
    }
  }
  if (!pruned) {
    rc = S <= 224 ? launch_tile<MODE_F32, 256>(X, n, (int)d, Q, nq, exclude_self, nullptr,
                                               nullptr, S, vec4, L.keys, stream)
                  : launch_tile<MODE_F32, 512>(X, n, (int)d, Q, nq, exclude_self, nullptr,
                                               nullptr, S, vec4, L.keys, stream);
    if (rc) return rc;
  }
  // (1+u)^(d+2) <= 1 + gamma for u = 2^-24
  // (the tensor-core passes hand over proven lower bounds: nothing to inflate)
  const double gamma =
      lb_keys ? 0.0 : (double)(d + 2) * 5.9604644775390625e-08 * 1.001 + 1e-12;
  const unsigned rgrid =
      (unsigned)std::min<int64_t>((nq + RR_WARPS - 1) / RR_WARPS, (int64_t)sms * 16);
  static int staged_env = -1;
  if (staged_env < 0) {
    const char *e = getenv("PGK_RERANK_STAGED");
    staged_env = (e && e[0] == '0') ? 0 : 1;
  }
  if (vec4 && staged_env) {
    const size_t rsm = sizeof(RerankSmem);
    PGK_CUDA(ensure_smem((const void *)rerank_staged_kernel, rsm));
    const unsigned sgrid =
        (unsigned)std::min<int64_t>((nq + RS_WARPS - 1) / RS_WARPS, (int64_t)sms * 8);
    rerank_staged_kernel<<<sgrid, RS_WARPS * 32, rsm, stream>>>(
        X, (int)d, Q, nq, L.keys, S, (int)k, gamma, gt_ids, pool_ids, pool_dists, L.fb_list,
        L.fb_count, pruned ? L.order : nullptr);
    PGK_CHECK_LAUNCH("rerank_staged_kernel");
  } else {
    rerank_kernel<<<rgrid, RR_WARPS * 32, 0, stream>>>(X, (int)d, Q, nq, L.keys, S, (int)k,
                                                       gamma, vec4, gt_ids, pool_ids,
                                                       pool_dists, L.fb_list, L.fb_count,
                                                       pruned ? L.order : nullptr);
    PGK_CHECK_LAUNCH("rerank_kernel");
  }
  fallback_kernel<<<(unsigned)sms * 8, FB_THREADS, 0, stream>>>(
      X, n, (int)d, Q, exclude_self, (int)k, vec4, L.fb_list, L.fb_count, gt_ids, pool_ids,
      pool_dists, pruned ? ft : FbTiles{});
  PGK_CHECK_LAUNCH("fallback_kernel");
  return PGK_OK;
}

// The staged (chunked) center assignment on the tile workspace inside a
// pgk_knn_pools workspace (U8 mode, self pool).
int knn_tiles_prepare(void *ws, size_t bytes, int64_t n, int64_t d, int64_t k,
                      const float *centers, cudaStream_t stream) {
  KnnLayout L = knn_layout(ws, bytes, n, n, d, k, PGK_POOL_U8);
  PGK_REQUIRE(L.total <= bytes && L.tws, "knn workspace has no tile pruning for this shape");
  return tiles_u8_prepare(L.tws, L.tws_bytes, n, (int)d, (int)k, centers, stream);
}

int knn_tiles_assign(void *ws, size_t bytes, int64_t n, int64_t d, int64_t k,
                     const uint8_t *rows_u8, const int32_t *norms, int64_t row0, int64_t nrows,
                     cudaStream_t stream) {
  KnnLayout L = knn_layout(ws, bytes, n, n, d, k, PGK_POOL_U8);
  PGK_REQUIRE(L.total <= bytes && L.tws, "knn workspace has no tile pruning for this shape");
  return tiles_u8_assign(L.tws, L.tws_bytes, n, (int)d, (int)k, rows_u8, norms, row0, nrows,
                         stream);
}

int detect_u8_async(const float *X, int64_t n, int64_t d, int *flag, cudaStream_t stream) {
  const int64_t total = n * d;
  if (total == 0) return PGK_OK;
  unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)num_sms() * 8);
  detect_u8_kernel<<<blocks, 256, 0, stream>>>(X, total, flag);
  PGK_CHECK_LAUNCH("detect_u8_kernel");
  return PGK_OK;
}

}  // namespace pgk
