// prune_gram_f32.cu -- the batched per-point C x C candidate-distance kernel
// for general fp32 data (configs 1, 3, 4): phase A and the phase-B re-prune
// (reference _kernels.py:364-427, prune.py:109-151) with the candidate Gram
// matrix on the tensor cores (tcgen05 kind::f16, bf16 hi/lo operands) and the
// reference's sequential fp32 squared_l2 evaluated only for the few pairs the
// tensor-core value cannot decide.
//
// The scan compares F = squared_l2(c_i, c_t) (fp32, index order, no FMA:
// _kernels.py:17-24) against dv = d(u, c_t) for pairs (kept c_i, c_t).  For
// one point u with cnt <= 128 candidates:
//   * producers (4 warps, thread = candidate) centre every candidate row on u,
//     c' = fl32(c - u), split it into two bf16 terms and write the SW128
//     operand tiles of one 64-dimension k-block per stage (hi and lo); they
//     also accumulate n_t = |c'_t|^2;
//   * the MMA warp accumulates G = C'C'^T ~ hi.hi + hi.lo + lo.hi over the
//     k-blocks (fp32 in TMEM);
//   * the mask warps (thread t = TMEM lane t) form A = n_t + n_i - 2 G[t][i]
//     for the lower triangle and classify each pair with the bound
//     |F - A| <= ee (n_t + n_i)  (operand truncation, truncating fp32
//     accumulation, centring and norm rounding, the sequential sum's own
//     rounding): certainly dominating (pm bit), certainly not, or AMBIGUOUS
//     (qm bit: also every pair whose F could be exactly 0);
//   * the greedy warps run the reference's scan on the pm masks, look which
//     ambiguous pairs the result actually depends on (kept c_i in front of
//     c_t's first certain dominator -- the pairs the lazy reference evaluates),
//     compute exactly those with the sequential fp32 chain from the original
//     rows, fold the verdicts into the masks and repeat until no relevant
//     ambiguous pair is left.  Kept sets, verdicts and the lazy dist_evals
//     counters (popcounts of the final masks) are then exactly the
//     reference's; about 5 of the ~8,000 pairs of a config-3 point need the
//     exact chain.
// Rows with more than 128 candidates are left to prune_kernel.  rng and
// the slack rule only (the alpha rule's float64 angle stays on prune_kernel).
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace pgk {
namespace gramf {

using namespace tc;

constexpr int C = 128;        // candidates per point (TMEM lanes)
constexpr int KBLK = 64;      // dimensions per k-block (128 B of bf16)
constexpr int STAGES = 3;     // operand ring (hi + lo tiles, 32 KB per stage)
constexpr int PW = 8;         // producer warps (16 candidate rows each)
#ifndef GRAMF_PF_AHEAD
#define GRAMF_PF_AHEAD 0  // measured: no gain in phase A, slower re-prune (3 / 5 blocks ahead)
#endif
constexpr int PF_AHEAD = GRAMF_PF_AHEAD;  // L1 prefetch distance in k-blocks
constexpr int NBUF = 3;       // mask buffers (point k uses k % NBUF)
constexpr int NG = 3;         // greedy warps (point k goes to warp k % NG)
constexpr int DMAX = 1024;    // largest dimension (u's row is staged in shared memory)
constexpr int THREADS = 32 * (PW + 4 + 1 + NG);  // 16 warps
constexpr int MASK_WARP = PW, MMA_WARP = PW + 4, GREEDY_WARP = PW + 5;
constexpr int TILE_B = C * 128;
constexpr int TMEM_COLS = 2 * C;
// kind::f16: D fp32, A/B bf16, K-major, M = 128; N = the point's candidate
// count rounded up to 16 (the re-prune's unions hold ~30 candidates)
constexpr uint32_t IDESC_BASE = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(C >> 4) << 24);

struct __align__(1024) Smem {
  uint8_t tile[STAGES][2][TILE_B];  // [stage][hi / lo], SW128 K-major
  alignas(16) float urow[2][DMAX];  // the point's own row, by point parity
  int32_t id[2][C];
  float dist[2][C];
  alignas(16) float nrm[2][C];      // |c'|^2
  int32_t cnt[2];                   // -1: end of this CTA's stream
  int32_t self[2];
  int64_t u[2];
  int32_t stage_end[STAGES];        // 1: end of stream; else 0
  int32_t stage_n[STAGES];          // MMA N of the stage's point
  alignas(16) uint32_t pm[NBUF][C][4];  // pm[t]: candidates i < t that certainly dominate c_t
  alignas(16) uint32_t qm[NBUF][C][4];  // qm[t]: undecided pairs
  alignas(16) uint32_t am[NBUF][C][4];  // am[t] (alpha rule): pairs whose test evaluates the angle
  uint32_t ex[NBUF][4];
  int32_t gid[NBUF][C];
  float gdist[NBUF][C];
  int64_t gu[NBUF];
  int32_t gcnt[NBUF];
  alignas(16) float pair[NG][2][DMAX];  // per greedy warp: the two rows of an undecided pair
  uint64_t full[STAGES], empty[STAGES];
  uint64_t tfull[2], tempty[2];
  uint64_t pfull[2], pempty[2];
  uint64_t mfull[NBUF], mempty[NBUF];
  uint32_t tmem_base;
};

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// two floats -> packed bf16x2 (low half = first), and the same two values
// back as floats
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t *>(&h);
}

// c_i dominates c_t given the exact F = squared_l2(c_i, c_t) (rng / slack;
// prune.cu's test_round)
__device__ __forceinline__ bool dominates_exact(float F, float dv, int strategy, double p) {
  if (F == 0.0f) return true;
  if (!(F < dv)) return false;
  return strategy == 0 ? true : p * (double)F < (double)dv;
}

// The alpha rule on an exact F (prune.cu's test_round): bit 0 = dominates,
// bit 1 = the angle was evaluated.
__device__ __forceinline__ int alpha_exact(float duw, float F, float dv, double cos_alpha) {
  if (F == 0.0f) return 1;
  if (!(F < dv)) return 0;
  return 2 | (cos_angle_from_sq(duw, F, dv) < cos_alpha ? 1 : 0);
}

// sign of duw + x - dv - 2 cos(alpha) sqrt(duw x): negative iff the angle test
// dominates (the cosine is increasing in x = dwv for x > duw - dv)
__device__ __forceinline__ double alpha_f(double duw, double x, double dv, double k2) {
  return (duw - dv) + x - k2 * sqrt(duw * x);
}

// PGK_GRAM_F32_STATS=1: cycles each role spends in its barrier waits
// (stats[4 + slot]); slots: 0 producer-pempty 1 producer-empty 2 producer-total
// 3 mma-full 4 mma-tempty 5 mma-total 6 mask-pfull 7 mask-tfull 8 mask-mempty
// 9 mask-total 10 greedy-mfull 11 greedy-resolve 12 greedy-total
#define GFWAIT(slot, expr)                                                      \
  do {                                                                          \
    if (stats) {                                                                \
      const long long t0_ = clock64();                                          \
      expr;                                                                     \
      tw[slot] += clock64() - t0_;                                              \
    } else {                                                                    \
      expr;                                                                     \
    }                                                                           \
  } while (0)

template <bool ALPHA>  // the alpha rule (strategy 1): angle masks and counters compiled in
__global__ void __launch_bounds__(THREADS, 1)
    prune_gram_f32_kernel(const float *__restrict__ X, int d, int64_t n_rows,
                          const int32_t *__restrict__ row_node,
                          const int32_t *__restrict__ row_order,
                          const int64_t *__restrict__ cand_off,
                          const int32_t *__restrict__ cand_counts,
                          const int32_t *__restrict__ cand_ids,
                          const float *__restrict__ cand_dists, int strategy, double p_slack,
                          float ee, double gseq, int M, int width, int32_t *__restrict__ out_ids,
                          float *__restrict__ out_dists, int32_t *__restrict__ out_counts,
                          int64_t *__restrict__ dist_evals, int64_t *__restrict__ angle_evals,
                          unsigned long long *__restrict__ stats) {
  extern __shared__ uint8_t smem_raw[];
  Smem &s = *reinterpret_cast<Smem *>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkb = (d + KBLK - 1) / KBLK;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&s.full[i], PW);
      mbar_init(&s.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s.tfull[i], 1);
      mbar_init(&s.tempty[i], 4);
      mbar_init(&s.pfull[i], PW);
      mbar_init(&s.pempty[i], 4);
    }
    for (int i = 0; i < NBUF; ++i) {
      mbar_init(&s.mfull[i], 4);
      mbar_init(&s.mempty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&s.tmem_base)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;
  long long tw[13] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const long long t_begin = stats ? clock64() : 0;

  if (warp < PW) {
    // ---------------- producers (PW warps) ----------------
    // Warp w owns candidate rows 16w .. 16w+15.  Per k-block a thread centres
    // and splits 4 pieces of 8 dimensions: lane l takes 16-byte bf16 chunk
    // l%4 of each line of rows g + 4*((l/4)%2) + 8*rg (g = l/8, rg = 0, 1), so
    // one STS.128 of a quarter warp covers two rows whose SW128 positions fall
    // into disjoint halves of the 128-byte bank span (conflict free), and the
    // 32-byte global reads of four lanes cover one 128-byte line.  The next
    // k-block's 8 float4 (the next point's first block at the end of a point)
    // are in flight while the current one is converted; 4 partial row norms
    // per thread, reduced over the row's 4 lanes at the end of a point.
    // Metadata pipeline over this CTA's points (i = blockIdx.x + k gridDim.x):
    // the node of point k+2 and the counts / offsets of point k+1 at the top
    // of point k, its candidate ids and own-row slice half way through it.
    const int t = threadIdx.x;
    const int c16 = lane & 3;
    const int rl = (lane >> 3) + 4 * ((lane >> 2) & 1);  // row within a group of 8
    const int wrow0 = warp * 16;
    const int d4 = d >> 2;
    const float4 *X4 = reinterpret_cast<const float4 *>(X);
    int stage = 0;
    uint32_t phase = 0;
    int64_t kp = 0;  // points published by this CTA
    const int64_t nb = blockIdx.x < n_rows ? (n_rows - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    auto rowu = [&](int64_t k) -> int64_t {
      if (k >= nb) return -1;
      const int64_t i = blockIdx.x + k * gridDim.x;
      return row_order ? (int64_t)row_order[i] : i;
    };
    // k-block kb of this thread's 4 pieces (piece i: row group i/2, line i%2)
    auto load_kb = [&](const int32_t (&rid)[2], int kb, float4 (&dst)[8]) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int e4 = kb * 16 + (i & 1) * 8 + c16 * 2;
        const float4 *src = X4 + (int64_t)(rid[i >> 1] < 0 ? 0 : rid[i >> 1]) * d4 + e4;
        const bool ok = rid[i >> 1] >= 0;
        dst[2 * i] = (ok && e4 < d4) ? __ldg(src) : make_float4(0.f, 0.f, 0.f, 0.f);
        dst[2 * i + 1] = (ok && e4 + 1 < d4) ? __ldg(src + 1) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    auto load_ids = [&](int64_t off, int cnt, int32_t (&rid)[2]) {
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const int r = wrow0 + 8 * g + rl;
        rid[g] = r < cnt ? cand_ids[off + r] : -1;
      }
    };
    int64_t u0 = rowu(0), u1 = rowu(1);
    int cnt0 = -1, cnt1 = -1;
    int64_t off0 = 0, off1 = 0;
    int32_t self0 = 0, self1 = 0, cid0 = -1, cid1 = -1;
    float dist0 = __int_as_float(0x7f800000), dist1 = dist0;
    int32_t rid0[2] = {-1, -1}, rid1[2] = {-1, -1};
    float4 us0 = make_float4(0.f, 0.f, 0.f, 0.f), us1 = us0;  // own-row slice (d4 <= 256)
    float4 xn[8];
    if (u0 >= 0) {
      cnt0 = cand_counts[u0];
      off0 = cand_off[u0];
      self0 = row_node ? row_node[u0] : (int32_t)u0;
      if (cnt0 <= C) {
        if (t < cnt0) {
          cid0 = cand_ids[off0 + t];
          dist0 = cand_dists[off0 + t];
        }
        load_ids(off0, cnt0, rid0);
        if (t < d4) us0 = __ldg(X4 + (int64_t)self0 * d4 + t);
      }
    }
    load_kb(rid0, 0, xn);
    for (int64_t k = 0; k < nb; ++k) {
      const int64_t u2 = rowu(k + 2);
      cnt1 = -1;
      if (u1 >= 0) {
        cnt1 = cand_counts[u1];
        off1 = cand_off[u1];
        self1 = row_node ? row_node[u1] : (int32_t)u1;
      }
      cid1 = -1;
      dist1 = __int_as_float(0x7f800000);
      bool have1 = false;
      auto fetch1 = [&]() {  // the second half of point k+1's metadata
        have1 = true;
        rid1[0] = rid1[1] = -1;
        us1 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (cnt1 >= 0 && cnt1 <= C) {
          if (t < cnt1) {
            cid1 = cand_ids[off1 + t];
            dist1 = cand_dists[off1 + t];
          }
          load_ids(off1, cnt1, rid1);
          if (t < d4) us1 = __ldg(X4 + (int64_t)self1 * d4 + t);
        }
      };
      if (cnt0 > C) {  // hub row: skipped here, taken by prune_kernel
        fetch1();
        load_kb(rid1, 0, xn);
      } else {
        const int par = (int)(kp & 1);
        GFWAIT(0, mbar_wait(&s.pempty[par], (uint32_t)(((kp >> 1) & 1) ^ 1)));
        if (t < C) {
          s.id[par][t] = cid0;
          s.dist[par][t] = dist0;
        }
        if (t == 0) {
          s.cnt[par] = cnt0;
          s.self[par] = self0;
          s.u[par] = u0;
        }
        if (t < nkb * (KBLK / 4)) reinterpret_cast<float4 *>(s.urow[par])[t] = us0;
        named_bar_sync(2, PW * 32);
        const bool wact = wrow0 < cnt0;  // this warp has rows
        float nacc[2] = {0.f, 0.f};
        for (int kb = 0; kb < nkb; ++kb) {
          float4 xv[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) xv[j] = xn[j];
          if (kb + 1 < nkb) {
            if (wact) load_kb(rid0, kb + 1, xn);
          } else {  // the next point's first k-block
            if (!have1) fetch1();
            load_kb(rid1, 0, xn);
          }
          if (kb == (nkb >> 1) - 1 && !have1) fetch1();
          {
            // L1 prefetch PF_AHEAD blocks ahead (the register prefetch covers one
            // block, less than the L2 latency when a point has few rows):
            // lane l of a row's 4 lanes takes the 128-byte line of piece l
            const int pk = kb + PF_AHEAD;
            const bool nxt = pk >= nkb;
            const int pb = nxt ? pk - nkb : pk;
            const int32_t ra = nxt ? rid1[0] : rid0[0], rb = nxt ? rid1[1] : rid0[1];
            const int32_t rr = (c16 >> 1) ? rb : ra;
            const int e4 = pb * 16 + (c16 & 1) * 8;
            if (PF_AHEAD > 0 && (!nxt || have1) && pb < nkb && rr >= 0 && e4 < d4)
              asm volatile("prefetch.global.L1 [%0];" ::"l"(X4 + (int64_t)rr * d4 + e4));
          }
          GFWAIT(1, mbar_wait(&s.empty[stage], phase ^ 1));
          if (t == 0) {
            s.stage_end[stage] = 0;
            s.stage_n[stage] = max(16, (cnt0 + 15) & ~15);
          }
          if (wact) {
            const float4 *us = reinterpret_cast<const float4 *>(s.urow[par] + kb * KBLK);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int g = i >> 1, line = i & 1;
              if (rid0[g] < 0) continue;
              const int r = wrow0 + 8 * g + rl;
              const float4 ua = us[line * 8 + c16 * 2], ub = us[line * 8 + c16 * 2 + 1];
              const float4 xa = xv[2 * i], xb = xv[2 * i + 1];
              const float v[8] = {__fsub_rn(xa.x, ua.x), __fsub_rn(xa.y, ua.y),
                                  __fsub_rn(xa.z, ua.z), __fsub_rn(xa.w, ua.w),
                                  __fsub_rn(xb.x, ub.x), __fsub_rn(xb.y, ub.y),
                                  __fsub_rn(xb.z, ub.z), __fsub_rn(xb.w, ub.w)};
              uint32_t hw[4], lw[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float a = v[2 * e], b = v[2 * e + 1];
                nacc[g] = fmaf(a, a, nacc[g]);
                nacc[g] = fmaf(b, b, nacc[g]);
                hw[e] = pack_bf16x2(a, b);
                lw[e] = pack_bf16x2(__fsub_rn(a, __uint_as_float(hw[e] << 16)),
                                    __fsub_rn(b, __uint_as_float(hw[e] & 0xffff0000u)));
              }
              // 16-byte chunk line*4 + c16 of tile row r
              const uint32_t pos = (uint32_t)((r >> 3) * 1024 + (r & 7) * 128) +
                                   ((((uint32_t)(line * 4 + c16)) ^ (uint32_t)(r & 7)) << 4);
              *reinterpret_cast<uint4 *>(s.tile[stage][0] + pos) =
                  make_uint4(hw[0], hw[1], hw[2], hw[3]);
              *reinterpret_cast<uint4 *>(s.tile[stage][1] + pos) =
                  make_uint4(lw[0], lw[1], lw[2], lw[3]);
            }
          }
          fence_proxy_async_smem();  // generic-proxy smem writes -> tensor-core reads
          __syncwarp();
          if (lane == 0) mbar_arrive(&s.full[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        // row norms: the 4 lanes of a row hold its partial sums
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          float v = nacc[g];
          v += __shfl_xor_sync(0xffffffffu, v, 1);
          v += __shfl_xor_sync(0xffffffffu, v, 2);
          if (c16 == 0) s.nrm[par][wrow0 + 8 * g + rl] = v;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&s.pfull[par]);
        ++kp;
      }
      u0 = u1; cnt0 = cnt1; off0 = off1; self0 = self1; cid0 = cid1; dist0 = dist1;
      us0 = us1;
      rid0[0] = rid1[0];
      rid0[1] = rid1[1];
      u1 = u2;
    }
    // end of stream: one sentinel stage for the MMA warp, one sentinel point
    // for the mask warps
    GFWAIT(1, mbar_wait(&s.empty[stage], phase ^ 1));
    if (t == 0) s.stage_end[stage] = 1;
    __syncwarp();
    if (lane == 0) mbar_arrive(&s.full[stage]);
    {
      const int par = (int)(kp & 1);
      mbar_wait(&s.pempty[par], (uint32_t)(((kp >> 1) & 1) ^ 1));
      if (t == 0) s.cnt[par] = -1;
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.pfull[par]);
    }
    if (stats && t == 0) {
      tw[2] = clock64() - t_begin;
      for (int i = 0; i < 3; ++i) atomicAdd(stats + 4 + i, (unsigned long long)tw[i]);
    }
  } else if (warp == MMA_WARP) {
    if (lane == 0) {
      // ---------------- MMA: G = C' C'^T over the k-blocks ----------------
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t kp = 0;; ++kp) {
        const int par = (int)(kp & 1);
        GFWAIT(3, mbar_wait_sleep(&s.full[stage], phase, 200));
        if (s.stage_end[stage]) break;
        GFWAIT(4, mbar_wait(&s.tempty[par], (uint32_t)(((kp >> 1) & 1) ^ 1)));
        const uint32_t dcol = tmem + par * C;
        const uint32_t idesc = IDESC_BASE | ((uint32_t)(s.stage_n[stage] >> 3) << 17);
        for (int kb = 0; kb < nkb; ++kb) {
          if (kb > 0) GFWAIT(3, mbar_wait_sleep(&s.full[stage], phase, 100));
          fence_proxy_async_smem();
          tc_fence_after();
          const uint64_t dh = sw128_desc(s.tile[stage][0]), dl = sw128_desc(s.tile[stage][1]);
#pragma unroll
          for (int kk = 0; kk < KBLK / 16; ++kk)
            mma_bf16(dcol, dh + 2 * kk, dh + 2 * kk, idesc, (kb | kk) != 0);
#pragma unroll
          for (int kk = 0; kk < KBLK / 16; ++kk) mma_bf16(dcol, dh + 2 * kk, dl + 2 * kk, idesc, 1);
#pragma unroll
          for (int kk = 0; kk < KBLK / 16; ++kk) mma_bf16(dcol, dl + 2 * kk, dh + 2 * kk, idesc, 1);
          tc_commit(&s.empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit(&s.tfull[par]);
      }
      if (stats) {
        tw[5] = clock64() - t_begin;
        for (int i = 3; i < 6; ++i) atomicAdd(stats + 4 + i, (unsigned long long)tw[i]);
      }
    }
  } else if (warp < MMA_WARP) {  // warps PW .. PW+3: warp & 3 = TMEM lane quarter
    // ---------------- masks: thread t = candidate t = TMEM lane t ----------
    const int q = warp & 3;
    const int t = q * 32 + lane;
    for (int64_t kp = 0;; ++kp) {
      const int par = (int)(kp & 1);
      const uint32_t pph = (uint32_t)((kp >> 1) & 1);
      const int mb = (int)(kp % NBUF);
      const uint32_t mphase = (uint32_t)((kp / NBUF) & 1);
      GFWAIT(6, mbar_wait_sleep(&s.pfull[par], pph, 500));
      const int cnt = s.cnt[par];
      if (cnt < 0) {  // end of stream: tell every greedy warp
        for (int64_t kk = kp; kk < kp + NG; ++kk) {
          const int b = (int)(kk % NBUF);
          mbar_wait(&s.mempty[b], ((uint32_t)((kk / NBUF) & 1)) ^ 1);
          if (t == 0) s.gcnt[b] = -1;
          __syncwarp();
          if (lane == 0) mbar_arrive(&s.mfull[b]);
        }
        break;
      }
      const float dv = s.dist[par][t];
      const float nt = s.nrm[par][t];
      const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16) + par * C;
      uint32_t pm[4] = {0, 0, 0, 0}, qm[4] = {0, 0, 0, 0}, gmm[4] = {0, 0, 0, 0};
      GFWAIT(7, mbar_wait_sleep(&s.tfull[par], pph, 100));
      tc_fence_after();
      const int clast = q * 32 >= cnt ? -1 : min(q, (cnt - 1) >> 5);
#pragma unroll 1
      for (int c = 0; c <= clast; ++c) {
        uint32_t g[32];
        tmem_ld32(tl + (uint32_t)(c * 32), g);
        const uint32_t zu = __ballot_sync(0xffffffffu, s.dist[par][c * 32 + lane] == 0.0f);
        const uint32_t valid = c < q ? 0xffffffffu : ((1u << lane) - 1u);
        tmem_wait_ld();
        uint32_t dm = 0, am = 0, gm = 0;  // dominates / undecided / angle evaluated
        const float4 *np = reinterpret_cast<const float4 *>(s.nrm[par] + c * 32);
        const float4 *dp4 = reinterpret_cast<const float4 *>(s.dist[par] + c * 32);
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const float4 w = np[v];
          const float ni[4] = {w.x, w.y, w.z, w.w};
          float du[4] = {0.f, 0.f, 0.f, 0.f};
          if (ALPHA) {
            const float4 dq = dp4[v];
            du[0] = dq.x; du[1] = dq.y; du[2] = dq.z; du[3] = dq.w;
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int k = 4 * v + e;
            const float S = nt + ni[e];
            const float A = fmaf(-2.0f, __uint_as_float(g[k]), S);
            const float hi = fmaf(ee, S, A), lo = fmaf(-ee, S, A);
            bool cd, cn;
            if (ALPHA) {
              // F < dv and F > 0 certain: the angle is evaluated; its verdict
              // from the sign of f at the interval's ends (fp32, with slack)
              const bool lt = hi < dv && lo > 0.0f;
              const float duw = du[e];
              const float base = duw - dv, kk = (float)(2.0 * p_slack);
              const float fhi = base + hi - kk * sqrtf(duw * hi);
              const float flo = base + lo - kk * sqrtf(duw * lo);
              const float eps = 2e-6f * (duw + dv + hi);
              const bool mono = lo > base;  // (always, for sorted rows: duw <= dv)
              cd = lt && mono && fhi < -eps;
              cn = (lo >= dv && lo > 0.0f) || (lt && mono && flo > eps);
              gm |= (lt && (cd || cn)) ? (1u << k) : 0u;
            } else if (strategy == 0) {
              cd = hi < dv;
              cn = lo >= dv && lo > 0.0f;
            } else {
              cd = hi < dv && p_slack * (double)hi * (1.0 + 1e-12) < (double)dv;
              cn = lo > 0.0f && (lo >= dv || p_slack * (double)lo * (1.0 - 1e-12) >= (double)dv);
            }
            dm |= cd ? (1u << k) : 0u;
            am |= (cd || cn) ? 0u : (1u << k);
          }
        }
        pm[c] = (dm | zu) & valid;
        qm[c] = am & ~zu & valid;
        if (ALPHA) gmm[c] = gm & ~zu & valid;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.tempty[par]);
      GFWAIT(8, mbar_wait(&s.mempty[mb], mphase ^ 1));
      *reinterpret_cast<uint4 *>(s.pm[mb][t]) = make_uint4(pm[0], pm[1], pm[2], pm[3]);
      *reinterpret_cast<uint4 *>(s.qm[mb][t]) = make_uint4(qm[0], qm[1], qm[2], qm[3]);
      if (ALPHA)
        *reinterpret_cast<uint4 *>(s.am[mb][t]) = make_uint4(gmm[0], gmm[1], gmm[2], gmm[3]);
      const int32_t myid = s.id[par][t];
      const unsigned exm = __ballot_sync(0xffffffffu, t < cnt && myid != s.self[par]);
      if (lane == 0) s.ex[mb][q] = exm;
      s.gid[mb][t] = myid;
      s.gdist[mb][t] = dv;
      if (t == 0) {
        s.gu[mb] = s.u[par];
        s.gcnt[mb] = cnt;
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&s.mfull[mb]);
        mbar_arrive(&s.pempty[par]);
      }
    }
    if (stats && t == 96) {  // the busiest mask warp (4 chunks)
      tw[9] = clock64() - t_begin;
      for (int i = 6; i < 10; ++i) atomicAdd(stats + 4 + i, (unsigned long long)tw[i]);
    }
  } else {
    // ---------------- greedy scan, lazy exact pairs, counters (NG warps) ----
    const int gw = warp - GREEDY_WARP;
    unsigned long long st_exact = 0, st_iter = 0, st_amb = 0, st_chain = 0;
    for (int64_t k = gw;; k += NG) {
      const int mb = (int)(k % NBUF);
      GFWAIT(10, mbar_wait_sleep(&s.mfull[mb], (uint32_t)((k / NBUF) & 1), 1000));
      if (s.gcnt[mb] < 0) break;
      const int64_t u = s.gu[mb];
      const int32_t *sid = s.gid[mb];
      const float *sdist = s.gdist[mb];
      uint32_t pw[4][4], qw[4][4];  // this lane's candidates c*32+lane: pm / qm rows
      uint32_t aw[ALPHA ? 4 : 1][4];  // ... and the angle-evaluated masks (alpha rule)
      uint32_t exv[4];
      int32_t idv[4];
      float dsv[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint4 a = *reinterpret_cast<const uint4 *>(s.pm[mb][c * 32 + lane]);
        const uint4 b = *reinterpret_cast<const uint4 *>(s.qm[mb][c * 32 + lane]);
        pw[c][0] = a.x; pw[c][1] = a.y; pw[c][2] = a.z; pw[c][3] = a.w;
        qw[c][0] = b.x; qw[c][1] = b.y; qw[c][2] = b.z; qw[c][3] = b.w;
        if (ALPHA) {
          const uint4 g4 = *reinterpret_cast<const uint4 *>(s.am[mb][c * 32 + lane]);
          aw[ALPHA ? c : 0][0] = g4.x; aw[ALPHA ? c : 0][1] = g4.y;
          aw[ALPHA ? c : 0][2] = g4.z; aw[ALPHA ? c : 0][3] = g4.w;
        }
        exv[c] = s.ex[mb][c];
        idv[c] = sid[c * 32 + lane];
        dsv[c] = sdist[c * 32 + lane];
        if (stats) st_amb += __popc(b.x) + __popc(b.y) + __popc(b.z) + __popc(b.w);
      }
      uint32_t zu[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) zu[c] = __ballot_sync(0xffffffffu, dsv[c] == 0.0f);
      uint32_t kept_m[4];
      int kept, stop_j;
      for (;;) {
        // the reference's scan on the certain masks
        kept_m[0] = kept_m[1] = kept_m[2] = kept_m[3] = 0;
        kept = 0;
        stop_j = C;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (stop_j != C) break;
          const bool blocked = (pw[c][0] & kept_m[0]) | (pw[c][1] & kept_m[1]) |
                               (pw[c][2] & kept_m[2]) | (pw[c][3] & kept_m[3]);
          const uint32_t pjc = pw[c][c];
          unsigned m = exv[c] & __ballot_sync(0xffffffffu, !blocked);
          uint32_t km = 0;
          while (m) {
            const int li = __ffs(m) - 1;
            km |= 1u << li;
            if (++kept == M) {  // _kernels.py:378: nothing after it is examined
              stop_j = c * 32 + li;
              break;
            }
            const unsigned dom = __ballot_sync(0xffffffffu, (pjc >> li) & 1u);
            m &= ~(dom | ((2u << li) - 1u));
          }
          kept_m[c] = km;
        }
        // undecided pairs the result depends on: kept c_i in front of c_j's
        // first certain dominator (or of c_j itself) -- resolved one at a
        // time by the whole warp
        bool any_work = false;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int j = c * 32 + lane;
          const bool exam = j <= stop_j && ((exv[c] >> lane) & 1u);
          int f = -1;
#pragma unroll
          for (int w = 0; w <= c; ++w) {
            const uint32_t dd = pw[c][w] & kept_m[w] & (w < c ? 0xffffffffu : lanemask_lt());
            if (f < 0 && dd) f = w * 32 + __ffs(dd) - 1;
          }
          const int end = f >= 0 ? f : j;
#pragma unroll
          for (int w = 0; w <= c; ++w) {
            const uint32_t lim = end >= (w + 1) * 32 ? 0xffffffffu
                                 : (end <= w * 32 ? 0u : ((1u << (end - w * 32)) - 1u));
            uint32_t rel = exam ? (qw[c][w] & kept_m[w] & lim) : 0u;
            unsigned has = __ballot_sync(0xffffffffu, rel != 0);
            while (has) {
              const long long tr0 = stats ? clock64() : 0;
              const int src = __ffs(has) - 1;
              const uint32_t r = __shfl_sync(0xffffffffu, rel, src);
              const int ib = __ffs(r) - 1;
              const int32_t ida = sid[w * 32 + ib];
              const int32_t idb = __shfl_sync(0xffffffffu, idv[c], src);
              const float dvb = __shfl_sync(0xffffffffu, dsv[c], src);
              // level 2: both rows staged (coalesced) and their float64
              // distance; F = D (1 + theta), |theta| <= gseq
              const float4 *a4 = reinterpret_cast<const float4 *>(X + (int64_t)ida * d);
              const float4 *b4 = reinterpret_cast<const float4 *>(X + (int64_t)idb * d);
              float4 *pa = reinterpret_cast<float4 *>(s.pair[gw][0]);
              float4 *pb = reinterpret_cast<float4 *>(s.pair[gw][1]);
              double acc = 0.0;
              for (int e0 = 0; e0 < (d >> 2); e0 += 128) {
                float4 xa[4], xb[4];
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                  const int e = e0 + q4 * 32 + lane;
                  if (e < (d >> 2)) {
                    xa[q4] = __ldg(a4 + e);
                    xb[q4] = __ldg(b4 + e);
                  }
                }
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) {
                  const int e = e0 + q4 * 32 + lane;
                  if (e < (d >> 2)) {
                    pa[e] = xa[q4];
                    pb[e] = xb[q4];
                    double tt;
                    tt = (double)xa[q4].x - (double)xb[q4].x; acc = fma(tt, tt, acc);
                    tt = (double)xa[q4].y - (double)xb[q4].y; acc = fma(tt, tt, acc);
                    tt = (double)xa[q4].z - (double)xb[q4].z; acc = fma(tt, tt, acc);
                    tt = (double)xa[q4].w - (double)xb[q4].w; acc = fma(tt, tt, acc);
                  }
                }
              }
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
              const double dlo = acc * (1.0 - gseq), dhi = acc * (1.0 + gseq);
              const double dvd = (double)dvb;
              const float duwf = sdist[w * 32 + ib];  // d(u, c_i)
              int verdict = -1;  // bit 0 dominates, bit 1 angle evaluated; -1 undecided
              if (acc > 1e-30) {
                if (ALPHA) {
                  if (dlo >= dvd) {
                    verdict = 0;
                  } else if (dhi < dvd && dlo > (double)duwf - dvd) {
                    const double k2 = 2.0 * p_slack, du = (double)duwf;
                    const double tol = 1e-11 * (du + dvd + dhi);
                    if (alpha_f(du, dhi, dvd, k2) < -tol) verdict = 3;
                    else if (alpha_f(du, dlo, dvd, k2) > tol) verdict = 2;
                  }
                } else if (strategy == 0) {
                  if (dhi < dvd) verdict = 1;
                  else if (dlo >= dvd) verdict = 0;
                } else {
                  if (dhi < dvd && p_slack * dhi * (1.0 + 1e-12) < dvd) verdict = 1;
                  else if (dlo >= dvd || p_slack * dlo * (1.0 - 1e-12) >= dvd) verdict = 0;
                }
              }
              if (stats) ++st_exact;
              if (verdict < 0) {
                // level 3: the reference's sequential fp32 chain, from the staged rows
                __syncwarp();
                float F = 0.0f;
                if (lane == 0) {
                  const float *ra = s.pair[gw][0], *rb = s.pair[gw][1];
#pragma unroll 8
                  for (int e = 0; e < d; ++e) F = sq_step(F, ra[e], rb[e]);
                }
                F = __shfl_sync(0xffffffffu, F, 0);
                verdict = ALPHA ? alpha_exact(duwf, F, dvb, p_slack)
                                : (dominates_exact(F, dvb, strategy, p_slack) ? 1 : 0);
                if (stats) ++st_chain;
              }
              __syncwarp();
              if (lane == src) {
                if (verdict & 1) pw[c][w] |= 1u << ib;
                if (ALPHA && (verdict & 2)) aw[ALPHA ? c : 0][w] |= 1u << ib;
                qw[c][w] &= ~(1u << ib);
                rel &= rel - 1;
              }
              any_work = true;
              has = __ballot_sync(0xffffffffu, rel != 0);
              if (stats) tw[11] += clock64() - tr0;
            }
          }
        }
        if (stats) ++st_iter;
        if (!any_work) break;
      }
      // the kept candidates in scan order, staged in this point's candidate
      // buffer, then written as whole padded rows
      {
        int32_t *oid = s.gid[mb];
        float *od = s.gdist[mb];
        __syncwarp();
        int base = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if ((kept_m[c] >> lane) & 1u) {
            const int pos = base + __popc(kept_m[c] & lanemask_lt());
            oid[pos] = idv[c];
            od[pos] = dsv[c];
          }
          base += __popc(kept_m[c]);
        }
        __syncwarp();
        for (int j = lane; j < width; j += 32) {
          const bool kk = j < kept;
          out_ids[u * width + j] = kk ? oid[j] : -1;
          out_dists[u * width + j] = kk ? od[j] : __int_as_float(0x7f800000);
        }
      }
      // exact lazy counters of every examined candidate
      const int kp1 = __popc(kept_m[0]), kp2 = kp1 + __popc(kept_m[1]),
                kp3 = kp2 + __popc(kept_m[2]);
      long long dsum = 0, asum = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int j = c * 32 + lane;
        if (j > stop_j || !((exv[c] >> lane) & 1u)) continue;
        int f = -1;
#pragma unroll
        for (int w = 0; w <= c; ++w) {
          const uint32_t dd = pw[c][w] & kept_m[w] & (w < c ? 0xffffffffu : lanemask_lt());
          if (f < 0 && dd) f = w * 32 + __ffs(dd) - 1;
        }
        const int end = f >= 0 ? f : j;
        const int ew = end >> 5;
        const uint32_t kw = ew == 0 ? kept_m[0] : ew == 1 ? kept_m[1] : ew == 2 ? kept_m[2] : kept_m[3];
        int ev = (ew == 0 ? 0 : ew == 1 ? kp1 : ew == 2 ? kp2 : kp3) +
                 __popc(kw & ((1u << (end & 31)) - 1u));
        if (f >= 0 && !((zu[f >> 5] >> (f & 31)) & 1u)) ev += 1;
        dsum += ev;
        if (ALPHA) {  // angle evaluations among the pairs the scan looked at
          int an = 0;
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            uint32_t lim = end >= (w + 1) * 32 ? 0xffffffffu
                                               : (end <= w * 32 ? 0u : ((1u << (end - w * 32)) - 1u));
            if (f >= 0 && (f >> 5) == w) lim |= 1u << (f & 31);
            an += __popc(aw[ALPHA ? c : 0][w] & kept_m[w] & lim);
          }
          asum += an;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
        if (ALPHA) asum += __shfl_xor_sync(0xffffffffu, asum, o);
      }
      if (lane == 0) {
        dist_evals[u] = dsum;
        angle_evals[u] = asum;
        out_counts[u] = kept;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.mempty[mb]);
    }
    if (stats) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) st_amb += __shfl_xor_sync(0xffffffffu, st_amb, o);
      if (lane == 0) {
        atomicAdd(stats, st_exact);
        atomicAdd(stats + 1, st_iter);
        atomicAdd(stats + 2, st_amb);
        atomicAdd(stats + 3, st_chain);
        if (gw == 0) {
          tw[12] = clock64() - t_begin;
          for (int i = 10; i < 13; ++i) atomicAdd(stats + 4 + i, (unsigned long long)tw[i]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(TMEM_COLS));
  }
}

}  // namespace gramf

// fp32 rows, d % 4 == 0, 16-byte aligned, 128 <= d <= 1024; rng, alpha and slack
bool gram_f32_supported(const float *X, int64_t d, int strategy) {
  static int env = -1;
  if (env < 0) {
    const char *e = getenv("PGK_GRAM_F32");
    env = (e && e[0] == '0') ? 0 : 1;
  }
  return env && strategy >= 0 && strategy <= 2 && d >= 128 && d <= gramf::DMAX && d % 4 == 0 &&
         ((uintptr_t)X % 16 == 0);
}

// Rows with more than 128 candidates are skipped (the caller's prune_kernel
// launch takes exactly those).
int launch_prune_gram_f32(const float *X, int64_t d, int64_t n, const int32_t *row_node,
                          const int32_t *row_order, const int64_t *cand_off,
                          const int32_t *cand_counts, const int32_t *cand_ids,
                          const float *cand_dists, int strategy, double cos_alpha, int64_t M,
                          int64_t width, int32_t *out_ids, float *out_dists,
                          int32_t *out_counts, int64_t *dist_evals, int64_t *angle_evals,
                          cudaStream_t stream) {
  using namespace gramf;
  const int nkb = (int)((d + KBLK - 1) / KBLK);
  const double dp = (double)nkb * KBLK;
  const double u24 = 5.9604644775390625e-08;
  // |F - A| <= ee (n_t + n_i): norm sums, the fp32 evaluation of A, centring
  // rounding, the sequential chain's own rounding; operand truncation and the
  // truncating fp32 accumulation of 3 dp products (a_t a_i <= (n_t + n_i) / 2)
  const double ee = (dp + 2.0 * (double)d + 16.0) * u24 * 1.02 +
                    (3.1 / 262144.0 + 4.0 * (dp + 16.0) / 8388608.0) + 8.0 * u24;
  const size_t smem = sizeof(Smem) + 1024;
  PGK_CUDA(ensure_smem((const void *)prune_gram_f32_kernel<false>, smem));
  PGK_CUDA(ensure_smem((const void *)prune_gram_f32_kernel<true>, smem));
  const unsigned grid = (unsigned)std::min<int64_t>(n, (int64_t)num_sms());
  // F = D (1 + theta): t = fl(a - b), t * t and d - 1 additions, each rounded
  const double gseq = ((double)d + 3.0) * u24 * 1.0001;
  static int stats_env = -1;
  if (stats_env < 0) {
    const char *e = getenv("PGK_GRAM_F32_STATS");
    stats_env = (e && e[0] == '1') ? 1 : 0;
  }
  unsigned long long *dstats = nullptr;
  if (stats_env) {
    PGK_CUDA(cudaMalloc(&dstats, 20 * sizeof(unsigned long long)));
    PGK_CUDA(cudaMemsetAsync(dstats, 0, 20 * sizeof(unsigned long long), stream));
  }
  if (strategy == 1)
    prune_gram_f32_kernel<true><<<grid, THREADS, smem, stream>>>(
        X, (int)d, n, row_node, row_order, cand_off, cand_counts, cand_ids, cand_dists, strategy,
        cos_alpha, (float)ee, gseq, (int)M, (int)width, out_ids, out_dists, out_counts, dist_evals,
        angle_evals, dstats);
  else
    prune_gram_f32_kernel<false><<<grid, THREADS, smem, stream>>>(
        X, (int)d, n, row_node, row_order, cand_off, cand_counts, cand_ids, cand_dists, strategy,
        cos_alpha, (float)ee, gseq, (int)M, (int)width, out_ids, out_dists, out_counts, dist_evals,
        angle_evals, dstats);
  PGK_CHECK_LAUNCH("prune_gram_f32_kernel");
  if (stats_env) {
    unsigned long long h[20];
    PGK_CUDA(cudaMemcpyAsync(h, dstats, sizeof(h), cudaMemcpyDeviceToHost, stream));
    PGK_CUDA(cudaStreamSynchronize(stream));
    cudaFree(dstats);
    fprintf(stderr,
            "[gram f32] %lld rows: undecided pairs %.1f per row, float64 pair evaluations %.2f, "
            "sequential chains %.3f, scan iterations %.2f per row\n",
            (long long)n, (double)h[2] / (double)n, (double)h[0] / (double)n,
            (double)h[3] / (double)n, (double)h[1] / (double)n);
    const double cg = (double)grid * 1e6;
    fprintf(stderr,
            "[gram f32] Mcycles per CTA: producer total %.2f (pempty %.2f, empty %.2f) | mma total "
            "%.2f (full %.2f, tempty %.2f) | mask total %.2f (pfull %.2f, tfull %.2f, mempty %.2f) "
            "| greedy total %.2f (mfull %.2f, resolve %.2f)\n",
            h[6] / cg, h[4] / cg, h[5] / cg, h[9] / cg, h[7] / cg, h[8] / cg, h[13] / cg, h[10] / cg,
            h[11] / cg, h[12] / cg, h[16] / cg, h[14] / cg, h[15] / cg);
  }
  return PGK_OK;
}

}  // namespace pgk
