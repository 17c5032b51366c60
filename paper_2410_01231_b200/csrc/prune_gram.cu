// prune_gram.cu -- the batched per-point C x C candidate-distance kernel on
// tcgen05 tensor cores, feeding the greedy RNG / alpha scan (phase A and the
// phase-B re-prune) for exact-integer data (values in [0,255], d <= 128).
//
// For one point u with cnt <= 128 candidates c_0..c_{cnt-1} (ascending
// (dist, id)):  the candidates' u8 rows are gathered into a 128 x 128-byte
// SW128 K-major tile, and ONE tcgen05.mma.kind::i8 (M=N=128, K=128 in 4
// steps) produces the Gram matrix G = C C^T (s32, exact) in TMEM.  Candidate
// t lives in TMEM lane t = thread t of the 4-warp scan group, so when c_e is
// kept every candidate reads G[t][e] from its own lane (tcgen05.ld.32x32b.x1
// at column e) and tests
//     squared_l2(c_e, c_t) = |c_e|^2 + |c_t|^2 - 2 G[t][e]
// -- bit-identical to the reference's sequential fp32 squared_l2 because
// every partial sum is an integer below 2^24 (_kernels.py:17-24).  The scan
// itself is the reference's (_kernels.py:364-409): the next kept neighbour is
// the first still-alive candidate, candidates are dropped the moment a kept
// neighbour dominates them, and each candidate's dist_evals / angle_evals are
// exactly the lazy pairs the reference evaluates (speculation past the M-th
// kept neighbour is discarded).  Rows with more than 128 candidates (hubs in
// phase B) are listed and left to prune_u8_kernel.
//
// CTA: warp 0 gathers (cp.async, zero-filled tails), warp 1 allocates TMEM and
// issues the MMA, warps 2-5 scan.  4 CTAs per SM share the tensor core
// (128 TMEM columns each).
#include "common.cuh"
#include "tc_ptx.cuh"

namespace pgk {
namespace gram {

using namespace tc;

constexpr int C = 128;          // candidates per point (TMEM lanes)
constexpr int STAGES = 2;       // gathered points in flight
constexpr int THREADS = 192;
constexpr int CTAS_PER_SM = 4;
constexpr int TMEM_COLS = 128;
constexpr uint32_t IDESC = (2u << 4) | ((uint32_t)(C >> 3) << 17) | ((uint32_t)(C >> 4) << 24);

struct __align__(1024) Smem {
  uint8_t tile[STAGES][C * 128];  // SW128 K-major: 8-row x 128-byte atoms
  int32_t id[STAGES][C];
  float dist[STAGES][C];
  int32_t nrm[STAGES][C];
  int64_t u[STAGES];
  int32_t cnt[STAGES];
  alignas(16) uint32_t pm[C][4];  // pm[j]: candidates i < j that dominate c_j if kept
  alignas(16) uint32_t am[C][4];  // am[j]: candidates i whose test of c_j evaluates the angle
  uint32_t ex[4];        // examinable candidates (in range, not u itself)
  uint64_t full[STAGES], empty[STAGES];
  uint64_t tfull, tempty;
  uint32_t tmem_base;
};

template <int STRATEGY>  // 0 = rng, 1 = alpha (compile-time: no angle code for rng)
__global__ void __launch_bounds__(THREADS, CTAS_PER_SM)
    prune_gram_kernel(const uint8_t *__restrict__ xu8, const int32_t *__restrict__ norms,
                      int64_t n_rows, const int32_t *__restrict__ row_node,
                      const int32_t *__restrict__ row_order,
                      const int64_t *__restrict__ cand_off,
                      const int32_t *__restrict__ cand_counts,
                      const int32_t *__restrict__ cand_ids,
                      const float *__restrict__ cand_dists, int strategy, double cos_alpha,
                      int M, int width, int32_t *__restrict__ out_ids,
                      float *__restrict__ out_dists, int32_t *__restrict__ out_counts,
                      int64_t *__restrict__ dist_evals, int64_t *__restrict__ angle_evals,
                      int32_t *__restrict__ long_rows, int32_t *__restrict__ long_count) {
  extern __shared__ uint8_t smem_raw[];
  Smem &s = *reinterpret_cast<Smem *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                      ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&s.full[i], 32);   // every gather lane arrives (cp.async.mbarrier)
      mbar_init(&s.empty[i], 4);   // every scan warp releases the stage
    }
    mbar_init(&s.tfull, 1);
    mbar_init(&s.tempty, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&s.tmem_base)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s.tmem_base;

  if (warp == 0) {
    // ---------------- gather: rows, ids, dists, norms of one point --------
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t i = blockIdx.x; i < n_rows; i += gridDim.x) {
      const int64_t u = row_order ? row_order[i] : i;
      const int cnt = cand_counts[u];
      if (cnt > C) {  // hub row: left to the per-warp kernel
        if (lane == 0) long_rows[atomicAdd(long_count, 1)] = (int32_t)u;
        continue;
      }
      mbar_wait(&s.empty[stage], phase ^ 1);
      const int64_t base = cand_off[u];
      uint8_t *tile = s.tile[stage];
#pragma unroll
      for (int k = 0; k < C / 32; ++k) {
        const int r = lane + 32 * k;
        const bool ok = r < cnt;
        const int32_t v = ok ? cand_ids[base + r] : 0;
        s.id[stage][r] = ok ? v : -1;
        s.dist[stage][r] = ok ? cand_dists[base + r] : 0.f;
        s.nrm[stage][r] = ok ? __ldg(norms + v) : 0;
        const uint8_t *src = xu8 + (int64_t)v * 128;
        uint8_t *dst = tile + (r >> 3) * 1024 + (r & 7) * 128;
#pragma unroll
        for (int ch = 0; ch < 8; ++ch)  // 128B swizzle: chunk ^ (row % 8)
          cp_async16_zfill(dst + ((ch ^ (r & 7)) << 4), src + ch * 16, ok ? 16u : 0u);
      }
      if (lane == 0) {
        s.u[stage] = u;
        s.cnt[stage] = cnt;
      }
      __syncwarp();
      cp_async_mbar_arrive(&s.full[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA: G = C C^T per gathered point ----------------
      int stage = 0;
      uint32_t phase = 0, tphase = 0;
      for (int64_t i = blockIdx.x; i < n_rows; i += gridDim.x) {
        const int64_t u = row_order ? row_order[i] : i;
        if (cand_counts[u] > C) continue;
        mbar_wait(&s.full[stage], phase);
        fence_proxy_async_smem();  // cp.async (generic proxy) -> tensor-core reads
        mbar_wait(&s.tempty, tphase ^ 1);
        tc_fence_after();
        const uint64_t desc = sw128_desc(s.tile[stage]);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_i8(tmem, desc + 2 * kk, desc + 2 * kk, IDESC, kk > 0);
        tc_commit(&s.tfull);
        tphase ^= 1;
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else {
    // ---------------- scan group: thread t = candidate t = TMEM lane t ----
    // 1. every candidate t reads its own Gram row G[t][*] from TMEM and
    //    builds two 128-bit masks over the candidates i < t:
    //      pm: c_i dominates c_t if c_i is kept (_kernels.py:385-397)
    //      am: the reference's test of c_t against kept c_i evaluates the angle
    // 2. one warp runs the greedy scan on the masks (kept = first candidate
    //    not dominated by an earlier kept one, stop at M) and derives every
    //    examined candidate's lazy dist / angle evaluation counts.
    const int q = warp & 3;               // TMEM lane quarter of this warp
    const int t = q * 32 + lane;          // candidate index
    const int sw = warp - 2;              // scan-warp slot 0..3
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    int stage = 0;
    uint32_t phase = 0, tphase = 0;
    for (int64_t i = blockIdx.x; i < n_rows; i += gridDim.x) {
      const int64_t u = row_order ? row_order[i] : i;
      const int cnt = cand_counts[u];
      if (cnt > C) continue;
      mbar_wait(&s.full[stage], phase);
      mbar_wait(&s.tfull, tphase);
      tc_fence_after();
      const int32_t self = row_node ? row_node[u] : (int32_t)u;
      const int32_t *sid = s.id[stage];
      const float *sdist = s.dist[stage];
      const int32_t *snrm = s.nrm[stage];
      const float dv = sdist[t];
      const int nv = snrm[t];
      uint32_t pm[4] = {0, 0, 0, 0}, am[4] = {0, 0, 0, 0};
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t g[32];
        tmem_ld32(tl + (uint32_t)(c * 32), g);
        tmem_wait_ld();
        // branch-free simple verdicts; the fp64 angle tests only for alpha
        uint32_t dm = 0, need = 0;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const int ci = c * 32 + k;
          const float duw = sdist[ci];
          const float dwv = (float)(snrm[ci] + nv - 2 * (int)g[k]);  // == squared_l2
          const bool valid = ci < t;
          const bool z = (duw == 0.0f) | (dwv == 0.0f);
          const bool lt = dwv < dv;
          if (STRATEGY == 0) {
            dm |= (valid & (z | lt)) ? (1u << k) : 0u;
          } else {
            dm |= (valid & z) ? (1u << k) : 0u;
            const bool ang = valid & !z & lt;
            need |= ang ? (1u << k) : 0u;
            if (ang && cos_angle_from_sq(duw, dwv, dv) < cos_alpha) dm |= 1u << k;
          }
        }
        am[c] = need;
        pm[c] = dm;
      }
      // TMEM is free for the next point's MMA
      tc_fence_before();
      named_bar_sync(1, 128);  // previous point's greedy warp is done with pm/am
      if (lane == 0) mbar_arrive(&s.tempty);
      *reinterpret_cast<uint4 *>(s.pm[t]) = make_uint4(pm[0], pm[1], pm[2], pm[3]);
      *reinterpret_cast<uint4 *>(s.am[t]) = make_uint4(am[0], am[1], am[2], am[3]);
      const unsigned exm = __ballot_sync(0xffffffffu, t < cnt && sid[t] != self);
      if (lane == 0) s.ex[q] = exm;
      named_bar_sync(1, 128);
      if (sw == 0) {
        // ---- greedy scan on the masks (warp 2) ----
        uint32_t kept_m[4] = {0, 0, 0, 0};
        int kept = 0, stop_j = C;
        for (int c = 0; c < 4 && stop_j == C; ++c) {
          const int j = c * 32 + lane;
          const uint4 pj = *reinterpret_cast<const uint4 *>(s.pm[j]);
          const bool blocked = (pj.x & kept_m[0]) | (pj.y & kept_m[1]) | (pj.z & kept_m[2]) |
                               (pj.w & kept_m[3]);
          const uint32_t pjc = c == 0 ? pj.x : c == 1 ? pj.y : c == 2 ? pj.z : pj.w;
          unsigned m = s.ex[c] & __ballot_sync(0xffffffffu, !blocked);
          while (m) {
            const int li = __ffs(m) - 1;  // next kept candidate, index c*32+li
            kept_m[c] |= 1u << li;
            if (lane == 0) {
              out_ids[u * width + kept] = sid[c * 32 + li];
              out_dists[u * width + kept] = sdist[c * 32 + li];
            }
            ++kept;
            if (kept == M) {  // _kernels.py:378: nothing after it is examined
              stop_j = c * 32 + li;
              break;
            }
            // later lanes of this chunk dominated by c_li
            const unsigned dom = __ballot_sync(0xffffffffu, (pjc >> li) & 1u);
            m &= ~(dom | ((2u << li) - 1u));
          }
        }
        // ---- exact lazy counters of every examined candidate ----
        long long dsum = 0, asum = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int j = c * 32 + lane;
          if (j > stop_j || !((s.ex[c] >> lane) & 1u)) continue;
          const uint4 pj = *reinterpret_cast<const uint4 *>(s.pm[j]);
          const uint4 aj = *reinterpret_cast<const uint4 *>(s.am[j]);
          const uint32_t pw[4] = {pj.x, pj.y, pj.z, pj.w}, aw[4] = {aj.x, aj.y, aj.z, aj.w};
          // kept candidates before j, in order, up to the first dominator
          int f = -1;
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            const uint32_t below = w < c ? 0xffffffffu : (w == c ? ((1u << lane) - 1u) : 0u);
            const uint32_t d = pw[w] & kept_m[w] & below;
            if (f < 0 && d) f = w * 32 + __ffs(d) - 1;
          }
          int ev = 0, an = 0;
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            uint32_t lim;  // kept candidates examined by c_j: before f (or before j)
            const int end = f >= 0 ? f : j;
            lim = end >= (w + 1) * 32 ? 0xffffffffu : (end <= w * 32 ? 0u : ((1u << (end - w * 32)) - 1u));
            ev += __popc(kept_m[w] & lim);
            const uint32_t lim_incl = f >= 0 && (f >> 5) == w ? (lim | (1u << (f & 31))) : lim;
            an += __popc(aw[w] & kept_m[w] & lim_incl);
          }
          if (f >= 0 && sdist[f] != 0.0f) ev += 1;  // the dominator's own test (not duw == 0)
          dsum += ev;
          asum += an;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
          asum += __shfl_xor_sync(0xffffffffu, asum, o);
        }
        for (int j = kept + lane; j < width; j += 32) {
          out_ids[u * width + j] = -1;
          out_dists[u * width + j] = __int_as_float(0x7f800000);
        }
        if (lane == 0) {
          dist_evals[u] = dsum;
          angle_evals[u] = asum;
          out_counts[u] = kept;
        }
        __syncwarp();
      }
      // stage (ids / dists / norms) released once the greedy warp is done
      if (sw == 0 && lane == 0) mbar_arrive(&s.empty[stage]);
      if (sw != 0 && lane == 0) mbar_arrive(&s.empty[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
      tphase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(TMEM_COLS));
  }
}

}  // namespace gram

int launch_prune_u8_rows(const uint8_t *xu8, const int32_t *norms, int64_t n,
                         const int32_t *n_dev, const int32_t *row_node, const int32_t *row_order,
                         const int64_t *cand_off, const int32_t *cand_counts,
                         const int32_t *cand_ids, const float *cand_dists, int strategy,
                         double cos_alpha, int64_t M, int64_t width, int32_t *out_ids,
                         float *out_dists, int32_t *out_counts, int64_t *dist_evals,
                         int64_t *angle_evals, cudaStream_t stream);

size_t gram_workspace(int64_t n) { return (size_t)(n + 64) * sizeof(int32_t); }

// Opt-in (PGK_GRAM=1): exact and parity-tested, but on config 2 the per-warp
// exact-integer kernel is faster today (12 vs 19 ms for phase A at 1M; the
// full C x C predicate matrix costs more than the reference's lazy pairs).
bool gram_enabled() {
  static int env = -1;
  if (env < 0) {
    const char *e = getenv("PGK_GRAM");
    env = (e && e[0] == '1') ? 1 : 0;
  }
  return env == 1;
}

// Phase-A / re-prune selection through the tensor-core Gram kernel; rows with
// more than 128 candidates go to prune_u8_kernel.  ws: gram_workspace(n) bytes.
int launch_prune_gram(const uint8_t *xu8, const int32_t *norms, int64_t n,
                      const int32_t *row_node, const int32_t *row_order,
                      const int64_t *cand_off, const int32_t *cand_counts,
                      const int32_t *cand_ids, const float *cand_dists, int strategy,
                      double cos_alpha, int64_t M, int64_t width, int32_t *out_ids,
                      float *out_dists, int32_t *out_counts, int64_t *dist_evals,
                      int64_t *angle_evals, void *ws, cudaStream_t stream) {
  if (n == 0) return PGK_OK;
  int32_t *long_count = reinterpret_cast<int32_t *>(ws);
  int32_t *long_rows = long_count + 32;
  PGK_CUDA(cudaMemsetAsync(long_count, 0, sizeof(int32_t), stream));
  const size_t smem = sizeof(gram::Smem) + 1024;
  static bool attr = false;
  if (!attr) {
    PGK_CUDA(cudaFuncSetAttribute(gram::prune_gram_kernel<0>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    PGK_CUDA(cudaFuncSetAttribute(gram::prune_gram_kernel<1>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  const unsigned grid =
      (unsigned)std::min<int64_t>(n, (int64_t)gram::CTAS_PER_SM * num_sms());
  if (strategy == 0)
    gram::prune_gram_kernel<0><<<grid, gram::THREADS, smem, stream>>>(
        xu8, norms, n, row_node, row_order, cand_off, cand_counts, cand_ids, cand_dists, 0,
        cos_alpha, (int)M, (int)width, out_ids, out_dists, out_counts, dist_evals, angle_evals,
        long_rows, long_count);
  else
    gram::prune_gram_kernel<1><<<grid, gram::THREADS, smem, stream>>>(
        xu8, norms, n, row_node, row_order, cand_off, cand_counts, cand_ids, cand_dists, 1,
        cos_alpha, (int)M, (int)width, out_ids, out_dists, out_counts, dist_evals, angle_evals,
        long_rows, long_count);
  PGK_CHECK_LAUNCH("prune_gram_kernel");
  // hub rows (> 128 candidates): the per-warp exact-integer kernel, over the
  // device-side list (its length is read on the device)
  return launch_prune_u8_rows(xu8, norms, n, long_count, row_node, long_rows, cand_off,
                              cand_counts, cand_ids, cand_dists, strategy, cos_alpha, M, width,
                              out_ids, out_dists, out_counts, dist_evals, angle_evals, stream);
}

}  // namespace pgk
