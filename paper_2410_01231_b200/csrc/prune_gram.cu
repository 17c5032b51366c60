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
// CTA: warp 0 gathers (TMA gather4 rows, register-pipelined metadata), warp 1 allocates TMEM and
// issues the MMA, warps 2-5 build the predicate masks (each its lower-
// triangle chunks of the Gram rows), warp 6 runs the greedy scan and the
// counters on double-buffered masks, overlapped with the next point's masks.
// 4 CTAs per SM share the tensor core (128 TMEM columns each).
#include <cuda.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace pgk {
namespace gram {

using namespace tc;

constexpr int C = 128;          // candidates per point (TMEM lanes)
#ifndef GRAM_STAGES
#define GRAM_STAGES 2
#endif
#ifndef GRAM_GROUPS
#define GRAM_GROUPS 1
#endif
#ifndef GRAM_CTAS
#define GRAM_CTAS 4
#endif
#ifndef GRAM_GREEDY
#define GRAM_GREEDY 2
#endif
#ifndef GRAM_ROWS_CPASYNC
#define GRAM_ROWS_CPASYNC 0  // candidate rows by 16-byte cp.async instead of TMA gather4
#endif
#ifndef GRAM_TMA_SINGLE
#define GRAM_TMA_SINGLE 0  // 1: lane 0 issues all gather4 ops from shared-memory ids
#endif
#ifndef GRAM_TMA_UNIFORM
#define GRAM_TMA_UNIFORM 0  // 1: warp-uniform gather4 issue loop (lane g's ids broadcast, lane 0 issues)
#endif
#ifndef GRAM_TMA_ROWS
#define GRAM_TMA_ROWS 64  // with GRAM_ROWS_CPASYNC: rows per point left to TMA gather4
#endif
#ifndef GRAM_NORMS_GATHER
#define GRAM_NORMS_GATHER 1  // 1: the gather warp fetches |c|^2 (cp.async); 0: mask warps compute it
#endif
#ifndef GRAM_NBUF
#define GRAM_NBUF 2  // measured: 3 buffers cost 5 % (less shared memory left to L1)
#endif
constexpr int STAGES = GRAM_STAGES;  // gathered points in flight
constexpr int GROUPS = GRAM_GROUPS;  // mask warpgroups = TMEM accumulators (point parity)
constexpr int NG = GRAM_GREEDY;      // greedy warps: point k goes to warp k % NG
constexpr int NBUF = GRAM_NBUF;      // mask buffers: point k uses k % NBUF
static_assert(NBUF >= NG, "every greedy warp needs a buffer");
constexpr int THREADS = 32 * (2 + 4 * GROUPS + NG);
constexpr int GREEDY_WARP = 2 + 4 * GROUPS;  // first greedy warp
constexpr int CTAS_PER_SM = GRAM_CTAS;
constexpr int TMEM_COLS = C * GROUPS;
constexpr uint32_t IDESC = (2u << 4) | ((uint32_t)(C >> 3) << 17) | ((uint32_t)(C >> 4) << 24);

template <int STRATEGY>
struct __align__(1024) Smem {
  uint8_t tile[STAGES][C * 128];  // SW128 K-major: 8-row x 128-byte atoms
  int32_t id[STAGES][C];
  float dist[STAGES][C];
  alignas(16) int32_t nrm[STAGES][C];
  // per stage, per point slot (PAIR mode: two points share a stage, rows
  // 0..63 and 64..127; otherwise slot 0 only)
  int32_t cnt[STAGES][2];   // [0] -1: end of this CTA's stream; 0: empty slot
  int32_t self[STAGES][2];
  int64_t u[STAGES][2];
  alignas(16) uint32_t pm[NBUF][C][4];  // pm[j]: candidates i < j that dominate c_j if kept
  // am[j]: candidates i whose test of c_j evaluates the angle (alpha only)
  alignas(16) uint32_t am[STRATEGY == 1 ? NBUF : 1][STRATEGY == 1 ? C : 1][4];
  uint32_t ex[NBUF][4];     // examinable candidates (in range, not u itself)
  int32_t gid[NBUF][C];     // the greedy warp's copy of the point (the gather
  float gdist[NBUF][C];     // stage is released as soon as the masks are built)
  int64_t gu[NBUF][2];     // -1: empty slot
  int32_t gcnt[NBUF][2];    // [0] -1: end of stream
  uint64_t full[STAGES], empty[STAGES];
  uint64_t tfull[GROUPS], tempty[GROUPS];
  uint64_t mfull[NBUF], mempty[NBUF];
  uint32_t tmem_base;
};

#ifndef GRAM_SLEEP
#define GRAM_SLEEP 0  // ns between polls of the roles waiting on the gather stream (0: spin)
#endif
#if GRAM_SLEEP > 0
#define GRAM_IDLE_WAIT(bar, par) mbar_wait_sleep(bar, par, GRAM_SLEEP)
#else
#define GRAM_IDLE_WAIT(bar, par) mbar_wait(bar, par)
#endif
#ifndef GRAM_STATS
#define GRAM_STATS 0
#endif
// GRAM_STATS=1 builds: per-role cycles spent in each mbarrier wait
// (slots: 0 gather-empty, 1 mma-full, 2 mma-tempty, 3 mask-full, 4 mask-tfull,
// 5 mask-mempty, 6 greedy-mfull, 7-10 total cycles of gather/mma/mask/greedy)
__device__ unsigned long long g_gram_stats[16];
#if GRAM_STATS
#define GWAIT(slot, expr)                                   \
  do {                                                      \
    const long long t0_ = clock64();                        \
    expr;                                                   \
    if (lane == 0) atomicAdd(&g_gram_stats[slot], (unsigned long long)(clock64() - t0_)); \
  } while (0)
#define GMARK(acc)                                            \
  do {                                                      \
    const long long t_ = clock64();                         \
    acc += t_ - gmark_;                                     \
    gmark_ = t_;                                            \
  } while (0)
#else
#define GWAIT(slot, expr) expr
#define GMARK(acc) do { } while (0)
#endif

// PAIR: two points of <= 64 candidates per stage / MMA (rows 0..63 and
// 64..127 of the tile; the diagonal 64 x 64 blocks of the Gram matrix are the
// two points' own): the phase-B re-prune, whose rows hold ~27 candidates, is
// bound by the per-point pipeline cost, which pairing halves.  Rows with more
// than 64 candidates are listed for the single-point kernel.
template <int STRATEGY, bool PAIR>  // 0 = rng, 1 = alpha (compile-time: no angle code for rng)
__global__ void __launch_bounds__(THREADS, CTAS_PER_SM)
    prune_gram_kernel(const __grid_constant__ CUtensorMap tmX,
                      const uint8_t *__restrict__ xrows, const int32_t *__restrict__ norms,
                      int64_t n_rows, const int32_t *__restrict__ row_node,
                      const int32_t *__restrict__ row_order,
                      const int64_t *__restrict__ cand_off,
                      const int32_t *__restrict__ cand_counts,
                      const int32_t *__restrict__ cand_ids,
                      const float *__restrict__ cand_dists, int strategy, double cos_alpha,
                      int M, int width, int32_t *__restrict__ out_ids,
                      float *__restrict__ out_dists, int32_t *__restrict__ out_counts,
                      int64_t *__restrict__ dist_evals, int64_t *__restrict__ angle_evals,
                      int32_t *__restrict__ long_rows, int32_t *__restrict__ long_count,
                      const int32_t *__restrict__ n_rows_dev) {
  static_assert(!PAIR || (GROUPS == 1 && NG == 2), "PAIR: one mask group, one greedy warp per slot");
  constexpr int PC = PAIR ? C / 2 : C;  // candidates per point
  if (n_rows_dev) n_rows = *n_rows_dev;  // rows listed on the device (a previous launch)
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned view, derived from the shared array itself so every access
  // compiles to LDS/STS (an integer round trip would leave generic LD/ST)
  Smem<STRATEGY> &s = *reinterpret_cast<Smem<STRATEGY> *>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&s.full[i], 33);   // gather: 32 cp.async arrivals + lane 0 (after the STS), + TMA bytes
      mbar_init(&s.empty[i], 4);   // released by the 4 mask warps
    }
    for (int i = 0; i < GROUPS; ++i) {
      mbar_init(&s.tfull[i], 1);
      mbar_init(&s.tempty[i], 4);
    }
    for (int i = 0; i < NBUF; ++i) {
      mbar_init(&s.mfull[i], 4);
      mbar_init(&s.mempty[i], PAIR ? 2 : 1);  // PAIR: each greedy warp frees its slot
    }
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
  const long long t_start = clock64();

  if (warp == 0) {
    // ---------------- gather: rows, ids, dists, norms of one point --------
    // This CTA's points are i = blockIdx.x + k * gridDim.x; their (u, cnt,
    // off, self) are loaded 32 at a time (lane j: point 32b + j), two
    // batches resident, the next one fetched in two steps (node ids, then
    // their counts / offsets) well before it is needed.  The only values
    // the warp itself waits for are each point's candidate ids (the TMA
    // gather's row coordinates), loaded GD points ahead; dists and norms go
    // global -> shared by cp.async, completed on the stage's full barrier
    // (32 asynchronous arrivals + lane 0's), so no dependent global round
    // trip sits in this loop.  Lane l holds candidates 4l..4l+3 (id -1 past
    // cnt); its gather4 fetches exactly those rows.
    constexpr int GD = 4;
    int stage = 0, half = 0;
    uint32_t phase = 0;
    const int64_t nb = blockIdx.x < n_rows ? (n_rows - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    int64_t bu0 = 0, bu1 = 0, bo0 = 0, bo1 = 0;
    int bc0 = 0, bc1 = 0, bs0 = 0, bs1 = 0;
    auto fetch_u = [&](int64_t b) {  // batch b, step 1: node ids
      const int64_t kk = b * 32 + lane;
      int64_t u = 0;
      if (kk < nb) {
        const int64_t i = blockIdx.x + kk * gridDim.x;
        u = row_order ? row_order[i] : i;
      }
      if (b & 1) bu1 = u; else bu0 = u;
    };
    auto fetch_rest = [&](int64_t b) {  // step 2: counts, offsets, self ids
      const int64_t kk = b * 32 + lane;
      const int64_t u = (b & 1) ? bu1 : bu0;
      int c = 0, sf = 0;
      int64_t o = 0;
      if (kk < nb) {
        c = cand_counts[u];
        o = cand_off[u];
        sf = row_node ? row_node[u] : (int32_t)u;
      }
      if (b & 1) { bc1 = c; bo1 = o; bs1 = sf; } else { bc0 = c; bo0 = o; bs0 = sf; }
    };
    struct PM {
      int64_t u, off;
      int cnt, self;  // cnt -1: past the stream
    };
    auto meta = [&](int64_t j) {
      PM m{0, 0, -1, 0};
      if (j < nb) {
        const bool odd = (j >> 5) & 1;
        const int src = (int)(j & 31);
        m.u = __shfl_sync(0xffffffffu, odd ? bu1 : bu0, src);
        m.off = __shfl_sync(0xffffffffu, odd ? bo1 : bo0, src);
        m.cnt = __shfl_sync(0xffffffffu, odd ? bc1 : bc0, src);
        m.self = __shfl_sync(0xffffffffu, odd ? bs1 : bs0, src);
      }
      return m;
    };
    auto ids_of = [&](const PM &m, int32_t (&o)[4]) {
      const int r = 4 * lane;
      if (m.cnt <= PC && r + 3 < m.cnt && (m.off & 3) == 0) {
        const int4 v = *reinterpret_cast<const int4 *>(cand_ids + m.off + r);
        o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          o[i] = (m.cnt <= PC && r + i < m.cnt) ? cand_ids[m.off + r + i] : -1;
      }
    };
    auto publish_end = [&]() {  // the stage is complete: 32 async + 1 arrivals
      cp_async_mbar_arrive(&s.full[stage]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.full[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    };
    fetch_u(0);
    fetch_rest(0);
    fetch_u(1);
    fetch_rest(1);
    // The id registers of GD points are NOT rotated (a rotation reads the
    // newest load's destination at the top of the next iteration, which
    // stalls the warp on a load issued one iteration earlier): the loop is
    // unrolled GD times over GD named register sets, and a set is reloaded
    // with point k + GD's ids right after point k has used it.
    int32_t ia[4], ib[4], ic[4], id4[4];
    ids_of(meta(0), ia);
    ids_of(meta(1), ib);
    ids_of(meta(2), ic);
    ids_of(meta(3), id4);
    static_assert(GD == 4, "four named id register sets below");
#if GRAM_STATS
    long long gmark_ = clock64(), g_meta = 0, g_tma = 0, g_cpa = 0, g_pub = 0, g_wait = 0;
#endif
    auto point = [&](const int64_t k, int32_t (&i0)[4]) {
      GMARK(g_pub);
      const int64_t b = k >> 5;
      if (b >= 1 && (k & 31) == 0) fetch_u(b + 1);
      if (b >= 1 && (k & 31) == 16) fetch_rest(b + 1);
      const PM m0 = meta(k);
      if (m0.cnt < 0) {
        // a row the fused merge kernel (reverse.cu) has already pruned
      } else if (m0.cnt > PC) {  // hub row (PAIR: > 64): left to the next kernel
        if (lane == 0) long_rows[atomicAdd(long_count, 1)] = (int32_t)m0.u;
      } else {
        GMARK(g_meta);
        if (half == 0) GWAIT(0, mbar_wait(&s.empty[stage], phase ^ 1));
        GMARK(g_wait);
        // candidate rows by TMA gather4 (4 rows of 128 B per instruction,
        // SW128 applied by the map; lane l's rows land at tile row r0 + 4l,
        // i.e. atom (r0 + 4l) / 8).  Rows past cnt keep stale bytes: their
        // Gram entries feed no mask bit that is ever read (t >= cnt is not
        // examinable, i >= cnt > t unused).
        const int r0 = half * 64;
        const int ng = (m0.cnt + 3) >> 2;
        // GRAM_ROWS_CPASYNC: rows [ncp0, cnt) by 16-byte cp.async (instruction m
        // moves 4 rows, 8 lanes per row: lane l takes row 4m + l/8, chunk
        // l%8 at SW128 position chunk ^ (row % 8); ids read back from the
        // stage), rows [0, ncp0) by TMA gather4: the two paths in parallel
        const int ncp0 = GRAM_ROWS_CPASYNC ? GRAM_TMA_ROWS : 4 * ng;
        const int ngt = min(ng, ncp0 >> 2);  // TMA gather4 instructions
        if (lane == 0 && ngt > 0) mbar_expect_tx_only(&s.full[stage], (uint32_t)ngt * 512u);
        if (GRAM_ROWS_CPASYNC && 4 * lane < PC)
          *reinterpret_cast<int4 *>(&s.id[stage][r0 + 4 * lane]) = make_int4(i0[0], i0[1], i0[2], i0[3]);
        __syncwarp();
#if GRAM_TMA_SINGLE
        // one thread issues every gather4 (row ids staged in shared memory:
        // no per-lane ELECT / R2UR serialisation loop)
        if (4 * lane < PC) {
          const int32_t a = i0[0];
          *reinterpret_cast<int4 *>(&s.id[stage][r0 + 4 * lane]) =
              make_int4(a, i0[1] >= 0 ? i0[1] : a, i0[2] >= 0 ? i0[2] : a, i0[3] >= 0 ? i0[3] : a);
        }
        __syncwarp();
        if (lane == 0) {
          const int4 *idv = reinterpret_cast<const int4 *>(&s.id[stage][r0]);
          uint8_t *tb = s.tile[stage] + (r0 >> 3) * 1024;
#pragma unroll 4
          for (int g = 0; g < ngt; ++g) {
            const int4 v = idv[g];
            tma_gather4(tb + (g >> 1) * 1024 + (g & 1) * 512, &tmX, &s.full[stage], 0, v.x, v.y,
                        v.z, v.w);
          }
        }
        __syncwarp();
#elif GRAM_TMA_UNIFORM
        // warp-uniform issue loop: pass g broadcasts lane g's four row ids and
        // lane 0 issues; no per-lane ELECT / branch waterfall, and the passes
        // are independent, so their register -> uniform-register moves overlap
        {
          uint8_t *tb = s.tile[stage] + (r0 >> 3) * 1024;
          uint64_t *fb = &s.full[stage];
#pragma unroll 4
          for (int g = 0; g < ngt; ++g) {
            const int32_t a = __shfl_sync(0xffffffffu, i0[0], g);
            const int32_t b1 = __shfl_sync(0xffffffffu, i0[1], g);
            const int32_t b2 = __shfl_sync(0xffffffffu, i0[2], g);
            const int32_t b3 = __shfl_sync(0xffffffffu, i0[3], g);
            if (lane == 0)
              tma_gather4(tb + (g >> 1) * 1024 + (g & 1) * 512, &tmX, fb, 0, a, b1 >= 0 ? b1 : a,
                          b2 >= 0 ? b2 : a, b3 >= 0 ? b3 : a);
          }
        }
#else
        if (lane < ngt) {
          const int32_t a = i0[0];
          tma_gather4(s.tile[stage] + ((r0 + 4 * lane) >> 3) * 1024 + (lane & 1) * 512, &tmX,
                      &s.full[stage], 0, a, i0[1] >= 0 ? i0[1] : a, i0[2] >= 0 ? i0[2] : a,
                      i0[3] >= 0 ? i0[3] : a);
        }
#endif
        if (GRAM_ROWS_CPASYNC) {
          const int j = lane & 7, rq = lane >> 3;
          for (int m = ngt; m < ng; ++m) {
            const int ra = r0 + 4 * m + rq;  // tile row
            const int32_t id = s.id[stage][ra];
            if (id >= 0)
              cp_async16_zfill(s.tile[stage] + (ra >> 3) * 1024 + (ra & 7) * 128 + ((j ^ (ra & 7)) << 4),
                               xrows + (int64_t)id * 128 + j * 16, 16);
          }
        }
        GMARK(g_tma);
        if (4 * lane < PC) {
          const int rb = r0 + 4 * lane;
          *reinterpret_cast<int4 *>(&s.id[stage][rb]) = make_int4(i0[0], i0[1], i0[2], i0[3]);
          // dists: asynchronous copies (id -1 past cnt: zeros); the norms
          // are computed by the mask warps from the gathered rows
#if GRAM_NORMS_GATHER
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (i0[i] >= 0) cp_async4(&s.nrm[stage][rb + i], norms + i0[i]);
            else s.nrm[stage][rb + i] = 0;
          }
#endif
          const float *dsrc = cand_dists + m0.off + 4 * lane;
          if (i0[3] >= 0 && ((uintptr_t)dsrc & 15) == 0) {
            cp_async16_zfill(&s.dist[stage][rb], dsrc, 16);
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              if (i0[i] >= 0) cp_async4(&s.dist[stage][rb + i], dsrc + i);
              else s.dist[stage][rb + i] = 0.f;
            }
          }
        }
        if (lane == 0) {
          s.u[stage][half] = m0.u;
          s.cnt[stage][half] = m0.cnt;
          s.self[stage][half] = m0.self;
        }
        GMARK(g_cpa);
        if (PAIR && half == 0) {
          half = 1;  // the next point fills the other half of this stage
        } else {
          publish_end();
          half = 0;
        }
      }
      ids_of(meta(k + GD), i0);  // this set's next point
    };
    for (int64_t k = 0; k < nb; k += GD) {
      point(k, ia);
      if (k + 1 < nb) point(k + 1, ib);
      if (k + 2 < nb) point(k + 2, ic);
      if (k + 3 < nb) point(k + 3, id4);
    }
    if (PAIR && half == 1) {  // a half-filled last stage: the second slot is empty
      if (lane == 0) {
        s.u[stage][1] = -1;
        s.cnt[stage][1] = 0;
      }
      if (4 * lane < PC) {
        *reinterpret_cast<int4 *>(&s.id[stage][64 + 4 * lane]) = make_int4(-1, -1, -1, -1);
        *reinterpret_cast<float4 *>(&s.dist[stage][64 + 4 * lane]) = make_float4(0.f, 0.f, 0.f, 0.f);
        *reinterpret_cast<int4 *>(&s.nrm[stage][64 + 4 * lane]) = make_int4(0, 0, 0, 0);
      }
      publish_end();
    }
#if GRAM_STATS
    if (lane == 0) {
      atomicAdd(&g_gram_stats[11], (unsigned long long)g_meta);
      atomicAdd(&g_gram_stats[12], (unsigned long long)g_tma);
      atomicAdd(&g_gram_stats[13], (unsigned long long)g_cpa);
      atomicAdd(&g_gram_stats[14], (unsigned long long)g_pub);
      atomicAdd(&g_gram_stats[15], (unsigned long long)g_wait);
    }
#endif
    // end of stream: one sentinel per mask group (each reads every other point)
    for (int g = 0; g < GROUPS; ++g) {
      GWAIT(0, mbar_wait(&s.empty[stage], phase ^ 1));
      if (lane == 0) s.cnt[stage][0] = g == 0 ? -1 : -2;
      publish_end();
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA: G = C C^T per gathered point ----------------
      int stage = 0, acc = 0;
      uint32_t phase = 0, tphase = 0;
      for (;;) {
        GWAIT(1, GRAM_IDLE_WAIT(&s.full[stage], phase));
        if (s.cnt[stage][0] < 0) break;
        fence_proxy_async_smem();  // generic-proxy smem writes -> tensor-core reads
        GWAIT(2, mbar_wait(&s.tempty[acc], tphase ^ 1));
        tc_fence_after();
        const uint64_t desc = sw128_desc(s.tile[stage]);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_i8(tmem + acc * C, desc + 2 * kk, desc + 2 * kk, IDESC, kk > 0);
        tc_commit(&s.tfull[acc]);
        if (++acc == GROUPS) { acc = 0; tphase ^= 1; }
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp < GREEDY_WARP) {
    // ---------------- masks: thread t = candidate t = TMEM lane t ----------
    // Candidate t reads its Gram row G[t][i] (i < t: the lower triangle, so
    // warp quarter q reads chunks 0..q only) and builds two 128-bit masks:
    //   pm: c_i dominates c_t if c_i is kept (_kernels.py:385-397)
    //   am: the reference's test of c_t against kept c_i evaluates the angle
    const int q = warp & 3;               // TMEM lane quarter of this warp
    const int grp = (warp - 2) >> 2;      // mask group: points k = grp (mod GROUPS)
    const int t = q * 32 + lane;          // candidate index
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16) + grp * C;
    uint32_t tphase = 0;
    for (int64_t k = grp;; k += GROUPS) {
      const int stage = (int)(k % STAGES);
      const uint32_t phase = (uint32_t)((k / STAGES) & 1);
      const int mb = (int)(k % NBUF);  // greedy buffer of point k
      const uint32_t mphase = (uint32_t)((k / NBUF) & 1);
      GWAIT(3, GRAM_IDLE_WAIT(&s.full[stage], phase));
      const int cnt0 = s.cnt[stage][0];
      if (cnt0 < 0) {  // end of stream: the first group to see it tells every greedy warp
        // (PAIR: both greedy warps read every buffer, one sentinel serves both)
        for (int64_t kk = k; cnt0 == -1 && kk < k + (PAIR ? 1 : NG); ++kk) {
          const int b = (int)(kk % NBUF);
          GWAIT(5, mbar_wait(&s.mempty[b], ((uint32_t)((kk / NBUF) & 1)) ^ 1));
          if (t == 0) s.gcnt[b][0] = -1;
          __syncwarp();
          if (lane == 0) mbar_arrive(&s.mfull[b]);
        }
        break;
      }
      const int P = PAIR ? (q >> 1) : 0;  // this warp's point slot
      const int ql = PAIR ? (q & 1) : q;  // its quarter within the point
      const int cb = PAIR ? 2 * P : 0;    // the point's first column chunk
      const int cnt = s.cnt[stage][P];
      const int32_t self = s.self[stage][P];
      const int32_t *sid = s.id[stage];
      const float *sdist = s.dist[stage];
      int32_t *snrm = s.nrm[stage];
      const float dv = sdist[t];
      // |c_t|^2 from the gathered row itself (SW128: 16-byte chunk j of tile
      // row t sits at atom t/8, row t%8, position j ^ (t%8)), published for
      // the other mask warps: no norm gather in the gather warp's loop.
      // Rows past cnt hold stale bytes; their norms feed no mask bit read.
#if GRAM_NORMS_GATHER
      const int nv = snrm[t];
#else
      unsigned nvu = 0;
      {
        const uint8_t *rowp = s.tile[stage] + (t >> 3) * 1024 + (t & 7) * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint4 w = *reinterpret_cast<const uint4 *>(rowp + ((j ^ (t & 7)) << 4));
          nvu = __dp4a(w.x, w.x, nvu);
          nvu = __dp4a(w.y, w.y, nvu);
          nvu = __dp4a(w.z, w.z, nvu);
          nvu = __dp4a(w.w, w.w, nvu);
        }
        snrm[t] = (int)nvu;
        if (GROUPS == 1) asm volatile("bar.sync 1, 128;" ::: "memory");
        else named_bar_sync(1 + grp, 128);
      }
      const int nv = (int)nvu;
#endif
      // c_i dominates c_t (rng) iff duw == 0 or dwv == 0 or dwv < dv, with
      // dwv = |c_i|^2 + |c_t|^2 - 2 G[t][i] an exact integer >= 0:
      //   dwv < dv  <=>  dwv <= ceil(dv) - 1;  dwv == 0  <=>  dwv <= 0
      // so with x = |c_i|^2 - 2 G[t][i]:  x <= max(ceil(dv) - 1, 0) - |c_t|^2
      // rng: dwv < dv; "slack" extension: s^2 * dwv < dv (s^2 = cos_alpha >= 1):
      // the largest integer x with p * x < dv, in the same float64 arithmetic
      int dle;
      if (dv >= 2.0e9f) {
        dle = 0x7fffffff;
      } else if (strategy != 2) {  // rng: the largest integer below dv, exactly
        const float fl = floorf(dv);
        const int x = (int)fl - (fl == dv ? 1 : 0);
        dle = x > 0 ? x : 0;
      } else {
        const double p = cos_alpha;
        int64_t x = (int64_t)floor((double)dv / p);
        while (x >= 0 && !(p * (double)x < (double)dv)) --x;
        while (p * (double)(x + 1) < (double)dv) ++x;
        dle = (int)(x > 0 ? x : 0);
      }
      const int thr = dle == 0x7fffffff ? 0x7fffffff : dle - nv;
      uint32_t pm[4] = {0, 0, 0, 0}, am[4] = {0, 0, 0, 0};
      GWAIT(4, mbar_wait(&s.tfull[grp], tphase));
      tc_fence_after();
      // lower-triangle chunks holding candidates; none when this warp's
      // candidates are all past cnt (their masks are never read)
      const int clast = ql * 32 >= cnt ? -1 : min(ql, (cnt - 1) >> 5);
#pragma unroll 1
      for (int c = 0; c <= clast; ++c) {
        const int gc = cb + c;  // column chunk of the tile
        uint32_t g[32];
        tmem_ld32(tl + (uint32_t)(gc * 32), g);
        const uint32_t zu = __ballot_sync(0xffffffffu, sdist[gc * 32 + lane] == 0.0f);
        const uint32_t valid = c < ql ? 0xffffffffu : ((1u << lane) - 1u);
        tmem_wait_ld();
        uint32_t dm = 0, need = 0;
        if (STRATEGY == 0) {
          const int4 *np = reinterpret_cast<const int4 *>(snrm + gc * 32);
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            const int4 w = np[v];
            dm |= (w.x - 2 * (int)g[4 * v] <= thr) ? (1u << (4 * v)) : 0u;
            dm |= (w.y - 2 * (int)g[4 * v + 1] <= thr) ? (1u << (4 * v + 1)) : 0u;
            dm |= (w.z - 2 * (int)g[4 * v + 2] <= thr) ? (1u << (4 * v + 2)) : 0u;
            dm |= (w.w - 2 * (int)g[4 * v + 3] <= thr) ? (1u << (4 * v + 3)) : 0u;
          }
          dm = (dm | zu) & valid;
        } else {
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const int ci = gc * 32 + k;
            const float duw = sdist[ci];
            const float dwv = (float)(snrm[ci] + nv - 2 * (int)g[k]);  // == squared_l2
            const bool z = (duw == 0.0f) | (dwv == 0.0f);
            const bool lt = dwv < dv;
            dm |= z ? (1u << k) : 0u;
            const bool ang = ((valid >> k) & 1u) & !z & lt;
            need |= ang ? (1u << k) : 0u;
            if (ang && cos_angle_from_sq(duw, dwv, dv) < cos_alpha) dm |= 1u << k;
          }
          dm &= valid;
        }
        am[c] = need;
        pm[c] = dm;
      }
      // TMEM is free for the next point's MMA
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.tempty[grp]);
      GWAIT(5, mbar_wait(&s.mempty[mb], mphase ^ 1));  // the greedy warp is done with buffer mb
      *reinterpret_cast<uint4 *>(s.pm[mb][t]) = make_uint4(pm[0], pm[1], pm[2], pm[3]);
      if (STRATEGY == 1)
        *reinterpret_cast<uint4 *>(s.am[mb][t]) = make_uint4(am[0], am[1], am[2], am[3]);
      const unsigned exm = __ballot_sync(0xffffffffu, ql * 32 + lane < cnt && sid[t] != self);
      if (lane == 0) s.ex[mb][q] = exm;
      s.gid[mb][t] = sid[t];
      s.gdist[mb][t] = dv;
      if (ql == 0 && lane == 0) {
        s.gu[mb][P] = s.u[stage][P];
        s.gcnt[mb][P] = cnt;
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&s.mfull[mb]);
        mbar_arrive(&s.empty[stage]);
      }
      tphase ^= 1;
    }
  } else {
    // ---------------- greedy scan + exact lazy counters (NG warps) ---------
    const int gw = warp - GREEDY_WARP;
    const int P = PAIR ? gw : 0;        // PAIR: greedy warp w takes slot w of every buffer
    const int base = P * PC;            // the slot's first tile row
    for (int64_t k = PAIR ? 0 : gw;; k += PAIR ? 1 : NG) {
      const int mb = (int)(k % NBUF);
      GWAIT(6, GRAM_IDLE_WAIT(&s.mfull[mb], (uint32_t)((k / NBUF) & 1)));
      if (s.gcnt[mb][0] < 0) break;
      const int64_t u = s.gu[mb][P];
      if (PAIR && u < 0) {  // empty slot (odd point count)
        __syncwarp();
        if (lane == 0) mbar_arrive(&s.mempty[mb]);
        continue;
      }
      const int32_t *sid = s.gid[mb];
      const float *sdist = s.gdist[mb];
      const uint32_t(*spm)[4] = s.pm[mb];
      const uint32_t(*sam)[4] = s.am[STRATEGY == 1 ? mb : 0];
      const uint32_t *sex = s.ex[mb];
      // everything this lane needs, loaded at once (one shared-memory latency)
      uint4 pjv[4];
      uint32_t exv[4];
      int32_t idv[4];
      float dsv[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (c * 32 < PC) {
          pjv[c] = *reinterpret_cast<const uint4 *>(spm[base + c * 32 + lane]);
          exv[c] = sex[(PAIR ? 2 * P : 0) + c];
          idv[c] = sid[base + c * 32 + lane];
          dsv[c] = sdist[base + c * 32 + lane];
        } else {  // PAIR: chunks 2, 3 are the other slot's
          pjv[c] = make_uint4(0, 0, 0, 0);
          exv[c] = 0;
          idv[c] = -1;
          dsv[c] = 0.0f;
        }
      }
      uint32_t zu[4];  // candidates with duw == 0 (no distance computed against them)
#pragma unroll
      for (int c = 0; c < 4; ++c) zu[c] = __ballot_sync(0xffffffffu, dsv[c] == 0.0f);
      uint32_t kept_m[4] = {0, 0, 0, 0};  // warp-uniform
      int kept = 0, stop_j = C;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (stop_j != C) break;
        const uint4 pj = pjv[c];
        const bool blocked = (pj.x & kept_m[0]) | (pj.y & kept_m[1]) | (pj.z & kept_m[2]) |
                             (pj.w & kept_m[3]);
        const uint32_t pjc = c == 0 ? pj.x : c == 1 ? pj.y : c == 2 ? pj.z : pj.w;
        unsigned m = exv[c] & __ballot_sync(0xffffffffu, !blocked);
        uint32_t km = 0;
        while (m) {
          const int li = __ffs(m) - 1;  // next kept candidate, index c*32+li
          km |= 1u << li;
          if (++kept == M) {  // _kernels.py:378: nothing after it is examined
            stop_j = c * 32 + li;
            break;
          }
          // later lanes of this chunk dominated by c_li
          const unsigned dom = __ballot_sync(0xffffffffu, (pjc >> li) & 1u);
          m &= ~(dom | ((2u << li) - 1u));
        }
        kept_m[c] = km;
      }
      // the kept candidates in scan order, staged in this point's (already
      // register-resident) candidate buffer, then written as whole padded
      // rows: one fully coalesced store sequence per row (whole 128-byte
      // lines also when the output is pinned host memory)
      {
        int32_t *oid = s.gid[mb] + base;
        float *od = s.gdist[mb] + base;
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
          const bool k = j < kept;
          out_ids[u * width + j] = k ? oid[j] : -1;
          out_dists[u * width + j] = k ? od[j] : __int_as_float(0x7f800000);
        }
      }
      // ---- exact lazy counters of every examined candidate ----
      const int kp1 = __popc(kept_m[0]), kp2 = kp1 + __popc(kept_m[1]),
                kp3 = kp2 + __popc(kept_m[2]);
      long long dsum = 0, asum = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int j = c * 32 + lane;
        if (j > stop_j || !((exv[c] >> lane) & 1u)) continue;
        const uint32_t pw[4] = {pjv[c].x, pjv[c].y, pjv[c].z, pjv[c].w};
        // the first kept candidate before j that dominates it
        int f = -1;
#pragma unroll
        for (int w = 0; w <= c; ++w) {
          const uint32_t d = pw[w] & kept_m[w] & (w < c ? 0xffffffffu : lanemask_lt());
          if (f < 0 && d) f = w * 32 + __ffs(d) - 1;
        }
        // kept candidates c_j was tested against: every kept one before the
        // first dominator (or before j), plus the dominator itself unless its
        // duw == 0 short-cut needed no distance
        const int end = f >= 0 ? f : j;
        const int ew = end >> 5;
        const uint32_t kw = ew == 0 ? kept_m[0] : ew == 1 ? kept_m[1] : ew == 2 ? kept_m[2] : kept_m[3];
        int ev = (ew == 0 ? 0 : ew == 1 ? kp1 : ew == 2 ? kp2 : kp3) +
                 __popc(kw & ((1u << (end & 31)) - 1u));
        if (f >= 0 && !((zu[f >> 5] >> (f & 31)) & 1u)) ev += 1;
        dsum += ev;
        if (STRATEGY == 1) {
          const uint4 aj = *reinterpret_cast<const uint4 *>(sam[base + j]);
          const uint32_t aw[4] = {aj.x, aj.y, aj.z, aj.w};
          int an = 0;
#pragma unroll
          for (int w = 0; w < 4; ++w) {
            uint32_t lim = end >= (w + 1) * 32 ? 0xffffffffu
                                               : (end <= w * 32 ? 0u : ((1u << (end - w * 32)) - 1u));
            if (f >= 0 && (f >> 5) == w) lim |= 1u << (f & 31);
            an += __popc(aw[w] & kept_m[w] & lim);
          }
          asum += an;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
        if (STRATEGY == 1) asum += __shfl_xor_sync(0xffffffffu, asum, o);
      }
      if (lane == 0) {
        dist_evals[u] = dsum;
        angle_evals[u] = asum;
        out_counts[u] = kept;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&s.mempty[mb]);
    }
  }
#if GRAM_STATS
  if (lane == 0 && (warp <= 2 || warp == GREEDY_WARP))
    atomicAdd(&g_gram_stats[7 + (warp == GREEDY_WARP ? 3 : warp)],
              (unsigned long long)(clock64() - t_start));
#endif
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

bool make_u8_row_map(CUtensorMap *tm, const uint8_t *base, int64_t rows, int box_rows);

size_t gram_workspace(int64_t n) { return (size_t)(2 * n + 128) * sizeof(int32_t); }

// Default selection path for exact-integer rows (PGK_GRAM=0 selects the
// per-warp prune_u8_kernel instead, e.g. for A/B timing).
bool gram_enabled() {
  static int env = -1;
  if (env < 0) {
    const char *e = getenv("PGK_GRAM");
    env = (e && e[0] == '0') ? 0 : 1;
  }
  return env == 1;
}

// Phase-A / re-prune selection through the tensor-core Gram kernel; rows with
// more than 128 candidates go to prune_u8_kernel.  ws: gram_workspace(n) bytes.
// pair: rows of <= 64 candidates two per MMA first (the phase-B re-prune),
// the longer ones listed on the device for the single-point kernel.
template <int STRATEGY, bool PAIR>
static int launch_gram_kernel(const CUtensorMap &tmX, const uint8_t *xu8, const int32_t *norms,
                              int64_t n,
                              const int32_t *n_dev, const int32_t *row_node,
                              const int32_t *row_order, const int64_t *cand_off,
                              const int32_t *cand_counts, const int32_t *cand_ids,
                              const float *cand_dists, int strategy, double cos_alpha, int64_t M,
                              int64_t width, int32_t *out_ids, float *out_dists,
                              int32_t *out_counts, int64_t *dist_evals, int64_t *angle_evals,
                              int32_t *long_rows, int32_t *long_count, cudaStream_t stream) {
  const size_t smem = sizeof(gram::Smem<STRATEGY>) + 1024;
  PGK_CUDA(ensure_smem((const void *)gram::prune_gram_kernel<STRATEGY, PAIR>, smem));
  const unsigned grid = (unsigned)std::min<int64_t>(n, (int64_t)gram::CTAS_PER_SM * num_sms());
  gram::prune_gram_kernel<STRATEGY, PAIR><<<grid, gram::THREADS, smem, stream>>>(
      tmX, xu8, norms, n, row_node, row_order, cand_off, cand_counts, cand_ids, cand_dists, strategy,
      cos_alpha, (int)M, (int)width, out_ids, out_dists, out_counts, dist_evals, angle_evals,
      long_rows, long_count, n_dev);
  PGK_CHECK_LAUNCH("prune_gram_kernel");
  return PGK_OK;
}

int launch_prune_gram(const uint8_t *xu8, const int32_t *norms, int64_t n,
                      const int32_t *row_node, const int32_t *row_order,
                      const int64_t *cand_off, const int32_t *cand_counts,
                      const int32_t *cand_ids, const float *cand_dists, int strategy,
                      double cos_alpha, int64_t M, int64_t width, int32_t *out_ids,
                      float *out_dists, int32_t *out_counts, int64_t *dist_evals,
                      int64_t *angle_evals, void *ws, cudaStream_t stream, bool pair) {
  if (n == 0) return PGK_OK;
  int32_t *long_count = reinterpret_cast<int32_t *>(ws);  // rows past the single kernel
  int32_t *pair_count = long_count + 1;                   // rows past the pair kernel
  int32_t *long_rows = long_count + 32;
  int32_t *pair_rows = long_rows + n + 32;
  PGK_CUDA(cudaMemsetAsync(long_count, 0, 2 * sizeof(int32_t), stream));
  // candidate ids index data rows (< 2^31 by the ABI); the gather map needs
  // no tighter row bound
  CUtensorMap tmX;
  if (!make_u8_row_map(&tmX, xu8, 0x7fffffff, 1)) {
    set_error("cuTensorMapEncodeTiled failed (gather4 map)");
    return PGK_ERR_CUDA;
  }
  const bool rng = strategy == 0 || strategy == 2;  // slack: the rng masks, another threshold
  const int sa = rng ? strategy : 1;
  int rc;
  if (pair) {
    rc = rng ? launch_gram_kernel<0, true>(tmX, xu8, norms, n, nullptr, row_node, row_order, cand_off,
                                           cand_counts, cand_ids, cand_dists, sa, cos_alpha, M,
                                           width, out_ids, out_dists, out_counts, dist_evals,
                                           angle_evals, pair_rows, pair_count, stream)
             : launch_gram_kernel<1, true>(tmX, xu8, norms, n, nullptr, row_node, row_order, cand_off,
                                           cand_counts, cand_ids, cand_dists, sa, cos_alpha, M,
                                           width, out_ids, out_dists, out_counts, dist_evals,
                                           angle_evals, pair_rows, pair_count, stream);
    if (rc) return rc;
  }
  // single-point kernel: every row, or (pair) the rows listed above
  const int32_t *order1 = pair ? pair_rows : row_order;
  const int32_t *n1_dev = pair ? pair_count : nullptr;
  rc = rng ? launch_gram_kernel<0, false>(tmX, xu8, norms, n, n1_dev, row_node, order1, cand_off,
                                          cand_counts, cand_ids, cand_dists, sa, cos_alpha, M,
                                          width, out_ids, out_dists, out_counts, dist_evals,
                                          angle_evals, long_rows, long_count, stream)
           : launch_gram_kernel<1, false>(tmX, xu8, norms, n, n1_dev, row_node, order1, cand_off,
                                          cand_counts, cand_ids, cand_dists, sa, cos_alpha, M,
                                          width, out_ids, out_dists, out_counts, dist_evals,
                                          angle_evals, long_rows, long_count, stream);
  if (rc) return rc;
  const unsigned grid = (unsigned)std::min<int64_t>(n, (int64_t)gram::CTAS_PER_SM * num_sms());
  (void)grid;
#if GRAM_STATS
  {
    unsigned long long h[16];
    PGK_CUDA(cudaStreamSynchronize(stream));
    PGK_CUDA(cudaMemcpyFromSymbol(h, gram::g_gram_stats, sizeof(h)));
    const double ctas = (double)grid;
    fprintf(stderr,
            "[gram stats] per CTA, Mcycles: total gather %.2f mma %.2f mask(w2) %.2f greedy %.2f | "
            "waits: gather-empty %.2f mma-full %.2f mma-tempty %.2f mask-full %.2f mask-tfull "
            "%.2f mask-mempty %.2f (per mask warp) greedy-mfull %.2f\n",
            h[7] / ctas / 1e6, h[8] / ctas / 1e6, h[9] / ctas / 1e6, h[10] / ctas / 1e6,
            h[0] / ctas / 1e6, h[1] / ctas / 1e6, h[2] / ctas / 1e6, h[3] / ctas / 4e6,
            h[4] / ctas / 4e6, h[5] / ctas / 4e6, h[6] / ctas / 1e6);
    fprintf(stderr, "[gram stats] gather loop per CTA, Mcycles: meta+ids %.2f empty-wait %.2f tma-issue %.2f "
            "cp.async+sts %.2f publish %.2f\n", h[11] / ctas / 1e6, h[15] / ctas / 1e6,
            h[12] / ctas / 1e6, h[13] / ctas / 1e6, h[14] / ctas / 1e6);
    unsigned long long z[16] = {0};
    PGK_CUDA(cudaMemcpyToSymbol(gram::g_gram_stats, z, sizeof(z)));
  }
#endif
  // hub rows (> 128 candidates): the per-warp exact-integer kernel, over the
  // device-side list (its length is read on the device)
  return launch_prune_u8_rows(xu8, norms, n, long_count, row_node, long_rows, cand_off,
                              cand_counts, cand_ids, cand_dists, strategy, cos_alpha, M, width,
                              out_ids, out_dists, out_counts, dist_evals, angle_evals, stream);
}

}  // namespace pgk
