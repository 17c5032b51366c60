// pool_tc.cu -- exact k-NN pools on the 5th-gen tensor cores (tcgen05,
// kind::i8) for integer-valued data in [0, 255] with d <= 128 (config 2).
//
// Why it is exact: with u8 operands and s32 accumulation every dot product is
// an exact integer, so dist = |q|^2 + |x|^2 - 2 q.x is the exact squared
// distance -- equal to the reference's float64 ranking value
// (oracle.py:52-58) and to its fp32 sequential squared_l2 (_kernels.py:17-24;
// all partial sums are integers < 2^24).  Top-K by packed (dist, id) key is
// therefore the reference's (dist, id) order, no rerank needed.
//
// Kernel shape (persistent, TC_CTAS = 2 CTAs / SM, 192 threads):
//   warp 0      TMA producer + dynamic block scheduler: the block's 128 query
//               rows (A, once per block) and a 2-stage ring of 128-point data
//               tiles (B), 128 B/row, SW128
//   warp 1      TMEM allocator + MMA issuer: D[128 x 128] (s32) = A . B^T,
//               4 x K=32 tcgen05.mma per 64-column part; TC_ACC = 2
//               accumulators by tile parity, so the epilogue warps may drift
//               a whole tile apart; bulk-loads each tile's |x|^2 and ids one
//               tile ahead (NYBUF ring)
//   warps 2..5  epilogue: warp q reads TMEM lanes 32q..32q+31, i.e. thread =
//               query row; per 32 columns one IADD + one compare per value
//               against the row's threshold (fast reject); survivors appended
//               to a per-row candidate buffer in global memory; the
//               massively parallel finalize kernel selects and sorts.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tc_ptx.cuh"
#include "tc_select.cuh"

namespace pgk {
namespace tc {

constexpr int BM = 128;   // query rows per block == TMEM lanes
constexpr int BN = 128;   // data points per tile == MMA N
constexpr int KB = 128;   // bytes per (padded) row
constexpr int STAGES = 2;       // B-tile ring depth
#ifndef TC_ACC
#define TC_ACC 2
#endif

constexpr int ACC = TC_ACC;     // TMEM accumulator stages (128 columns each, by tile)
#ifndef TC_PARTS
#define TC_PARTS 2
#endif
constexpr int HALVES = TC_PARTS;  // each accumulator is filled / drained in column parts
constexpr int HN = BN / HALVES;
constexpr int CPP = HN / 32;      // 32-column epilogue chunks per part
#ifndef TC_CTAS
#define TC_CTAS 2
#endif
constexpr int CTAS_PER_SM = TC_CTAS;  // co-resident CTAs share the tensor core
constexpr int TILE_BYTES = BN * KB;
constexpr int NYBUF = ACC + 2;  // the MMA runs up to ACC tiles ahead of the epilogue
#ifndef TC_CAP
#define TC_CAP 512  // same pass-2 / finalize times as 1,024 at config 2, half the buffers
#endif
constexpr int CAP = TC_CAP;  // per-row candidate buffer (keys, global memory)
constexpr int THREADS = 192;  // warp 0 TMA, warp 1 TMEM alloc + MMA, warps 2-5 epilogue
constexpr int TMEM_COLS = ACC * BN;
constexpr int GUESSED = 1 << 30;  // row_cnt flag: the row ran under a guessed threshold

struct __align__(1024) Smem {
  uint8_t a[BM * KB];
  uint8_t b[STAGES][TILE_BYTES];
#ifndef TC_APPEND_UNROLL
#define TC_APPEND_UNROLL 2
#endif
#ifndef TC_PAIR_APPEND
#define TC_PAIR_APPEND 1  // survivors of a 64-column part appended in one loop (K > 1 pass 2):
                          // 3.51 -> 3.22 ms at config 2; 0 = one loop per 32-column chunk
#endif
  // per epilogue warp: one chunk (TC_PAIR_APPEND: one part = two chunks) of dot
  // products per lane
  int32_t sv[4][32 * (TC_PAIR_APPEND ? 68 : 36)];  // lane stride = 4 (mod 32) words: conflict-free STS.128
  // |x|^2 and original ids (pruned path) of the tile's columns, 3 buffers by
  // running tile count: the MMA warp prefetches tile g+1's while the
  // epilogue may still read tile g-1's
  alignas(16) int32_t ny[NYBUF][BN];
  alignas(16) int32_t pid[NYBUF][BN];
  uint64_t nfull[NYBUF];
  uint64_t full[STAGES], empty[STAGES];
  uint64_t tfull[ACC][HALVES], tempty[ACC][HALVES];  // per accumulator slot and part
  uint64_t a_full, a_empty;
  uint32_t tmem_base;
  int32_t blk[2];  // dynamic schedule: block index per A-tile phase (-1 = done)
};

// kind::i8 instruction descriptor: D s32, A/B u8, K-major, M=128, N=BN
// half-width (N = 64) MMAs: half h of a tile lands in TMEM columns h*64..h*64+63,
// so the MMA of the next tile's first half overlaps the epilogue's second half
constexpr uint32_t IDESC_H =
    (2u << 4) | ((uint32_t)(HN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

// Register bitonic sort of 32*NPL keys (element i = slot*32 + lane).
template <int NPL>
__device__ __forceinline__ void reg_bitonic(uint64_t (&e)[NPL], int lane) {
  constexpr int SIZE = 32 * NPL;
#pragma unroll
  for (int k = 2; k <= SIZE; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
        const int js = j >> 5;
#pragma unroll
        for (int s0 = 0; s0 < NPL; ++s0) {
          if (s0 & js) continue;
          const int s1 = s0 ^ js;
          const bool up = (((s0 << 5) | lane) & k) == 0;
          const uint64_t a = e[s0], b = e[s1];
          const bool sw = (a > b) == up;
          e[s0] = sw ? b : a;
          e[s1] = sw ? a : b;
        }
      } else {
        const bool lower = (lane & j) == 0;
#pragma unroll
        for (int s0 = 0; s0 < NPL; ++s0) {
          const uint64_t o = __shfl_xor_sync(0xffffffffu, e[s0], j);
          const bool up = (((s0 << 5) | lane) & k) == 0;
          const uint64_t mn = e[s0] < o ? e[s0] : o, mx = e[s0] < o ? o : e[s0];
          e[s0] = (lower == up) ? mn : mx;
        }
      }
    }
  }
}

// Final per-row output: best K keys, ascending, in the library's packed
// (float dist, id) key format.
template <int NPL>
__device__ __forceinline__ void emit_sorted(const uint64_t *buf, int cnt, int K,
                                            uint64_t *out, int lane) {
  uint64_t e[NPL];
#pragma unroll
  for (int s0 = 0; s0 < NPL; ++s0) {
    const int idx = s0 * 32 + lane;
    e[s0] = idx < cnt && idx < K ? buf[idx] : KEY_MAX;
  }
  reg_bitonic<NPL>(e, lane);
#pragma unroll
  for (int s0 = 0; s0 < NPL; ++s0) {
    const int idx = s0 * 32 + lane;
    if (idx < K)
      out[idx] = e[s0] == KEY_MAX ? KEY_MAX : pack_key((float)khi(e[s0]), (int32_t)(uint32_t)e[s0]);
  }
}

__device__ __forceinline__ int tau_prefilter(uint64_t tau, int nx) {
  if (tau == KEY_MAX) return 0x7fffffff;
  return (int)khi(tau) - nx;
}

// s-value prefilter bound of a row: K == 1 keeps dist <= khi(tau) (then the
// exact key compare), K > 1 keeps dist < khi(tau) (tau = T << 32, exact).
__device__ __forceinline__ int row_tp(uint64_t tau, int nx, int K) {
  if (tau == KEY_MAX) return 0x7fffffff;
  return (int)khi(tau) - nx - (K > 1 ? 1 : 0);
}

// Optional epilogue instrumentation (PGK_TC_STATS=1): cycles / event counts.
enum { ST_WAIT, ST_MAIN, ST_SLOW, ST_COMPACT, ST_FINAL, ST_NSLOW, ST_NCOMPACT, ST_NAPPEND,
       ST_COUNT };

// DENSE (pass-1 bound mode): no threshold, no survivor lists -- every row
// stores every column's distance, densely, as u16 ceil(dist / 2^DENSE_Q)
// (exact u8 distances are < 2^23; the top value = invalid), at most
// DENSE_TILES tiles per row in the row's CAP x 8-byte slot, for
// tc_kth_dense_kernel.  2^DENSE_Q x the K-th smallest stored value bounds the
// K-th smallest distance from above (within 2^DENSE_Q of it): half the bytes
// of u32.
constexpr int DENSE_TILES = 16;  // u16 values: 16 tiles x 128 x 2 B = 4 KB of the row's slot
static_assert(DENSE_TILES * BN * 2 <= CAP * 8, "dense pass-1 values must fit the row's buffer");
#ifndef TC_DENSE_NOVALID
#define TC_DENSE_NOVALID 0  // 1: no per-value validity tests in the dense pass-1 epilogue
#endif
#ifndef TC_DENSE_PACKED
#define TC_DENSE_PACKED 1  // 15-bit values (dist / 2^8), counted two per instruction in the K-th search
#endif
#if TC_DENSE_PACKED
// values < 2^15 (u8 distances < 2^23; 0x7fff = invalid): two per 32-bit word,
// and (mid + 0x8000 - v) has bit 15 set iff v <= mid with no borrow between
// the halves, so one subtraction compares both
constexpr int DENSE_Q = 8;  // quantisation: dist / 2^8, rounded up
constexpr uint32_t DENSE_INVALID = 0x7fffu, DENSE_VMAX = 0x7ffeu;
#else
constexpr int DENSE_Q = 7;  // quantisation: dist / 2^7, rounded up
constexpr uint32_t DENSE_INVALID = 0xffffu, DENSE_VMAX = 0xfffeu;
#endif

__device__ __forceinline__ uint32_t dense_val(int dist, int64_t col, int64_t n, int32_t pid,
                                              bool self) {
  return (col < n && pid >= 0 && !self)
             ? min(((uint32_t)dist + ((1u << DENSE_Q) - 1u)) >> DENSE_Q, DENSE_VMAX)
             : DENSE_INVALID;
}

// K1: the K = 1 (nearest neighbour) instantiation; the K > 1 one carries no
// K = 1 code (registers and scheduling of the pass-2 epilogue).
template <bool STATS, bool DENSE, bool K1 = false>
// 112 registers keeps CTAS_PER_SM = 3 resident (3 x 6 warps x 112 x 32 <= 64K)
__global__ void __maxnreg__(TC_CTAS == 3 ? 112 : 168)
    tc_pool_u8_kernel(const __grid_constant__ CUtensorMap tmX,
                      const __grid_constant__ CUtensorMap tmQ, int64_t n, int64_t nq,
                      int exclude_self, const int32_t *__restrict__ xnorm,
                      const int32_t *__restrict__ qnorm, int K, uint64_t *__restrict__ bufs,
                      uint64_t *__restrict__ out_keys, unsigned long long *stats,
                      const int32_t *__restrict__ tlist, const int32_t *__restrict__ tlen,
                      int64_t tstride, const int32_t *__restrict__ perm,
                      const uint64_t *__restrict__ init_keys, float shrink,
                      int32_t *__restrict__ row_cnt, uint64_t *__restrict__ row_tau,
                      int32_t *__restrict__ sched, const uint8_t *__restrict__ row_mask,
                      int k1_direct, const int32_t *__restrict__ gate, int gate_min) {
  // a device-side switch: run only when *gate >= gate_min (the re-run of
  // failing rows on the tensor cores, taken when they are too many for the
  // SIMT rescan)
  if (gate && *gate < gate_min) return;
  // K == 1 paths: compiled in for the K1 instantiation (and the STATS one)
  const bool isk1 = K1 ? true : (STATS ? K == 1 : false);
  unsigned long long st[ST_COUNT] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long t_prev = STATS ? clock64() : 0;
#define PGK_TICK(slot)                          \
  do {                                          \
    if (STATS) {                                \
      long long t_ = clock64();                 \
      st[slot] += (unsigned long long)(t_ - t_prev); \
      t_prev = t_;                              \
    }                                           \
  } while (0)
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned view, derived from the shared array itself so every access
  // compiles to LDS/STS (an integer round trip would leave generic LD/ST)
  Smem &s = *reinterpret_cast<Smem *>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nblocks = (int)((nq + BM - 1) / BM);
  const int ntiles = (int)((n + BN - 1) / BN);

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&s.full[i], 1);
      mbar_init(&s.empty[i], 1);
    }
    for (int i = 0; i < HALVES; ++i) {
      for (int a = 0; a < ACC; ++a) {
        mbar_init(&s.tfull[a][i], 1);
        mbar_init(&s.tempty[a][i], 4);
      }
    }
    for (int i = 0; i < NYBUF; ++i) mbar_init(&s.nfull[i], 1);
    mbar_init(&s.a_full, 1);
    // the A tile / block slot is free once the MMA is done with it AND every
    // epilogue warp has taken the block index: otherwise, with one-tile
    // blocks, a_full could run two phases ahead of the epilogue (parity alias)
    mbar_init(&s.a_empty, 1 + 4);
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
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmX) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmQ) : "memory");
      int stage = 0;
      uint32_t phase = 0;
      // dynamic block schedule: claim the next block with work, publish its
      // index in the 2-slot ring s.blk (read by MMA + epilogue after a_full);
      // -1 ends the CTA
      for (int it = 0;; ++it) {
        int b, len = 0;
        do {
          b = atomicAdd(sched, 1);
          if (b < nblocks) len = tlist ? tlen[b] : ntiles;
        } while (b < nblocks && len == 0);
        mbar_wait(&s.a_empty, (it & 1) ^ 1);
        s.blk[it & 1] = b < nblocks ? b : -1;
        if (b >= nblocks) {
          mbar_arrive(&s.a_full);
          break;
        }
        mbar_expect_tx(&s.a_full, BM * KB);
        tma_load_2d(s.a, &tmQ, &s.a_full, 0, b * BM);
        for (int t = 0; t < len; ++t) {
          const int tid = tlist ? tlist[(int64_t)b * tstride + t] : t;
          mbar_wait(&s.empty[stage], phase ^ 1);
          mbar_expect_tx(&s.full[stage], TILE_BYTES);
          tma_load_2d(s.b[stage], &tmX, &s.full[stage], 0, tid * BN);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      int stage = 0;
      uint32_t phase = 0;
      uint32_t g = 0;  // tiles issued by this CTA (accumulator g % ACC, norm buffer g % NYBUF)
      // the tile's |x|^2 (xnorm is padded to a multiple of BN) and ids into
      // buffer gi % NYBUF, one tile ahead of the MMA
      auto load_norms = [&](uint32_t gi, int tid) {
        const int nb = (int)(gi % NYBUF);
        mbar_expect_tx(&s.nfull[nb], perm ? BN * 8 : BN * 4);
        bulk_load(s.ny[nb], xnorm + (int64_t)tid * BN, BN * 4, &s.nfull[nb]);
        if (perm) bulk_load(s.pid[nb], perm + (int64_t)tid * BN, BN * 4, &s.nfull[nb]);
      };
      for (int it = 0;; ++it) {
        mbar_wait(&s.a_full, it & 1);
        const int b = s.blk[it & 1];
        if (b < 0) break;
        const int len = tlist ? tlen[b] : ntiles;
        tc_fence_after();
        const uint64_t adesc = sw128_desc(s.a);
        // buffer g % NYBUF last served tile g - NYBUF; the epilogue finished it
        // before releasing tile g-1-ACC's last part (waited on for tile g-1)
        int tid_nx = tlist ? tlist[(int64_t)b * tstride] : 0;
        load_norms(g, tid_nx);
        for (int t = 0; t < len; ++t, ++g) {
          const int tid = tid_nx;
          if (t + 1 < len) tid_nx = tlist ? tlist[(int64_t)b * tstride + t + 1] : t + 1;
#pragma unroll
          for (int h = 0; h < HALVES; ++h) {
            mbar_wait(&s.tempty[g % ACC][h], ((g / ACC) & 1) ^ 1);
            if (h == 0) {
              // the epilogue has released tile g-ACC's first part (this slot's
              // previous use), so it is done with tile g-ACC-1 = g+1-NYBUF:
              // that norm buffer takes tile g+1's
              if (t + 1 < len) load_norms(g + 1, tid_nx);
              mbar_wait(&s.full[stage], phase);
            }
            tc_fence_after();
            // rows h*64.. of the B tile: 8 SW128 atoms of 1024 B further on
            const uint64_t bdesc = sw128_desc(s.b[stage] + h * HN * KB);
#pragma unroll
            for (int kk = 0; kk < KB / 32; ++kk)  // K = 32 bytes per MMA; +32 B = +2 (16 B units)
              mma_i8(tmem + (g % ACC) * BN + h * HN, adesc + 2 * kk, bdesc + 2 * kk, IDESC_H, kk > 0);
            tc_commit(&s.tfull[g % ACC][h]);
          }
          tc_commit(&s.empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit(&s.a_empty);
      }
    }
  } else if (warp >= 2) {
    // ---------------- epilogue ----------------
    const int q = warp & 3;  // TMEM lane quarter this warp may access (warp % 4)
    int32_t *const svw = s.sv[warp - 2];  // this warp's staging: lane l at svw[l * 36]
    int32_t *sv = svw + lane * (TC_PAIR_APPEND ? 68 : 36);
    uint32_t g = 0;  // tiles consumed by this CTA (accumulator g % ACC, norm buffer g % NYBUF)
    for (int it = 0;; ++it) {
      mbar_wait(&s.a_full, it & 1);
      const int b = s.blk[it & 1];
      if (b < 0) break;
      if (lane == 0) mbar_arrive(&s.a_empty);  // block index taken
      const int64_t row = (int64_t)b * BM + q * 32 + lane;
      // padding rows (and, in a re-run, rows already finished): no pool
      const bool row_ok =
          row < nq && (!perm || perm[row] >= 0) && (!row_mask || row_mask[row]);
      // per-row candidate buffers (global memory, CAP keys per row)
      uint64_t *wbuf = bufs + ((int64_t)b * BM + q * 32) * CAP;  // this warp's rows
      const int len = tlist ? tlen[b] : ntiles;
      int tid_next = tlist ? tlist[(int64_t)b * tstride] : 0;  // prefetched one tile ahead
      const int nx = row_ok ? qnorm[row] : 0;
      int cnt = 0;
      bool guessed = false;
      // Row threshold.  K == 1: tau is the exact best key (keep key < tau).
      // K > 1: tau = T << 32 with T an exclusive DISTANCE bound (keep dist < T),
      // so the per-value prefilter below is the whole test.
      uint64_t tau = KEY_MAX;
      if (row_ok && init_keys) {
        // a previous pass's K-th key of this row (library key format) bounds
        // its true K-th key from above
        const uint64_t k0 = init_keys[(perm ? (int64_t)perm[row] : row) * K + K - 1];
        if (k0 != KEY_MAX) {
          const uint32_t d0 = (uint32_t)key_dist(k0);
          if (isk1) {
            tau = (((uint64_t)d0 << 32) | (uint32_t)key_id(k0)) + 1;
          } else {
            // optionally a GUESS below the bound (shrink < 1): exact iff the
            // pass still finds >= K keys under it, which finalize verifies
            uint32_t t = d0 + 1;
            if (shrink < 1.0f) {
              const uint32_t g = (uint32_t)((double)d0 * (double)shrink);
              if (g < t) {
                t = g;
                guessed = true;
              }
            }
            tau = (uint64_t)t << 32;
          }
        }
      }
      int tp = row_ok ? row_tp(tau, nx, K) : -0x7fffffff;  // invalid rows never pass
      int smax = -0x7fffffff;  // largest buffered s value while no threshold is set
      for (int t = 0; t < len; ++t) {
        const int tid = tlist ? tid_next : t;
        if (tlist && t + 1 < len) tid_next = tlist[(int64_t)b * tstride + t + 1];
        const int64_t col0 = (int64_t)tid * BN;
        const int tpar = (int)(g % NYBUF);
        const int aslot = (int)(g % ACC);
        const uint32_t acc_phase = (g / ACC) & 1;
        const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + aslot * BN;
#if TC_PAIR_APPEND
        if (!STATS && !DENSE && !K1) {
          // One 64-column part at a time: both chunks' survivor masks first (raw
          // dot products of chunks with survivors staged per lane), the part
          // handed back to the MMA, then ONE append loop over the part's
          // survivors: its trip count is the warp's maximum per-row survivor
          // count of the part (less than the sum of the two chunks' maxima) and
          // the per-chunk ballots / reductions are paid once.
          static_assert(CPP == 2, "a part is two 32-column chunks");
          static_assert(CAP >= 256 + 64, "room for K <= 256 plus one part");
#pragma unroll 1
          for (int part = 0; part < HALVES; ++part) {
            if (part == 0) mbar_wait(&s.nfull[tpar], (g / NYBUF) & 1);  // the tile's norms / ids
            mbar_wait(&s.tfull[aslot][part], acc_phase);
            tc_fence_after();
            uint32_t mk[2];
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
              const int c = part * 2 + cc;
              uint32_t r[32];
              tmem_ld32(tbase + c * 32, r);
              tmem_wait_ld();
              const int64_t cb = col0 + c * 32;
              const int4 *nyp = reinterpret_cast<const int4 *>(s.ny[tpar] + c * 32);
              uint32_t mask = 0;
#pragma unroll
              for (int v = 0; v < 8; ++v) {
                const int4 w = nyp[v];
                mask |= ((w.x - 2 * (int)r[4 * v]) <= tp) ? (1u << (4 * v)) : 0u;
                mask |= ((w.y - 2 * (int)r[4 * v + 1]) <= tp) ? (1u << (4 * v + 1)) : 0u;
                mask |= ((w.z - 2 * (int)r[4 * v + 2]) <= tp) ? (1u << (4 * v + 2)) : 0u;
                mask |= ((w.w - 2 * (int)r[4 * v + 3]) <= tp) ? (1u << (4 * v + 3)) : 0u;
              }
              if (__any_sync(0xffffffffu, mask != 0)) {
                if (__any_sync(0xffffffffu, tp >= 0x3f000000)) {  // rows without a threshold
                  const int64_t colj = cb + lane;
                  const int32_t cidj = perm ? s.pid[tpar][c * 32 + lane] : (int32_t)colj;
                  mask &= __ballot_sync(0xffffffffu, colj < n && cidj >= 0);
                }
                if (exclude_self && row >= cb && row < cb + 32) mask &= ~(1u << (int)(row - cb));
                if (mask) {
#pragma unroll
                  for (int v = 0; v < 8; ++v)
                    reinterpret_cast<int4 *>(sv + cc * 32)[v] = make_int4(
                        (int)r[4 * v], (int)r[4 * v + 1], (int)r[4 * v + 2], (int)r[4 * v + 3]);
                }
              }
              mk[cc] = mask;
            }
            // the part's columns are consumed (registers / staging): the MMA may reuse it
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.tempty[aslot][part]);
            const uint32_t m0 = mk[0], m1 = mk[1];
            if (__any_sync(0xffffffffu, (m0 | m1) != 0)) {
              const int32_t *tny = s.ny[tpar] + part * 64;
              const int32_t *tpid = s.pid[tpar] + part * 64;
              const int64_t cb = col0 + part * 64;
              const int np = __popc(m0) + __popc(m1);
              const bool track = tau == KEY_MAX && np;
              if (track) {  // rare: rows still without a threshold
                for (unsigned mm = m0; mm; mm &= mm - 1) {
                  const int j = __ffs(mm) - 1;
                  smax = max(smax, tny[j] - 2 * sv[j]);
                }
                for (unsigned mm = m1; mm; mm &= mm - 1) {
                  const int j = __ffs(mm) - 1;
                  smax = max(smax, tny[32 + j] - 2 * sv[32 + j]);
                }
              }
              unsigned need = __ballot_sync(0xffffffffu, cnt + np > CAP);
              while (need) {
                const int src = __ffs(need) - 1;
                need &= need - 1;
                const int c_src = __shfl_sync(0xffffffffu, cnt, src);
                const uint64_t t_src = __shfl_sync(0xffffffffu, tau, src);
                const uint64_t nt = select_k(wbuf + (size_t)src * CAP, c_src, K,
                                             t_src == KEY_MAX ? 0xffffffffu : khi(t_src), lane);
                if (lane == src) {
                  cnt = K;
                  tau = (uint64_t)(khi(nt) + 1) << 32;
                  tp = row_tp(tau, nx, K);
                }
              }
              uint64_t *mybuf = wbuf + (size_t)lane * CAP + cnt;
              const int trips = (int)__reduce_max_sync(0xffffffffu, (unsigned)np);
              unsigned mm0 = m0, mm1 = m1;
#if TC_APPEND_UNROLL == 4
#pragma unroll 4
#elif TC_APPEND_UNROLL == 1
#pragma unroll 1
#else
#pragma unroll 2
#endif
              for (int it = 0; it < trips; ++it) {
                const bool a0 = mm0 != 0;
                const unsigned mc = a0 ? mm0 : mm1;
                const bool act = mc != 0;
                const int j = act ? __ffs(mc) - 1 : 0;
                const int cj = (a0 ? 0 : 32) + j;   // column within the part = staging slot
                const int32_t cid = perm ? tpid[cj] : (int32_t)(cb + cj);
                const uint64_t key =
                    ((uint64_t)(uint32_t)(tny[cj] - 2 * sv[cj] + nx) << 32) | (uint32_t)cid;
                if (act) *mybuf = key;
                mybuf += act ? 1 : 0;
                const unsigned nm = mc & (mc - 1);
                mm0 = a0 ? nm : mm0;
                mm1 = a0 ? mm1 : nm;
              }
              cnt += np;
              if (track && cnt >= K) {
                tau = (uint64_t)((uint32_t)(smax + nx) + 1) << 32;
                tp = row_tp(tau, nx, K);
              }
              __syncwarp();
            }
          }
          ++g;
          continue;
        }
#endif
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          if (c == 0) mbar_wait(&s.nfull[tpar], (g / NYBUF) & 1);  // the tile's norms / ids
          if (c % CPP == 0) {  // entering part c/CPP: wait for its MMAs
            if (c > 0) {  // the previous half is in registers: let the MMA reuse it
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&s.tempty[aslot][c / CPP - 1]);
            }
            PGK_TICK(ST_MAIN);
            mbar_wait(&s.tfull[aslot][c / CPP], acc_phase);
            tc_fence_after();
            PGK_TICK(ST_WAIT);
          }
          uint32_t r[32];
          // (co-resident CTAs hide the TMEM-load latency; one chunk in flight;
          // two loads per round trip measured no faster)
          tmem_ld32(tbase + c * 32, r);
          tmem_wait_ld();
          const int64_t cb = col0 + c * 32;
          const int4 *nyp = reinterpret_cast<const int4 *>(s.ny[tpar] + c * 32);
          if (DENSE) {
            if (row_ok && t < DENSE_TILES) {
              uint2 *dst = reinterpret_cast<uint2 *>(reinterpret_cast<uint16_t *>(bufs + row * CAP) +
                                                     t * BN + c * 32);
#if TC_DENSE_NOVALID
              // (measured and left off: the dense pass is not bound by these
              // instructions, 0.767 vs 0.764 ms, and the padding values widen the
              // K-th search's range, so its 1/1024 tolerance loosens the seeds:
              // pool 9.81 -> 10.71 ms)
              // Columns that are no points (padding slots of the tile sort,
              // columns past n) carry |x|^2 = 0x3f3f3f3f: their value clamps to
              // DENSE_VMAX, above every real distance, so counting them cannot
              // lower a row's K-th value below its K-th real distance -- no
              // per-value validity test.  Only the row's own column must not
              // count, and it lies in one chunk (rows of a warp share row / 32).
              uint32_t a[32];
#pragma unroll
              for (int v = 0; v < 8; ++v) {
                const int4 w = nyp[v];
                a[4 * v] = min((uint32_t)(w.x - 2 * (int)r[4 * v] + nx + 255) >> DENSE_Q, DENSE_VMAX);
                a[4 * v + 1] = min((uint32_t)(w.y - 2 * (int)r[4 * v + 1] + nx + 255) >> DENSE_Q, DENSE_VMAX);
                a[4 * v + 2] = min((uint32_t)(w.z - 2 * (int)r[4 * v + 2] + nx + 255) >> DENSE_Q, DENSE_VMAX);
                a[4 * v + 3] = min((uint32_t)(w.w - 2 * (int)r[4 * v + 3] + nx + 255) >> DENSE_Q, DENSE_VMAX);
              }
              if (exclude_self && row >= cb && row < cb + 32) {
                const int sj = (int)(row - cb);
#pragma unroll
                for (int j = 0; j < 32; ++j) a[j] = j == sj ? DENSE_INVALID : a[j];
              }
#pragma unroll
              for (int v = 0; v < 8; ++v)
                dst[v] = make_uint2(a[4 * v] | (a[4 * v + 1] << 16), a[4 * v + 2] | (a[4 * v + 3] << 16));
#else
              const int4 *pp = reinterpret_cast<const int4 *>(s.pid[tpar] + c * 32);
              const bool es = exclude_self != 0;
#pragma unroll
              for (int v = 0; v < 8; ++v) {
                const int4 w = nyp[v];
                const int4 pd = perm ? pp[v] : make_int4(0, 0, 0, 0);
                const int64_t cj = cb + 4 * v;
                const uint32_t a0 = dense_val(w.x - 2 * (int)r[4 * v] + nx, cj, n, pd.x, es && row == cj);
                const uint32_t a1 = dense_val(w.y - 2 * (int)r[4 * v + 1] + nx, cj + 1, n, pd.y, es && row == cj + 1);
                const uint32_t a2 = dense_val(w.z - 2 * (int)r[4 * v + 2] + nx, cj + 2, n, pd.z, es && row == cj + 2);
                const uint32_t a3 = dense_val(w.w - 2 * (int)r[4 * v + 3] + nx, cj + 3, n, pd.w, es && row == cj + 3);
                dst[v] = make_uint2(a0 | (a1 << 16), a2 | (a3 << 16));
              }
#endif
            }
            continue;
          }
          if (isk1) {
            // nearest neighbour only (the center assignment): the chunk's
            // minimum s_j (3-input min tree), then -- only when some row
            // improves -- the smallest id among the columns at that minimum.
            // Same result as the survivor-mask path below, ~half the work.
#pragma unroll
            for (int v = 0; v < 8; ++v) {
              const int4 w = nyp[v];
              r[4 * v] = (uint32_t)(w.x - 2 * (int)r[4 * v]);
              r[4 * v + 1] = (uint32_t)(w.y - 2 * (int)r[4 * v + 1]);
              r[4 * v + 2] = (uint32_t)(w.z - 2 * (int)r[4 * v + 2]);
              r[4 * v + 3] = (uint32_t)(w.w - 2 * (int)r[4 * v + 3]);
            }
            if (__any_sync(0xffffffffu, tp >= 0x3f000000)) {  // rows without a threshold yet
              const int64_t colj = cb + lane;
              const int32_t cidj = perm ? s.pid[tpar][c * 32 + lane] : (int32_t)colj;
              const uint32_t ok = __ballot_sync(0xffffffffu, colj < n && cidj >= 0);
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (!((ok >> j) & 1u)) r[j] = 0x7fffffffu;
            }
            if (exclude_self && __any_sync(0xffffffffu, row >= cb && row < cb + 32)) {
              const int sj = (row >= cb && row < cb + 32) ? (int)(row - cb) : -1;
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (j == sj) r[j] = 0x7fffffffu;
            }
            int smin = 0x7fffffff;
#pragma unroll
            for (int j = 0; j < 32; j += 2) smin = min(smin, min((int)r[j], (int)r[j + 1]));
            const bool imp = smin <= tp;
            if (__any_sync(0xffffffffu, imp)) {
              uint32_t idm = 0xffffffffu;
              const int4 *pp = reinterpret_cast<const int4 *>(s.pid[tpar] + c * 32);
#pragma unroll
              for (int v = 0; v < 8; ++v) {
                const int4 pd = perm ? pp[v] : make_int4((int)(cb + 4 * v), (int)(cb + 4 * v + 1),
                                                         (int)(cb + 4 * v + 2), (int)(cb + 4 * v + 3));
                idm = (int)r[4 * v] == smin ? min(idm, (uint32_t)pd.x) : idm;
                idm = (int)r[4 * v + 1] == smin ? min(idm, (uint32_t)pd.y) : idm;
                idm = (int)r[4 * v + 2] == smin ? min(idm, (uint32_t)pd.z) : idm;
                idm = (int)r[4 * v + 3] == smin ? min(idm, (uint32_t)pd.w) : idm;
              }
              const uint64_t key = ((uint64_t)(uint32_t)(smin + nx) << 32) | idm;
              if (imp && key < tau) {
                tau = key;
                tp = tau_prefilter(tau, nx);
              }
            }
            continue;
          }
          // s_j = |x_j|^2 - 2 q.x_j ; pass iff s_j <= tp
          uint32_t mask = 0;
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            const int4 w = nyp[v];
            mask |= ((w.x - 2 * (int)r[4 * v]) <= tp) ? (1u << (4 * v)) : 0u;
            mask |= ((w.y - 2 * (int)r[4 * v + 1]) <= tp) ? (1u << (4 * v + 1)) : 0u;
            mask |= ((w.z - 2 * (int)r[4 * v + 2]) <= tp) ? (1u << (4 * v + 2)) : 0u;
            mask |= ((w.w - 2 * (int)r[4 * v + 3]) <= tp) ? (1u << (4 * v + 3)) : 0u;
          }
          if (__any_sync(0xffffffffu, mask != 0)) {
            PGK_TICK(ST_MAIN);
            if (STATS) st[ST_NSLOW]++;
            // exact survivor masks: lane j vouches for column cb + j (inside
            // the data, not a padding slot of the tile sort), and a row never
            // keeps itself
            // padding slots and columns past n carry a huge |x|^2 (0x3f3f3f3f),
            // so no finite threshold passes them; only rows still without one
            // need the explicit column check
            if (__any_sync(0xffffffffu, tp >= 0x3f000000)) {
              const int64_t colj = cb + lane;
              const int32_t cidj = perm ? s.pid[tpar][c * 32 + lane] : (int32_t)colj;
              mask &= __ballot_sync(0xffffffffu, colj < n && cidj >= 0);
            }
            if (exclude_self && row >= cb && row < cb + 32) mask &= ~(1u << (int)(row - cb));
            if (isk1) {  // nearest neighbour only: the threshold IS the answer
              // branch-free minimum (dist, id) key over the chunk's survivors
              uint64_t best = KEY_MAX;
              const int4 *pp = reinterpret_cast<const int4 *>(s.pid[tpar] + c * 32);
#pragma unroll
              for (int v = 0; v < 8; ++v) {
                const int4 w = nyp[v];
                const int4 pd = perm ? pp[v] : make_int4((int)(cb + 4 * v), (int)(cb + 4 * v + 1),
                                                         (int)(cb + 4 * v + 2), (int)(cb + 4 * v + 3));
                const int wv[4] = {w.x, w.y, w.z, w.w};
                const int pv[4] = {pd.x, pd.y, pd.z, pd.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const int j = 4 * v + e;
                  const uint64_t key = ((uint64_t)(uint32_t)(wv[e] - 2 * (int)r[j] + nx) << 32) |
                                       (uint32_t)pv[e];
                  best = ((mask >> j) & 1u) && key < best ? key : best;
                }
              }
              if (best < tau) {
                tau = best;
                tp = tau_prefilter(tau, nx);
              }
              continue;
            }
            const bool track = !isk1 && tau == KEY_MAX && mask;
            // stage the raw dot products (s_j = |x_j|^2 - 2 sv[j] is formed
            // per survivor from the tile's norms)
            if (mask) {
#pragma unroll
              for (int v = 0; v < 8; ++v)
                reinterpret_cast<int4 *>(sv)[v] =
                    make_int4((int)r[4 * v], (int)r[4 * v + 1], (int)r[4 * v + 2], (int)r[4 * v + 3]);
            }
            __syncwarp();
            const int32_t *tny = s.ny[tpar] + c * 32;
            if (track) {  // rare: rows still without a threshold
              for (unsigned mm = mask; mm; mm &= mm - 1) {
                const int j = __ffs(mm) - 1;
                smax = max(smax, tny[j] - 2 * sv[j]);
              }
            }
            // room for this chunk's survivors in every row of the warp
            unsigned need = __ballot_sync(0xffffffffu, cnt + __popc(mask) > CAP);
            if (STATS) st[ST_NCOMPACT] += __popc(need);
            while (need) {
              const int src = __ffs(need) - 1;
              need &= need - 1;
              const int c_src = __shfl_sync(0xffffffffu, cnt, src);
              const uint64_t t_src = __shfl_sync(0xffffffffu, tau, src);
              const uint64_t nt = select_k(wbuf + (size_t)src * CAP, c_src, K,
                                           t_src == KEY_MAX ? 0xffffffffu : khi(t_src), lane);
              if (lane == src) {
                cnt = K;
                tau = (uint64_t)(khi(nt) + 1) << 32;
                tp = row_tp(tau, nx, K);
              }
            }
            PGK_TICK(ST_COMPACT);
            {
              // every lane appends its own survivors (per-row serial loops
              // across the warp measured 2.8x slower than these per-lane
              // appends), in a warp-uniform loop of max-over-lanes trips with
              // predicated stores: no divergent branch to resolve per survivor
              uint64_t *mybuf = wbuf + (size_t)lane * CAP + cnt;
              const int trips = (int)__reduce_max_sync(0xffffffffu, (unsigned)__popc(mask));
              unsigned mm = mask;
#pragma unroll 2
              for (int it = 0; it < trips; ++it) {
                const bool act = mm != 0;
                const int j = act ? __ffs(mm) - 1 : 0;
                const int32_t cid = perm ? s.pid[tpar][c * 32 + j] : (int32_t)(cb + j);
                const uint64_t key =
                    ((uint64_t)(uint32_t)(tny[j] - 2 * sv[j] + nx) << 32) | (uint32_t)cid;
                if (act) *mybuf = key;
                mybuf += act ? 1 : 0;
                mm &= mm - 1;
              }
            }
            cnt += __popc(mask);
            if (STATS) st[ST_NAPPEND] += __popc(mask);
            // no threshold yet but K keys buffered: their largest distance + 1
            // bounds the K-th distance from above (exclusive)
            if (track && cnt >= K) {
              tau = (uint64_t)((uint32_t)(smax + nx) + 1) << 32;
              tp = row_tp(tau, nx, K);
            }
            __syncwarp();
            PGK_TICK(ST_SLOW);
          }
        }
        // last half and the tile's norms / ids consumed: hand them back
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&s.tempty[aslot][HALVES - 1]);
        ++g;
      }
      // block done: record each row's buffer fill and threshold; selection
      // and sorting run in the massively parallel finalize kernel
      PGK_TICK(ST_MAIN);
      if (DENSE) cnt = min(len, DENSE_TILES) * BN;
      if (row < nq) {
        row_cnt[row] = row_ok ? (cnt | (guessed ? GUESSED : 0)) : -1;
        row_tau[row] = tau;
        // K == 1: the threshold is the answer; each lane writes its own row
        // (no finalize pass)
        if (isk1 && k1_direct && row_ok) {
          const int64_t orow = perm ? (int64_t)perm[row] : row;
          out_keys[orow] =
              tau == KEY_MAX ? KEY_MAX : pack_key((float)khi(tau), (int32_t)(uint32_t)tau);
        }
      }
      PGK_TICK(ST_FINAL);
    }
    if (STATS) {
      for (int i = 0; i < ST_COUNT; ++i) {
        unsigned long long v = st[i];
        if (i == ST_NAPPEND) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        }
        if (lane == 0) atomicAdd(stats + i, v);
      }
    }
  }
#undef PGK_TICK
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// Finalize: warp per (sorted) row.  Radix selection on the register-resident
// buffer (8-bit digits of the row's value range, one 256-bin shared-memory
// histogram per warp), then the K survivors sorted by a lane-contiguous
// bitonic network.
// ---------------------------------------------------------------------------
constexpr int FIN_WARPS = 8;
constexpr int FIN_STAGE = 256;  // max K

struct FinOut {          // optional direct pool output (pool_simt's arrays)
  int32_t *gt_ids;       // may be null
  int32_t *ids;
  float *dists;
};

// The need-th smallest participating value (ON_ID: ids of the keys whose
// distance is tie_d; else distances), need 1-based and updated to the rank
// left inside the returned value.  With max_passes too small to resolve every
// digit (exact = false) the result is the upper edge of the selected bucket:
// an upper bound on the need-th value.
template <int KPL, bool ON_ID>
__device__ __forceinline__ uint32_t radix_pick(const uint64_t (&kk)[KPL], int cnt, uint32_t tie_d,
                                               int &need, uint32_t *hist, int lane,
                                               int max_passes, bool &exact,
                                               uint32_t *lo_edge = nullptr) {
  uint32_t vmin = 0xffffffffu, vmax = 0;
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    const bool p = i * 32 + lane < cnt && (!ON_ID || khi(kk[i]) == tie_d);
    const uint32_t v = ON_ID ? (uint32_t)kk[i] : khi(kk[i]);
    if (p) {
      vmin = min(vmin, v);
      vmax = max(vmax, v);
    }
  }
  vmin = __reduce_min_sync(0xffffffffu, vmin);
  vmax = __reduce_max_sync(0xffffffffu, vmax);
  const uint32_t range = vmax - vmin;
  int shift = range ? 32 - __clz(range) : 0;
  uint32_t prefix = 0;
  for (int pass = 0; shift > 0 && pass < max_passes; ++pass) {
    const int dig = min(8, shift);
    shift -= dig;
#pragma unroll
    for (int t = 0; t < 8; ++t) hist[t * 32 + lane] = 0;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const bool p = i * 32 + lane < cnt && (!ON_ID || khi(kk[i]) == tie_d);
      const uint32_t v = ((ON_ID ? (uint32_t)kk[i] : khi(kk[i])) - vmin) >> shift;
      if (p && (v >> dig) == prefix) atomicAdd(&hist[v & ((1u << dig) - 1)], 1u);
    }
    __syncwarp();
    uint32_t c[8], sum = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      c[t] = hist[lane * 8 + t];
      sum += c[t];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t excl = incl - sum, nd = (uint32_t)need;
    const int src = __ffs(__ballot_sync(0xffffffffu, excl < nd && nd <= incl)) - 1;
    int found = 0;
    uint32_t acc = excl, below = 0;
    bool done = false;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if (!done && acc + c[t] >= nd) {
        found = t;
        below = acc;
        done = true;
      }
      acc += c[t];
    }
    const int bsel = __shfl_sync(0xffffffffu, lane * 8 + found, src);
    need -= (int)__shfl_sync(0xffffffffu, below, src);
    prefix = (prefix << dig) | (uint32_t)bsel;
    __syncwarp();
  }
  exact = shift == 0;
  if (lo_edge) *lo_edge = vmin + (prefix << shift);
  return exact ? vmin + prefix : vmin + (((prefix + 1) << shift) - 1);
}

// exact K-th smallest (dist, id) key of cnt > K register-resident keys
template <int KPL>
__device__ __forceinline__ uint64_t radix_kth(const uint64_t (&kk)[KPL], int cnt, int K,
                                              uint32_t *hist, int lane);

// The same, faster in the common case: ONE 8-bit radix pass over the row's
// distance range isolates the bucket holding the K-th key; when that bucket
// holds at most 32 keys (a few, typically) they are compacted into `scratch`
// and the K-th is found by ranking them against each other -- full (dist, id)
// keys, so distance ties need no separate id pass.  Otherwise the full radix.
template <int KPL>
__device__ __forceinline__ uint64_t radix_kth_fast(const uint64_t (&kk)[KPL], int cnt, int K,
                                                   uint32_t *hist, uint64_t *scratch, int lane) {
  int need = K;
  bool exact;
  uint32_t lo = 0;
  const uint32_t hi = radix_pick<KPL, false>(kk, cnt, 0, need, hist, lane, 1, exact, &lo);
  int bc = 0;
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    const uint32_t dv = khi(kk[i]);
    bc += __popc(__ballot_sync(0xffffffffu, i * 32 + lane < cnt && dv >= lo && dv <= hi));
  }
  if (bc > 32) return radix_kth<KPL>(kk, cnt, K, hist, lane);
  int base = 0;
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    const uint32_t dv = khi(kk[i]);
    const bool in = i * 32 + lane < cnt && dv >= lo && dv <= hi;
    const unsigned b = __ballot_sync(0xffffffffu, in);
    if (in) scratch[base + __popc(b & lanemask_lt())] = kk[i];
    base += __popc(b);
  }
  __syncwarp();
  const uint64_t mine = lane < bc ? scratch[lane] : KEY_MAX;
  int rank = 0;
  for (int o = 0; o < bc; ++o) rank += scratch[o] < mine;
  const unsigned hit = __ballot_sync(0xffffffffu, lane < bc && rank == need - 1);
  __syncwarp();
  return __shfl_sync(0xffffffffu, mine, __ffs(hit) - 1);
}

template <int KPL>
__device__ __forceinline__ uint64_t radix_kth(const uint64_t (&kk)[KPL], int cnt, int K,
                                              uint32_t *hist, int lane) {
  int need = K;
  bool exact;
  const uint32_t td = radix_pick<KPL, false>(kk, cnt, 0, need, hist, lane, 4, exact);
  int ties = 0;
  uint32_t idmax = 0;
#pragma unroll
  for (int i = 0; i < KPL; ++i)
    if (i * 32 + lane < cnt && khi(kk[i]) == td) {
      ++ties;
      idmax = max(idmax, (uint32_t)kk[i]);
    }
  ties = (int)__reduce_add_sync(0xffffffffu, (unsigned)ties);
  uint32_t tid;
  if (ties == need) {  // every key at the K-th distance is in: the largest id
    tid = __reduce_max_sync(0xffffffffu, idmax);
  } else {             // ties straddle the cut: smallest ids win
    tid = radix_pick<KPL, true>(kk, cnt, td, need, hist, lane, 4, exact);
  }
  return ((uint64_t)td << 32) | tid;
}

// bitonic sort of 32*NPL u32 keys, lane-contiguous (element lane*NPL + s):
// the (k, j) stage loops stay rolled (one copy of each stage body, I-cache)
template <int NPL, int J>
__device__ __forceinline__ void bitonic_reg_stage(uint32_t (&e)[NPL], int k, int lane) {
#pragma unroll
  for (int s0 = 0; s0 < NPL; ++s0) {
    if (s0 & J) continue;
    const int s1 = s0 | J;
    const bool up = ((lane * NPL + s0) & k) == 0;
    const uint32_t a = e[s0], b = e[s1];
    const bool sw = (a > b) == up;
    e[s0] = sw ? b : a;
    e[s1] = sw ? a : b;
  }
}

#ifndef TC_SORT_UNROLL
#define TC_SORT_UNROLL 1  // measured: rolled stage loops cost 6 % of the finalize
#endif
template <int NPL>
__device__ __forceinline__ void bitonic_contig(uint32_t (&e)[NPL], int lane) {
#if TC_SORT_UNROLL
#pragma unroll
#else
#pragma unroll 1
#endif
  for (int k = 2; k <= 32 * NPL; k <<= 1) {
#if TC_SORT_UNROLL
#pragma unroll
#else
#pragma unroll 1
#endif
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= NPL) {
        const int lj = j / NPL;
        const bool lower = (lane & lj) == 0;
#pragma unroll
        for (int s0 = 0; s0 < NPL; ++s0) {
          const uint32_t o = __shfl_xor_sync(0xffffffffu, e[s0], lj);
          const bool up = ((lane * NPL + s0) & k) == 0;
          e[s0] = (lower == up) ? min(e[s0], o) : max(e[s0], o);
        }
      } else if (NPL > 4 && j == 4) {
        bitonic_reg_stage<NPL, (NPL > 4 ? 4 : 1)>(e, k, lane);
      } else if (NPL > 2 && j == 2) {
        bitonic_reg_stage<NPL, (NPL > 2 ? 2 : 1)>(e, k, lane);
      } else {
        bitonic_reg_stage<NPL, 1>(e, k, lane);
      }
    }
  }
}

// Sort the staged keys (KEY_MAX padded to 32*NPL) and write the row.  The
// network sorts u32 (dist << 8 | slot) -- exact u8 distances are < 2^23 and
// K <= 256 -- then odd-even transposition passes on the gathered 64-bit keys
// put equal distances into id order (runs of ties are short: ~2 passes).
template <int NPL>
__device__ __noinline__ void sort_emit(const uint64_t *stage, int K, int64_t orow,
                                       uint64_t *out_keys, FinOut fo, int lane) {
  uint32_t e[NPL];
#pragma unroll
  for (int s0 = 0; s0 < NPL; ++s0) {
    const int idx = lane * NPL + s0;
    const uint64_t k = stage[idx];
    e[s0] = k == KEY_MAX ? 0xffffffffu : (khi(k) << 8) | (uint32_t)idx;
  }
  bitonic_contig<NPL>(e, lane);
  uint64_t k[NPL];
#pragma unroll
  for (int s0 = 0; s0 < NPL; ++s0) k[s0] = e[s0] == 0xffffffffu ? KEY_MAX : stage[e[s0] & 0xffu];
  int quiet = 0;
#pragma unroll 1
  for (int par = 0; quiet < 2; par ^= 1) {
    bool sw = false;
#pragma unroll
    for (int s0 = 0; s0 + 1 < NPL; ++s0)
      if (((lane * NPL + s0) & 1) == par && k[s0] > k[s0 + 1]) {
        const uint64_t t = k[s0];
        k[s0] = k[s0 + 1];
        k[s0 + 1] = t;
        sw = true;
      }
    const uint64_t nxt = __shfl_down_sync(0xffffffffu, k[0], 1);
    const uint64_t prv = __shfl_up_sync(0xffffffffu, k[NPL - 1], 1);
    if (lane < 31 && ((lane * NPL + NPL - 1) & 1) == par && k[NPL - 1] > nxt) {
      k[NPL - 1] = nxt;
      sw = true;
    }
    if (lane > 0 && (((lane - 1) * NPL + NPL - 1) & 1) == par && prv > k[0]) k[0] = prv;
    quiet = __any_sync(0xffffffffu, sw) ? 0 : quiet + 1;
  }
#pragma unroll
  for (int s0 = 0; s0 < NPL; ++s0) {
    const int idx = lane * NPL + s0;
    if (idx >= K) continue;
    const uint64_t kk = k[s0];
    if (fo.ids) {
      const int32_t id = kk == KEY_MAX ? -1 : (int32_t)(uint32_t)kk;
      fo.ids[orow * K + idx] = id;
      fo.dists[orow * K + idx] = kk == KEY_MAX ? __int_as_float(0x7f800000) : (float)khi(kk);
      if (fo.gt_ids) fo.gt_ids[orow * K + idx] = id;
    } else {
      out_keys[orow * K + idx] =
          kk == KEY_MAX ? KEY_MAX : pack_key((float)khi(kk), (int32_t)(uint32_t)kk);
    }
  }
}

// select (cnt > K) and stage the row's best min(cnt, K) keys, or (kth_only)
// write the pass-1 bound; returns true when the staged keys need sort_emit
template <int KPL>
__device__ __noinline__ bool select_stage(const uint64_t *__restrict__ buf, int cnt, int K,
                                          bool kth_only, int64_t orow, uint64_t *out_keys,
                                          uint32_t *hist, uint64_t *stage, int npl32,
                                          int lane) {
  uint64_t kk[KPL];
#pragma unroll
  for (int i = 0; i < KPL; ++i) kk[i] = i * 32 + lane < cnt ? buf[i * 32 + lane] : KEY_MAX;
  if (kth_only) {
    // pass-1 bound: any key >= the true K-th serves; one histogram pass
    // gives the K-th distance to within 1/256 of the row's range
    uint64_t kth = KEY_MAX;
    if (cnt >= K) {
      int need = K;
      bool exact;
      const uint32_t d = radix_pick<KPL, false>(kk, cnt, 0, need, hist, lane, 1, exact);
      kth = pack_key((float)d, 0x7fffffff);
    }
    if (lane == 0) out_keys[orow * K + K - 1] = kth;
    return false;
  }
  const uint64_t tau = cnt > K ? radix_kth_fast<KPL>(kk, cnt, K, hist, stage, lane) : KEY_MAX;
  int base = 0;
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    const bool keep = i * 32 + lane < cnt && kk[i] <= tau;
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (keep) stage[base + __popc(bal & lanemask_lt())] = kk[i];
    base += __popc(bal);
  }
  for (int j = base + lane; j < npl32; j += 32) stage[j] = KEY_MAX;
  __syncwarp();
  return true;
}

#ifndef FIN_MID_SIZES
#define FIN_MID_SIZES 0  // measured: 6- and 12-key-per-lane instantiations 2.91 ms vs 2.73 ms without (code size)
#endif
template <int NPL>
__device__ __forceinline__ void finalize_row(const uint64_t *buf, int cnt, int K, bool kth_only,
                                             int64_t orow, uint64_t *out_keys, FinOut fo,
                                             uint32_t *hist, uint64_t *stage, int lane) {
  bool sort;
  // (the buffered counts cluster around 1.9 K: intermediate sizes save a
  // quarter of the per-key work for the rows just above a power of two)
  if (cnt <= 128)
    sort = select_stage<4>(buf, cnt, K, kth_only, orow, out_keys, hist, stage, 32 * NPL, lane);
#if FIN_MID_SIZES == 1
  else if (cnt <= 192)
    sort = select_stage<6>(buf, cnt, K, kth_only, orow, out_keys, hist, stage, 32 * NPL, lane);
#endif
  else if (cnt <= 256)
    sort = select_stage<8>(buf, cnt, K, kth_only, orow, out_keys, hist, stage, 32 * NPL, lane);
#if FIN_MID_SIZES
  else if (cnt <= 384)
    sort = select_stage<12>(buf, cnt, K, kth_only, orow, out_keys, hist, stage, 32 * NPL, lane);
#endif
  else if (cnt <= 512)
    sort = select_stage<16>(buf, cnt, K, kth_only, orow, out_keys, hist, stage, 32 * NPL, lane);
  else
    sort = select_stage<CAP / 32>(buf, cnt, K, kth_only, orow, out_keys, hist, stage, 32 * NPL,
                                  lane);
  if (sort) sort_emit<NPL>(stage, K, orow, out_keys, fo, lane);
  __syncwarp();
}

#ifndef FIN_PREFETCH
#define FIN_PREFETCH 0  // measured: L2 prefetch of the next row 3.08 ms vs 2.72 ms without
#endif
#ifndef FIN_MINB
#define FIN_MINB 2  // 128 registers, no spills: 2.96 -> 2.83 ms at config 2
#endif
__global__ void __launch_bounds__(FIN_WARPS * 32, FIN_MINB)
    tc_finalize_kernel(const uint64_t *__restrict__ bufs, const int32_t *__restrict__ row_cnt,
                       const uint64_t *__restrict__ row_tau, int64_t nrows, int K,
                       const int32_t *__restrict__ perm, int kth_only,
                       uint64_t *__restrict__ out_keys, int32_t *__restrict__ fail_blocks,
                       uint8_t *__restrict__ fail_rows, const int32_t *__restrict__ tlen,
                       FinOut fo, const int32_t *__restrict__ gate = nullptr,
                       int gate_min = 0) {
  if (gate && *gate < gate_min) return;
  __shared__ uint32_t s_hist[FIN_WARPS][256];
  __shared__ uint64_t s_stage[FIN_WARPS][FIN_STAGE];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t step = (int64_t)gridDim.x * FIN_WARPS;
  for (int64_t r = (int64_t)blockIdx.x * FIN_WARPS + warp; r < nrows; r += step) {
#if FIN_PREFETCH
    // pull the next row's keys (and its metadata) into L2 while this row is
    // worked on: the buffers (~2 KB per row, 2 GB in all) stream from DRAM
    if (r + step < nrows) {
      if (lane < 16)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(bufs + (r + step) * CAP + lane * 16));
      else if (lane == 16)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(row_cnt + r + step));
      else if (lane == 17 && perm)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(perm + r + step));
    }
#endif
    if (tlen && tlen[r / BM] == 0) continue;  // block not scheduled in this launch
    const int raw = row_cnt[r];
    if (raw < 0) continue;  // padding row
    const int cnt = raw & ~GUESSED;
    if ((raw & GUESSED) && cnt < K) {
      // the guessed threshold was too tight: leave the row's seed in place
      // and have its block re-run with the true bound
      if (lane == 0) {
        fail_blocks[r / BM] = 1;
        fail_rows[r] = 1;
      }
      continue;
    }
    const int64_t orow = perm ? (int64_t)perm[r] : r;
#ifdef TC_DEBUG
    if (lane == 0 && (cnt > CAP || orow < 0 || orow >= nrows))
      printf("[tc_finalize] r=%lld raw=%d cnt=%d orow=%lld K=%d nrows=%lld\n", (long long)r, raw,
             cnt, (long long)orow, K, (long long)nrows);
#endif
    if (K == 1) {  // the kernel's threshold is the answer
      const uint64_t tau = row_tau[r];
      if (lane == 0) {
        if (fo.ids && !kth_only) {
          fo.ids[orow] = tau == KEY_MAX ? -1 : (int32_t)(uint32_t)tau;
          fo.dists[orow] = tau == KEY_MAX ? __int_as_float(0x7f800000) : (float)khi(tau);
          if (fo.gt_ids) fo.gt_ids[orow] = fo.ids[orow];
        } else {
          out_keys[orow] =
              tau == KEY_MAX ? KEY_MAX : pack_key((float)khi(tau), (int32_t)(uint32_t)tau);
        }
      }
      continue;
    }
    const uint64_t *b = bufs + r * CAP;
    uint32_t *hist = s_hist[warp];
    uint64_t *stage = s_stage[warp];
    if (K <= 32) finalize_row<1>(b, cnt, K, kth_only, orow, out_keys, fo, hist, stage, lane);
    else if (K <= 64) finalize_row<2>(b, cnt, K, kth_only, orow, out_keys, fo, hist, stage, lane);
    else if (K <= 128) finalize_row<4>(b, cnt, K, kth_only, orow, out_keys, fo, hist, stage, lane);
    else finalize_row<8>(b, cnt, K, kth_only, orow, out_keys, fo, hist, stage, lane);
  }
}

// K-th smallest of a row's dense pass-1 values (u16; 0xffff = invalid), to
// within 1/1024 of the row's value range from above: a warp-wide binary
// search over register-resident values (per step one compare per value and
// one REDUX count), keeping count(v <= hi) >= K.  Returns hi.
template <int VPL>
__device__ __noinline__ uint32_t kth_dense(const uint16_t *__restrict__ buf, int cnt, int K,
                                           int lane) {
  static_assert(VPL % 2 == 0, "values are loaded in u16 pairs");
  const uint32_t *buf2 = reinterpret_cast<const uint32_t *>(buf);  // cnt is a multiple of 128
#if TC_DENSE_PACKED
  // words of two 15-bit values; invalid (0x7fff) never counts: mid stays
  // below it.  Past cnt: two invalid values.
  uint32_t w2[VPL / 2];
  int nv = 0;
  uint32_t vmin = 0xffffffffu, vmax = 0;
#pragma unroll
  for (int i = 0; i < VPL / 2; ++i) {
    const int idx = i * 32 + lane;  // word: values 2 idx, 2 idx + 1 (order is irrelevant)
    const uint32_t w = 2 * idx < cnt ? buf2[idx] : 0x7fff7fffu;
    w2[i] = w;
    const uint32_t a = w & 0xffffu, b = w >> 16;
    if (a != DENSE_INVALID) {
      ++nv;
      vmin = min(vmin, a);
      vmax = max(vmax, a);
    }
    if (b != DENSE_INVALID) {
      ++nv;
      vmin = min(vmin, b);
      vmax = max(vmax, b);
    }
  }
  if ((int)__reduce_add_sync(0xffffffffu, (unsigned)nv) < K) return 0xffffffffu;
  uint32_t lo = __reduce_min_sync(0xffffffffu, vmin);
  uint32_t hi = __reduce_max_sync(0xffffffffu, vmax);
  const uint32_t tol = (hi - lo) >> 10;
  while (hi - lo > tol) {
    const uint32_t mid = lo + ((hi - lo) >> 1);
    const uint32_t m2 = (mid | (mid << 16)) + 0x80008000u;
    uint32_t c2 = 0;  // two 16-bit counters (VPL / 2 <= 32 words per lane)
#pragma unroll
    for (int i = 0; i < VPL / 2; ++i) c2 += ((m2 - w2[i]) >> 15) & 0x00010001u;
    const unsigned c = (c2 & 0xffffu) + (c2 >> 16);
    if ((int)__reduce_add_sync(0xffffffffu, c) >= K) hi = mid;
    else lo = mid + 1;
  }
  return hi;
#else
  uint32_t v[VPL];
  int nv = 0;
  uint32_t vmin = 0xffffffffu, vmax = 0;
#pragma unroll
  for (int i = 0; i < VPL / 2; ++i) {
    const int idx = i * 32 + lane;  // word: values 2 idx, 2 idx + 1 (order is irrelevant)
    const uint32_t w = 2 * idx < cnt ? buf2[idx] : 0xffffffffu;
    v[2 * i] = (w & 0xffffu) == 0xffffu ? 0xffffffffu : (w & 0xffffu);
    v[2 * i + 1] = (w >> 16) == 0xffffu ? 0xffffffffu : (w >> 16);
  }
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    if (v[i] != 0xffffffffu) {
      ++nv;
      vmin = min(vmin, v[i]);
      vmax = max(vmax, v[i]);
    }
  }
  if ((int)__reduce_add_sync(0xffffffffu, (unsigned)nv) < K) return 0xffffffffu;
  uint32_t lo = __reduce_min_sync(0xffffffffu, vmin);
  uint32_t hi = __reduce_max_sync(0xffffffffu, vmax);
  const uint32_t tol = (hi - lo) >> 10;
  while (hi - lo > tol) {
    const uint32_t mid = lo + ((hi - lo) >> 1);
    int c = 0;
#pragma unroll
    for (int i = 0; i < VPL; ++i) c += v[i] <= mid;
    if ((int)__reduce_add_sync(0xffffffffu, (unsigned)c) >= K) hi = mid;
    else lo = mid + 1;
  }
  return hi;
#endif
}

// Pass-1 bound of every row from its dense distances (warp per row): an
// upper bound of the K-th smallest valid distance, itself an upper bound of
// the true K-th neighbour distance (the row met real points only), in the library's key
// format at out_keys[orig_row * K + K - 1].
__global__ void __launch_bounds__(FIN_WARPS * 32, 4)
    tc_kth_dense_kernel(const uint64_t *__restrict__ bufs, const int32_t *__restrict__ row_cnt,
                        int64_t nrows, int K, const int32_t *__restrict__ perm,
                        uint64_t *__restrict__ out_keys, uint32_t *__restrict__ ostat) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t r = (int64_t)blockIdx.x * FIN_WARPS + warp; r < nrows;
       r += (int64_t)gridDim.x * FIN_WARPS) {
    const int cnt = row_cnt[r];
    if (cnt < 0) continue;  // padding row
    const uint16_t *b = reinterpret_cast<const uint16_t *>(bufs + r * CAP);
    uint32_t kth;
    if (cnt <= 512) kth = kth_dense<16>(b, cnt, K, lane);
    else if (cnt <= 768) kth = kth_dense<24>(b, cnt, K, lane);
    else if (cnt <= 1024) kth = kth_dense<32>(b, cnt, K, lane);
    else kth = kth_dense<64>(b, cnt, K, lane);
    const int64_t orow = perm ? (int64_t)perm[r] : r;
    if (lane == 0)
      out_keys[orow * K + K - 1] =
          kth == 0xffffffffu ? KEY_MAX : pack_key((float)(kth << DENSE_Q), 0x7fffffff);
    if (ostat) {  // instrumentation: order statistics K/8, K/4, K/2, K (PGK_TILES_STATS)
      for (int j = 0; j < 4; ++j) {
        const int kj = max(1, K >> (3 - j));
        const uint32_t x = cnt <= 1024 ? kth_dense<32>(b, cnt, kj, lane) : kth_dense<64>(b, cnt, kj, lane);
        if (lane == 0) ostat[orow * 4 + j] = x == 0xffffffffu ? x : x << DENSE_Q;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Rows whose guessed pass-2 threshold proved too tight (fail_rows != 0, ~0.2 %
// of the rows): an exact rescan on the SIMT cores instead of re-running their
// whole 128-row blocks on the tensor cores.  Block per failing row: the 8
// warps share the full-radius tile list of the row's block; every key with
// dist <= the row's pass-1 seed (an upper bound of its true K-th distance,
// the seed is the row's untouched pass-1 key) goes to the row's buffer, which
// is compacted to the K best (select_k) whenever the next round could
// overflow it; warp 0 then finalizes the row (finalize_row).  Distances are
// the same exact integers as the tensor-core path (dp4a on the u8 rows).
// ---------------------------------------------------------------------------
__global__ void fail_list_kernel(const uint8_t *__restrict__ fail_rows, int64_t nrows,
                                 int32_t *__restrict__ list, int32_t *__restrict__ count) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows;
       r += (int64_t)gridDim.x * blockDim.x)
    if (fail_rows[r]) list[atomicAdd(count, 1)] = (int32_t)r;
}

constexpr int RR_THREADS = FIN_WARPS * 32;
constexpr int RR_ROUND = FIN_WARPS * BN;  // keys one round (a tile per warp) can produce
__global__ void __launch_bounds__(RR_THREADS, 2)
    rerun_rows_kernel(const uint8_t *__restrict__ xs, const int32_t *__restrict__ ns,
                      const int32_t *__restrict__ perm, const int32_t *__restrict__ list,
                      const int32_t *__restrict__ count, const int32_t *__restrict__ tlist,
                      const int32_t *__restrict__ tlen, int64_t tstride,
                      const uint64_t *__restrict__ seeds, int K, uint64_t *__restrict__ bufs,
                      uint64_t *__restrict__ out_keys, FinOut fo, int max_rows) {
  __shared__ uint32_t s_hist[256];
  __shared__ uint64_t s_stage[FIN_STAGE];
  __shared__ uint64_t s_round[RR_ROUND];
  if (*count > max_rows) return;  // too many: the tensor-core block re-run takes them  // this round's survivors
  __shared__ int s_rc, s_cnt;
  __shared__ uint32_t s_t;  // exclusive distance bound
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nl = *count;
  for (int li = blockIdx.x; li < nl; li += gridDim.x) {
    const int64_t r = list[li];
    const int64_t orow = perm[r];
    uint64_t *buf = bufs + r * CAP;
    // the query row (u8, 128 B) in registers, word w = bytes 4w..4w+3
    uint32_t q[32];
    const uint4 *qr = reinterpret_cast<const uint4 *>(xs + r * KB);
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const uint4 w = qr[v];
      q[4 * v] = w.x; q[4 * v + 1] = w.y; q[4 * v + 2] = w.z; q[4 * v + 3] = w.w;
    }
    const int nq = ns[r];
    if (threadIdx.x == 0) {
      const uint64_t k0 = seeds[orow * K + K - 1];
      s_t = k0 == KEY_MAX ? 0xffffffffu : (uint32_t)key_dist(k0) + 1u;
      s_cnt = 0;
      s_rc = 0;
    }
    __syncthreads();
    const int64_t b = r / BM;
    const int len = tlen[b];
    const int32_t *tl = tlist + b * tstride;
    for (int t0 = 0; t0 < len; t0 += FIN_WARPS) {
      const int ti = t0 + warp;
      const uint32_t tb = s_t;
      if (ti < len) {
        const int64_t tile = tl[ti];
#pragma unroll 1
        for (int i = 0; i < 4; ++i) {
          const int64_t col = tile * BN + i * 32 + lane;
          const int32_t id = perm[col];
          const uint4 *xr = reinterpret_cast<const uint4 *>(xs + col * KB);
          uint32_t dot = 0;
#pragma unroll
          for (int v = 0; v < 8; ++v) {
            const uint4 w = xr[v];
            dot = __dp4a(w.x, q[4 * v], dot);
            dot = __dp4a(w.y, q[4 * v + 1], dot);
            dot = __dp4a(w.z, q[4 * v + 2], dot);
            dot = __dp4a(w.w, q[4 * v + 3], dot);
          }
          const uint32_t dist = (uint32_t)(ns[col] + nq - 2 * (int)dot);
          const bool keep = id >= 0 && id != (int32_t)orow && dist < tb;
          const unsigned bal = __ballot_sync(0xffffffffu, keep);
          int base = 0;
          if (lane == 0 && bal) base = atomicAdd(&s_rc, __popc(bal));
          base = __shfl_sync(0xffffffffu, base, 0);
          if (keep) s_round[base + __popc(bal & lanemask_lt())] = ((uint64_t)dist << 32) | (uint32_t)id;
        }
      }
      __syncthreads();
      if (warp == 0) {  // move the round into the row's buffer, compacting when full
        int cnt = s_cnt;
        uint32_t t = s_t;
        const int rc = s_rc;
        for (int i0 = 0; i0 < rc; i0 += 32) {
          if (cnt + 32 > CAP) {
            const uint64_t nt = select_k(buf, cnt, K, t, lane);
            cnt = K;
            t = min(t, khi(nt) + 1u);
          }
          const uint64_t key = i0 + lane < rc ? s_round[i0 + lane] : KEY_MAX;
          const bool keep = key != KEY_MAX && khi(key) < t;
          const unsigned bal = __ballot_sync(0xffffffffu, keep);
          if (keep) buf[cnt + __popc(bal & lanemask_lt())] = key;
          cnt += __popc(bal);
        }
        __syncwarp();
        if (lane == 0) {
          s_cnt = cnt;
          s_t = t;
          s_rc = 0;
        }
      }
      __syncthreads();
    }
    if (warp == 0) {
      const int cnt = s_cnt;
      if (K <= 32) finalize_row<1>(buf, cnt, K, false, orow, out_keys, fo, s_hist, s_stage, lane);
      else if (K <= 64) finalize_row<2>(buf, cnt, K, false, orow, out_keys, fo, s_hist, s_stage, lane);
      else if (K <= 128) finalize_row<4>(buf, cnt, K, false, orow, out_keys, fo, s_hist, s_stage, lane);
      else finalize_row<8>(buf, cnt, K, false, orow, out_keys, fo, s_hist, s_stage, lane);
    }
    __syncthreads();
  }
}

// float (integer-valued, d <= 128) -> u8 rows padded to 128 bytes
__global__ void to_u8_kernel(const float *__restrict__ X, int64_t n, int d,
                             uint8_t *__restrict__ out) {
  const int64_t total = n * KB;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / KB;
    int c = (int)(e - r * KB);
    out[e] = c < d ? (uint8_t)__float2int_rn(X[r * d + c]) : (uint8_t)0;
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

static bool make_map(CUtensorMap *tm, const uint8_t *base, int64_t rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)KB, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)KB};
  cuuint32_t box[2] = {(cuuint32_t)KB, (cuuint32_t)BN};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void *)base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace tc

// (128-byte rows x rows) u8 tensor map with a (128 x box_rows) box, SW128;
// box_rows = 1 is the TMA gather4 form (prune_gram.cu)
#ifndef GRAM_L2_PROMO
#define GRAM_L2_PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif
bool make_u8_row_map(CUtensorMap *tm, const uint8_t *base, int64_t rows, int box_rows) {
  auto fn = tc::encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)tc::KB, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)tc::KB};
  cuuint32_t box[2] = {(cuuint32_t)tc::KB, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void *)base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  GRAM_L2_PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// (rows x cols) bf16 row-major tensor map with a (64 x 128) box, SW128: the
// operand blocks of the float pool (pool_tc_f32.cu)
bool make_bf16_tile_map(CUtensorMap *tm, const void *base, int64_t rows, int64_t cols) {
  auto fn = tc::encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// instrumentation (PGK_TILES_STATS): pass-1 order statistics per row
uint32_t *g_dense_ostat = nullptr;

// k1: the K = 1 pass whose epilogue writes the answer itself (the center
// assignment) buffers no candidates: no per-row buffers (8 KB per row)
size_t tc_pool_workspace(int64_t n, int64_t nq, bool self, bool k1) {
  size_t b = (size_t)n * tc::KB + 1024;
  if (!self) b += (size_t)nq * tc::KB + 1024;
  const int64_t rows = (nq + tc::BM - 1) / tc::BM * tc::BM;
  if (!k1) b += (size_t)rows * tc::CAP * sizeof(uint64_t) + 1024;  // per-row candidate buffers
  b += (size_t)rows * (sizeof(int32_t) + sizeof(uint64_t)) + 2048;
  b += 256;  // dynamic block-schedule counter
  return b;
}

bool tc_pool_supported(int64_t d, int64_t k) {
  static_assert(tc::CAP >= 256 + 32, "CAP must leave room for K <= 256 plus one chunk");
  static_assert(tc::CAP <= tc::SEL_CAP, "select_k holds CAP keys in registers");
  static_assert(tc::FIN_STAGE >= 256, "finalize stages up to K = 256 keys");
  static int env = -1;
  if (env < 0) {
    const char *e = getenv("PGK_DISABLE_TC");
    env = (e && e[0] == '1') ? 1 : 0;
  }
  return !env && d <= tc::KB && k >= 1 && k <= 256;
}

int launch_pool_tc_u8_lists(const float *X, int64_t n, int d, const float *Q, int64_t nq,
                            int exclude_self, const int32_t *xnorm, const int32_t *qnorm,
                            int K, uint64_t *keys, void *tc_ws, size_t tc_bytes,
                            cudaStream_t stream, const uint8_t *xs_sorted,
                            const int32_t *tlist, const int32_t *tlen, int64_t tstride,
                            const int32_t *perm, bool *handled, const uint64_t *init_keys,
                            int kth_only, float shrink, int32_t *fail_blocks,
                            const PoolOut *out, uint8_t *fail_rows, const uint8_t *row_mask,
                            const uint8_t *qu8_in, const int32_t *gate, int gate_min) {
  *handled = false;
  if (shrink < 1.0f && (!fail_blocks || !fail_rows)) {
    set_error("guessed thresholds need a fail-block array");
    return PGK_ERR_INVALID;
  }
  if (!tc_pool_supported(d, K)) return PGK_OK;
  const bool self = (Q == X);
  // K == 1 into keys (not the pool arrays): the epilogue writes the answer
  const int k1_direct = (K == 1 && !(out && !kth_only)) ? 1 : 0;
  if (tc_bytes < tc_pool_workspace(n, nq, self, k1_direct != 0)) {
    set_error("tc pool workspace too small");
    return PGK_ERR_NOMEM;
  }
  Carve c(tc_ws, tc_bytes);
  uint8_t *xu8 = c.take<uint8_t>((size_t)n * tc::KB);
  uint8_t *qu8 = self ? xu8 : c.take<uint8_t>((size_t)nq * tc::KB);
  const int sms = num_sms();
  const int64_t rows = (nq + tc::BM - 1) / tc::BM * tc::BM;
  uint64_t *bufs = k1_direct ? nullptr : c.take<uint64_t>((size_t)rows * tc::CAP);
  int32_t *row_cnt = c.take<int32_t>(rows);
  uint64_t *row_tau = c.take<uint64_t>(rows);
  int32_t *sched = c.take<int32_t>(1);
  const unsigned cg = (unsigned)std::min<int64_t>((n * tc::KB + 255) / 256, (int64_t)sms * 16);
  if (xs_sorted) {
    xu8 = qu8 = const_cast<uint8_t *>(xs_sorted);  // already u8, permuted by the tile sort
  } else {
    tc::to_u8_kernel<<<cg, 256, 0, stream>>>(X, n, d, xu8);
    PGK_CHECK_LAUNCH("to_u8_kernel");
  }
  if (!self && qu8_in) {
    qu8 = const_cast<uint8_t *>(qu8_in);  // the caller's u8 rows (128 B each)
  } else if (!self) {
    tc::to_u8_kernel<<<cg, 256, 0, stream>>>(Q, nq, d, qu8);
    PGK_CHECK_LAUNCH("to_u8_kernel");
  }
  // pad |x|^2 to a multiple of BN with a huge value (0x3f3f3f3f > any distance):
  // the kernel bulk-copies whole 128-entry tiles of it
  const int64_t n_pad = (n + tc::BN - 1) / tc::BN * tc::BN;
  if (n_pad > n && !xs_sorted)
    PGK_CUDA(cudaMemsetAsync(const_cast<int32_t *>(xnorm) + n, 0x3f, (n_pad - n) * 4, stream));
  CUtensorMap tmX, tmQ;
  if (!tc::make_map(&tmX, xu8, n) || !tc::make_map(&tmQ, qu8, nq)) {
    set_error("cuTensorMapEncodeTiled failed");
    return PGK_ERR_CUDA;
  }
  const size_t smem = sizeof(tc::Smem) + 1024;
  PGK_CUDA(ensure_smem((const void *)tc::tc_pool_u8_kernel<false, false>, smem));
  PGK_CUDA(ensure_smem((const void *)tc::tc_pool_u8_kernel<true, false>, smem));
  PGK_CUDA(ensure_smem((const void *)tc::tc_pool_u8_kernel<false, true>, smem));
  PGK_CUDA(ensure_smem((const void *)tc::tc_pool_u8_kernel<false, false, true>, smem));
  const int nblocks = (int)((nq + tc::BM - 1) / tc::BM);
  const unsigned grid = (unsigned)std::min<int64_t>(nblocks, (int64_t)tc::CTAS_PER_SM * sms);
  PGK_CUDA(cudaMemsetAsync(sched, 0, sizeof(int32_t), stream));
  // pass-1 bounds over tile lists: dense distances + exact K-th selection
  const bool dense = kth_only && K > 1 && tlist;
  const char *se = getenv("PGK_TC_STATS");
  if (dense) {
    tc::tc_pool_u8_kernel<false, true><<<grid, tc::THREADS, smem, stream>>>(
        tmX, tmQ, n, nq, exclude_self, xnorm, qnorm, K, bufs, keys, nullptr, tlist, tlen,
        tstride, perm, init_keys, shrink, row_cnt, row_tau, sched, row_mask, 0, gate, gate_min);
    PGK_CHECK_LAUNCH("tc_pool_u8_kernel<dense>");
    const unsigned fgrid =
        (unsigned)std::min<int64_t>((nq + tc::FIN_WARPS - 1) / tc::FIN_WARPS, (int64_t)sms * 8);
    tc::tc_kth_dense_kernel<<<fgrid, tc::FIN_WARPS * 32, 0, stream>>>(bufs, row_cnt, nq, K, perm,
                                                                      keys, g_dense_ostat);
    PGK_CHECK_LAUNCH("tc_kth_dense_kernel");
    *handled = true;
    return PGK_OK;
  }
  if (se && se[0] == '1') {
    unsigned long long *dstats = nullptr;
    PGK_CUDA(cudaMalloc(&dstats, sizeof(unsigned long long) * tc::ST_COUNT));
    PGK_CUDA(cudaMemsetAsync(dstats, 0, sizeof(unsigned long long) * tc::ST_COUNT, stream));
    tc::tc_pool_u8_kernel<true, false><<<grid, tc::THREADS, smem, stream>>>(
        tmX, tmQ, n, nq, exclude_self, xnorm, qnorm, K, bufs, keys, dstats, tlist, tlen,
        tstride, perm, init_keys, shrink, row_cnt, row_tau, sched, row_mask, k1_direct, gate,
        gate_min);
    PGK_CHECK_LAUNCH("tc_pool_u8_kernel<stats>");
    unsigned long long h[tc::ST_COUNT];
    PGK_CUDA(cudaMemcpyAsync(h, dstats, sizeof(h), cudaMemcpyDeviceToHost, stream));
    PGK_CUDA(cudaStreamSynchronize(stream));
    cudaFree(dstats);
    const double warps = 4.0 * grid;
    fprintf(stderr,
            "[tc stats] per epilogue warp: wait %.3g main %.3g slow %.3g compact %.3g final %.3g "
            "cycles; slow-chunks %.3g compactions %.3g; appends/row-block %.1f\n",
            h[0] / warps, h[1] / warps, h[2] / warps, h[3] / warps, h[4] / warps, h[5] / warps,
            h[6] / warps, (double)h[7] / (double)nq);
    if (k1_direct) {
      *handled = true;
      return PGK_OK;
    }
  } else {
    if (K == 1)
      tc::tc_pool_u8_kernel<false, false, true><<<grid, tc::THREADS, smem, stream>>>(
          tmX, tmQ, n, nq, exclude_self, xnorm, qnorm, K, bufs, keys, nullptr, tlist, tlen,
          tstride, perm, init_keys, shrink, row_cnt, row_tau, sched, row_mask, k1_direct, gate,
          gate_min);
    else
      tc::tc_pool_u8_kernel<false, false><<<grid, tc::THREADS, smem, stream>>>(
          tmX, tmQ, n, nq, exclude_self, xnorm, qnorm, K, bufs, keys, nullptr, tlist, tlen,
          tstride, perm, init_keys, shrink, row_cnt, row_tau, sched, row_mask, k1_direct, gate,
          gate_min);
    PGK_CHECK_LAUNCH("tc_pool_u8_kernel");
    if (k1_direct) {
      *handled = true;
      return PGK_OK;
    }
  }
  tc::FinOut fo{nullptr, nullptr, nullptr};
  if (out && !kth_only) fo = tc::FinOut{out->gt_ids, out->ids, out->dists};
  const unsigned fgrid =
      (unsigned)std::min<int64_t>((nq + tc::FIN_WARPS - 1) / tc::FIN_WARPS, (int64_t)sms * 8);
  tc::tc_finalize_kernel<<<fgrid, tc::FIN_WARPS * 32, 0, stream>>>(
      bufs, row_cnt, row_tau, nq, K, perm, kth_only, keys, fail_blocks, fail_rows,
      tlist ? tlen : nullptr, fo, gate, gate_min);
  PGK_CHECK_LAUNCH("tc_finalize_kernel");
  *handled = true;
  return PGK_OK;
}

// The failing rows of the last guessed pass 2 (see rerun_rows_kernel), on
// the same tc workspace (its per-row buffers), xs / ns / perm the tile-sorted
// rows, norms and permutation, tlist / tlen / tstride their full-radius lists.
int launch_rerun_rows(int64_t np, void *tc_ws, size_t tc_bytes, const uint8_t *xs,
                      const int32_t *ns, const int32_t *perm, const uint8_t *fail_rows,
                      const int32_t *tlist, const int32_t *tlen, int64_t tstride,
                      const uint64_t *seeds, int K, uint64_t *keys, const PoolOut *out,
                      int32_t *scratch, int max_rows, cudaStream_t stream) {
  Carve c(tc_ws, tc_bytes);
  c.take<uint8_t>((size_t)np * tc::KB);  // the tc launcher's u8 copy (unused with xs)
  const int64_t rows = (np + tc::BM - 1) / tc::BM * tc::BM;
  uint64_t *bufs = c.take<uint64_t>((size_t)rows * tc::CAP);
  int32_t *count = scratch, *list = scratch + 32;
  const int sms = num_sms();
  PGK_CUDA(cudaMemsetAsync(count, 0, sizeof(int32_t), stream));
  tc::fail_list_kernel<<<(unsigned)sms * 4, 256, 0, stream>>>(fail_rows, np, list, count);
  PGK_CHECK_LAUNCH("fail_list_kernel");
  tc::FinOut fo{nullptr, nullptr, nullptr};
  if (out) fo = tc::FinOut{out->gt_ids, out->ids, out->dists};
  tc::rerun_rows_kernel<<<(unsigned)sms * 8, tc::RR_THREADS, 0, stream>>>(
      xs, ns, perm, list, count, tlist, tlen, tstride, seeds, K, bufs, keys, fo, max_rows);
  PGK_CHECK_LAUNCH("rerun_rows_kernel");
  return PGK_OK;
}

}  // namespace pgk
