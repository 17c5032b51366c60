// reverse.cu -- phase B: reverse-edge insertion + re-prune
// (prune.add_reverse_and_prune, prune.py:129-151).
//
// Reference: bincount of all live phase-A targets + cumsum (prune.py:134-138),
// a serial owner-ascending scatter of (owner, owner's stored dist)
// (_kernels.scatter_reverse :530-541), a per-node sort_pairs of the reverse
// slice, a merge with the node's own row (own first on equal (dist, id)) that
// drops consecutive duplicate ids (_kernels.merge_with_reverse :544-588), and
// prune_all of every merged row with the same params.
//
// GPU pipeline (all on one stream, no host sync):
//   1. count    : atomic in-degree histogram                      (rev_cnt)
//   2. scan     : mrg_off = exclusive_scan(counts + rev_cnt)  (block scan,
//                 recursive over block totals)
//   3. scatter  : own entries to the front of each merged slice, reverse
//                 entries after them at mrg_off[v] + counts[v] + atomic slot,
//                 as packed (dist, id) keys
//   4. sort     : per node, ascending sort of the whole slice (warp bitonic in
//                 shared memory; long slices: block bitonic in global scratch)
//                 then drop consecutive duplicate ids.  Sorting the union by
//                 (dist, id) yields the same sequence as the reference's merge
//                 (entries with equal (dist, id) are identical), so the atomic
//                 arrival order never shows: the output is deterministic.
//   5. re-prune : prune_kernel on the merged CSR.
#include "common.cuh"

namespace pgk {

size_t prune_workspace(int64_t n_rows);
int launch_prune(const float *X, const uint8_t *xu8, const int32_t *norms, int64_t n,
                 int64_t d, const int32_t *row_node, const int32_t *row_order, void *ws,
                 size_t ws_bytes, const int64_t *cand_off,
                 const int32_t *cand_counts, const int32_t *cand_ids,
                 const float *cand_dists, int strategy, double cos_alpha,
                 int64_t M, int64_t width, int32_t *out_ids, float *out_dists,
                 int32_t *out_counts, int64_t *dist_evals, int64_t *angle_evals,
                 cudaStream_t stream, bool short_rows = false);

size_t gram_workspace(int64_t n);
bool gram_enabled();

// PGK_REV_FUSED=0: every merged row goes to the tcgen05 kernels (A/B timing)
static bool rev_fused_enabled() {
  static int env = -1;
  if (env < 0) {
    const char *e = getenv("PGK_REV_FUSED");
    env = (e && e[0] == '0') ? 0 : 1;
  }
  return env == 1;
}

constexpr int SORT_WARPS = 8;
#ifndef SCATTER_PASSES
#define SCATTER_PASSES 1  // measured: 4 node-range passes 1.05 ms vs 0.68 ms for one
#endif
constexpr int SORT_SMEM_KEYS = 512;  // per-warp in-register sort capacity (16 keys per lane)

// warp per phase-A row, lane per entry (no per-element division)
__global__ void rev_count_kernel(const int32_t *__restrict__ ids,
                                 const int32_t *__restrict__ counts, int64_t n,
                                 int width, int32_t *__restrict__ rev_cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < n; u += nw) {
    const int c = counts[u];
    for (int j = lane; j < c; j += 32) {
      const int32_t v = ids[u * width + j];
      if ((uint64_t)v < (uint64_t)n) atomicAdd(rev_cnt + v, 1);  // out-of-range ids: no edge
    }
  }
}

// merged-slice capacity of node u: own entries + reverse entries (index n
// holds 0 so an (n+1)-item exclusive scan also yields the total).
__global__ void cap_kernel(const int32_t *__restrict__ counts,
                           const int32_t *__restrict__ rev, int64_t n,
                           int64_t *__restrict__ cap) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u <= n;
       u += (int64_t)gridDim.x * blockDim.x)
    cap[u] = u < n ? (int64_t)counts[u] + rev[u] : 0;
}

// Exclusive scan of int64: 1024 threads x 4 items per block, block totals
// scanned recursively, then added back.
constexpr int SCAN_T = 1024, SCAN_ITEMS = 4, SCAN_TILE = SCAN_T * SCAN_ITEMS;

__global__ void __launch_bounds__(SCAN_T)
    scan_block_kernel(const int64_t *__restrict__ in, int64_t *__restrict__ out,
                      int64_t m, int64_t *__restrict__ bsum) {
  __shared__ int64_t warp_tot[SCAN_T / 32];
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
  int64_t v[SCAN_ITEMS], run = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    v[i] = base + i < m ? in[base + i] : 0;
    run += v[i];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int64_t w = warp_tot[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    warp_tot[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  int64_t pre = incl - run + (warp > 0 ? warp_tot[warp - 1] : 0);
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    if (base + i < m) out[base + i] = pre;
    pre += v[i];
  }
  if (threadIdx.x == SCAN_T - 1) bsum[blockIdx.x] = pre;
}

__global__ void scan_add_kernel(int64_t *__restrict__ out, int64_t m,
                                const int64_t *__restrict__ boff) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m;
       e += (int64_t)gridDim.x * blockDim.x)
    out[e] += boff[e / SCAN_TILE];
}

size_t scan_scratch(int64_t m) {
  size_t tot = 0;
  while (m > 1) {
    int64_t nb = (m + SCAN_TILE - 1) / SCAN_TILE;
    tot += 2 * (size_t)nb;
    m = nb;
  }
  return tot + 2;
}

int exclusive_scan(const int64_t *in, int64_t *out, int64_t m, int64_t *scratch,
                          cudaStream_t stream) {
  const int64_t nb = (m + SCAN_TILE - 1) / SCAN_TILE;
  int64_t *bsum = scratch, *boff = scratch + nb;
  scan_block_kernel<<<(unsigned)nb, SCAN_T, 0, stream>>>(in, out, m, bsum);
  PGK_CHECK_LAUNCH("scan_block_kernel");
  if (nb > 1) {
    int rc = exclusive_scan(bsum, boff, nb, scratch + 2 * nb, stream);
    if (rc) return rc;
    unsigned g = (unsigned)std::min<int64_t>((m + 255) / 256, (int64_t)num_sms() * 16);
    scan_add_kernel<<<g, 256, 0, stream>>>(out, m, boff);
    PGK_CHECK_LAUNCH("scan_add_kernel");
  }
  return PGK_OK;
}

// own entries and reverse entries into the merged slices: warp per two
// phase-A rows (lane per entry), so each lane has two slot atomics in flight
__global__ void scatter_kernel(const int32_t *__restrict__ ids,
                               const float *__restrict__ dists,
                               const int32_t *__restrict__ counts, int64_t n,
                               int width, const int64_t *__restrict__ mrg_off,
                               int32_t *__restrict__ rev_left,
                               uint64_t *__restrict__ keys, int64_t vlo, int64_t vhi) {
  // one pass of SCATTER_PASSES: only entries whose target slice (v for a
  // reverse entry, u for an own entry) lies in [vlo, vhi) are written, so
  // the pass's scattered 8-byte writes stay inside an L2-sized part of the
  // key array (no partial-sector write-backs to DRAM)
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < n; u += 2 * nw) {
    const int64_t u2 = u + nw;
    const int c1 = counts[u], c2 = u2 < n ? counts[u2] : 0;
    const int64_t o1 = mrg_off[u], o2 = u2 < n ? mrg_off[u2] : 0;
    for (int j = lane; j < max(c1, c2); j += 32) {
      const bool p1 = j < c1, p2 = j < c2;
      int32_t v1 = p1 ? ids[u * width + j] : 0, v2 = p2 ? ids[u2 * width + j] : 0;
      const float d1 = p1 ? dists[u * width + j] : 0.f, d2 = p2 ? dists[u2 * width + j] : 0.f;
      // an id outside [0, n) (a precondition violation the host shim rejects
      // with ValueError) becomes the row's own id, which the scan skips: no
      // write or gather ever leaves the buffers
      const bool r1 = p1 && (uint64_t)v1 < (uint64_t)n, r2 = p2 && (uint64_t)v2 < (uint64_t)n;
      if (p1 && !r1) v1 = (int32_t)u;
      if (p2 && !r2) v2 = (int32_t)u2;
      const bool w1 = r1 && v1 >= vlo && v1 < vhi, w2 = r2 && v2 >= vlo && v2 < vhi;
      int s1 = 0, s2 = 0;
      if (w1) s1 = atomicSub(rev_left + v1, 1) - 1;
      if (w2) s2 = atomicSub(rev_left + v2, 1) - 1;
      const int64_t b1 = w1 ? mrg_off[v1] + counts[v1] : 0;
      const int64_t b2 = w2 ? mrg_off[v2] + counts[v2] : 0;
      if (p1 && u >= vlo && u < vhi) keys[o1 + j] = pack_key(d1, v1);     // own entry
      if (w1) keys[b1 + s1] = pack_key(d1, (int32_t)u);                   // reverse
      if (p2 && u2 >= vlo && u2 < vhi) keys[o2 + j] = pack_key(d2, v2);
      if (w2) keys[b2 + s2] = pack_key(d2, (int32_t)u2);
    }
  }
}

// Drop consecutive duplicate ids from a sorted key run, writing ids/dists at
// out; returns the kept count.  Warp-cooperative.
__device__ __forceinline__ int warp_dedupe(const uint64_t *s, int len,
                                           int32_t *out_ids, float *out_d,
                                           int lane) {
  int m = 0;
  for (int b = 0; b < len; b += 32) {
    int i = b + lane;
    bool keep = false;
    uint64_t k = 0;
    if (i < len) {
      k = s[i];
      keep = (i == 0) || key_id(s[i - 1]) != key_id(k);
    }
    unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      int p = m + __popc(bal & lanemask_lt());
      out_ids[p] = key_id(k);
      out_d[p] = key_dist(k);
    }
    m += __popc(bal);
  }
  return m;
}

// Register bitonic sort of 32*NPL keys (element i = slot*32 + lane), then the
// consecutive-duplicate-id removal of warp_dedupe on the sorted registers.
template <int NPL>
__device__ __forceinline__ int reg_sort_dedupe(const uint64_t *__restrict__ keys, int len,
                                               int32_t *__restrict__ out_ids,
                                               float *__restrict__ out_d, int lane) {
  constexpr int SIZE = 32 * NPL;
  uint64_t e[NPL];
#pragma unroll
  for (int s0 = 0; s0 < NPL; ++s0) {
    const int i = s0 * 32 + lane;
    e[s0] = i < len ? keys[i] : KEY_MAX;
  }
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
  int m = 0;
  uint64_t last = 0;  // previous slot's lane-31 key
#pragma unroll
  for (int s0 = 0; s0 < NPL; ++s0) {
    if (s0 * 32 >= len) break;
    uint64_t prev = __shfl_up_sync(0xffffffffu, e[s0], 1);
    if (lane == 0) prev = last;
    last = __shfl_sync(0xffffffffu, e[s0], 31);
    const int i = s0 * 32 + lane;
    const bool keep = i < len && (i == 0 || key_id(prev) != key_id(e[s0]));
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      const int p = m + __popc(bal & lanemask_lt());
      out_ids[p] = key_id(e[s0]);
      out_d[p] = key_dist(e[s0]);
    }
    m += __popc(bal);
  }
  return m;
}

// A slice of own <= 32 entries (the phase-A row, already ascending) and
// rev <= 32 reverse entries (arrival order): sort only the reverse part (one
// key per lane), then one bitonic merge with the own part -- 26 shuffle
// stages against 40 for sorting all 64 -- and the same duplicate drop.
// (register core: e0 = the ascending own part, r = the unsorted reverse part,
// KEY_MAX past their lengths; len = own + rev)
__device__ __forceinline__ int merge_own_rev_regs(uint64_t e0, uint64_t r, int len, int nr,
                                                  int32_t *__restrict__ out_ids,
                                                  float *__restrict__ out_d, int lane) {
  // nr keys sit in lanes 0..nr-1 of r (KEY_MAX behind them): the network only
  // has to sort the first power-of-two block that holds them (warp-uniform)
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
    if ((k >> 1) >= nr) break;
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint64_t o = __shfl_xor_sync(0xffffffffu, r, j);
      const bool up = (lane & k) == 0, lower = (lane & j) == 0;
      const uint64_t mn = r < o ? r : o, mx = r < o ? o : r;
      r = (lower == up) ? mn : mx;
    }
  }
  // own ascending ++ reverse descending is bitonic (64 keys, slot*32 + lane)
  uint64_t e1 = __shfl_sync(0xffffffffu, r, 31 - lane);
  {
    const uint64_t mn = e0 < e1 ? e0 : e1, mx = e0 < e1 ? e1 : e0;
    e0 = mn;
    e1 = mx;
  }
#pragma unroll
  for (int j = 16; j > 0; j >>= 1) {
    const bool lower = (lane & j) == 0;
    const uint64_t o0 = __shfl_xor_sync(0xffffffffu, e0, j);
    const uint64_t o1 = __shfl_xor_sync(0xffffffffu, e1, j);
    e0 = lower ? (e0 < o0 ? e0 : o0) : (e0 < o0 ? o0 : e0);
    e1 = lower ? (e1 < o1 ? e1 : o1) : (e1 < o1 ? o1 : e1);
  }
  int m = 0;
  uint64_t last = 0;
#pragma unroll
  for (int s0 = 0; s0 < 2; ++s0) {
    const uint64_t v = s0 == 0 ? e0 : e1;
    if (s0 * 32 >= len) break;
    uint64_t prev = __shfl_up_sync(0xffffffffu, v, 1);
    if (lane == 0) prev = last;
    last = __shfl_sync(0xffffffffu, v, 31);
    const int i = s0 * 32 + lane;
    const bool keep = i < len && (i == 0 || key_id(prev) != key_id(v));
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      const int p = m + __popc(bal & lanemask_lt());
      out_ids[p] = key_id(v);
      out_d[p] = key_dist(v);
    }
    m += __popc(bal);
  }
  return m;
}

__device__ __forceinline__ int merge_own_rev(const uint64_t *__restrict__ keys, int own, int rev,
                                             int32_t *__restrict__ out_ids,
                                             float *__restrict__ out_d, int lane) {
  const uint64_t e0 = lane < own ? keys[lane] : KEY_MAX;
  const uint64_t r = lane < rev ? keys[own + lane] : KEY_MAX;
  return merge_own_rev_regs(e0, r, own + rev, rev, out_ids, out_d, lane);
}

// ---------------------------------------------------------------------------
// Fused merge + re-prune of short unions (exact-integer rows, rng / slack).
// At config 2 68 % of the merged rows hold <= 32 candidates: too little work
// for the tcgen05 Gram pipeline, whose per-point hand-offs (gather -> MMA ->
// masks -> greedy) cost more than the row itself.  Here the warp that merged
// the slice keeps it in registers and prunes it on the spot:
//   * lane t = candidate t; lane (g, tig) = (lane / 4, lane % 4) loads 32 bytes
//     of each of the rows g, g + 8, g + 16, g + 24 (two LDG.128 per row);
//   * the 32 x 32 Gram matrix C C^T (exact s32) by warp-level
//     mma.sync.m16n8k32.u8.u8 on exactly those registers -- a lane's rows are
//     both its A fragments (rows g, g + 8 of an m-tile) and its B fragments
//     (column g of an n-tile), and the k order is the same lane-local word
//     order on both sides, so no data moves between lanes; lower-triangle
//     tiles only;
//   * the dominance masks, the greedy scan and the lazy-evaluation counters of
//     prune_gram_kernel (prune_gram.cu: same integer compare, same popcount
//     formulas), on one 32-bit mask per candidate.
// No shared-memory tiles, no TMEM, no barriers; the merged row never travels
// through HBM.  Rows with more than 32 merged candidates are written to the
// merged CSR as before for the tcgen05 kernels; slices too long for the
// two-part merge are listed (todo) for merge_sort_kernel.
__device__ __forceinline__ void mma_u8_16832(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                             uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

struct FusedOut {
  const uint8_t *xu8;      // (N, 128) exact-integer rows
  const int32_t *norms;    // |x|^2
  int strategy;            // 0 rng, 2 slack
  double p;                // slack: s^2
  int M, width;
  int32_t *out_ids;
  float *out_dists;
  int32_t *out_counts;
  int64_t *dist_evals, *angle_evals;
};

// lane t holds candidate t (id < 0 past m), m <= 32, ascending (dist, id)
__device__ __forceinline__ void warp_prune_u8(const FusedOut &o, int64_t u, int m, int32_t id,
                                              float dv, int lane) {
  const int g = lane >> 2, tig = lane & 3;
  const int nv = id >= 0 ? o.norms[id] : 0;
  // rows g + 8q, 32 bytes each: words 0..3 = bytes 16 tig.., 4..7 = bytes 64 + 16 tig..
  uint32_t w[4][8];
  const int nq = (m + 7) >> 3;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int32_t rid = __shfl_sync(0xffffffffu, id, g + 8 * q);
    uint4 lo = make_uint4(0, 0, 0, 0), hi = lo;
    if (q < nq && rid >= 0) {
      const uint4 *rp = reinterpret_cast<const uint4 *>(o.xu8 + (int64_t)rid * 128);
      lo = __ldg(rp + tig);
      hi = __ldg(rp + 4 + tig);
    }
    w[q][0] = lo.x; w[q][1] = lo.y; w[q][2] = lo.z; w[q][3] = lo.w;
    w[q][4] = hi.x; w[q][5] = hi.y; w[q][6] = hi.z; w[q][7] = hi.w;
  }
  // c_i dominates c_t iff |c_i|^2 - 2 G[t][i] <= thr_t (prune_gram.cu: dle - |c_t|^2)
  int dle;
  if (dv >= 2.0e9f) {
    dle = 0x7fffffff;
  } else if (o.strategy != 2) {
    const float fl = floorf(dv);
    const int x = (int)fl - (fl == dv ? 1 : 0);
    dle = x > 0 ? x : 0;
  } else {
    const double p = o.p;
    int64_t x = (int64_t)floor((double)dv / p);
    while (x >= 0 && !(p * (double)x < (double)dv)) --x;
    while (p * (double)(x + 1) < (double)dv) ++x;
    dle = (int)(x > 0 ? x : 0);
  }
  const int thr = dle == 0x7fffffff ? 0x7fffffff : dle - nv;
  // Gram tiles (m-tile mt: rows 16 mt.., n-tile j: columns 8 j..), lower
  // triangle; one m-tile at a time (its accumulators become mask bits before
  // the next one is computed).  This lane's columns are 8 j + 2 tig + e, its
  // rows g + 8 q.
  int ncol[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    ncol[j][0] = __shfl_sync(0xffffffffu, nv, 8 * j + 2 * tig);
    ncol[j][1] = __shfl_sync(0xffffffffu, nv, 8 * j + 2 * tig + 1);
  }
  uint32_t mine = 0;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    if (mt == 1 && m <= 16) break;  // warp-uniform
    int acc[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j > 2 * mt + 1) continue;  // upper triangle: never read
        mma_u8_16832(acc[j], w[2 * mt][2 * ks], w[2 * mt + 1][2 * ks], w[2 * mt][2 * ks + 1],
                     w[2 * mt + 1][2 * ks + 1], w[j][2 * ks], w[j][2 * ks + 1]);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int q = 2 * mt + h;
      const int thq = __shfl_sync(0xffffffffu, thr, g + 8 * q);
      uint32_t pmq = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j > 2 * mt + 1) continue;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const bool dom = ncol[j][e] - 2 * acc[j][2 * h + e] <= thq;
          pmq |= dom ? (1u << (8 * j + 2 * tig + e)) : 0u;
        }
      }
      pmq |= __shfl_xor_sync(0xffffffffu, pmq, 1);
      pmq |= __shfl_xor_sync(0xffffffffu, pmq, 2);
      // candidate t = g' + 8 q' reads row slot q' of lane 4 g'
      const uint32_t got = __shfl_sync(0xffffffffu, pmq, 4 * (lane & 7));
      if ((lane >> 3) == q) mine = got;
    }
  }
  const uint32_t zu = __ballot_sync(0xffffffffu, dv == 0.0f);  // duw == 0: no distance computed
  const uint32_t pm = (mine | zu) & lanemask_lt();
  const uint32_t ex = __ballot_sync(0xffffffffu, lane < m && id != (int32_t)u);
  // greedy scan (_kernels.py:364-427): first candidate not dominated by a kept one
  uint32_t km = 0, mm = ex;
  int kept = 0, stop_j = 32;
  while (mm) {
    const int li = __ffs(mm) - 1;
    km |= 1u << li;
    if (++kept == o.M) {
      stop_j = li;
      break;
    }
    const uint32_t dom = __ballot_sync(0xffffffffu, (pm >> li) & 1u);
    mm &= ~(dom | ((2u << li) - 1u));
  }
  // kept candidates in scan order as one padded row
  {
    const int src_lane = __fns(km, 0, lane + 1);  // lane of the (lane+1)-th kept candidate
    const int32_t kid = __shfl_sync(0xffffffffu, id, src_lane & 31);
    const float kd = __shfl_sync(0xffffffffu, dv, src_lane & 31);
    for (int j = lane; j < o.width; j += 32) {
      const bool has = j < kept;  // kept <= 32: only j == lane can be kept
      o.out_ids[u * o.width + j] = has ? kid : -1;
      o.out_dists[u * o.width + j] = has ? kd : __int_as_float(0x7f800000);
    }
  }
  // exact lazy counters of every examined candidate
  long long ev = 0;
  if (lane <= stop_j && ((ex >> lane) & 1u)) {
    const uint32_t d = pm & km;  // pm holds only earlier candidates
    const int f = d ? __ffs(d) - 1 : -1;
    const int end = f >= 0 ? f : lane;
    ev = __popc(km & ((1u << end) - 1u));
    if (f >= 0 && !((zu >> f) & 1u)) ev += 1;
  }
#pragma unroll
  for (int of = 16; of > 0; of >>= 1) ev += __shfl_xor_sync(0xffffffffu, ev, of);
  if (lane == 0) {
    o.dist_evals[u] = ev;
    o.angle_evals[u] = 0;
    o.out_counts[u] = kept;
  }
}

// FUSED: slices whose merged row holds <= 32 candidates are pruned by the
// merging warp itself (warp_prune_u8) and marked mrg_counts = -1, which the
// tcgen05 kernels skip; rows are walked in the caller's locality order.
// the general register sort of one slice (every length up to SORT_SMEM_KEYS)
__device__ __forceinline__ int sort_slice(const uint64_t *__restrict__ keys, int own, int len,
                                          int32_t *__restrict__ out_ids,
                                          float *__restrict__ out_d, int lane) {
  if (len > 32 && own <= 32 && len - own <= 32)
    return merge_own_rev(keys, own, len - own, out_ids, out_d, lane);
  if (len <= 32) return reg_sort_dedupe<1>(keys, len, out_ids, out_d, lane);
  if (len <= 64) return reg_sort_dedupe<2>(keys, len, out_ids, out_d, lane);
  if (len <= 128) return reg_sort_dedupe<4>(keys, len, out_ids, out_d, lane);
  if (len <= 256) return reg_sort_dedupe<8>(keys, len, out_ids, out_d, lane);
  return reg_sort_dedupe<16>(keys, len, out_ids, out_d, lane);
}

__global__ void __launch_bounds__(SORT_WARPS * 32)
    merge_sort_kernel(const int64_t *__restrict__ mrg_off, int64_t n,
                      const int32_t *__restrict__ own_counts,
                      const uint64_t *__restrict__ keys,
                      int32_t *__restrict__ mrg_ids, float *__restrict__ mrg_d,
                      int32_t *__restrict__ mrg_counts,
                      int32_t *__restrict__ long_list,
                      int32_t *__restrict__ long_count,
                      const int32_t *__restrict__ todo, const int32_t *__restrict__ todo_count) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // after merge_prune_kernel: only the slices it listed (todo), else every row
  const int64_t rows = todo ? (int64_t)*todo_count : n;
  for (int64_t i = (int64_t)blockIdx.x * SORT_WARPS + warp; i < rows;
       i += (int64_t)gridDim.x * SORT_WARPS) {
    const int64_t u = todo ? (int64_t)todo[i] : i;
    const int64_t lo = mrg_off[u];
    const int len = (int)(mrg_off[u + 1] - lo);
    if (len > SORT_SMEM_KEYS) {
      if (lane == 0) long_list[atomicAdd(long_count, 1)] = (int32_t)u;
      continue;
    }
    const int m = sort_slice(keys + lo, own_counts[u], len, mrg_ids + lo, mrg_d + lo, lane);
    if (lane == 0) mrg_counts[u] = m;
  }
}

// Fused form: slices whose merged row holds <= 32 candidates are pruned by the
// merging warp itself (warp_prune_u8) and marked mrg_counts = -1, which the
// tcgen05 kernels skip; rows are walked in the caller's locality order.  A
// warp's rows come in batches of 32 (lane l loads row l's id, offsets and own
// count: one exposed latency per 32 rows) and the next row's keys are loaded
// while the current row is merged and pruned.
constexpr int FUSED_WARPS = 8;
#ifndef FUSED_MINB
#define FUSED_MINB 3
#endif
__global__ void __launch_bounds__(FUSED_WARPS * 32, FUSED_MINB)
    merge_prune_kernel(const int64_t *__restrict__ mrg_off, int64_t n,
                       const int32_t *__restrict__ own_counts,
                       const uint64_t *__restrict__ keys,
                       int32_t *__restrict__ mrg_ids, float *__restrict__ mrg_d,
                       int32_t *__restrict__ mrg_counts, int32_t *__restrict__ todo,
                       int32_t *__restrict__ todo_count,
                       const int32_t *__restrict__ row_order, const FusedOut fo) {
  __shared__ int32_t sh_ids[FUSED_WARPS][64];
  __shared__ float sh_d[FUSED_WARPS][64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t *si = sh_ids[warp];
  float *sd = sh_d[warp];
  const int64_t i0 = (int64_t)blockIdx.x * FUSED_WARPS + warp;
  const int64_t stride = (int64_t)gridDim.x * FUSED_WARPS;
  const int64_t nw = i0 < n ? (n - 1 - i0) / stride + 1 : 0;  // this warp's rows
  for (int64_t kb = 0; kb < nw; kb += 32) {
    int64_t bu = 0, blo = 0;
    int blen = 0, bown = 0;
    if (kb + lane < nw) {
      const int64_t i = i0 + (kb + lane) * stride;
      bu = row_order ? (int64_t)row_order[i] : i;
      blo = mrg_off[bu];
      blen = (int)(mrg_off[bu + 1] - blo);
      bown = own_counts[bu];
    }
    const int nb = (int)min((int64_t)32, nw - kb);
    // keys of a short slice: A = own part (or the whole slice when len <= 32),
    // B = reverse part of a two-part slice
    auto load_keys = [&](int64_t lo, int len, int own, uint64_t &A, uint64_t &B) {
      const bool two = len > 32 && own <= 32 && len - own <= 32;
      A = B = KEY_MAX;
      if (two) {
        if (lane < own) A = keys[lo + lane];
        if (lane < len - own) B = keys[lo + own + lane];
      } else if (len <= 32) {
        if (lane < len) A = keys[lo + lane];
      }
    };
    uint64_t ka, kr;
    load_keys(__shfl_sync(0xffffffffu, blo, 0), __shfl_sync(0xffffffffu, blen, 0),
              __shfl_sync(0xffffffffu, bown, 0), ka, kr);
    for (int j = 0; j < nb; ++j) {
      const int64_t u = __shfl_sync(0xffffffffu, bu, j);
      const int64_t lo = __shfl_sync(0xffffffffu, blo, j);
      const int len = __shfl_sync(0xffffffffu, blen, j);
      const int own = __shfl_sync(0xffffffffu, bown, j);
      uint64_t na = KEY_MAX, nr = KEY_MAX;
      if (j + 1 < nb)
        load_keys(__shfl_sync(0xffffffffu, blo, j + 1), __shfl_sync(0xffffffffu, blen, j + 1),
                  __shfl_sync(0xffffffffu, bown, j + 1), na, nr);
      const bool two = len > 32 && own <= 32 && len - own <= 32;
      if (two || len <= 32) {
        // len <= 32: the whole slice sits in the part that gets sorted
        const int m = merge_own_rev_regs(two ? ka : KEY_MAX, two ? kr : ka, len,
                                         two ? len - own : len, si, sd, lane);
        __syncwarp();
        if (m <= 32) {
          const int32_t id = lane < m ? si[lane] : -1;
          const float dv = lane < m ? sd[lane] : 0.0f;
          __syncwarp();
          warp_prune_u8(fo, u, m, id, dv, lane);
          if (lane == 0) mrg_counts[u] = -1;  // done here
        } else {
          for (int t = lane; t < m; t += 32) {
            mrg_ids[lo + t] = si[t];
            mrg_d[lo + t] = sd[t];
          }
          if (lane == 0) mrg_counts[u] = m;
          __syncwarp();
        }
      } else if (lane == 0) {
        todo[atomicAdd(todo_count, 1)] = (int32_t)u;  // longer slices: merge_sort_kernel, next launch
      }
      ka = na;
      kr = nr;
    }
  }
}

// Long slices (in-degree beyond the shared-memory capacity; hubs): one block
// per node, bitonic sort in a pow2-padded global scratch, warp 0 dedupes.
__global__ void long_sort_kernel(const int64_t *__restrict__ mrg_off,
                                 const uint64_t *__restrict__ keys,
                                 uint64_t *__restrict__ scratch,
                                 const int32_t *__restrict__ long_list,
                                 const int32_t *__restrict__ long_count,
                                 int32_t *__restrict__ mrg_ids,
                                 float *__restrict__ mrg_d,
                                 int32_t *__restrict__ mrg_counts) {
  const int nl = *long_count;
  for (int li = blockIdx.x; li < nl; li += gridDim.x) {
    const int64_t u = long_list[li];
    const int64_t lo = mrg_off[u];
    const int len = (int)(mrg_off[u + 1] - lo);
    const int size = next_pow2(len);
    // scratch region for this node: keys slice of 2*len >= size entries is
    // reserved at 2*lo (the workspace holds 2x the key capacity)
    uint64_t *g = scratch + 2 * lo;
    for (int i = threadIdx.x; i < size; i += blockDim.x) g[i] = i < len ? keys[lo + i] : KEY_MAX;
    __syncthreads();
    for (int k = 2; k <= size; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = threadIdx.x; i < size; i += blockDim.x) {
          int ixj = i ^ j;
          if (ixj > i) {
            uint64_t a = g[i], b = g[ixj];
            bool up = (i & k) == 0;
            if ((a > b) == up) { g[i] = b; g[ixj] = a; }
          }
        }
        __syncthreads();
      }
    }
    if (threadIdx.x < 32) {
      int m = warp_dedupe(g, len, mrg_ids + lo, mrg_d + lo, threadIdx.x);
      if (threadIdx.x == 0) mrg_counts[u] = m;
    }
    __syncthreads();
  }
}

struct RevLayout {
  int32_t *rev_cnt, *rev_left, *long_list, *long_count, *todo_list, *todo_count;
  int64_t *mrg_off;
  uint64_t *keys, *scratch;
  int32_t *mrg_ids, *mrg_counts;
  float *mrg_d;
  int64_t *cap, *scan_tmp;
  void *prune_ws;
  size_t prune_bytes;
  size_t total;
};

static RevLayout rev_layout(void *ws, size_t ws_bytes, int64_t n, int64_t width) {
  RevLayout L{};
  Carve c(ws, ws_bytes);
  const int64_t cap = 2 * n * width;  // own + reverse entries <= 2 * sum(counts)
  L.rev_cnt = c.take<int32_t>(n);
  L.rev_left = c.take<int32_t>(n);
  L.long_list = c.take<int32_t>(n);
  L.long_count = c.take<int32_t>(1);
  L.todo_list = c.take<int32_t>(n);
  L.todo_count = c.take<int32_t>(1);
  L.mrg_off = c.take<int64_t>(n + 1);
  L.mrg_counts = c.take<int32_t>(n);
  L.keys = c.take<uint64_t>(cap);
  L.scratch = c.take<uint64_t>(2 * cap + 2);
  L.mrg_ids = c.take<int32_t>(cap);
  L.mrg_d = c.take<float>(cap);
  L.cap = c.take<int64_t>(n + 1);
  L.scan_tmp = c.take<int64_t>(scan_scratch(n + 1));
  L.prune_bytes = prune_workspace(n);
  L.prune_ws = c.take<char>(L.prune_bytes);
  L.total = c.off;
  return L;
}

int reverse_workspace(int64_t n, int64_t width, size_t *bytes) {
  *bytes = rev_layout(nullptr, 0, n, width).total;
  return PGK_OK;
}

int add_reverse_and_prune(const float *X, const uint8_t *xu8, const int32_t *norms,
                          const int32_t *row_order, int64_t n, int64_t d,
                          const int32_t *a_ids, const float *a_dists,
                          const int32_t *a_counts, int64_t a_width, int strategy,
                          double cos_alpha, int64_t M, int64_t out_width,
                          int32_t *out_ids, float *out_dists, int32_t *out_counts,
                          int64_t *dist_evals, int64_t *angle_evals, void *ws,
                          size_t ws_bytes, cudaStream_t stream) {
  if (n == 0) return PGK_OK;
  RevLayout L = rev_layout(ws, ws_bytes, n, a_width);
  if (L.total > ws_bytes) {
    set_error("reverse workspace too small: need %zu bytes, got %zu", L.total, ws_bytes);
    return PGK_ERR_NOMEM;
  }
  const int sms = num_sms();
  const int64_t edges = n * a_width;
  const unsigned eblocks = (unsigned)std::min<int64_t>((edges + 255) / 256, (int64_t)sms * 16);
  // warp-per-row kernels (rev_count, scatter): one warp per 2 rows at most
  const unsigned rblocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 15) / 16, (int64_t)sms * 16));

  PGK_CUDA(cudaMemsetAsync(L.rev_cnt, 0, sizeof(int32_t) * n, stream));
  PGK_CUDA(cudaMemsetAsync(L.long_count, 0, sizeof(int32_t), stream));
  PGK_CUDA(cudaMemsetAsync(L.todo_count, 0, sizeof(int32_t), stream));
  rev_count_kernel<<<rblocks, 256, 0, stream>>>(a_ids, a_counts, n, (int)a_width, L.rev_cnt);
  PGK_CHECK_LAUNCH("rev_count_kernel");

  // mrg_off[u] = sum_{t<u} (counts[t] + rev_cnt[t]); mrg_off[n] = total
  cap_kernel<<<eblocks, 256, 0, stream>>>(a_counts, L.rev_cnt, n, L.cap);
  PGK_CHECK_LAUNCH("cap_kernel");
  int rc = exclusive_scan(L.cap, L.mrg_off, n + 1, L.scan_tmp, stream);
  if (rc) return rc;
  PGK_CUDA(cudaMemcpyAsync(L.rev_left, L.rev_cnt, sizeof(int32_t) * n,
                           cudaMemcpyDeviceToDevice, stream));

  // key array (2 n R entries, 8 B) in node-range passes of <= ~64 MB each
  const int64_t passes = std::max<int64_t>(1, std::min<int64_t>(SCATTER_PASSES,
                                                                 (16 * n * a_width) >> 26));
  for (int64_t p = 0; p < passes; ++p) {
    const int64_t vlo = n * p / passes, vhi = n * (p + 1) / passes;
    scatter_kernel<<<rblocks, 256, 0, stream>>>(a_ids, a_dists, a_counts, n, (int)a_width,
                                                L.mrg_off, L.rev_left, L.keys, vlo, vhi);
    PGK_CHECK_LAUNCH("scatter_kernel");
  }

  const unsigned sblocks =
      (unsigned)std::min<int64_t>((n + SORT_WARPS - 1) / SORT_WARPS, (int64_t)sms * 8);
  // exact-integer rows on the tensor-core selection path, rng / slack, phase-A
  // rows of <= 32 entries: short unions are pruned by the merging warp itself
  FusedOut fo{xu8, norms, strategy, cos_alpha, (int)M, (int)out_width, out_ids, out_dists,
              out_counts, dist_evals, angle_evals};
  const bool fused = rev_fused_enabled() && xu8 && norms && d <= 128 && gram_enabled() &&
                     L.prune_bytes >= gram_workspace(n) && strategy != 1 && M >= 1 &&
                     out_width >= 1;
  if (fused) {
    const unsigned fblocks =
        (unsigned)std::min<int64_t>((n + FUSED_WARPS - 1) / FUSED_WARPS, (int64_t)sms * FUSED_MINB);
    merge_prune_kernel<<<fblocks, FUSED_WARPS * 32, 0, stream>>>(
        L.mrg_off, n, a_counts, L.keys, L.mrg_ids, L.mrg_d, L.mrg_counts, L.todo_list,
        L.todo_count, row_order, fo);
    PGK_CHECK_LAUNCH("merge_prune_kernel");
    merge_sort_kernel<<<sblocks, SORT_WARPS * 32, 0, stream>>>(
        L.mrg_off, n, a_counts, L.keys, L.mrg_ids, L.mrg_d, L.mrg_counts, L.long_list,
        L.long_count, L.todo_list, L.todo_count);
  } else {
    merge_sort_kernel<<<sblocks, SORT_WARPS * 32, 0, stream>>>(
        L.mrg_off, n, a_counts, L.keys, L.mrg_ids, L.mrg_d, L.mrg_counts, L.long_list,
        L.long_count, nullptr, nullptr);
  }
  PGK_CHECK_LAUNCH("merge_sort_kernel");
  long_sort_kernel<<<(unsigned)sms, 512, 0, stream>>>(L.mrg_off, L.keys, L.scratch,
                                                      L.long_list, L.long_count,
                                                      L.mrg_ids, L.mrg_d, L.mrg_counts);
  PGK_CHECK_LAUNCH("long_sort_kernel");

  return launch_prune(X, xu8, norms, n, d, nullptr, row_order, L.prune_ws, L.prune_bytes,
                      L.mrg_off, L.mrg_counts, L.mrg_ids, L.mrg_d, strategy,
                      cos_alpha, M, out_width, out_ids, out_dists, out_counts,
                      dist_evals, angle_evals, stream, /*short_rows=*/true);
}

}  // namespace pgk
