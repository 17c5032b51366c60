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
__device__ __forceinline__ int merge_own_rev(const uint64_t *__restrict__ keys, int own, int rev,
                                             int32_t *__restrict__ out_ids,
                                             float *__restrict__ out_d, int lane) {
  uint64_t e0 = lane < own ? keys[lane] : KEY_MAX;
  uint64_t r = lane < rev ? keys[own + lane] : KEY_MAX;
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
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
  const int len = own + rev;
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

__global__ void __launch_bounds__(SORT_WARPS * 32)
    merge_sort_kernel(const int64_t *__restrict__ mrg_off, int64_t n,
                      const int32_t *__restrict__ own_counts,
                      const uint64_t *__restrict__ keys,
                      int32_t *__restrict__ mrg_ids, float *__restrict__ mrg_d,
                      int32_t *__restrict__ mrg_counts,
                      int32_t *__restrict__ long_list,
                      int32_t *__restrict__ long_count) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t u = (int64_t)blockIdx.x * SORT_WARPS + warp; u < n;
       u += (int64_t)gridDim.x * SORT_WARPS) {
    const int64_t lo = mrg_off[u];
    const int len = (int)(mrg_off[u + 1] - lo);
    if (len > SORT_SMEM_KEYS) {
      if (lane == 0) long_list[atomicAdd(long_count, 1)] = (int32_t)u;
      continue;
    }
    int m;
    const int own = own_counts[u];
    if (len > 32 && own <= 32 && len - own <= 32)
      m = merge_own_rev(keys + lo, own, len - own, mrg_ids + lo, mrg_d + lo, lane);
    else if (len <= 32) m = reg_sort_dedupe<1>(keys + lo, len, mrg_ids + lo, mrg_d + lo, lane);
    else if (len <= 64) m = reg_sort_dedupe<2>(keys + lo, len, mrg_ids + lo, mrg_d + lo, lane);
    else if (len <= 128) m = reg_sort_dedupe<4>(keys + lo, len, mrg_ids + lo, mrg_d + lo, lane);
    else if (len <= 256) m = reg_sort_dedupe<8>(keys + lo, len, mrg_ids + lo, mrg_d + lo, lane);
    else m = reg_sort_dedupe<16>(keys + lo, len, mrg_ids + lo, mrg_d + lo, lane);
    if (lane == 0) mrg_counts[u] = m;
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
  int32_t *rev_cnt, *rev_left, *long_list, *long_count;
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
  merge_sort_kernel<<<sblocks, SORT_WARPS * 32, 0, stream>>>(
      L.mrg_off, n, a_counts, L.keys, L.mrg_ids, L.mrg_d, L.mrg_counts, L.long_list, L.long_count);
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
