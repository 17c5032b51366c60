// search.cu -- beam search and phase-C plumbing.
//
// Beam search (_kernels.py:49-135 _search_core, :193-245 extract_results /
// search_one / search_many): a pool of capacity L sorted by (dist, id) with
// "expanded" flags; repeatedly expand the first unexpanded entry u, offering
// every not-yet-visited neighbour v of u (adjacency order) with the
// reference's sequential fp32 squared_l2(data[v], q).  A bounded sorted pool
// that keeps the L smallest offers and rejects duplicates ends up with the L
// smallest (dist, id) of everything offered, whatever the insertion order, so
// the GPU offers one adjacency chunk at a time: lanes compute the chunk's
// distances in parallel, the warp sorts the (<= 32) new keys and merges them
// into the pool with flags carried along -- identical pool states, visited
// sets, distance counts and expansion order to the reference's loop.
//
// One warp per query (persistent over queries); pool in shared memory; the
// visited set is a per-warp-slot stamp array in global memory (stamp = query
// index + 1 within a call, zeroed per call for the slots in use).
//
// Phase C (prune.py:165-199): reachability as a one-CTA BFS over a
// 32-bit bitmap (graph.py:112-123 marks every node reachable by directed
// edges; the visiting order does not change the set), the first unreached id
// by a min-reduction, and a deterministic float64 centroid (core.py:153-155)
// for the entry point.
#include "common.cuh"

namespace pgk {
namespace srch {

constexpr int WARPS = 4;       // queries per CTA
constexpr int LMAX = 256;      // pool capacity bound (reference L)
constexpr int MAX_SLOTS = 4 * 148;

struct WarpPool {
  uint64_t key[2][LMAX];  // packed (orderable dist, id), double-buffered merge
  uint8_t flag[2][LMAX];
  uint64_t batch[32];
};

__device__ __forceinline__ int32_t kid(uint64_t k) { return (int32_t)(uint32_t)k; }

// rank of key x among sorted a[0..na): number of entries < x
__device__ __forceinline__ int lower_rank(const uint64_t *a, int na, uint64_t x) {
  int lo = 0, hi = na;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(WARPS * 32)
    beam_search_kernel(const float *__restrict__ X, int64_t n, int d,
                       const int32_t *__restrict__ adj, int width,
                       const int32_t *__restrict__ counts, const float *__restrict__ Q,
                       int64_t nq, int k, int L, const int32_t *__restrict__ eps, int32_t ep,
                       int32_t exclude, int32_t *__restrict__ out_ids,
                       float *__restrict__ out_dists, int64_t *__restrict__ dist_counts,
                       int64_t *__restrict__ n_expanded, int32_t *__restrict__ stamps,
                       int nslots, int32_t *__restrict__ exp_out, int exp_cap,
                       uint64_t *__restrict__ exp_worst) {
  __shared__ WarpPool pools[WARPS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = blockIdx.x * WARPS + warp;
  if (slot >= nslots) return;
  WarpPool &P = pools[warp];
  int32_t *vis = stamps + (int64_t)slot * n;
  for (int64_t qi = slot; qi < nq; qi += nslots) {
    const int32_t stamp = (int32_t)(qi / nslots) + 1;  // unique per slot in this call
    const float *q = Q + qi * d;
    const int32_t e0 = eps ? eps[qi] : ep;
    int cur = 0, size = 0;
    int64_t dc = 0, nexp = 0;
    // the entry point
    if (lane == 0) {
      vis[e0] = stamp;
      P.key[0][0] = pack_key(sql2_seq<false>(X + (int64_t)e0 * d, q, d), e0);
      P.flag[0][0] = 0;
    }
    size = 1;
    dc = 1;
    __syncwarp();
    for (;;) {
      // first unexpanded entry among the first min(size, L)
      int idx = -1;
      for (int b = 0; b < size && idx < 0; b += 32) {
        const int i = b + lane;
        const unsigned m = __ballot_sync(0xffffffffu, i < size && !P.flag[cur][i]);
        if (m) idx = b + __ffs(m) - 1;
      }
      if (idx < 0) break;
      const int32_t u = kid(P.key[cur][idx]);
      if (lane == 0) {
        P.flag[cur][idx] = 1;
        // expansion order record (phase-C speculation checks it)
        if (exp_out && nexp < exp_cap) exp_out[qi * exp_cap + nexp] = u;
      }
      ++nexp;
      __syncwarp();
      const int cu = counts[u];
      for (int j0 = 0; j0 < cu; j0 += 32) {
        const int j = j0 + lane;
        int32_t v = -1;
        if (j < cu) {
          v = adj[(int64_t)u * width + j];
          // rows hold distinct ids, so lanes never race on the same v
          if (vis[v] == stamp) v = -1;
          else vis[v] = stamp;
        }
        const unsigned m = __ballot_sync(0xffffffffu, v >= 0);
        dc += __popc(m);
        const uint64_t key =
            v >= 0 ? pack_key(sql2_seq<false>(X + (int64_t)v * d, q, d), v) : KEY_MAX;
        P.batch[lane] = key;
        __syncwarp();
        warp_bitonic_sort(P.batch, 32, lane);
        const int nb = __popc(m);
        // merge pool[cur] (size) with batch (nb) -> pool[cur^1], first L
        const int tot = min(size + nb, L);
        for (int i = lane; i < size; i += 32) {
          const uint64_t x = P.key[cur][i];
          const int pos = i + lower_rank(P.batch, nb, x);
          if (pos < tot) {
            P.key[cur ^ 1][pos] = x;
            P.flag[cur ^ 1][pos] = P.flag[cur][i];
          }
        }
        if (lane < nb) {
          const uint64_t x = P.batch[lane];
          const int pos = lane + lower_rank(P.key[cur], size, x);
          if (pos < tot) {
            P.key[cur ^ 1][pos] = x;
            P.flag[cur ^ 1][pos] = 0;
          }
        }
        __syncwarp();
        cur ^= 1;
        size = tot;
      }
      // the pool's admission bound once u's neighbours are in (phase-C
      // speculation: an extra neighbour offered last is rejected iff its
      // key is >= this; KEY_MAX while the pool is not full)
      if (exp_worst && lane == 0 && nexp - 1 < exp_cap)
        exp_worst[qi * exp_cap + nexp - 1] = size == L ? P.key[cur][size - 1] : KEY_MAX;
    }
    // results: the first k pool entries, skipping `exclude` (-2: the query's
    // own index, batch_self_search, _kernels.py:252-281)
    const int32_t ex = exclude == -2 ? (int32_t)qi : exclude;
    int m = 0;
    for (int b = 0; b < size && m < k; b += 32) {
      const int i = b + lane;
      const bool take = i < size && kid(P.key[cur][i]) != ex;
      const unsigned bal = __ballot_sync(0xffffffffu, take);
      const int pos = m + __popc(bal & lanemask_lt());
      if (take && pos < k) {
        const uint64_t x = P.key[cur][i];
        out_ids[qi * k + pos] = kid(x);
        out_dists[qi * k + pos] = key_dist(x);
      }
      m += __popc(bal);
    }
    for (int i = max(m, 0) + lane; i < k; i += 32) {
      out_ids[qi * k + i] = -1;
      out_dists[qi * k + i] = __int_as_float(0x7f800000);
    }
    if (lane == 0) {
      if (dist_counts) dist_counts[qi] = dc;
      if (n_expanded) n_expanded[qi] = nexp;
    }
    __syncwarp();
  }
}

// ---- reachability -------------------------------------------------------
// BFS body shared by the single-start and the component-heads kernels:
// marks everything reachable from the nodes in cur[0..n_cur) through unseen
// nodes (cur already marked).
__device__ void bfs_from(const int32_t *__restrict__ adj, int width,
                         const int32_t *__restrict__ counts, uint32_t *__restrict__ seen,
                         int32_t *cur, int32_t *nxt, int *n_cur, int *n_next) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x / 32;
  while (*n_cur > 0) {
    if (threadIdx.x == 0) *n_next = 0;
    __syncthreads();
    const int nc = *n_cur;
    for (int f = warp; f < nc; f += nwarps) {
      const int32_t u = cur[f];
      const int cu = counts[u];
      for (int j = lane; j < cu; j += 32) {
        const int32_t v = adj[(int64_t)u * width + j];
        const uint32_t bit = 1u << (v & 31);
        if (seen[v >> 5] & bit) continue;
        const uint32_t old = atomicOr(seen + (v >> 5), bit);
        if (!(old & bit)) nxt[atomicAdd(n_next, 1)] = v;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) *n_cur = *n_next;
    int32_t *t = cur;
    cur = nxt;
    nxt = t;
    __syncthreads();
  }
}

// Phase C's component heads in the reference's order (prune.py:174-199): the
// first unreached id, everything it reaches, the next first unreached id...
// The sequence does not depend on the repair edges (they leave nodes that are
// already reached), so one CTA computes it up front.
__global__ void __launch_bounds__(1024)
    component_heads_kernel(const int32_t *__restrict__ adj, int width,
                           const int32_t *__restrict__ counts, int64_t n,
                           uint32_t *__restrict__ seen, int32_t *__restrict__ qa,
                           int32_t *__restrict__ qb, int32_t *__restrict__ heads,
                           int32_t *__restrict__ n_heads) {
  __shared__ int n_cur, n_next, s_found;
  __shared__ int64_t s_word;
  const int64_t nwords = (n + 31) >> 5;
  int64_t w0 = 0;
  int m = 0;
  for (;;) {
    // first word at or after w0 with an unseen bit (blockwide scan)
    if (threadIdx.x == 0) {
      s_word = nwords;
      s_found = 0;
    }
    __syncthreads();
    for (int64_t base = w0; base < nwords && !s_found; base += blockDim.x) {
      const int64_t w = base + threadIdx.x;
      if (w < nwords) {
        uint32_t miss = ~seen[w];
        const int64_t hi = n - w * 32;
        if (hi < 32) miss &= (1u << hi) - 1u;
        if (miss) atomicMin((unsigned long long *)&s_word, (unsigned long long)w);
      }
      __syncthreads();
      if (threadIdx.x == 0 && s_word < nwords) s_found = 1;
      __syncthreads();
    }
    if (!s_found) break;
    const int64_t w = s_word;
    w0 = w;
    if (threadIdx.x == 0) {
      uint32_t miss = ~seen[w];
      const int64_t hi = n - w * 32;
      if (hi < 32) miss &= (1u << hi) - 1u;
      const int32_t v = (int32_t)(w * 32 + __ffs(miss) - 1);
      heads[m] = v;
      atomicOr(seen + (v >> 5), 1u << (v & 31));
      qa[0] = v;
      n_cur = 1;
    }
    ++m;
    __syncthreads();
    bfs_from(adj, width, counts, seen, qa, qb, &n_cur, &n_next);
  }
  if (threadIdx.x == 0) *n_heads = m;
}

// One CTA runs the whole BFS (device-side level loop over a global-memory
// queue): no host round trip per level, so deep / chain-like components
// (phase C on near-duplicate data) cost no more than their size.
constexpr int BFS_THREADS = 1024;
__global__ void __launch_bounds__(BFS_THREADS)
    bfs_block_kernel(const int32_t *__restrict__ adj, int width,
                     const int32_t *__restrict__ counts, int32_t start,
                     uint32_t *__restrict__ seen, int32_t *__restrict__ qa,
                     int32_t *__restrict__ qb) {
  __shared__ int n_cur, n_next;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = BFS_THREADS / 32;
  if (threadIdx.x == 0) {
    const uint32_t bit = 1u << (start & 31);
    const uint32_t old = atomicOr(seen + (start >> 5), bit);
    n_cur = (old & bit) ? 0 : 1;
    qa[0] = start;
  }
  __syncthreads();
  int32_t *cur = qa, *nxt = qb;
  while (n_cur > 0) {
    if (threadIdx.x == 0) n_next = 0;
    __syncthreads();
    const int nc = n_cur;
    for (int f = warp; f < nc; f += nwarps) {
      const int32_t u = cur[f];
      const int cu = counts[u];
      for (int j = lane; j < cu; j += 32) {
        const int32_t v = adj[(int64_t)u * width + j];
        const uint32_t bit = 1u << (v & 31);
        if (seen[v >> 5] & bit) continue;
        const uint32_t old = atomicOr(seen + (v >> 5), bit);
        if (!(old & bit)) nxt[atomicAdd(&n_next, 1)] = v;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) n_cur = n_next;
    int32_t *t = cur;
    cur = nxt;
    nxt = t;
    __syncthreads();
  }
}

__global__ void first_unseen_kernel(const uint32_t *__restrict__ seen, int64_t n,
                                    int32_t *__restrict__ out) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w * 32 < n;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t miss = ~seen[w];
    const int64_t hi = n - w * 32;
    if (hi < 32) miss &= (1u << hi) - 1u;
    if (miss) atomicMin(out, (int32_t)(w * 32 + __ffs(miss) - 1));
  }
}

// ---- centroid: deterministic float64 column means ---------------------
// numpy's mean(axis=0, dtype=float64) on a C-contiguous (n, d) array adds the
// rows to the float64 accumulator in order (core.py:153-155): one thread per
// column does exactly that, rows loaded 8 ahead (the adds are a dependent
// chain; the loads are not).
__global__ void centroid_seq_kernel(const float *__restrict__ X, int64_t n, int d,
                                    float *__restrict__ out) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= d) return;
  double s = 0.0;
  int64_t r = 0;
  for (; r + 8 <= n; r += 8) {
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = X[(r + i) * d + col];
#pragma unroll
    for (int i = 0; i < 8; ++i) s += (double)v[i];
  }
  for (; r < n; ++r) s += (double)X[r * d + col];
  out[col] = (float)(s / (double)n);
}

}  // namespace srch

size_t search_workspace(int64_t n, int64_t nq) {
  const int64_t slots = std::min<int64_t>(std::max<int64_t>(nq, 1), srch::MAX_SLOTS);
  return (size_t)slots * n * sizeof(int32_t) + 256;
}

int beam_search(const float *X, int64_t n, int64_t d, const int32_t *adj, int64_t width,
                const int32_t *counts, const float *Q, int64_t nq, int64_t k, int64_t L,
                const int32_t *eps, int32_t ep, int32_t exclude, int32_t *out_ids,
                float *out_dists, int64_t *dist_counts, int64_t *n_expanded, void *ws,
                size_t ws_bytes, cudaStream_t stream, int32_t *exp_out, int64_t exp_cap,
                uint64_t *exp_worst) {
  PGK_REQUIRE(n >= 1 && d >= 1 && width >= 1, "empty graph");
  PGK_REQUIRE(k >= 1, "k must be >= 1");
  PGK_REQUIRE(k <= L, "k must not exceed the pool width L");
  PGK_REQUIRE(L <= srch::LMAX, "pool width L=%lld exceeds %d", (long long)L, srch::LMAX);
  PGK_REQUIRE(eps || (ep >= 0 && ep < n), "entry point out of range");
  if (nq == 0) return PGK_OK;
  PGK_REQUIRE(ws_bytes >= search_workspace(n, nq), "search workspace too small");
  const int64_t slots = std::min<int64_t>(nq, srch::MAX_SLOTS);
  int32_t *stamps = reinterpret_cast<int32_t *>(ws);
  PGK_CUDA(cudaMemsetAsync(stamps, 0, (size_t)slots * n * sizeof(int32_t), stream));
  const unsigned grid = (unsigned)((slots + srch::WARPS - 1) / srch::WARPS);
  srch::beam_search_kernel<<<grid, srch::WARPS * 32, 0, stream>>>(
      X, n, (int)d, adj, (int)width, counts, Q, nq, (int)k, (int)L, eps, ep, exclude, out_ids,
      out_dists, dist_counts, n_expanded, stamps, (int)slots, exp_out, (int)exp_cap,
      exp_worst);
  PGK_CHECK_LAUNCH("beam_search_kernel");
  return PGK_OK;
}

size_t reach_workspace(int64_t n) { return (size_t)(2 * n + 64) * sizeof(int32_t) + 512; }

// Extend the reachability bitmap `seen` ((n + 31) / 32 words) by everything
// reachable from `start` through unseen nodes (start itself included).
// Enqueued on the stream (no host sync).
int mark_reachable(const int32_t *adj, int64_t width, const int32_t *counts, int64_t n,
                   int32_t start, uint32_t *seen, void *ws, size_t ws_bytes,
                   cudaStream_t stream) {
  PGK_REQUIRE(start >= 0 && start < n, "start node out of range");
  PGK_REQUIRE(ws_bytes >= reach_workspace(n), "reach workspace too small");
  Carve c(ws, ws_bytes);
  c.take<int32_t>(64);
  int32_t *fa = c.take<int32_t>(n), *fb = c.take<int32_t>(n);
  srch::bfs_block_kernel<<<1, srch::BFS_THREADS, 0, stream>>>(adj, (int)width, counts, start,
                                                              seen, fa, fb);
  PGK_CHECK_LAUNCH("bfs_block_kernel");
  return PGK_OK;
}

// All component heads of the unreached remainder, in order (marks them and
// what they reach in `seen`); *n_heads_host receives the count (blocking).
int component_heads(const int32_t *adj, int64_t width, const int32_t *counts, int64_t n,
                    uint32_t *seen, int32_t *heads, int32_t *n_heads_host, void *ws,
                    size_t ws_bytes, cudaStream_t stream) {
  PGK_REQUIRE(ws_bytes >= reach_workspace(n), "reach workspace too small");
  Carve c(ws, ws_bytes);
  int32_t *cnt = c.take<int32_t>(64);
  int32_t *fa = c.take<int32_t>(n), *fb = c.take<int32_t>(n);
  srch::component_heads_kernel<<<1, 1024, 0, stream>>>(adj, (int)width, counts, n, seen, fa, fb,
                                                       heads, cnt);
  PGK_CHECK_LAUNCH("component_heads_kernel");
  PGK_CUDA(cudaMemcpyAsync(n_heads_host, cnt, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
  PGK_CUDA(cudaStreamSynchronize(stream));
  return PGK_OK;
}

// Smallest id whose bit is clear in `seen`, or -1 (blocking).
int first_unseen(const uint32_t *seen, int64_t n, int32_t *out_host, void *ws,
                 cudaStream_t stream) {
  int32_t *dv = reinterpret_cast<int32_t *>(ws);
  const int32_t big = 0x7fffffff;
  PGK_CUDA(cudaMemcpyAsync(dv, &big, sizeof(int32_t), cudaMemcpyHostToDevice, stream));
  srch::first_unseen_kernel<<<(unsigned)num_sms() * 4, 256, 0, stream>>>(seen, n, dv);
  PGK_CHECK_LAUNCH("first_unseen_kernel");
  int32_t h = big;
  PGK_CUDA(cudaMemcpyAsync(&h, dv, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
  PGK_CUDA(cudaStreamSynchronize(stream));
  *out_host = h == big ? -1 : h;
  return PGK_OK;
}

// squared_l2(data[a[i]], data[b[i]]) (the reference's sequential fp32)
__global__ void pair_dists_kernel(const float *__restrict__ X, int d, const int32_t *__restrict__ a,
                                  const int32_t *__restrict__ b, int64_t m,
                                  float *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = sql2_seq<false>(X + (int64_t)a[i] * d, X + (int64_t)b[i] * d, d);
}

int pair_dists(const float *X, int64_t d, const int32_t *a, const int32_t *b, int64_t m,
               float *out, cudaStream_t stream) {
  if (m == 0) return PGK_OK;
  pair_dists_kernel<<<(unsigned)std::min<int64_t>((m + 255) / 256, (int64_t)num_sms() * 8), 256,
                      0, stream>>>(X, (int)d, a, b, m, out);
  PGK_CHECK_LAUNCH("pair_dists_kernel");
  return PGK_OK;
}

size_t centroid_workspace(int64_t n, int64_t d) {
  (void)n;
  (void)d;
  return 256;  // (kept in the ABI: the sequential kernel needs none)
}

int centroid(const float *X, int64_t n, int64_t d, float *out, void *ws, size_t ws_bytes,
             cudaStream_t stream) {
  PGK_REQUIRE(n >= 1 && d >= 1, "empty dataset");
  PGK_REQUIRE(ws_bytes >= centroid_workspace(n, d), "centroid workspace too small");
  (void)ws;
  srch::centroid_seq_kernel<<<(unsigned)((d + 63) / 64), 64, 0, stream>>>(X, n, (int)d, out);
  PGK_CHECK_LAUNCH("centroid_seq_kernel");
  return PGK_OK;
}

}  // namespace pgk
