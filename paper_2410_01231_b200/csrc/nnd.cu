// nnd.cu -- NN-Descent k0-NN graph (knng.py:40-125 and
// _kernels.py:737-946) plus the FastNSG list bookkeeping (mark_fresh,
// _kernels.py:722-733).
//
// Semantics kept exactly (the stop rule reads the update count, so the
// counts must be the reference's, not just the rows):
//   * init: each row takes the first k0 distinct draws (self skipped by the
//     x >= u shift), then is sorted by (dist, id) with the reference's
//     sequential fp32 squared_l2(data[v], data[u]);
//   * reverse lists: every (u -> v, dist, flag) lands in v's list; each list
//     keeps its rcap closest by (dist, id) (ids are distinct per list, so any
//     sort order of the scatter gives the same result);
//   * join sets: forward and reverse rows merged by (dist, id) (forward
//     first on equal keys), consecutive duplicate ids dropped, at most
//     cap_new flagged-new and cap_old old entries -- one set per node per
//     round, computed once and shared by every node that joins through it;
//   * join: node u scans its join set in order and, for each member v, v's
//     join set in order, skipping pairs with no new hop and ids already seen
//     (u included); each surviving w is inserted into u's row (strictly
//     better than the current worst, no duplicates).  The row's final
//     content does not depend on insertion order, the accepted-insert count
//     does, so the warp computes a chunk's distances in parallel and then
//     replays the inserts in the reference's order.
#include "common.cuh"

namespace pgk {
namespace nnd {

constexpr int MAXK = 128;  // k0 bound (row width)

// ---- init ----------------------------------------------------------------
// One thread per row picks ids (sequential by definition); a second pass
// (warp per row) computes distances and sorts.
__global__ void init_pick_kernel(const int64_t *__restrict__ draws, int64_t n, int D, int k0,
                                 int32_t *__restrict__ ids, int32_t *__restrict__ shortfall) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
       u += (int64_t)gridDim.x * blockDim.x) {
    int32_t *row = ids + u * k0;  // kept ascending by id while picking
    int cnt = 0;
    for (int t = 0; t < D && cnt < k0; ++t) {
      int64_t x = draws[u * D + t];
      if (x >= u) ++x;
      int lo = 0, hi = cnt;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (row[mid] < x) lo = mid + 1;
        else hi = mid;
      }
      if (lo < cnt && row[lo] == x) continue;
      for (int b = cnt; b > lo; --b) row[b] = row[b - 1];
      row[lo] = (int32_t)x;
      ++cnt;
    }
    shortfall[u] = k0 - cnt;
  }
}

// rows (all, or the listed ones): dists to the row's node, sorted by (dist, id)
__global__ void row_dists_sort_kernel(const float *__restrict__ X, int d, int64_t nrows,
                                      const int32_t *__restrict__ which, int k0,
                                      const int32_t *__restrict__ shortfall,
                                      int32_t *__restrict__ ids, float *__restrict__ dists) {
  __shared__ uint64_t sk[8][MAXK];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K2 = next_pow2(k0);
  for (int64_t r = (int64_t)blockIdx.x * 8 + warp; r < nrows; r += (int64_t)gridDim.x * 8) {
    const int64_t u = which ? (int64_t)which[r] : r;
    if (!which && shortfall && shortfall[u] != 0) continue;  // repaired later
    for (int j = lane; j < K2; j += 32) {
      uint64_t key = KEY_MAX;
      if (j < k0) {
        const int32_t v = ids[u * k0 + j];
        key = pack_key(sql2_seq<false>(X + (int64_t)v * d, X + u * d, d), v);
      }
      sk[warp][j] = key;
    }
    __syncwarp();
    warp_bitonic_sort(sk[warp], K2, lane);
    for (int j = lane; j < k0; j += 32) {
      ids[u * k0 + j] = key_id(sk[warp][j]);
      dists[u * k0 + j] = key_dist(sk[warp][j]);
    }
    __syncwarp();
  }
}

// ---- reverse lists ---------------------------------------------------------
__global__ void widen_kernel(const int32_t *__restrict__ in, int64_t m, int64_t *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

__global__ void rev_hist_kernel(const int32_t *__restrict__ ids, int64_t total,
                                int32_t *__restrict__ cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(cnt + ids[e], 1);
}

__global__ void rev_scatter_kernel(const int32_t *__restrict__ ids,
                                   const float *__restrict__ dists,
                                   const uint8_t *__restrict__ flags, int64_t n, int k0,
                                   const int64_t *__restrict__ off, int32_t *__restrict__ fill,
                                   uint64_t *__restrict__ slots) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * k0;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = e / k0;
    const int32_t v = ids[e];
    // (dist, id, flag) packed so key order == (dist, id) order
    const uint64_t key = ((uint64_t)f32_orderable(dists[e]) << 32) |
                         ((uint64_t)(uint32_t)u << 1) | (uint64_t)(flags[e] ? 1u : 0u);
    slots[off[v] + atomicAdd(fill + v, 1)] = key;
  }
}

// warp per node: sort its reverse slice, keep the rcap closest
constexpr int RSORT = 1024;  // shared staging per warp (longer lists sort in place)
__global__ void rev_cap_kernel(uint64_t *__restrict__ slots, const int64_t *__restrict__ off,
                               int64_t n, int rcap, int32_t *__restrict__ r_ids,
                               float *__restrict__ r_dists, uint8_t *__restrict__ r_flags,
                               int32_t *__restrict__ r_cnt) {
  __shared__ uint64_t sk[4][RSORT];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t v = (int64_t)blockIdx.x * 4 + warp; v < n; v += (int64_t)gridDim.x * 4) {
    const int64_t lo = off[v];
    const int m = (int)(off[v + 1] - lo);
    uint64_t *s = m <= RSORT ? sk[warp] : slots + lo;
    const int M2 = next_pow2(max(m, 1));
    if (m <= RSORT) {
      for (int j = lane; j < M2; j += 32) s[j] = j < m ? slots[lo + j] : KEY_MAX;
      __syncwarp();
      warp_bitonic_sort(s, M2, lane);
    } else {
      // rare hub: repeated selection of the minimum, rcap times (in place)
      for (int t = 0; t < rcap; ++t) {
        uint64_t best = KEY_MAX;
        int bi = -1;
        for (int j = t + lane; j < m; j += 32)
          if (s[j] < best) { best = s[j]; bi = j; }
        for (int o = 16; o > 0; o >>= 1) {
          const uint64_t ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ob < best) { best = ob; bi = oi; }
        }
        if (lane == 0) {
          const uint64_t tmp = s[t];
          s[t] = s[bi];
          s[bi] = tmp;
        }
        __syncwarp();
      }
    }
    const int keep = min(m, rcap);
    for (int j = lane; j < rcap; j += 32) {
      const uint64_t k = j < keep ? s[j] : KEY_MAX;
      r_ids[v * rcap + j] = j < keep ? (int32_t)((uint32_t)k >> 1) : -1;
      r_dists[v * rcap + j] = j < keep ? f32_from_orderable((uint32_t)(k >> 32))
                                       : __int_as_float(0x7f800000);
      r_flags[v * rcap + j] = j < keep ? (uint8_t)(k & 1u) : 0;
    }
    if (lane == 0) r_cnt[v] = keep;
    __syncwarp();
  }
}

// ---- join sets (_select_join) ---------------------------------------------
__global__ void join_set_kernel(const int32_t *__restrict__ ids, const float *__restrict__ dists,
                                const uint8_t *__restrict__ flags, int64_t n, int k0,
                                const int32_t *__restrict__ r_ids,
                                const float *__restrict__ r_dists,
                                const uint8_t *__restrict__ r_flags,
                                const int32_t *__restrict__ r_cnt, int rcap, int cap_new,
                                int cap_old, int32_t *__restrict__ js_ids,
                                uint8_t *__restrict__ js_new, int32_t *__restrict__ js_pos,
                                int32_t *__restrict__ js_cnt) {
  const int cap = cap_new + cap_old;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t *fi = ids + v * k0;
    const float *fd = dists + v * k0;
    const uint8_t *ff = flags + v * k0;
    const int32_t *ri = r_ids + v * rcap;
    const float *rd = r_dists + v * rcap;
    const uint8_t *rf = r_flags + v * rcap;
    const int rc = r_cnt[v];
    int i = 0, j = 0, m = 0, n_new = 0, n_old = 0;
    int32_t last = -1;
    while ((i < k0 || j < rc) && (n_new < cap_new || n_old < cap_old)) {
      bool take_f;
      if (j >= rc) take_f = true;
      else if (i < k0) take_f = fd[i] < rd[j] || (fd[i] == rd[j] && fi[i] <= ri[j]);
      else take_f = false;
      int32_t cid, cpos;
      bool cfl;
      if (take_f) {
        cid = fi[i];
        cfl = ff[i] != 0;
        cpos = i;
        ++i;
      } else {
        cid = ri[j];
        cfl = rf[j] != 0;
        cpos = -1;
        ++j;
      }
      if (cid == last) continue;
      last = cid;
      if (cfl ? n_new < cap_new : n_old < cap_old) {
        js_ids[v * cap + m] = cid;
        js_new[v * cap + m] = cfl;
        js_pos[v * cap + m] = cpos;
        ++m;
        if (cfl) ++n_new;
        else ++n_old;
      }
    }
    js_cnt[v] = m;
  }
}

// ---- join round ------------------------------------------------------------
constexpr int JWARPS = 4;
__global__ void __launch_bounds__(JWARPS * 32)
    join_kernel(const float *__restrict__ X, int64_t n, int d, int k0,
                const int32_t *__restrict__ ids, const float *__restrict__ dists,
                const uint8_t *__restrict__ flags, const int32_t *__restrict__ js_ids,
                const uint8_t *__restrict__ js_new, const int32_t *__restrict__ js_pos,
                const int32_t *__restrict__ js_cnt, int cap, int32_t *__restrict__ out_ids,
                float *__restrict__ out_dists, uint8_t *__restrict__ out_flags,
                int64_t *__restrict__ upd_counts, int64_t *__restrict__ dist_evals,
                int32_t *__restrict__ stamps, int nslots) {
  __shared__ uint64_t rk[JWARPS][MAXK];  // u's row, (dist, id) keys ascending
  __shared__ uint8_t rf[JWARPS][MAXK];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = blockIdx.x * JWARPS + warp;
  if (slot >= nslots) return;
  int32_t *seen = stamps + (int64_t)slot * n;
  uint64_t *R = rk[warp];
  uint8_t *F = rf[warp];
  for (int64_t u = slot; u < n; u += nslots) {
    const int32_t stamp = (int32_t)(u / nslots) + 1;
    for (int j = lane; j < k0; j += 32) {
      R[j] = pack_key(dists[u * k0 + j], ids[u * k0 + j]);
      F[j] = flags[u * k0 + j];
    }
    if (lane == 0) seen[u] = stamp;
    __syncwarp();
    const int nb = js_cnt[u];
    // sampled new forward edges become old for the next round
    for (int b = lane; b < nb; b += 32)
      if (js_new[u * cap + b] && js_pos[u * cap + b] >= 0) F[js_pos[u * cap + b]] = 0;
    __syncwarp();
    int64_t upd = 0, ev = 0;
    for (int b = 0; b < nb; ++b) {
      const int32_t v = js_ids[u * cap + b];
      const bool bnew = js_new[u * cap + b] != 0;
      const int nt = js_cnt[v];
      for (int t0 = 0; t0 < nt; t0 += 32) {
        const int t = t0 + lane;
        int32_t w = -1;
        if (t < nt && (bnew || js_new[v * cap + t])) {
          w = js_ids[v * cap + t];
          // ids are distinct within a join set: no two lanes share a w
          if (seen[w] == stamp) w = -1;
          else seen[w] = stamp;
        }
        const unsigned live = __ballot_sync(0xffffffffu, w >= 0);
        ev += __popc(live);
        uint64_t key =
            w >= 0 ? pack_key(sql2_seq<false>(X + u * d, X + (int64_t)w * d, d), w) : KEY_MAX;
        // replay row_insert in candidate (lane) order: a candidate is taken
        // iff it beats the current worst and is not already in the row
        unsigned todo = live;
        while (todo) {
          const uint64_t worst = R[k0 - 1];
          todo &= __ballot_sync(0xffffffffu, key < worst);
          if (!todo) break;
          const int src = __ffs(todo) - 1;
          todo &= todo - 1;
          const uint64_t x = __shfl_sync(0xffffffffu, key, src);
          // lower bound of x in R (k0 <= 128: 4 entries per lane)
          int below = 0;
          for (int j = lane; j < k0; j += 32) below += R[j] < x;
          const int pos = (int)__reduce_add_sync(0xffffffffu, (unsigned)below);
          if (R[pos] == x) continue;  // already present: rejected, not counted
          // shift R[pos..k0-2] one up (descending copy by lanes in two passes)
          uint64_t mv[MAXK / 32];
          uint8_t mf[MAXK / 32];
#pragma unroll
          for (int q = 0; q < MAXK / 32; ++q) {
            const int j = q * 32 + lane;
            mv[q] = (j >= pos && j < k0 - 1) ? R[j] : 0;
            mf[q] = (j >= pos && j < k0 - 1) ? F[j] : 0;
          }
          __syncwarp();
#pragma unroll
          for (int q = 0; q < MAXK / 32; ++q) {
            const int j = q * 32 + lane;
            if (j >= pos && j < k0 - 1) {
              R[j + 1] = mv[q];
              F[j + 1] = mf[q];
            }
          }
          if (lane == 0) {
            R[pos] = x;
            F[pos] = 1;
          }
          __syncwarp();
          ++upd;
        }
      }
    }
    for (int j = lane; j < k0; j += 32) {
      out_ids[u * k0 + j] = key_id(R[j]);
      out_dists[u * k0 + j] = key_dist(R[j]);
      out_flags[u * k0 + j] = F[j];
    }
    if (lane == 0) {
      upd_counts[u] = upd;
      dist_evals[u] = ev;
    }
    __syncwarp();
  }
}

// ---- mark_fresh: candidate ids absent from the row's previous list ---------
__global__ void mark_fresh_kernel(const int32_t *__restrict__ cand, int cw,
                                  const int32_t *__restrict__ ccnt,
                                  const int32_t *__restrict__ prev, int pw,
                                  const int32_t *__restrict__ pcnt, int64_t n,
                                  uint8_t *__restrict__ fresh) {
  __shared__ int32_t sp[8][512];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t u = (int64_t)blockIdx.x * 8 + warp; u < n; u += (int64_t)gridDim.x * 8) {
    const int pc = pcnt[u];
    const int P2 = next_pow2(max(pc, 1));
    for (int j = lane; j < P2; j += 32) sp[warp][j] = j < pc ? prev[u * pw + j] : 0x7fffffff;
    __syncwarp();
    warp_bitonic_sort(sp[warp], P2, lane);
    const int cc = ccnt[u];
    for (int j = lane; j < cw; j += 32) {
      bool f = false;
      if (j < cc) {
        const int32_t x = cand[u * cw + j];
        int lo = 0, hi = pc;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (sp[warp][mid] < x) lo = mid + 1;
          else hi = mid;
        }
        f = !(lo < pc && sp[warp][lo] == x);
      }
      fresh[u * cw + j] = f;
    }
    __syncwarp();
  }
}

}  // namespace nnd

size_t scan_scratch(int64_t m);
int exclusive_scan(const int64_t *in, int64_t *out, int64_t m, int64_t *scratch,
                   cudaStream_t stream);

int knng_init(const float *X, int64_t n, int64_t d, const int64_t *draws, int64_t D, int64_t k0,
              int32_t *ids, float *dists, int32_t *shortfall, cudaStream_t stream) {
  PGK_REQUIRE(k0 >= 1 && k0 <= nnd::MAXK && k0 < n, "need 1 <= k0 < n, k0 <= %d", nnd::MAXK);
  const unsigned g = (unsigned)num_sms() * 8;
  nnd::init_pick_kernel<<<g, 256, 0, stream>>>(draws, n, (int)D, (int)k0, ids, shortfall);
  PGK_CHECK_LAUNCH("init_pick_kernel");
  nnd::row_dists_sort_kernel<<<g, 256, 0, stream>>>(X, (int)d, n, nullptr, (int)k0, shortfall,
                                                    ids, dists);
  PGK_CHECK_LAUNCH("row_dists_sort_kernel");
  return PGK_OK;
}

int knng_sort_rows(const float *X, int64_t d, const int32_t *rows, int64_t nrows, int64_t k0,
                   int32_t *ids, float *dists, cudaStream_t stream) {
  if (nrows == 0) return PGK_OK;
  PGK_REQUIRE(k0 >= 1 && k0 <= nnd::MAXK, "bad k0");
  nnd::row_dists_sort_kernel<<<(unsigned)num_sms() * 8, 256, 0, stream>>>(
      X, (int)d, nrows, rows, (int)k0, nullptr, ids, dists);
  PGK_CHECK_LAUNCH("row_dists_sort_kernel");
  return PGK_OK;
}

size_t knng_round_workspace(int64_t n, int64_t k0, int64_t cap) {
  Carve c(nullptr, ~size_t(0));
  c.take<int32_t>(n + 1);            // reverse counts
  c.take<int32_t>(n + 1);            // fill cursors
  c.take<int64_t>(n + 1);            // offsets
  c.take<int64_t>(scan_scratch(n + 1));
  c.take<uint64_t>((size_t)n * k0);  // scattered reverse keys
  c.take<int32_t>((size_t)n * k0);   // capped reverse rows
  c.take<float>((size_t)n * k0);
  c.take<uint8_t>((size_t)n * k0);
  c.take<int32_t>(n);
  c.take<int32_t>((size_t)n * cap);  // join sets
  c.take<uint8_t>((size_t)n * cap);
  c.take<int32_t>((size_t)n * cap);
  c.take<int32_t>(n);
  const int64_t slots = std::min<int64_t>(n, 4 * 148);
  c.take<int32_t>((size_t)slots * n);  // seen stamps
  return c.off + 256;
}

// One NN-Descent round (knng.py:64-101): new rows / flags and per-node
// update and distance counts.
int knng_round(const float *X, int64_t n, int64_t d, int64_t k0, const int32_t *ids,
               const float *dists, const uint8_t *flags, int64_t cap_new, int64_t cap_old,
               int32_t *out_ids, float *out_dists, uint8_t *out_flags, int64_t *upd,
               int64_t *evals, void *ws, size_t ws_bytes, cudaStream_t stream) {
  PGK_REQUIRE(k0 >= 1 && k0 <= nnd::MAXK, "bad k0");
  const int64_t cap = cap_new + cap_old;
  PGK_REQUIRE(ws_bytes >= knng_round_workspace(n, k0, cap), "knng workspace too small");
  Carve c(ws, ws_bytes);
  int32_t *rcount = c.take<int32_t>(n + 1);
  int32_t *fill = c.take<int32_t>(n + 1);
  int64_t *off = c.take<int64_t>(n + 1);
  int64_t *scan_tmp = c.take<int64_t>(scan_scratch(n + 1));
  uint64_t *slots = c.take<uint64_t>((size_t)n * k0);
  int32_t *r_ids = c.take<int32_t>((size_t)n * k0);
  float *r_d = c.take<float>((size_t)n * k0);
  uint8_t *r_f = c.take<uint8_t>((size_t)n * k0);
  int32_t *r_cnt = c.take<int32_t>(n);
  int32_t *js_ids = c.take<int32_t>((size_t)n * cap);
  uint8_t *js_new = c.take<uint8_t>((size_t)n * cap);
  int32_t *js_pos = c.take<int32_t>((size_t)n * cap);
  int32_t *js_cnt = c.take<int32_t>(n);
  const int64_t nslots = std::min<int64_t>(n, 4 * 148);
  int32_t *stamps = c.take<int32_t>((size_t)nslots * n);
  const unsigned g = (unsigned)num_sms() * 8;
  PGK_CUDA(cudaMemsetAsync(rcount, 0, (n + 1) * 4, stream));
  PGK_CUDA(cudaMemsetAsync(fill, 0, (n + 1) * 4, stream));
  nnd::rev_hist_kernel<<<g, 256, 0, stream>>>(ids, n * k0, rcount);
  PGK_CHECK_LAUNCH("rev_hist_kernel");
  nnd::widen_kernel<<<g, 256, 0, stream>>>(rcount, n + 1, off);
  PGK_CHECK_LAUNCH("widen_kernel");
  int rc = exclusive_scan(off, off, n + 1, scan_tmp, stream);
  if (rc) return rc;
  nnd::rev_scatter_kernel<<<g, 256, 0, stream>>>(ids, dists, flags, n, (int)k0, off, fill,
                                                 slots);
  PGK_CHECK_LAUNCH("rev_scatter_kernel");
  const int rcap = (int)k0;  // knng.py:79-81: reverse rows capped at k0
  nnd::rev_cap_kernel<<<g, 128, 0, stream>>>(slots, off, n, rcap, r_ids, r_d, r_f, r_cnt);
  PGK_CHECK_LAUNCH("rev_cap_kernel");
  nnd::join_set_kernel<<<g, 256, 0, stream>>>(ids, dists, flags, n, (int)k0, r_ids, r_d, r_f,
                                              r_cnt, rcap, (int)cap_new, (int)cap_old, js_ids,
                                              js_new, js_pos, js_cnt);
  PGK_CHECK_LAUNCH("join_set_kernel");
  PGK_CUDA(cudaMemsetAsync(stamps, 0, (size_t)nslots * n * sizeof(int32_t), stream));
  const unsigned jg = (unsigned)((nslots + nnd::JWARPS - 1) / nnd::JWARPS);
  nnd::join_kernel<<<jg, nnd::JWARPS * 32, 0, stream>>>(
      X, n, (int)d, (int)k0, ids, dists, flags, js_ids, js_new, js_pos, js_cnt, (int)cap, out_ids,
      out_dists, out_flags, upd, evals, stamps, (int)nslots);
  PGK_CHECK_LAUNCH("join_kernel");
  return PGK_OK;
}

int mark_fresh(const int32_t *cand, int64_t cw, const int32_t *ccnt, const int32_t *prev,
               int64_t pw, const int32_t *pcnt, int64_t n, uint8_t *fresh,
               cudaStream_t stream) {
  PGK_REQUIRE(pw <= 512, "previous list width %lld > 512", (long long)pw);
  nnd::mark_fresh_kernel<<<(unsigned)num_sms() * 8, 256, 0, stream>>>(cand, (int)cw, ccnt, prev,
                                                                      (int)pw, pcnt, n, fresh);
  PGK_CHECK_LAUNCH("mark_fresh_kernel");
  return PGK_OK;
}

}  // namespace pgk
