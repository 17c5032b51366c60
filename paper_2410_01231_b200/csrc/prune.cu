// prune.cu -- phase-A edge selection (the reference's _prune_row /
// prune_batch, _kernels.py:364-427) as a warp-per-point sm_100a kernel.
//
// Layout: one warp owns one point u.  The candidate slice is processed in
// windows of W entries held in shared memory (id, dist, per-entry counters)
// plus an order-preserving "alive" index list.  The greedy scan is run as
// rounds over the kept set: whenever a candidate w is kept, every still-alive
// later candidate is tested against w in parallel (one candidate per lane,
// each lane computing the full fp32 sequential distance).  A candidate leaves
// the alive list the moment some kept w dominates it.
//
// That evaluates exactly the reference's lazy pair set -- for each examined v,
// the kept w's in kept order up to and including the first dominator -- so the
// per-node dist_evals / angle_evals counters come out identical, and because
// every pair distance uses the reference's arithmetic the verdicts (and thus
// the adjacency) are bit-identical.  Entries after the point where the M-th
// neighbour is kept are never examined by the reference; their counters are
// discarded (their distances may have been computed speculatively).
#include "common.cuh"

namespace pgk {

constexpr int PRUNE_WARPS = 8;
constexpr int PRUNE_W = 256;  // window entries per warp
constexpr int DC = 32;        // dimensions per staged chunk
constexpr int SROW = DC + 4;  // staged row stride (floats): == 4 mod 32 -> LDS.128 conflict-free

struct PruneSmem {
  int32_t id[PRUNE_WARPS][PRUNE_W];
  float dist[PRUNE_WARPS][PRUNE_W];
  int32_t de[PRUNE_WARPS][PRUNE_W];
  int32_t ae[PRUNE_WARPS][PRUNE_W];
  int16_t alive[PRUNE_WARPS][PRUNE_W];
  alignas(16) float stage[PRUNE_WARPS][2][32 * SROW];  // 32 candidate rows x 2 chunks
};

// Test alive entries alive[a0 .. n_alive) against kept neighbour w; returns
// the new alive count (survivors compacted to alive[0..), order kept).
//
// One lane per candidate; each lane accumulates its full squared distance in
// the reference's sequential fp32 order.  VEC4 (d % 4 == 0, aligned rows):
// the batch's 32 candidate rows are staged through shared memory 64 dims at a
// time with coalesced float4 loads (two rows per warp instruction) and read
// back conflict-free, instead of 32 scattered per-lane row walks.
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// MODE 0: scalar fp32 rows; MODE 1: float4-staged fp32 rows (d % 4 == 0);
// MODE 2: exact-integer rows (every value an integer in [0,255], d <= 128):
// the reference's sequential fp32 squared_l2 only ever holds integers below
// 2^24 there, so it equals |w|^2 + |v|^2 - 2 w.v computed with u8 dp4a on
// 128-byte rows -- bit-identical, ~10x fewer instructions, 4x fewer bytes.
template <int MODE>
__device__ __forceinline__ int test_round(
    const float *__restrict__ X, const uint8_t *__restrict__ xu8,
    const int32_t *__restrict__ norms, int d, int32_t w, float duw, int strategy,
    double cos_alpha, int a0, int n_alive, int32_t *s_id, float *s_dist,
    int32_t *s_de, int32_t *s_ae, int16_t *s_alive, float *stage, int lane) {
  if (duw == 0.0f) return 0;  // _kernels.py:387-389: dominated, no evaluation
  const float *xw = X + (int64_t)w * d;
  uint4 wr[8] = {};
  int nw = 0;
  if (MODE == 2) {
    const uint4 *p = reinterpret_cast<const uint4 *>(xu8 + (int64_t)w * 128);
#pragma unroll
    for (int i = 0; i < 8; ++i) wr[i] = __ldg(p + i);
    nw = __ldg(norms + w);
  }
  int new_n = 0;
  for (int base = a0; base < n_alive; base += 32) {
    const int a = base + lane;
    const bool act = a < n_alive;
    const int nb = min(32, n_alive - base);
    const int j = act ? s_alive[a] : s_alive[base];
    const int32_t v = s_id[j];
    float dwv = 0.0f;  // _kernels.py:390: squared_l2(data[w], data[v])
    if (MODE == 2) {
      uint8_t *st8 = reinterpret_cast<uint8_t *>(stage);
      const int l8 = lane & 7, rsub = lane >> 3;
      __syncwarp();
#pragma unroll
      for (int e0 = 0; e0 < 32; e0 += 4) {
        const int e = e0 + rsub;
        const int32_t ve = __shfl_sync(0xffffffffu, v, e);
        if (e < nb) cp_async16(st8 + e * 144 + 16 * l8, xu8 + (int64_t)ve * 128 + 16 * l8);
      }
      cp_async_commit();
      int nv = act ? __ldg(norms + v) : 0;
      cp_async_wait<0>();
      __syncwarp();
      if (act) {
        const uint4 *sr = reinterpret_cast<const uint4 *>(st8 + lane * 144);
        unsigned dot = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint4 b = sr[i];
          dot = __dp4a(wr[i].x, b.x, dot);
          dot = __dp4a(wr[i].y, b.y, dot);
          dot = __dp4a(wr[i].z, b.z, dot);
          dot = __dp4a(wr[i].w, b.w, dot);
        }
        dwv = (float)(nw + nv - 2 * (int)dot);
      }
    } else if (MODE == 1) {
      // stage chunk c0 of the batch's rows: 8 lanes per row, 4 rows per
      // instruction, all 8 cp.async instructions in flight together
      const int l8 = lane & 7, rsub = lane >> 3;
      auto issue = [&](int c0, float *buf) {
        const int dc = min(DC, d - c0);
#pragma unroll
        for (int e0 = 0; e0 < 32; e0 += 4) {
          const int e = e0 + rsub;
          const int32_t ve = __shfl_sync(0xffffffffu, v, e);
          if (e < nb && 4 * l8 < dc)
            cp_async16(buf + e * SROW + 4 * l8, X + (int64_t)ve * d + c0 + 4 * l8);
        }
        cp_async_commit();
      };
      __syncwarp();
      issue(0, stage);
      int cur = 0;
      for (int c0 = 0; c0 < d; c0 += DC) {
        const bool more = c0 + DC < d;
        if (more) {
          issue(c0 + DC, stage + (cur ^ 1) * 32 * SROW);
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        __syncwarp();
        if (act) {
          const int dc = min(DC, d - c0);
          const float *srow = stage + cur * 32 * SROW + lane * SROW;
          const float4 *w4 = reinterpret_cast<const float4 *>(xw + c0);
#pragma unroll 4
          for (int k = 0; k < dc; k += 4) {
            const float4 x = __ldg(w4 + (k >> 2));
            const float4 y = *reinterpret_cast<const float4 *>(srow + k);
            dwv = sq_step(dwv, x.x, y.x);
            dwv = sq_step(dwv, x.y, y.y);
            dwv = sq_step(dwv, x.z, y.z);
            dwv = sq_step(dwv, x.w, y.w);
          }
        }
        __syncwarp();
        cur ^= 1;
      }
    } else if (act) {
      dwv = sql2_seq<false>(xw, X + (int64_t)v * d, d);
    }
    bool survive = false;
    if (act) {
      const float dv = s_dist[j];
      s_de[j] += 1;
      bool dom;
      if (dwv == 0.0f) {
        dom = true;
      } else if (dwv < dv) {
        if (strategy == 0) {
          dom = true;
        } else if (strategy == 2) {  // "slack" extension: s^2 * dwv < dv
          dom = cos_alpha * (double)dwv < (double)dv;
        } else {
          double c = cos_angle_from_sq(duw, dwv, dv);
          s_ae[j] += 1;
          dom = c < cos_alpha;
        }
      } else {
        dom = false;
      }
      survive = !dom;
    }
    unsigned b = __ballot_sync(0xffffffffu, survive);
    if (survive) s_alive[new_n + __popc(b & lanemask_lt())] = (int16_t)j;
    new_n += __popc(b);
  }
  __syncwarp();
  return new_n;
}

// Speculative in-window rounds (MODE 1, fp32 rows).  The next kept
// neighbours can only be the first alive entries, so one staged pass over the
// alive rows computes every alive entry's distance to each of the first SPEC
// alive entries (SPEC = 3 independent sequential fp32 chains per lane: bit-
// identical values, SPEC x fewer row reads, SPEC-way ILP), and the rounds are
// then resolved in order from registers.  A distance is counted (s_de / s_ae)
// only when its round happens, i.e. for kept neighbours, so verdicts, the kept
// set and the lazy counters are exactly the sequential rounds'.  Returns the
// new alive count; kept / stop / stop_j are updated as the caller's loop does.
#ifndef PRUNE_SPEC
#define PRUNE_SPEC 3
#endif
constexpr int SPEC = PRUNE_SPEC;
constexpr int SB = PRUNE_W / 32;

__device__ __forceinline__ int spec_block(const float *__restrict__ X, int d, int strategy,
                                          double cos_alpha, int n_alive, int32_t *s_id,
                                          float *s_dist, int32_t *s_de, int32_t *s_ae,
                                          int16_t *s_alive, float *stage, int32_t *orow,
                                          float *odrow, int &kept, int M, bool &stop,
                                          int &stop_j, int lane) {
  const int nw = min(SPEC, n_alive);
  int32_t wid[SPEC];
  float wdu[SPEC];
#pragma unroll
  for (int i = 0; i < SPEC; ++i) {
    const int e = s_alive[i < nw ? i : 0];
    wid[i] = s_id[e];
    wdu[i] = s_dist[e];
  }
  float dr[SB][SPEC];
  const int l8 = lane & 7, rsub = lane >> 3;
#pragma unroll
  for (int b = 0; b < SB; ++b) {
#pragma unroll
    for (int i = 0; i < SPEC; ++i) dr[b][i] = 0.0f;
    const int base = b * 32;
    if (base >= n_alive) continue;
    const int nb = min(32, n_alive - base);
    const bool act = lane < nb;
    const int32_t v = s_id[s_alive[act ? base + lane : base]];
    auto issue = [&](int c0, float *buf) {
      const int dc = min(DC, d - c0);
#pragma unroll
      for (int e0 = 0; e0 < 32; e0 += 4) {
        const int e = e0 + rsub;
        const int32_t ve = __shfl_sync(0xffffffffu, v, e);
        if (e < nb && 4 * l8 < dc)
          cp_async16(buf + e * SROW + 4 * l8, X + (int64_t)ve * d + c0 + 4 * l8);
      }
      cp_async_commit();
    };
    float acc[SPEC];
#pragma unroll
    for (int i = 0; i < SPEC; ++i) acc[i] = 0.0f;
    __syncwarp();
    issue(0, stage);
    int cur = 0;
    for (int c0 = 0; c0 < d; c0 += DC) {
      if (c0 + DC < d) {
        issue(c0 + DC, stage + (cur ^ 1) * 32 * SROW);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncwarp();
      if (act) {
        const int dc = min(DC, d - c0);
        const float *srow = stage + cur * 32 * SROW + lane * SROW;
#pragma unroll 2
        for (int k = 0; k < dc; k += 4) {
          const float4 y = *reinterpret_cast<const float4 *>(srow + k);
#pragma unroll
          for (int i = 0; i < SPEC; ++i) {
            if (i < nw) {
              // squared_l2(data[w], data[v]) (_kernels.py:390)
              const float4 x =
                  __ldg(reinterpret_cast<const float4 *>(X + (int64_t)wid[i] * d + c0 + k));
              acc[i] = sq_step(acc[i], x.x, y.x);
              acc[i] = sq_step(acc[i], x.y, y.y);
              acc[i] = sq_step(acc[i], x.z, y.z);
              acc[i] = sq_step(acc[i], x.w, y.w);
            }
          }
        }
      }
      __syncwarp();
      cur ^= 1;
    }
#pragma unroll
    for (int i = 0; i < SPEC; ++i) dr[b][i] = acc[i];
  }
  // resolve the rounds in order
  unsigned am[SB];
#pragma unroll
  for (int b = 0; b < SB; ++b) am[b] = __ballot_sync(0xffffffffu, b * 32 + lane < n_alive);
  int pos = 0, last = 0;
#pragma unroll
  for (int i = 0; i < SPEC; ++i) {
    if (i >= nw) break;
    if (pos != i) continue;  // entry i was dominated: the next kept lies further on
    // alive entry i is the next kept neighbour (_kernels.py:396-399)
    if (lane == 0) {
      orow[kept] = wid[i];
      odrow[kept] = wdu[i];
    }
    ++kept;
    last = i;
    if (kept == M) {  // _kernels.py:378: later candidates never examined
      stop = true;
      stop_j = s_alive[i];
      return 0;
    }
    const float duw = wdu[i];
#pragma unroll
    for (int b = 0; b < SB; ++b) {
      const int p = b * 32 + lane;
      bool live = (am[b] >> lane) & 1u;
      if (live && p > i) {
        if (duw == 0.0f) {  // _kernels.py:387-389: dominated, no evaluation
          live = false;
        } else {
          const int j = s_alive[p];
          const float dv = s_dist[j];
          const float dwv = dr[b][i];
          s_de[j] += 1;
          bool dom;
          if (dwv == 0.0f) {
            dom = true;
          } else if (dwv < dv) {
            if (strategy == 0) {
              dom = true;
            } else if (strategy == 2) {  // "slack" extension: s^2 * dwv < dv
              dom = cos_alpha * (double)dwv < (double)dv;
            } else {
              double c = cos_angle_from_sq(duw, dwv, dv);
              s_ae[j] += 1;
              dom = c < cos_alpha;
            }
          } else {
            dom = false;
          }
          live = !dom;
        }
      }
      am[b] = __ballot_sync(0xffffffffu, live);
    }
    // next kept: the first alive entry after i
    int nxt = n_alive;
#pragma unroll
    for (int b = SB - 1; b >= 0; --b) {
      const int sh = i - b * 32;  // bits 0..sh of batch b are at or before entry i
      const unsigned after = sh < 0 ? 0xffffffffu : (sh >= 31 ? 0u : ~((2u << sh) - 1u));
      const unsigned m = am[b] & after;
      if (m) nxt = b * 32 + __ffs(m) - 1;
    }
    pos = nxt;
  }
  // compact: alive entries after the last kept one, order kept
  int16_t keep_e[SB];
#pragma unroll
  for (int b = 0; b < SB; ++b) {
    const int p = b * 32 + lane;
    keep_e[b] = p < n_alive ? s_alive[p] : (int16_t)0;
  }
  __syncwarp();
  int new_n = 0;
#pragma unroll
  for (int b = 0; b < SB; ++b) {
    const int p = b * 32 + lane;
    const bool k = ((am[b] >> lane) & 1u) && p > last;
    const unsigned bb = __ballot_sync(0xffffffffu, k);
    if (k) s_alive[new_n + __popc(bb & lanemask_lt())] = keep_e[b];
    new_n += __popc(bb);
  }
  __syncwarp();
  return new_n;
}

template <int MODE>
__global__ void __launch_bounds__(PRUNE_WARPS * 32, 2)
    prune_kernel(const float *__restrict__ X, const uint8_t *__restrict__ xu8,
                 const int32_t *__restrict__ norms, int64_t n, int d,
                 const int32_t *__restrict__ row_node, const int32_t *__restrict__ row_order,
                 const int64_t *__restrict__ cand_off,
                 const int32_t *__restrict__ cand_counts,
                 const int32_t *__restrict__ cand_ids,
                 const float *__restrict__ cand_dists, int strategy,
                 double cos_alpha, int M, int width, int32_t *__restrict__ out_ids,
                 float *__restrict__ out_dists, int32_t *__restrict__ out_counts,
                 int64_t *__restrict__ dist_evals,
                 int64_t *__restrict__ angle_evals, int min_cnt) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PruneSmem &sm = *reinterpret_cast<PruneSmem *>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t *s_id = sm.id[warp];
  float *s_dist = sm.dist[warp];
  int32_t *s_de = sm.de[warp];
  int32_t *s_ae = sm.ae[warp];
  int16_t *s_alive = sm.alive[warp];
  float *stage = sm.stage[warp][0];

  for (int64_t i = (int64_t)blockIdx.x * PRUNE_WARPS + warp; i < n;
       i += (int64_t)gridDim.x * PRUNE_WARPS) {
    const int64_t u = row_order ? row_order[i] : i;
    const int cnt = cand_counts[u];
    if (cnt <= min_cnt) continue;  // rows the tensor-core kernel has done
    const int64_t base = cand_off[u];
    const int32_t self = row_node ? row_node[u] : (int32_t)u;
    int32_t *orow = out_ids + u * width;
    float *odrow = out_dists + u * width;
    int kept = 0;
    bool stop = false;
    long long de_tot = 0, ae_tot = 0;

    for (int s = 0; s < cnt && !stop; s += PRUNE_W) {
      const int wn = min(PRUNE_W, cnt - s);
      __syncwarp();
      for (int j = lane; j < wn; j += 32) {
        s_id[j] = cand_ids[base + s + j];
        s_dist[j] = cand_dists[base + s + j];
        s_de[j] = 0;
        s_ae[j] = 0;
      }
      __syncwarp();
      // alive = examined candidates other than u itself (_kernels.py:380-382)
      int n_alive = 0;
      for (int j0 = 0; j0 < wn; j0 += 32) {
        int j = j0 + lane;
        bool al = j < wn && s_id[j] != self;
        unsigned b = __ballot_sync(0xffffffffu, al);
        if (al) s_alive[n_alive + __popc(b & lanemask_lt())] = (int16_t)j;
        n_alive += __popc(b);
      }
      __syncwarp();
      // rounds against neighbours kept in earlier windows
      for (int kj = 0; kj < kept && n_alive > 0; ++kj) {
        int32_t w = orow[kj];
        float duw = odrow[kj];
        n_alive = test_round<MODE>(X, xu8, norms, d, w, duw, strategy, cos_alpha, 0, n_alive,
                                   s_id, s_dist, s_de, s_ae, s_alive, stage, lane);
      }
      // in-window greedy: the first alive entry is the next kept neighbour
      int stop_j = wn - 1;
      if (MODE == 1) {  // speculative rounds (same verdicts, counters, order)
        while (n_alive > 0 && !stop)
          n_alive = spec_block(X, d, strategy, cos_alpha, n_alive, s_id, s_dist, s_de, s_ae,
                               s_alive, stage, orow, odrow, kept, M, stop, stop_j, lane);
      }
      while (MODE != 1 && n_alive > 0) {
        const int e = s_alive[0];
        const int32_t w = s_id[e];
        const float duw = s_dist[e];
        if (lane == 0) {
          orow[kept] = w;
          odrow[kept] = duw;
        }
        ++kept;
        if (kept == M) {  // _kernels.py:378: later candidates never examined
          stop = true;
          stop_j = e;
          break;
        }
        n_alive = test_round<MODE>(X, xu8, norms, d, w, duw, strategy, cos_alpha, 1, n_alive,
                                   s_id, s_dist, s_de, s_ae, s_alive, stage, lane);
      }
      __syncwarp();
      long long de = 0, ae = 0;
      for (int j = lane; j <= stop_j; j += 32) {
        de += s_de[j];
        ae += s_ae[j];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        de += __shfl_xor_sync(0xffffffffu, de, o);
        ae += __shfl_xor_sync(0xffffffffu, ae, o);
      }
      de_tot += de;
      ae_tot += ae;
    }
    __syncwarp();
    for (int j = kept + lane; j < width; j += 32) {
      orow[j] = -1;
      odrow[j] = __int_as_float(0x7f800000);
    }
    if (lane == 0) {
      out_counts[u] = kept;
      dist_evals[u] = de_tot;
      angle_evals[u] = ae_tot;
    }
  }
}

// ---------------------------------------------------------------------------
// Exact-integer selection with window-resident rows.  Same scan, rounds and
// counters as prune_kernel, but a window of up to 128 candidates keeps its
// u8 rows (128 B each) in shared memory for all rounds: one cp.async burst per
// window instead of a global round trip per round.
// ---------------------------------------------------------------------------
constexpr int U8_WARPS = 16;
constexpr int U8_W = 64;
constexpr int U8_ROW = 144;  // padded row stride (36 words == 4 mod 32)

struct PruneU8Smem {
  int32_t id[U8_WARPS][U8_W];
  float dist[U8_WARPS][U8_W];
  int32_t de[U8_WARPS][U8_W];
  int32_t ae[U8_WARPS][U8_W];
  int32_t nrm[U8_WARPS][U8_W];
  int16_t alive[U8_WARPS][U8_W];
  alignas(16) uint8_t rows[U8_WARPS][U8_W * U8_ROW];
};

// test alive[a0..n_alive) against kept w (row wr in registers, norm nw)
__device__ __forceinline__ int test_round_u8(const uint4 (&wr)[8], int nw, float duw,
                                             int strategy, double cos_alpha, int a0,
                                             int n_alive, const float *s_dist, int32_t *s_de,
                                             int32_t *s_ae, int16_t *s_alive,
                                             const int32_t *s_nrm, const uint8_t *rows,
                                             int lane) {
  if (duw == 0.0f) return 0;  // _kernels.py:387-389
  int new_n = 0;
  for (int base = a0; base < n_alive; base += 32) {
    const int a = base + lane;
    const bool act = a < n_alive;
    bool survive = false;
    int j = 0;
    if (act) {
      j = s_alive[a];
      const uint4 *sr = reinterpret_cast<const uint4 *>(rows + j * U8_ROW);
      unsigned d0 = 0, d1 = 0, d2 = 0, d3 = 0;  // 4 independent chains
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint4 b = sr[i];
        d0 = __dp4a(wr[i].x, b.x, d0);
        d1 = __dp4a(wr[i].y, b.y, d1);
        d2 = __dp4a(wr[i].z, b.z, d2);
        d3 = __dp4a(wr[i].w, b.w, d3);
      }
      const unsigned dot = (d0 + d1) + (d2 + d3);
      // == squared_l2(data[w], data[v]) exactly (integers < 2^24)
      const float dwv = (float)(nw + s_nrm[j] - 2 * (int)dot);
      const float dv = s_dist[j];
      s_de[j] += 1;
      bool dom;
      if (dwv == 0.0f) {
        dom = true;
      } else if (dwv < dv) {
        if (strategy == 0) {
          dom = true;
        } else if (strategy == 2) {  // "slack" extension: s^2 * dwv < dv
          dom = cos_alpha * (double)dwv < (double)dv;
        } else {
          const double c = cos_angle_from_sq(duw, dwv, dv);
          s_ae[j] += 1;
          dom = c < cos_alpha;
        }
      } else {
        dom = false;
      }
      survive = !dom;
    }
    const unsigned b = __ballot_sync(0xffffffffu, survive);
    if (survive) s_alive[new_n + __popc(b & lanemask_lt())] = (int16_t)j;
    new_n += __popc(b);
  }
  __syncwarp();
  return new_n;
}

__global__ void __launch_bounds__(U8_WARPS * 32, 1)
    prune_u8_kernel(const uint8_t *__restrict__ xu8, const int32_t *__restrict__ norms,
                    int64_t n, const int32_t *__restrict__ n_dev,
                    const int32_t *__restrict__ row_node,
                    const int32_t *__restrict__ row_order,
                    const int64_t *__restrict__ cand_off,
                    const int32_t *__restrict__ cand_counts,
                    const int32_t *__restrict__ cand_ids, const float *__restrict__ cand_dists,
                    int strategy, double cos_alpha, int M, int width,
                    int32_t *__restrict__ out_ids, float *__restrict__ out_dists,
                    int32_t *__restrict__ out_counts, int64_t *__restrict__ dist_evals,
                    int64_t *__restrict__ angle_evals) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PruneU8Smem &sm = *reinterpret_cast<PruneU8Smem *>(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int32_t *s_id = sm.id[warp];
  float *s_dist = sm.dist[warp];
  int32_t *s_de = sm.de[warp];
  int32_t *s_ae = sm.ae[warp];
  int32_t *s_nrm = sm.nrm[warp];
  int16_t *s_alive = sm.alive[warp];
  uint8_t *rows = sm.rows[warp];
  if (n_dev) n = *n_dev;  // row count produced on the device (hub list)

  for (int64_t i = (int64_t)blockIdx.x * U8_WARPS + warp; i < n;
       i += (int64_t)gridDim.x * U8_WARPS) {
    const int64_t u = row_order ? row_order[i] : i;
    const int cnt = cand_counts[u];
    const int64_t base = cand_off[u];
    const int32_t self = row_node ? row_node[u] : (int32_t)u;
    int32_t *orow = out_ids + u * width;
    float *odrow = out_dists + u * width;
    int kept = 0;
    bool stop = false;
    long long de_tot = 0, ae_tot = 0;

    for (int s = 0; s < cnt && !stop; s += U8_W) {
      const int wn = min(U8_W, cnt - s);
      __syncwarp();
      // window: ids first (coalesced), then every candidate row in one
      // cp.async burst, then norms / dists while the rows land
      for (int j = lane; j < wn; j += 32) s_id[j] = cand_ids[base + s + j];
      __syncwarp();
#pragma unroll 4
      for (int j0 = 0; j0 < wn; j0 += 4) {
        const int j = j0 + (lane >> 3);
        if (j < wn)
          cp_async16(rows + j * U8_ROW + 16 * (lane & 7),
                     xu8 + (int64_t)s_id[j] * 128 + 16 * (lane & 7));
      }
      cp_async_commit();
      for (int j = lane; j < wn; j += 32) {
        s_dist[j] = cand_dists[base + s + j];
        s_nrm[j] = __ldg(norms + s_id[j]);
        s_de[j] = 0;
        s_ae[j] = 0;
      }
      __syncwarp();
      int n_alive = 0;
      for (int j0 = 0; j0 < wn; j0 += 32) {
        const int j = j0 + lane;
        const bool al = j < wn && s_id[j] != self;  // _kernels.py:380-382
        const unsigned b = __ballot_sync(0xffffffffu, al);
        if (al) s_alive[n_alive + __popc(b & lanemask_lt())] = (int16_t)j;
        n_alive += __popc(b);
      }
      cp_async_wait<0>();
      __syncwarp();
      // rounds against neighbours kept in earlier windows (rows from global)
      for (int kj = 0; kj < kept && n_alive > 0; ++kj) {
        const int32_t w = orow[kj];
        uint4 wr[8];
        const uint4 *gp = reinterpret_cast<const uint4 *>(xu8 + (int64_t)w * 128);
#pragma unroll
        for (int i = 0; i < 8; ++i) wr[i] = __ldg(gp + i);
        n_alive = test_round_u8(wr, __ldg(norms + w), odrow[kj], strategy, cos_alpha, 0, n_alive,
                                s_dist, s_de, s_ae, s_alive, s_nrm, rows, lane);
      }
      // in-window greedy: the first alive entry is the next kept neighbour
      int stop_j = wn - 1;
      while (n_alive > 0) {
        const int e = s_alive[0];
        const float duw = s_dist[e];
        if (lane == 0) {
          orow[kept] = s_id[e];
          odrow[kept] = duw;
        }
        ++kept;
        if (kept == M) {  // _kernels.py:378
          stop = true;
          stop_j = e;
          break;
        }
        uint4 wr[8];
        const uint4 *sp = reinterpret_cast<const uint4 *>(rows + e * U8_ROW);
#pragma unroll
        for (int i = 0; i < 8; ++i) wr[i] = sp[i];
        n_alive = test_round_u8(wr, s_nrm[e], duw, strategy, cos_alpha, 1, n_alive, s_dist, s_de,
                                s_ae, s_alive, s_nrm, rows, lane);
      }
      __syncwarp();
      long long de = 0, ae = 0;
      for (int j = lane; j <= stop_j; j += 32) {
        de += s_de[j];
        ae += s_ae[j];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        de += __shfl_xor_sync(0xffffffffu, de, o);
        ae += __shfl_xor_sync(0xffffffffu, ae, o);
      }
      de_tot += de;
      ae_tot += ae;
    }
    __syncwarp();
    for (int j = kept + lane; j < width; j += 32) {
      orow[j] = -1;
      odrow[j] = __int_as_float(0x7f800000);
    }
    if (lane == 0) {
      out_counts[u] = kept;
      dist_evals[u] = de_tot;
      angle_evals[u] = ae_tot;
    }
  }
}

int launch_prune_u8_rows(const uint8_t *xu8, const int32_t *norms, int64_t n,
                         const int32_t *n_dev, const int32_t *row_node,
                         const int32_t *row_order, const int64_t *cand_off,
                     const int32_t *cand_counts, const int32_t *cand_ids,
                     const float *cand_dists, int strategy, double cos_alpha, int64_t M,
                     int64_t width, int32_t *out_ids, float *out_dists, int32_t *out_counts,
                     int64_t *dist_evals, int64_t *angle_evals, cudaStream_t stream) {
  const size_t smem = sizeof(PruneU8Smem);
  PGK_CUDA(ensure_smem((const void *)prune_u8_kernel, smem));
  int64_t blocks = (n + U8_WARPS - 1) / U8_WARPS;
  const int64_t cap = (int64_t)num_sms();  // one ~210 KB block per SM
  if (blocks > cap) blocks = cap;
  prune_u8_kernel<<<(unsigned)blocks, U8_WARPS * 32, smem, stream>>>(
      xu8, norms, n, n_dev, row_node, row_order, cand_off, cand_counts, cand_ids, cand_dists,
      strategy, cos_alpha,
      (int)M, (int)width, out_ids, out_dists, out_counts, dist_evals, angle_evals);
  PGK_CHECK_LAUNCH("prune_u8_kernel");
  return PGK_OK;
}

template <int MODE>
static int launch_mode(const float *X, const uint8_t *xu8, const int32_t *norms, int64_t n,
                       int64_t d, const int32_t *row_node, const int32_t *row_order,
                       const int64_t *cand_off,
                       const int32_t *cand_counts, const int32_t *cand_ids,
                       const float *cand_dists, int strategy, double cos_alpha, int64_t M,
                       int64_t width, int32_t *out_ids, float *out_dists, int32_t *out_counts,
                       int64_t *dist_evals, int64_t *angle_evals, cudaStream_t stream,
                       int min_cnt = -1) {
  const size_t smem = sizeof(PruneSmem);
  int64_t blocks = (n + PRUNE_WARPS - 1) / PRUNE_WARPS;
  const int64_t cap = (int64_t)num_sms() * 2;  // 2 resident blocks per SM (~110 KB smem each)
  if (blocks > cap) blocks = cap;
  PGK_CUDA(ensure_smem((const void *)prune_kernel<MODE>, smem));
  prune_kernel<MODE><<<(unsigned)blocks, PRUNE_WARPS * 32, smem, stream>>>(
      X, xu8, norms, n, (int)d, row_node, row_order, cand_off, cand_counts, cand_ids, cand_dists,
      strategy,
      cos_alpha, (int)M, (int)width, out_ids, out_dists, out_counts, dist_evals, angle_evals,
      min_cnt);
  PGK_CHECK_LAUNCH("prune_kernel");
  return PGK_OK;
}

// xu8 / norms (optional): the exact-integer copy of X (rows of 128 bytes,
// zero padded) and its integer squared norms -- valid only when every value
// of X is an integer in [0,255] and d <= 128 (pgk_detect_u8).
bool gram_enabled();
size_t gram_workspace(int64_t n);
int launch_prune_gram(const uint8_t *xu8, const int32_t *norms, int64_t n,
                      const int32_t *row_node, const int32_t *row_order,
                      const int64_t *cand_off, const int32_t *cand_counts,
                      const int32_t *cand_ids, const float *cand_dists, int strategy,
                      double cos_alpha, int64_t M, int64_t width, int32_t *out_ids,
                      float *out_dists, int32_t *out_counts, int64_t *dist_evals,
                      int64_t *angle_evals, void *ws, cudaStream_t stream, bool pair);

bool gram_f32_supported(const float *X, int64_t d, int strategy);
int launch_prune_gram_f32(const float *X, int64_t d, int64_t n, const int32_t *row_node,
                          const int32_t *row_order, const int64_t *cand_off,
                          const int32_t *cand_counts, const int32_t *cand_ids,
                          const float *cand_dists, int strategy, double cos_alpha, int64_t M,
                          int64_t width, int32_t *out_ids, float *out_dists,
                          int32_t *out_counts, int64_t *dist_evals, int64_t *angle_evals,
                          cudaStream_t stream);

size_t prune_workspace(int64_t n_rows) { return gram_workspace(n_rows); }

int launch_prune(const float *X, const uint8_t *xu8, const int32_t *norms, int64_t n,
                 int64_t d, const int32_t *row_node, const int32_t *row_order, void *ws,
                 size_t ws_bytes, const int64_t *cand_off,
                 const int32_t *cand_counts, const int32_t *cand_ids, const float *cand_dists,
                 int strategy, double cos_alpha, int64_t M, int64_t width, int32_t *out_ids,
                 float *out_dists, int32_t *out_counts, int64_t *dist_evals,
                 int64_t *angle_evals, cudaStream_t stream, bool short_rows) {
  if (n == 0) return PGK_OK;
  if (xu8 && norms && d <= 128 && ws && ws_bytes >= gram_workspace(n) && gram_enabled())
    return launch_prune_gram(xu8, norms, n, row_node, row_order, cand_off, cand_counts, cand_ids,
                             cand_dists, strategy, cos_alpha, M, width, out_ids, out_dists,
                             out_counts, dist_evals, angle_evals, ws, stream, short_rows);
  if (xu8 && norms && d <= 128)
    return launch_prune_u8_rows(xu8, norms, n, nullptr, row_node, row_order, cand_off,
                     cand_counts, cand_ids, cand_dists,
                     strategy, cos_alpha, M, width, out_ids, out_dists, out_counts, dist_evals,
                     angle_evals, stream);
  if (ws && ws_bytes >= gram_workspace(n) && gram_f32_supported(X, d, strategy)) {
    // fp32 rows: the candidate Gram matrix on the tensor cores, exact chains
    // only for undecided pairs (prune_gram_f32.cu); rows with more than 128
    // candidates are skipped there and taken by prune_kernel, in the same
    // (locality) order
    int rc = launch_prune_gram_f32(X, d, n, row_node, row_order, cand_off, cand_counts, cand_ids,
                                   cand_dists, strategy, cos_alpha, M, width, out_ids, out_dists,
                                   out_counts, dist_evals, angle_evals, stream);
    if (rc) return rc;
    return launch_mode<1>(X, nullptr, nullptr, n, d, row_node, row_order, cand_off, cand_counts,
                          cand_ids, cand_dists, strategy, cos_alpha, M, width, out_ids, out_dists,
                          out_counts, dist_evals, angle_evals, stream, 128);
  }
  if ((d % 4 == 0) && ((uintptr_t)X % 16 == 0))
    return launch_mode<1>(X, nullptr, nullptr, n, d, row_node, row_order, cand_off, cand_counts,
                          cand_ids,
                          cand_dists, strategy, cos_alpha, M, width, out_ids, out_dists,
                          out_counts, dist_evals, angle_evals, stream);
  return launch_mode<0>(X, nullptr, nullptr, n, d, row_node, row_order, cand_off, cand_counts,
                        cand_ids,
                        cand_dists, strategy, cos_alpha, M, width, out_ids, out_dists,
                        out_counts, dist_evals, angle_evals, stream);
}

// float (integer-valued) -> u8 rows padded to 128 bytes + integer norms
__global__ void make_u8_kernel(const float *__restrict__ X, int64_t n, int d,
                               uint8_t *__restrict__ out, int32_t *__restrict__ norms) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < n;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int acc = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = lane + 32 * k;
      const int v = c < d ? (int)(uint8_t)__float2int_rn(X[r * d + c]) : 0;  // norm of the stored byte
      out[r * 128 + c] = (uint8_t)v;
      acc += v * v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) norms[r] = acc;
  }
}

int make_u8(const float *X, int64_t n, int64_t d, uint8_t *out, int32_t *norms,
            cudaStream_t stream) {
  if (d > 128) {
    set_error("exact-integer rows need d <= 128");
    return PGK_ERR_UNSUPPORTED;
  }
  if (n == 0) return PGK_OK;
  make_u8_kernel<<<(unsigned)num_sms() * 8, 256, 0, stream>>>(X, n, (int)d, out, norms);
  PGK_CHECK_LAUNCH("make_u8_kernel");
  return PGK_OK;
}

}  // namespace pgk
