// pool_tiles.cu -- exact tile pruning for the self k-NN pool (U8 path).
//
// The brute-force pool touches all N^2 pairs.  For a provably sufficient
// subset: points are grouped into spatially coherent 128-row tiles -- every
// point is assigned to its nearest "center" (every 512th data row; the
// tcgen05 kernel itself with K = 1), points are counting-sorted by center and
// each center's run is padded to a multiple of 128 rows with inert rows
// (zero vector, huge norm, no output) so no tile straddles two cells -- and
// every tile gets a centroid c_T and radius r_T = max |x - c_T| over its real
// rows (float64).  For a query tile Q and any q in Q, x in T:
//      |q - x| >= |c_Q - c_T| - r_Q - r_T  =: lb(Q,T)      (triangle inequality)
//      |q - x| <= |c_Q - c_T| + r_Q + r_T  =: ub(Q,T)
// Pass 1 runs the exact top-K of every query tile over its 8 nearest tiles
// (by centroid distance); U_Q = the largest K-th distance found in Q is an
// upper bound of every row's true K-th neighbour distance, so no point
// farther than U_Q from a row of Q can be in its pool.  Q's candidate tiles
// are {T : lb(Q,T) <= U_Q}, and pass 2 recomputes the exact top-K over them.  The tcgen05 kernel
// then runs unchanged over each query tile's candidate list; results are
// identical to the full scan (ids are mapped back through the permutation and
// ties still break on the original id).  All bounds are float64 with explicit
// relative margins, far above the float64 rounding of the inputs.
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace pgk {

size_t scan_scratch(int64_t m);
int exclusive_scan(const int64_t *in, int64_t *out, int64_t m, int64_t *scratch,
                   cudaStream_t stream);

// PGK_DEBUG_SYNC=1: synchronise and report after every stage (hang hunting)
static void dbg_stage(const char *what, cudaStream_t stream) {
  static int env = -1;
  if (env < 0) {
    const char *e = getenv("PGK_DEBUG_SYNC");
    env = (e && e[0] == '1') ? 1 : 0;
  }
  if (!env) return;
  const cudaError_t err = cudaStreamSynchronize(stream);
  fprintf(stderr, "[pgk debug] %s: %s\n", what, cudaGetErrorString(err));
}

namespace tiles {

constexpr int TB = 128;  // tile size (== tc::BN == tc::BM)
constexpr double MARGIN = 1e-9;

#ifndef TILES_CSTRIDE
#define TILES_CSTRIDE 512
#endif
constexpr int CSTRIDE = TILES_CSTRIDE;  // one center per CSTRIDE rows

__global__ void gather_centers_kernel(const float *__restrict__ X, int64_t n, int d, int64_t C,
                                      float *__restrict__ cen) {
  const int64_t total = C * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = e / d;
    const int k = (int)(e - c * d);
    cen[e] = X[(c * CSTRIDE) * d + k];
  }
}

__global__ void assign_hist_kernel(const uint64_t *__restrict__ keys, int64_t n,
                                   int32_t *__restrict__ hist, int32_t *__restrict__ assign) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = key_id(keys[i]);
    assign[i] = c;
    atomicAdd(hist + c, 1);
  }
}

// padded run lengths: each center's run rounded up to whole tiles
__global__ void padded_len_kernel(const int32_t *__restrict__ hist, int64_t C,
                                  int64_t *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= C;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = i < C ? (int64_t)(hist[i] + TB - 1) / TB * TB : 0;
}

__global__ void fill_i32_kernel(int32_t *__restrict__ p, int64_t m, int32_t v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void assign_scatter_kernel(const int32_t *__restrict__ assign, int64_t n,
                                      const int64_t *__restrict__ off,
                                      int32_t *__restrict__ cursor,
                                      int32_t *__restrict__ perm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = assign[i];
    perm[off[c] + atomicAdd(cursor + c, 1)] = (int32_t)i;
  }
}

// sorted u8 rows (128 B) and norms; padding rows (perm < 0) are zero with a
// huge norm so they never enter a pool
__global__ void gather_sorted_kernel(const float *__restrict__ X, int d,
                                     const int32_t *__restrict__ perm,
                                     const int32_t *__restrict__ xnorm, int64_t np,
                                     uint8_t *__restrict__ xs, int32_t *__restrict__ ns) {
  // (from fp32 rows; gather_sorted_u8_kernel below copies existing u8 rows)
  const int64_t total = np * 128;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e >> 7;
    const int c = (int)(e & 127);
    const int32_t src = perm[r];
    xs[e] = (src >= 0 && c < d) ? (uint8_t)__float2int_rn(X[(int64_t)src * d + c]) : (uint8_t)0;
    if (c == 0) ns[r] = src >= 0 ? xnorm[src] : 0x3f3f3f3f;
  }
}

// the same from the caller's u8 rows (128 B each): 16-byte copies
__global__ void gather_sorted_u8_kernel(const uint8_t *__restrict__ xu8,
                                        const int32_t *__restrict__ perm,
                                        const int32_t *__restrict__ xnorm, int64_t np,
                                        uint8_t *__restrict__ xs, int32_t *__restrict__ ns) {
  const int64_t total = np * 8;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e >> 3;
    const int c = (int)(e & 7);
    const int32_t src = perm[r];
    reinterpret_cast<uint4 *>(xs)[e] =
        src >= 0 ? reinterpret_cast<const uint4 *>(xu8)[(int64_t)src * 8 + c] : make_uint4(0, 0, 0, 0);
    if (c == 0) ns[r] = src >= 0 ? xnorm[src] : 0x3f3f3f3f;
  }
}

// block (TB threads) per tile: centroid of the real rows (thread = dimension:
// an exact integer column sum, divided in float64 and stored fp32) and the
// radius against the stored centroid (thread = row: float64 squared distance,
// block max, inflated).  Padding rows are all-zero bytes.
__global__ void __launch_bounds__(TB) tile_stats_kernel(const uint8_t *__restrict__ xs,
                                                        const int32_t *__restrict__ perm, int d,
                                                        int64_t ntiles, float *__restrict__ cent,
                                                        double *__restrict__ rad,
                                                        int32_t *__restrict__ size) {
  __shared__ float c_s[TB];
  __shared__ uint8_t ok_s[TB];
  __shared__ double wmax[TB / 32];
  const int j = threadIdx.x, lane = j & 31;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t r0 = t * TB;
    const bool ok = perm[r0 + j] >= 0;
    ok_s[j] = ok;
    const int cnt = __syncthreads_count(ok);
    int sum = 0;
#pragma unroll 8
    for (int i = 0; i < TB; ++i)
      if (ok_s[i]) sum += xs[(r0 + i) * 128 + j];
    const float c = (cnt && j < d) ? (float)((double)sum / cnt) : 0.f;
    if (j < d) cent[t * d + j] = c;
    c_s[j] = c;
    __syncthreads();
    double s = 0.0;
    if (ok) {
      const uint4 *row = reinterpret_cast<const uint4 *>(xs + (r0 + j) * 128);
#pragma unroll 2
      for (int v = 0; v < 8; ++v) {
        const uint4 w = row[v];
        const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const double t_ = (double)((ww[q >> 2] >> (8 * (q & 3))) & 0xffu) - (double)c_s[16 * v + q];
          s += t_ * t_;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
    if (lane == 0) wmax[j >> 5] = s;
    __syncthreads();
    if (j == 0) {
      double rmax = 0.0;
#pragma unroll
      for (int w = 0; w < TB / 32; ++w) rmax = fmax(rmax, wmax[w]);
      rad[t] = sqrt(rmax) * (1.0 + MARGIN) + 1e-12;
      size[t] = cnt;
    }
    __syncthreads();
  }
}

// dc[Q][T] = |c_Q - c_T| for all tile pairs, register-tiled fp32.
//  * direct difference (GRAM = false): FSUB + FFMA per term, relative error
//    <= (d+2) 2^-24 on dc^2, covered by DC_MARGIN;
//  * norm expansion (GRAM = true; u8 centroids, whose norms are only ~25x the
//    distances): one FFMA per term, |approx - dc^2| <= (d+8) 2^-24 (|c_Q|^2 +
//    |c_T|^2) (the dot, the norms' and the final roundings), subtracted before
//    the square root, so dc is a lower bound (DC_MARGIN covers the sqrt).
constexpr double DC_MARGIN = 2e-5;
constexpr int DB = 64, DK = 32;
template <bool GRAM>
__global__ void __launch_bounds__(256)
    tile_dist_kernel(const float *__restrict__ cent, int64_t T, int d, float *__restrict__ dc,
                     const float *__restrict__ cn) {
  // rows padded to 68 floats: 16-byte aligned, so each thread's 4 rows and 4
  // columns of a k-step are one LDS.128 each
  __shared__ __align__(16) float sa[DK][DB + 4];
  __shared__ __align__(16) float sb[DK][DB + 4];
  __shared__ float st[DB][DB + 1];  // transposed block (mirror write)
  // dc is symmetric bit for bit ((a-b)^2 == (b-a)^2, same FMA order): only
  // blocks on or above the diagonal are computed, and mirrored
  if (blockIdx.x < blockIdx.y) return;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t q0 = (int64_t)blockIdx.y * DB, t0 = (int64_t)blockIdx.x * DB;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < d; k0 += DK) {
    for (int e = threadIdx.x; e < DB * DK; e += 256) {
      const int r = e / DK, k = e % DK;
      sa[k][r] = (q0 + r < T && k0 + k < d) ? cent[(q0 + r) * d + k0 + k] : 0.f;
      sb[k][r] = (t0 + r < T && k0 + k < d) ? cent[(t0 + r) * d + k0 + k] : 0.f;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < DK; ++k) {
      const float4 a4 = *reinterpret_cast<const float4 *>(&sa[k][ty * 4]);
      const float4 b4 = *reinterpret_cast<const float4 *>(&sb[k][tx * 4]);
      const float a[4] = {a4.x, a4.y, a4.z, a4.w}, b[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (GRAM) {
            acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
          } else {
            const float t_ = a[i] - b[j];
            acc[i][j] = fmaf(t_, t_, acc[i][j]);
          }
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t q = q0 + ty * 4 + i, t = t0 + tx * 4 + j;
      float v;
      if (GRAM) {
        const double nn = (q < T && t < T) ? (double)cn[q] + (double)cn[t] : 0.0;
        const double e = (double)(d + 8) * 5.9604644775390625e-08 * 1.01 * nn;
        v = (float)sqrt(fmax(nn - 2.0 * (double)acc[i][j] - e, 0.0));
      } else {
        v = sqrtf(acc[i][j]);
      }
      st[tx * 4 + j][ty * 4 + i] = v;
      if (q < T && t < T) dc[q * T + t] = v;
    }
  if (blockIdx.x == blockIdx.y) return;
  __syncthreads();
  for (int e = threadIdx.x; e < DB * DB; e += 256) {
    const int r = e / DB, c = e % DB;  // mirror row t0 + r, column q0 + c
    if (t0 + r < T && q0 + c < T) dc[(t0 + r) * T + q0 + c] = st[r][c];
  }
}

// fp32 squared norms of the (fp32) centroids, float64 sums rounded once
__global__ void cent_norms_kernel(const float *__restrict__ cent, int64_t T, int d,
                                  float *__restrict__ cn) {
  const int lane = threadIdx.x & 31;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < T;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double s = 0.0;
    for (int k = lane; k < d; k += 32) {
      const double v = (double)cent[t * d + k];
      s += v * v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) cn[t] = (float)s;
  }
}

// pass-1 list: the nearest tiles of every query tile by centroid distance,
// as many as needed to hold >= P1_MULT * K points (at most NEAR tiles)
constexpr int NEAR = 16;
#ifndef TILES_P1_MULT
#define TILES_P1_MULT 4
#endif
constexpr int P1_MULT = TILES_P1_MULT;
__global__ void tile_nearest_kernel(const float *__restrict__ dc, const int32_t *__restrict__ size,
                                    int64_t T, int K, int32_t *__restrict__ lists,
                                    int32_t *__restrict__ lens,
                                    unsigned long long *__restrict__ total) {
  const int lane = threadIdx.x & 31;
  for (int64_t Q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; Q < T;
       Q += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    // per-lane best NEAR (sorted insertion), then a warp sort of 32*NEAR keys
    uint64_t best[NEAR];
#pragma unroll
    for (int i = 0; i < NEAR; ++i) best[i] = KEY_MAX;
    const bool qreal = size[Q] > 0;
    // four columns per lane per trip, loads issued together
    for (int64_t t0 = lane; qreal && t0 < T; t0 += 128) {
      uint64_t kq[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t t = t0 + 32 * u;
        kq[u] = (t < T && size[t] > 0)
                    ? ((uint64_t)__float_as_uint(dc[Q * T + t]) << 32) | (uint32_t)t
                    : KEY_MAX;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint64_t k = kq[u];
        if (k < best[NEAR - 1]) {  // sorted insertion (branch-free shift)
#pragma unroll
          for (int i = NEAR - 1; i > 0; --i)
            best[i] = k < best[i - 1] ? best[i - 1] : (k < best[i] ? k : best[i]);
          best[0] = k < best[0] ? k : best[0];
        }
      }
    }
    // the warp's NEAR smallest keys in order: each lane's list is sorted, so
    // the next one is the warp minimum of the lanes' heads (keys are unique);
    // stop once the tiles hold P1_MULT * K points
    int m = 0, pts = 0;
    uint32_t mine = 0;  // lane i: the i-th nearest tile
    for (int i = 0; i < NEAR; ++i) {
      uint64_t mn = best[0];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t y = __shfl_xor_sync(0xffffffffu, mn, o);
        mn = y < mn ? y : mn;
      }
      if (mn == KEY_MAX) break;
      if (best[0] == mn) {  // pop the owner's head
#pragma unroll
        for (int j = 0; j + 1 < NEAR; ++j) best[j] = best[j + 1];
        best[NEAR - 1] = KEY_MAX;
      }
      if (lane == i) mine = (uint32_t)mn;
      pts += size[(uint32_t)mn];
      m = i + 1;
      if (pts >= P1_MULT * K) break;
    }
    if (lane < m) lists[Q * T + lane] = (int32_t)mine;
    if (lane == 0) {
      lens[Q] = m;
      atomicAdd(total, (unsigned long long)m);
    }
    __syncwarp();
  }
}

// U_Q = max over the tile's rows of the pass-1 K-th neighbour distance
__global__ void tile_ubound_kernel(const uint64_t *__restrict__ keys, int K,
                                   const int32_t *__restrict__ perm, int64_t T,
                                   double *__restrict__ U, double inflate = 1.0) {
  const int lane = threadIdx.x & 31;
  for (int64_t Q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; Q < T;
       Q += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    double m = 0.0;
    for (int r = lane; r < TB; r += 32) {
      const int64_t pos = Q * TB + r;
      if (perm[pos] < 0) continue;
      const uint64_t k = keys[(int64_t)perm[pos] * K + K - 1];
      const double dd = k == KEY_MAX ? __longlong_as_double(0x7ff0000000000000ll)
                                     : (double)key_dist(k);
      m = fmax(m, dd);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    // inflate: approximate pass-1 distances (F32 path) bound the exact K-th
    // one from above only after dividing by (1 - gamma)
    if (lane == 0) U[Q] = sqrt(m * inflate) * (1.0 + MARGIN) + 1e-9;
  }
}

// pass-2 list: every tile T with lb(Q,T) <= scale * U_Q (+1e-9), ascending T;
// with `only`, just the tiles Q with only[Q] != 0 (the others get no list)
__global__ void tile_filter_kernel(const float *__restrict__ dc, const double *__restrict__ rad,
                                   const int32_t *__restrict__ size, const double *__restrict__ U,
                                   int64_t T, int32_t *__restrict__ lists,
                                   int32_t *__restrict__ lens,
                                   unsigned long long *__restrict__ total,
                                   double dc_margin = DC_MARGIN, double scale = 1.0,
                                   const int32_t *__restrict__ only = nullptr) {
  const int lane = threadIdx.x & 31;
  for (int64_t Q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; Q < T;
       Q += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    if (only && only[Q] == 0) {
      if (lane == 0) lens[Q] = 0;
      continue;
    }
    const double rQ = rad[Q], UQ = U[Q] * scale + 1e-9;
    int base = 0;
    const bool qreal = size[Q] > 0;
    // four 32-column chunks per trip, their loads issued together (the
    // per-chunk ballot chain would otherwise expose one global latency each)
    for (int64_t t0 = 0; qreal && t0 < T; t0 += 128) {
      bool keep[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t t = t0 + 32 * u + lane;
        keep[u] = false;
        if (t < T) {
          const int32_t sz = size[t];
          const double lb = (double)dc[Q * T + t] * (1.0 - dc_margin) - rQ - rad[t];
          keep[u] = sz > 0 && lb <= UQ;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const unsigned bal = __ballot_sync(0xffffffffu, keep[u]);
        if (keep[u]) lists[Q * T + base + __popc(bal & lanemask_lt())] = (int32_t)(t0 + 32 * u + lane);
        base += __popc(bal);
      }
    }
    if (lane == 0) {
      lens[Q] = base;
      if (total) atomicAdd(total, (unsigned long long)base);
    }
  }
}

// ---------------------------------------------------------------------------
// Cell-level bounds (sparse tile lists, no T x T centroid-distance matrix).
// Tiles come in cells (every tile lies inside one center's run), so a cell
// is a ball around g_A (the size-weighted mean of its tile centroids, fp32)
// of radius R_A = max_{T in A} (|g_A - c_T| + r_T), and every tile Q of A is
// inside the ball around g_A of radius rho_Q = |c_Q - g_A| + r_Q.  For
// q in Q and x in any tile of cell B:
//     |q - x| >= |g_A - g_B| - rho_Q - R_B =: lbC(Q, B)
// so a whole cell is skipped when lbC > U_Q; only the tiles of the remaining
// cells get their centroid distance (computed on the fly, the same fp32
// norm-expansion lower bound as tile_dist_kernel) and the tile test.
// ---------------------------------------------------------------------------

// tile -> cell map (cells own contiguous tile runs: off is in padded rows)
__global__ void tile_cell_kernel(const int64_t *__restrict__ off, int64_t C,
                                 int32_t *__restrict__ tcell) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < C;
       c += (int64_t)gridDim.x * blockDim.x)
    for (int64_t t = off[c] / TB; t < off[c + 1] / TB; ++t) tcell[t] = (int32_t)c;
}

// block (TB threads, thread = dimension) per cell: g_A, then (warp 0) the
// cell radius and every tile's radius around g_A, in float64 from the fp32
// centroids, inflated by a relative margin
__global__ void __launch_bounds__(TB) cell_stats_kernel(const float *__restrict__ cent,
                                                        const double *__restrict__ rad,
                                                        const int32_t *__restrict__ size,
                                                        const int64_t *__restrict__ off,
                                                        int64_t C, int d, float *__restrict__ g,
                                                        double *__restrict__ Rc,
                                                        double *__restrict__ rho) {
  __shared__ float gs[TB];
  const int j = threadIdx.x, lane = j & 31;
  for (int64_t c = blockIdx.x; c < C; c += gridDim.x) {
    const int64_t t0 = off[c] / TB, t1 = off[c + 1] / TB;
    double acc = 0.0, w = 0.0;
    for (int64_t t = t0; t < t1; ++t) {
      const int sz = size[t];
      if (sz > 0 && j < d) acc += (double)sz * (double)cent[t * d + j];
      w += sz;
    }
    const float gj = (w > 0 && j < d) ? (float)(acc / w) : 0.f;
    if (j < d) g[c * d + j] = gj;
    gs[j] = gj;
    __syncthreads();
    if (j < 32) {
      double R = w > 0 ? 0.0 : -1.0;  // -1: an empty cell, never a candidate
      for (int64_t t = t0; t < t1; ++t) {
        double s2 = 0.0;
        for (int k = lane; k < d; k += 32) {
          const double dd = (double)cent[t * d + k] - (double)gs[k];
          s2 += dd * dd;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        const double rr = sqrt(s2) * (1.0 + 1e-9) + 1e-12 + rad[t];
        if (lane == 0) rho[t] = rr;
        if (size[t] > 0) R = fmax(R, rr);
      }
      if (lane == 0) Rc[c] = R;
    }
    __syncthreads();
  }
}

// lower bound of |c_Q - c_T| from the fp32 centroids (tile_dist_kernel<true>'s
// formula: FMA dot in dimension order, error <= (d+8) 2^-24 (|c_Q|^2+|c_T|^2))
__device__ __forceinline__ float dc_lower(const float *__restrict__ cq, const float *__restrict__ ct,
                                          float cnq, float cnt, int d) {
  float acc = 0.f;
  if ((d & 3) == 0) {
    for (int k = 0; k < d; k += 4) {
      const float4 a = *reinterpret_cast<const float4 *>(cq + k);
      const float4 b = *reinterpret_cast<const float4 *>(ct + k);
      acc = fmaf(a.x, b.x, acc);
      acc = fmaf(a.y, b.y, acc);
      acc = fmaf(a.z, b.z, acc);
      acc = fmaf(a.w, b.w, acc);
    }
  } else {
    for (int k = 0; k < d; ++k) acc = fmaf(cq[k], ct[k], acc);
  }
  const double nn = (double)cnq + (double)cnt;
  const double e = (double)(d + 8) * 5.9604644775390625e-08 * 1.01 * nn;
  return (float)sqrt(fmax(nn - 2.0 * (double)acc - e, 0.0));
}

// pass-1 lists from cells: Q's own cell and its nearest cells (by the cell
// centroid distance) supply the candidate tiles; the nearest of those by
// centroid distance, as many as hold >= P1_MULT * K points (<= NEAR tiles).
// Any real points bound the K-th distance from above, so this is an
// efficiency choice only.  Lists stride NEAR.
constexpr int P1_CELLS = 6;
__global__ void tile_nearest_cells_kernel(const float *__restrict__ cent,
                                          const float *__restrict__ cn,
                                          const int32_t *__restrict__ size,
                                          const int32_t *__restrict__ tcell,
                                          const int64_t *__restrict__ off,
                                          const float *__restrict__ dcc,
                                          const double *__restrict__ Rc, int64_t C, int64_t T,
                                          int d, int K, int32_t *__restrict__ lists,
                                          int32_t *__restrict__ lens,
                                          unsigned long long *__restrict__ total) {
  __shared__ uint64_t ck[8][64];  // 256 threads: per-warp candidate slots
  const int lane = threadIdx.x & 31;
  for (int64_t Q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; Q < T;
       Q += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    if (size[Q] <= 0) {
      if (lane == 0) lens[Q] = 0;
      continue;
    }
    const int32_t A = tcell[Q];
    // the P1_CELLS nearest non-empty cells (A itself at distance 0 first):
    // per-lane best list, then warp minima
    uint64_t best[P1_CELLS];
#pragma unroll
    for (int i = 0; i < P1_CELLS; ++i) best[i] = KEY_MAX;
    for (int64_t b = lane; b < C; b += 32) {
      if (Rc[b] < 0.0) continue;
      const float v = b == A ? 0.f : dcc[(int64_t)A * C + b];
      const uint64_t k = ((uint64_t)__float_as_uint(v) << 32) | (uint32_t)b;
      if (k < best[P1_CELLS - 1]) {
#pragma unroll
        for (int i = P1_CELLS - 1; i > 0; --i)
          best[i] = k < best[i - 1] ? best[i - 1] : (k < best[i] ? k : best[i]);
        best[0] = k < best[0] ? k : best[0];
      }
    }
    // candidate tiles (<= 64): (dc, tile) keys staged in this warp's slots
    uint64_t *mk = ck[threadIdx.x >> 5];
    int nc = 0;
    for (int i = 0; i < P1_CELLS; ++i) {
      uint64_t mn = best[0];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t y = __shfl_xor_sync(0xffffffffu, mn, o);
        mn = y < mn ? y : mn;
      }
      if (mn == KEY_MAX) break;
      if (best[0] == mn) {
#pragma unroll
        for (int j = 0; j + 1 < P1_CELLS; ++j) best[j] = best[j + 1];
        best[P1_CELLS - 1] = KEY_MAX;
      }
      const int64_t bc = (uint32_t)mn;
      const int64_t ta = off[bc] / TB, tb = off[bc + 1] / TB;
      for (int64_t t0 = ta; t0 < tb && nc < 64; t0 += 32) {
        const int64_t t = t0 + lane;
        const bool ok = t < tb && size[t] > 0;
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        const int pos = nc + __popc(bal & ((1u << lane) - 1u));
        if (ok && pos < 64) {
          const float v = dc_lower(cent + Q * d, cent + t * d, cn[Q], cn[t], d);
          mk[pos] = ((uint64_t)__float_as_uint(v) << 32) | (uint32_t)t;
        }
        nc = min(64, nc + __popc(bal));
      }
    }
    __syncwarp();
    uint64_t cand[2] = {lane < nc ? mk[lane] : KEY_MAX, lane + 32 < nc ? mk[lane + 32] : KEY_MAX};
    __syncwarp();
    // the nearest candidates in order until P1_MULT * K points
    int m = 0, pts = 0;
    uint32_t mine = 0;
    for (int i = 0; i < NEAR; ++i) {
      uint64_t a = cand[0] < cand[1] ? cand[0] : cand[1];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t y = __shfl_xor_sync(0xffffffffu, a, o);
        a = y < a ? y : a;
      }
      if (a == KEY_MAX) break;
      if (cand[0] == a) cand[0] = KEY_MAX;
      else if (cand[1] == a) cand[1] = KEY_MAX;
      if (lane == i) mine = (uint32_t)a;
      pts += size[(uint32_t)a];
      m = i + 1;
      if (pts >= P1_MULT * K) break;
    }
    if (lane < m) lists[Q * NEAR + lane] = (int32_t)mine;
    if (lane == 0) {
      lens[Q] = m;
      atomicAdd(total, (unsigned long long)m);
    }
    __syncwarp();
  }
}

// pass-2 lists from cells: every tile T with lb(Q,T) <= scale * U_Q, ascending
// T (cells in order, tiles in order), skipping whole cells by lbC; lists
// stride T as before.  `only`: just the tiles Q with only[Q] != 0.
__global__ void tile_filter_cells_kernel(const float *__restrict__ cent,
                                         const float *__restrict__ cn,
                                         const double *__restrict__ rad,
                                         const double *__restrict__ rho,
                                         const int32_t *__restrict__ size,
                                         const int32_t *__restrict__ tcell,
                                         const int64_t *__restrict__ off,
                                         const float *__restrict__ dcc,
                                         const double *__restrict__ Rc,
                                         const double *__restrict__ U, int64_t C, int64_t T,
                                         int d, int32_t *__restrict__ lists,
                                         int32_t *__restrict__ lens,
                                         unsigned long long *__restrict__ total,
                                         double dc_margin, double scale,
                                         const int32_t *__restrict__ only) {
  const int lane = threadIdx.x & 31;
  for (int64_t Q = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; Q < T;
       Q += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    if ((only && only[Q] == 0) || size[Q] <= 0) {
      if (lane == 0) lens[Q] = 0;
      continue;
    }
    const int32_t A = tcell[Q];
    const double rQ = rad[Q], rhoQ = rho[Q], UQ = U[Q] * scale + 1e-9;
    int base = 0;
    for (int64_t b0 = 0; b0 < C; b0 += 32) {
      const int64_t b = b0 + lane;
      bool cell = false;
      if (b < C && Rc[b] >= 0.0) {
        const double lbc = (b == A ? 0.0 : (double)dcc[(int64_t)A * C + b] * (1.0 - dc_margin)) -
                           rhoQ - Rc[b];
        cell = lbc <= UQ;
      }
      unsigned cm = __ballot_sync(0xffffffffu, cell);
      while (cm) {  // candidate cells in ascending order
        const int64_t bb = b0 + __ffs(cm) - 1;
        cm &= cm - 1;
        const int64_t ta = off[bb] / TB, tb = off[bb + 1] / TB;
        for (int64_t t0 = ta; t0 < tb; t0 += 32) {
          const int64_t t = t0 + lane;
          bool keep = false;
          if (t < tb && size[t] > 0) {
            const float v = dc_lower(cent + Q * d, cent + t * d, cn[Q], cn[t], d);
            keep = (double)v * (1.0 - dc_margin) - rQ - rad[t] <= UQ;
          }
          const unsigned bal = __ballot_sync(0xffffffffu, keep);
          if (keep) lists[Q * T + base + __popc(bal & ((1u << lane) - 1u))] = (int32_t)t;
          base += __popc(bal);
        }
      }
    }
    if (lane == 0) {
      lens[Q] = base;
      if (total) atomicAdd(total, (unsigned long long)base);
    }
  }
}

// Pass-2 threshold guess: seed * SHRINK (exclusive squared-distance bound).
// In high dimension the final K-th distance is a near-constant fraction of
// the pass-1 seed (config 2: 0.86-0.92), so the guess cuts the buffered
// survivors ~2.5x; rows where it proves too tight re-run with the seed.
static float seed_shrink() {
  static float v = -1.0f;
  if (v < 0.0f) {
    const char *e = getenv("PGK_SEED_SHRINK");
    v = e ? (float)atof(e) : 0.93f;
    if (!(v > 0.0f && v <= 1.0f)) v = 1.0f;
  }
  return v;
}

struct Layout {
  float *cen, *cent, *cn, *gcell, *gcn, *dcc;
  double *Rc, *rho;
  int32_t *tcell, *rr;
  int32_t *cnorm, *hist, *cursor, *assign, *perm, *ns, *size, *lists, *lens, *fail, *lens2;
  uint8_t *fail_rows;
  int64_t *off, *scan_tmp;
  uint64_t *akeys;
  double *rad, *U;
  unsigned long long *total;
  uint8_t *xs;
  void *sub_ws;
  size_t sub_bytes, bytes;
  int64_t C, NPmax, Tmax;
};

}  // namespace tiles

size_t tc_pool_workspace(int64_t n, int64_t nq, bool self, bool k1 = false);
int launch_norms_u8(const float *X, int64_t n, int d, int32_t *out, cudaStream_t stream);
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

static tiles::Layout tiles_layout(void *ws, size_t bytes, int64_t n, int64_t d) {
  using namespace tiles;
  Layout L{};
  Carve c(ws, bytes);
  L.C = (n + CSTRIDE - 1) / CSTRIDE;
  L.NPmax = (n + TB - 1) / TB * TB + L.C * TB;  // padded rows, worst case
  L.Tmax = L.NPmax / TB;
  const int64_t C = L.C, NP = L.NPmax, T = L.Tmax;
  L.cen = c.take<float>((size_t)C * d);
  L.cnorm = c.take<int32_t>(C + 128);
  L.akeys = c.take<uint64_t>(n);
  L.hist = c.take<int32_t>(C);
  L.cursor = c.take<int32_t>(C);
  L.assign = c.take<int32_t>(n);
  L.off = c.take<int64_t>(C + 1);
  L.scan_tmp = c.take<int64_t>(scan_scratch(C + 1));
  L.perm = c.take<int32_t>(NP);
  L.xs = c.take<uint8_t>((size_t)NP * 128);
  L.ns = c.take<int32_t>(NP + 128);
  L.cent = c.take<float>((size_t)T * d);
  L.cn = c.take<float>(T);
  L.rad = c.take<double>(T);
  L.size = c.take<int32_t>(T);
  L.lists = c.take<int32_t>((size_t)T * T);
  L.lens = c.take<int32_t>(T);
  L.fail = c.take<int32_t>(T);
  L.lens2 = c.take<int32_t>(T);
  L.fail_rows = c.take<uint8_t>(NP);
  L.gcell = c.take<float>((size_t)C * d);
  L.gcn = c.take<float>(C);
  L.Rc = c.take<double>(C);
  L.rho = c.take<double>(T);
  L.tcell = c.take<int32_t>(T);
  L.dcc = c.take<float>((size_t)C * C);
  L.rr = c.take<int32_t>(NP + 32);
  L.U = c.take<double>(T);
  L.total = c.take<unsigned long long>(4);
  L.sub_bytes = tc_pool_workspace(C, n, false, true);  // K = 1 assignment only
  L.sub_ws = c.take<char>(L.sub_bytes);
  L.bytes = c.off;
  return L;
}

bool tiles_supported(int64_t n, int64_t d, int64_t k) {
  static int env = -1;
  if (env < 0) {
    const char *e = getenv("PGK_DISABLE_PRUNE");
    env = (e && e[0] == '1') ? 1 : 0;
  }
  const int64_t T = ((n + 127) / 128 * 128 + (n + tiles::CSTRIDE - 1) / tiles::CSTRIDE * 128) / 128;
  // the T x T list storage (4 B / tile pair: 6 GB at 4M points) stays
  // bounded; the bounds themselves are per cell pair (no T x T matrix)
  return !env && d <= 128 && k <= 256 && n >= 8 * tiles::TB && T <= 65536;
}

size_t tiles_workspace(int64_t n, int64_t d) { return tiles_layout(nullptr, 0, n, d).bytes; }

// rows of the padded, tile-sorted problem (the tc workspace must cover them)
int64_t tiles_rows(int64_t n) { return tiles_layout(nullptr, 0, n, 1).NPmax; }

// Staged center assignment for rows that arrive in chunks: the centers
// (rows 0, CSTRIDE, 2 CSTRIDE, ... of the data, fp32, device) first, then each
// chunk of exact-integer rows (128 B each) with its norms as it lands.
int64_t tiles_center_stride() { return tiles::CSTRIDE; }

int tiles_u8_prepare(void *tws, size_t tws_bytes, int64_t n, int d, int K, const float *centers,
                     cudaStream_t stream) {
  using namespace tiles;
  PGK_REQUIRE(tiles_supported(n, d, K), "tile pruning does not apply to this shape");
  Layout L = tiles_layout(tws, tws_bytes, n, d);
  PGK_REQUIRE(L.bytes <= tws_bytes, "tile workspace too small");
  PGK_CUDA(cudaMemcpyAsync(L.cen, centers, (size_t)L.C * d * sizeof(float),
                           cudaMemcpyDeviceToDevice, stream));
  return launch_norms_u8(L.cen, L.C, d, L.cnorm, stream);
}

int tiles_u8_assign(void *tws, size_t tws_bytes, int64_t n, int d, int K, const uint8_t *rows_u8,
                    const int32_t *norms, int64_t row0, int64_t nrows, cudaStream_t stream) {
  using namespace tiles;
  PGK_REQUIRE(tiles_supported(n, d, K), "tile pruning does not apply to this shape");
  PGK_REQUIRE(row0 >= 0 && nrows >= 0 && row0 + nrows <= n, "row range out of bounds");
  if (nrows == 0) return PGK_OK;
  Layout L = tiles_layout(tws, tws_bytes, n, d);
  PGK_REQUIRE(L.bytes <= tws_bytes, "tile workspace too small");
  bool h = false;
  // queries = the chunk's u8 rows (the fp32 query pointer is never read)
  const int rc = launch_pool_tc_u8_lists(L.cen, L.C, d, reinterpret_cast<const float *>(rows_u8),
                                         nrows, 0, L.cnorm, norms, 1, L.akeys + row0, L.sub_ws,
                                         L.sub_bytes, stream, nullptr, nullptr, nullptr, 0,
                                         nullptr, &h, nullptr, 0, 1.0f, nullptr, nullptr, nullptr,
                                         nullptr, rows_u8);
  if (rc) return rc;
  PGK_REQUIRE(h, "tensor-core assignment unavailable");
  return PGK_OK;
}

int launch_rerun_rows(int64_t np, void *tc_ws, size_t tc_bytes, const uint8_t *xs,
                      const int32_t *ns, const int32_t *perm, const uint8_t *fail_rows,
                      const int32_t *tlist, const int32_t *tlen, int64_t tstride,
                      const uint64_t *seeds, int K, uint64_t *keys, const PoolOut *out,
                      int32_t *scratch, int max_rows, cudaStream_t stream);

// Runs the whole pruned pool.  *handled = false when pruning does not apply.
extern uint32_t *g_dense_ostat;

int launch_pool_tiles_u8(const float *X, int64_t n, int d, const int32_t *xnorm, int K,
                         uint64_t *keys, void *tc_ws, size_t tc_bytes, void *tws,
                         size_t tws_bytes, cudaStream_t stream, bool *handled,
                         unsigned long long *pairs_out, const PoolOut *out,
                         const uint8_t *xu8_in, bool assigned) {
  using namespace tiles;
  *handled = false;
  if (!tiles_supported(n, d, K)) return PGK_OK;
  Layout L = tiles_layout(tws, tws_bytes, n, d);
  if (L.bytes > tws_bytes) {
    set_error("tile workspace too small");
    return PGK_ERR_NOMEM;
  }
  const int sms = num_sms();
  const int64_t C = L.C;
  const unsigned g = (unsigned)sms * 8;
  // 1. centers (every CSTRIDE-th row) + exact nearest center of every point
  // (K = 1); `assigned`: already done chunk by chunk (tiles_u8_prepare /
  // tiles_u8_assign, the host-data pipeline)
  int rc = PGK_OK;
  if (!assigned) {
  gather_centers_kernel<<<g, 256, 0, stream>>>(X, n, d, C, L.cen);
  PGK_CHECK_LAUNCH("gather_centers_kernel");
  dbg_stage("gather_centers_kernel", stream);
  rc = launch_norms_u8(L.cen, C, d, L.cnorm, stream);
  if (rc) return rc;
  bool h = false;
  rc = launch_pool_tc_u8_lists(L.cen, C, d, X, n, 0, L.cnorm, xnorm, 1, L.akeys, L.sub_ws,
                               L.sub_bytes, stream, nullptr, nullptr, nullptr, 0, nullptr, &h,
                               nullptr, 0, 1.0f, nullptr, nullptr, nullptr, nullptr, xu8_in);
  if (rc) return rc;
  dbg_stage("assign tc", stream);
  if (!h) return PGK_OK;
  }
  // 2. counting sort by center, every run padded to whole tiles (perm = -1)
  PGK_CUDA(cudaMemsetAsync(L.hist, 0, C * 4, stream));
  PGK_CUDA(cudaMemsetAsync(L.cursor, 0, C * 4, stream));
  assign_hist_kernel<<<g, 256, 0, stream>>>(L.akeys, n, L.hist, L.assign);
  PGK_CHECK_LAUNCH("assign_hist_kernel");
  dbg_stage("assign_hist_kernel", stream);
  padded_len_kernel<<<g, 256, 0, stream>>>(L.hist, C, L.off);
  PGK_CHECK_LAUNCH("padded_len_kernel");
  dbg_stage("padded_len_kernel", stream);
  rc = exclusive_scan(L.off, L.off, C + 1, L.scan_tmp, stream);
  if (rc) return rc;
  // the padded total lives on the device; kernels below run over the
  // worst-case size and treat tiles past the real total as empty
  fill_i32_kernel<<<g, 256, 0, stream>>>(L.perm, L.NPmax, -1);
  PGK_CHECK_LAUNCH("fill_i32_kernel");
  assign_scatter_kernel<<<g, 256, 0, stream>>>(L.assign, n, L.off, L.cursor, L.perm);
  PGK_CHECK_LAUNCH("assign_scatter_kernel");
  dbg_stage("assign_scatter_kernel", stream);
  const int64_t NP = L.NPmax, T = L.Tmax;
  // 3. sorted u8 rows / norms, tile summaries, centroid distances
  if (xu8_in) {
    gather_sorted_u8_kernel<<<g, 256, 0, stream>>>(xu8_in, L.perm, xnorm, NP, L.xs, L.ns);
    PGK_CHECK_LAUNCH("gather_sorted_u8_kernel");
  } else {
    gather_sorted_kernel<<<g, 256, 0, stream>>>(X, d, L.perm, xnorm, NP, L.xs, L.ns);
    PGK_CHECK_LAUNCH("gather_sorted_kernel");
  }
  dbg_stage("gather_sorted_kernel", stream);
  fill_i32_kernel<<<1, 128, 0, stream>>>(L.ns + NP, 128, 0x3f3f3f3f);
  PGK_CHECK_LAUNCH("fill_i32_kernel");
  tile_stats_kernel<<<(unsigned)std::min<int64_t>(T, (int64_t)sms * 16), TB, 0, stream>>>(
      L.xs, L.perm, d, T, L.cent, L.rad, L.size);
  PGK_CHECK_LAUNCH("tile_stats_kernel");
  dbg_stage("tile_stats_kernel", stream);
  PGK_CUDA(cudaMemsetAsync(L.total, 0, 4 * sizeof(unsigned long long), stream));
  cent_norms_kernel<<<g, 256, 0, stream>>>(L.cent, T, d, L.cn);
  PGK_CHECK_LAUNCH("cent_norms_kernel");
  // cells as balls (g_A, R_A), tiles' radii around their cell, and the C x C
  // cell-centroid distances: the bounds of the sparse tile lists
  tile_cell_kernel<<<g, 256, 0, stream>>>(L.off, C, L.tcell);
  PGK_CHECK_LAUNCH("tile_cell_kernel");
  cell_stats_kernel<<<(unsigned)std::min<int64_t>(C, (int64_t)sms * 16), TB, 0, stream>>>(
      L.cent, L.rad, L.size, L.off, C, d, L.gcell, L.Rc, L.rho);
  PGK_CHECK_LAUNCH("cell_stats_kernel");
  cent_norms_kernel<<<g, 256, 0, stream>>>(L.gcell, C, d, L.gcn);
  PGK_CHECK_LAUNCH("cent_norms_kernel");
  tile_dist_kernel<true><<<dim3((unsigned)((C + DB - 1) / DB), (unsigned)((C + DB - 1) / DB)),
                            256, 0, stream>>>(L.gcell, C, d, L.dcc, L.gcn);
  PGK_CHECK_LAUNCH("tile_dist_kernel (cells)");
  dbg_stage("cell bounds", stream);
  // 4. pass 1: exact top-K over each query tile's nearest tiles (from its
  // own and the nearest cells) -> U_Q; lists of stride NEAR
  tile_nearest_cells_kernel<<<g, 256, 0, stream>>>(L.cent, L.cn, L.size, L.tcell, L.off, L.dcc,
                                                   L.Rc, C, T, d, K, L.lists, L.lens, L.total + 1);
  PGK_CHECK_LAUNCH("tile_nearest_cells_kernel");
  dbg_stage("tile_nearest_cells_kernel", stream);
  const char *se0 = getenv("PGK_TILES_STATS");
  uint32_t *ostat = nullptr;
  if (se0 && se0[0] == '1') {  // pass-1 order statistics for the guess analysis
    PGK_CUDA(cudaMalloc(&ostat, (size_t)n * 4 * sizeof(uint32_t)));
    g_dense_ostat = ostat;
  }
  rc = launch_pool_tc_u8_lists(X, NP, d, X, NP, 1, L.ns, L.ns, K, keys, tc_ws, tc_bytes, stream,
                               L.xs, L.lists, L.lens, NEAR, L.perm, handled, nullptr, 1);
  g_dense_ostat = nullptr;
  if (rc) return rc;
  dbg_stage("pass 1 tc", stream);
  if (!*handled) return PGK_OK;
  tile_ubound_kernel<<<g, 256, 0, stream>>>(keys, K, L.perm, T, L.U);
  PGK_CHECK_LAUNCH("tile_ubound_kernel");
  dbg_stage("tile_ubound_kernel", stream);
  // 5. pass 2: every tile that can hold a pool member, then the full top-K.
  // With a guessed threshold g <= shrink * seed a row is exact only when it
  // finds >= K points below g (verified), and every point below g lies
  // within sqrt(shrink) * U_Q of the tile: the list can be cut to that
  // radius; rows failing the guess re-run on the full-radius list (step 6).
  const float shrink = seed_shrink();
  tile_filter_cells_kernel<<<g, 256, 0, stream>>>(
      L.cent, L.cn, L.rad, L.rho, L.size, L.tcell, L.off, L.dcc, L.Rc, L.U, C, T, d, L.lists,
      L.lens, L.total, DC_MARGIN, shrink < 1.0f ? sqrt((double)shrink) : 1.0, nullptr);
  PGK_CHECK_LAUNCH("tile_filter_cells_kernel");
  dbg_stage("tile_filter_kernel", stream);
  const char *se = getenv("PGK_TILES_STATS");
  const bool stats = se && se[0] == '1';
  std::vector<uint64_t> seed_k;
  if (stats) {  // each row's pass-1 K-th key (the pass-2 seed)
    seed_k.resize(n);
    PGK_CUDA(cudaMemcpy2DAsync(seed_k.data(), 8, keys + K - 1, (size_t)K * 8, 8, n,
                               cudaMemcpyDeviceToHost, stream));
  }
  PGK_CUDA(cudaMemsetAsync(L.fail, 0, T * 4, stream));
  PGK_CUDA(cudaMemsetAsync(L.fail_rows, 0, NP, stream));
  rc = launch_pool_tc_u8_lists(X, NP, d, X, NP, 1, L.ns, L.ns, K, keys, tc_ws, tc_bytes, stream,
                               L.xs, L.lists, L.lens, T, L.perm, handled, keys, 0, shrink,
                               L.fail, out, L.fail_rows);
  if (rc) return rc;
  dbg_stage("pass 2 tc", stream);
  if (shrink < 1.0f) {
    // 6. re-run the rows whose guess was too tight (their blocks, row mask),
    // seeded by their untouched pass-1 key, on the full-radius list
    tile_filter_cells_kernel<<<g, 256, 0, stream>>>(
        L.cent, L.cn, L.rad, L.rho, L.size, L.tcell, L.off, L.dcc, L.Rc, L.U, C, T, d, L.lists,
        L.lens2, nullptr, DC_MARGIN, 1.0, L.fail);
    PGK_CHECK_LAUNCH("tile_filter_cells_kernel (re-run)");
  dbg_stage("tile_filter_kernel (re-run)", stream);
    if (stats) {
      std::vector<int32_t> hf(T);
      PGK_CUDA(cudaMemcpyAsync(hf.data(), L.fail, T * 4, cudaMemcpyDeviceToHost, stream));
      PGK_CUDA(cudaStreamSynchronize(stream));
      int64_t nf = 0;
      for (auto f : hf) nf += f != 0;
      fprintf(stderr, "[tiles] guess %.3f: %lld of %lld blocks re-run\n", shrink, (long long)nf,
              (long long)T);
    }
    // the failing rows alone, exact SIMT rescans over their full-radius
    // lists (their whole blocks on the tensor cores cost ~4x more)
    // (when they are more than 1/32 of the rows -- a dataset the 0.93 guess
    // does not fit -- their blocks re-run on the tensor cores instead: both
    // launches read the failing-row count on the device and one exits)
    const int max_rows = (int)std::max<int64_t>(1024, n / 32);
    rc = launch_rerun_rows(NP, tc_ws, tc_bytes, L.xs, L.ns, L.perm, L.fail_rows, L.lists,
                           L.lens2, T, keys, K, keys, out, L.rr, max_rows, stream);
    if (rc) return rc;
    rc = launch_pool_tc_u8_lists(X, NP, d, X, NP, 1, L.ns, L.ns, K, keys, tc_ws, tc_bytes,
                                 stream, L.xs, L.lists, L.lens2, T, L.perm, handled, keys, 0,
                                 1.0f, nullptr, out, nullptr, L.fail_rows, nullptr, L.rr,
                                 max_rows + 1);
    if (rc) return rc;
  }
  if (stats && out) {  // final K-th distance (pool output) over the pass-2 seed
    std::vector<float> final_d(n);
    PGK_CUDA(cudaMemcpy2DAsync(final_d.data(), 4, out->dists + K - 1, (size_t)K * 4, 4, n,
                               cudaMemcpyDeviceToHost, stream));
    PGK_CUDA(cudaStreamSynchronize(stream));
    std::vector<double> ratio;
    for (int64_t i = 0; i < n; ++i) {
      const uint32_t a = (uint32_t)(seed_k[i] >> 32) & 0x7fffffffu;
      float fa;
      memcpy(&fa, &a, 4);
      if (fa > 0) ratio.push_back(final_d[i] / fa);
    }
    std::sort(ratio.begin(), ratio.end());
    auto qq = [&](double f) { return ratio.empty() ? 0.0 : ratio[(size_t)(f * (ratio.size() - 1))]; };
    fprintf(stderr, "[tiles] final/seed K-th dist ratio p1/p10/p50/p90/p99 %.3f %.3f %.3f %.3f %.3f max %.3f\n",
            qq(.01), qq(.1), qq(.5), qq(.9), qq(.99), qq(1.0));
    for (double f : {0.90, 0.92, 0.93, 0.94, 0.95, 0.96}) {
      const size_t above = ratio.end() - std::lower_bound(ratio.begin(), ratio.end(), f);
      fprintf(stderr, "[tiles]   rows with ratio >= %.2f: %zu\n", f, above);
    }
    if (ostat) {  // predictors: pass-1 order statistics K/8, K/4, K/2, K
      std::vector<uint32_t> os((size_t)n * 4);
      PGK_CUDA(cudaMemcpy(os.data(), ostat, os.size() * 4, cudaMemcpyDeviceToHost));
      for (int j = 0; j < 4; ++j) {
        std::vector<double> rr;
        for (int64_t i = 0; i < n; ++i)
          if (os[i * 4 + j] > 0 && os[i * 4 + j] != 0xffffffffu)
            rr.push_back(final_d[i] / (double)os[i * 4 + j]);
        std::sort(rr.begin(), rr.end());
        auto q = [&](double f) { return rr.empty() ? 0.0 : rr[(size_t)(f * (rr.size() - 1))]; };
        const double f = q(0.998);  // guess factor failing 0.2 % of rows
        double surv = 0;  // mean (guess / final)^12.9: relative buffered survivors
        for (double x : rr) surv += pow(f / x, 12.9);
        fprintf(stderr, "[tiles] predictor rank K>>%d: final/pred p1 %.3f p50 %.3f p99.8 %.3f "
                "-> survivors x%.2f of exact\n", 3 - j, q(0.01), q(0.5), f, surv / rr.size());
      }
      cudaFree(ostat);
    }
  }
  {  // work record: [0] pass-2 tile pairs, [1] pass-1 pairs, [2] assignment pairs, [3] done
    const unsigned long long rec[2] = {
        (unsigned long long)((n + TB - 1) / TB) * (unsigned long long)((C + TB - 1) / TB), 1ull};
    PGK_CUDA(cudaMemcpyAsync(L.total + 2, rec, sizeof(rec), cudaMemcpyHostToDevice, stream));
  }
  if (stats) {
    unsigned long long tot = 0;
    PGK_CUDA(cudaMemcpyAsync(&tot, L.total, sizeof(tot), cudaMemcpyDeviceToHost, stream));
    std::vector<double> hr(T), hu(T);
    std::vector<int32_t> hs(T);
    PGK_CUDA(cudaMemcpyAsync(hr.data(), L.rad, T * 8, cudaMemcpyDeviceToHost, stream));
    PGK_CUDA(cudaMemcpyAsync(hu.data(), L.U, T * 8, cudaMemcpyDeviceToHost, stream));
    PGK_CUDA(cudaMemcpyAsync(hs.data(), L.size, T * 4, cudaMemcpyDeviceToHost, stream));
    PGK_CUDA(cudaStreamSynchronize(stream));
    std::vector<double> r2, u2;
    int64_t real = 0;
    for (int64_t t = 0; t < T; ++t)
      if (hs[t] > 0) { r2.push_back(hr[t]); u2.push_back(hu[t]); ++real; }
    auto q = [](std::vector<double> v, double f) {
      std::sort(v.begin(), v.end());
      return v.empty() ? 0.0 : v[(size_t)(f * (v.size() - 1))];
    };
    fprintf(stderr,
            "[tiles] %lld non-empty tiles (padded rows %.1f%%); candidate pairs %llu = %.3f%% of "
            "N^2 tiles, mean list %.1f | radius p50/p90/max %.1f %.1f %.1f | U_Q p50/p90 %.1f "
            "%.1f\n",
            (long long)real, 100.0 * (real * 128.0 - n) / (real * 128.0), tot,
            100.0 * tot / ((double)real * real), (double)tot / real, q(r2, .5), q(r2, .9),
            q(r2, 1.0), q(u2, .5), q(u2, .9));
  }
  if (pairs_out) *pairs_out = 0;
  return PGK_OK;
}

// ===========================================================================
// F32 path (general float data: configs 1, 3, 4).  Same tiles and bounds; the
// tile passes run the SIMT direct-difference kernel over candidate lists and
// keep S = K + margin approximate survivors per row, which pool_simt.cu's
// float64 rerank then proves exact (or sends to the exact fallback).  Points
// with exact distance > U_Q are excluded by the bound, so the rerank's proof
// only has to cover the candidates it saw.
//   * assignment: the first <= 128 dimensions quantised to u8 by one global
//     affine map feed the tcgen05 K = 1 kernel -- only an efficiency
//     heuristic, correctness rests on the float64 radii of step 3;
//   * dc: fp32 direct-difference centroid distances, relative error
//     <= (d+2) 2^-24 on dc^2 (margin scaled with d);
//   * U_Q: the pass-1 K-th *approximate* distance a_K bounds the exact K-th
//     one by a_K / (1 - gamma), gamma = (d+2) 2^-24 (the rerank's bound).
// ===========================================================================
namespace tiles {

constexpr int DA = 128;  // assignment dimensions
// one center per 256 rows: mixture data with many components (config 4: 1000
// components, 2M points) still gets a center in practically every component
// (P(miss) ~ e^-7.8), which keeps cells -- hence tiles -- single-component
constexpr int CSTRIDE_F = 256;

__device__ __forceinline__ uint32_t f2ord(float f) {
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t o) {
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

// global min / max over the first da dimensions (orderable-uint atomics)
__global__ void minmax_kernel(const float *__restrict__ X, int64_t n, int d, int da,
                              uint32_t *__restrict__ mm) {
  uint32_t lo = 0xffffffffu, hi = 0u;
  const int64_t total = n * da;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / da;
    const uint32_t o = f2ord(X[r * d + (e - r * da)]);
    lo = min(lo, o);
    hi = max(hi, o);
  }
  lo = __reduce_min_sync(0xffffffffu, lo);
  hi = __reduce_max_sync(0xffffffffu, hi);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mm, lo);
    atomicMax(mm + 1, hi);
  }
}

// rows (every `stride`-th from `first` of X) -> da integer-valued floats in [0, 255]
__global__ void quantize_kernel(const float *__restrict__ X, int64_t rows, int64_t stride,
                                int d, int da, const uint32_t *__restrict__ mm,
                                float *__restrict__ out) {
  const float lo = ord2f(mm[0]), hi = ord2f(mm[1]);
  const float scale = hi > lo ? 255.0f / (hi - lo) : 0.0f;
  const int64_t total = rows * da;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / da;
    const float v = X[r * stride * d + (e - r * da)];
    out[e] = fminf(255.0f, fmaxf(0.0f, rintf((v - lo) * scale)));
  }
}

// tile-sorted float rows; padding rows are zero (perm < 0 keeps them out)
__global__ void gather_sorted_f32_kernel(const float *__restrict__ X, int d,
                                         const int32_t *__restrict__ perm, int64_t np,
                                         float *__restrict__ xs) {
  const int64_t total = np * d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / d;
    const int32_t src = perm[r];
    xs[e] = src >= 0 ? X[(int64_t)src * d + (e - r * d)] : 0.0f;
  }
}

// warp per tile: float64 centroid of the real rows (stored fp32), radius
// against the stored centroid in float64 (inflated)
__global__ void tile_stats_f32_kernel(const float *__restrict__ xs,
                                      const int32_t *__restrict__ perm, int d, int64_t ntiles,
                                      float *__restrict__ cent, double *__restrict__ rad,
                                      int32_t *__restrict__ size) {
  const int lane = threadIdx.x & 31;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < ntiles;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t r0 = t * TB;
    int cnt = 0;
    for (int i = 0; i < TB; ++i) cnt += perm[r0 + i] >= 0;
    for (int k0 = 0; k0 < d; k0 += 32) {
      const int k = k0 + lane;
      double acc = 0.0;
      if (k < d)
        for (int i = 0; i < TB; ++i)
          if (perm[r0 + i] >= 0) acc += (double)xs[(r0 + i) * d + k];
      if (k < d) cent[t * d + k] = cnt ? (float)(acc / cnt) : 0.f;
    }
    __syncwarp();
    double rmax = 0.0;
    for (int i = 0; i < TB; ++i) {
      if (perm[r0 + i] < 0) continue;
      double s = 0.0;
      for (int k = lane; k < d; k += 32) {
        const double t_ = (double)xs[(r0 + i) * d + k] - (double)cent[t * d + k];
        s += t_ * t_;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      rmax = fmax(rmax, s);
    }
    if (lane == 0) {
      rad[t] = sqrt(rmax) * (1.0 + MARGIN) + 1e-12;
      size[t] = cnt;
    }
  }
}

struct LayoutF32 {
  float *cen_q, *xq, *cent, *dcm, *xs;
  int32_t *cnorm, *xnorm, *hist, *cursor, *assign, *perm, *size, *lists, *lens;
  uint32_t *mm;
  int64_t *off, *scan_tmp;
  uint64_t *akeys, *keys1;
  double *rad, *U;
  unsigned long long *total;
  void *sub_ws, *tcf_ws;
  size_t sub_bytes, tcf_bytes, bytes;
  int64_t C, NPmax, Tmax;
};

}  // namespace tiles

bool tcf32_supported(int64_t d, int64_t k);
size_t tcf32_workspace(int64_t np, int64_t T, int64_t d);
int tcf32_prepare(const float *xs, const int32_t *perm, const float *cent, const double *rad,
                  const int32_t *size, int64_t np, int64_t T, int d, void *ws, size_t bytes,
                  cudaStream_t stream);
int tcf32_tau_from_keys(const uint64_t *keys1, int K, const int32_t *perm, int64_t np, int64_t T,
                        int d, double inflate, void *ws, size_t bytes, cudaStream_t stream);
int tcf32_pass(const float *xs, int64_t np, int64_t T, int d, const int32_t *perm, const int32_t *tlist,
               const int32_t *tlen, int64_t tstride, int K, int ub, double *U, uint64_t *keys,
               void *ws, size_t bytes, cudaStream_t stream);

static tiles::LayoutF32 tiles_layout_f32(void *ws, size_t bytes, int64_t n, int64_t d,
                                         int64_t K) {
  using namespace tiles;
  LayoutF32 L{};
  Carve c(ws, bytes);
  L.C = (n + CSTRIDE_F - 1) / CSTRIDE_F;
  L.NPmax = (n + TB - 1) / TB * TB + L.C * TB;
  L.Tmax = L.NPmax / TB;
  const int64_t C = L.C, NP = L.NPmax, T = L.Tmax;
  // layout prefix shared with Layout: size / perm / total / akeys are what
  // the order and work helpers read (tiles_order_ptrs)
  L.total = c.take<unsigned long long>(4);
  L.mm = c.take<uint32_t>(2);
  L.cen_q = c.take<float>((size_t)C * DA);
  L.xq = c.take<float>((size_t)n * DA);
  L.cnorm = c.take<int32_t>(C + 128);
  L.xnorm = c.take<int32_t>(n + 128);
  L.akeys = c.take<uint64_t>(n);
  L.hist = c.take<int32_t>(C);
  L.cursor = c.take<int32_t>(C);
  L.assign = c.take<int32_t>(n);
  L.off = c.take<int64_t>(C + 1);
  L.scan_tmp = c.take<int64_t>(scan_scratch(C + 1));
  L.perm = c.take<int32_t>(NP);
  L.xs = c.take<float>((size_t)NP * d);
  L.cent = c.take<float>((size_t)T * d);
  L.rad = c.take<double>(T);
  L.size = c.take<int32_t>(T);
  L.lists = c.take<int32_t>((size_t)T * T);
  L.lens = c.take<int32_t>(T);
  L.dcm = c.take<float>((size_t)T * T);
  L.U = c.take<double>(T);
  L.keys1 = c.take<uint64_t>((size_t)n * K);
  L.sub_bytes = tc_pool_workspace(C, n, false, true);  // K = 1 assignment only
  L.sub_ws = c.take<char>(L.sub_bytes);
  L.tcf_bytes = tcf32_supported(d, K) ? tcf32_workspace(NP, T, d) : 0;
  L.tcf_ws = L.tcf_bytes ? c.take<char>(L.tcf_bytes) : nullptr;
  L.bytes = c.off;
  return L;
}

bool tiles_f32_supported(int64_t n, int64_t d, int64_t k) {
  static int env = -1;
  if (env < 0) {
    const char *e = getenv("PGK_DISABLE_PRUNE");
    env = (e && e[0] == '1') ? 1 : 0;
  }
  const int64_t T = ((n + 127) / 128 * 128 + (n + 255) / 256 * 128) / 128;
  return !env && k <= 384 && n >= 8 * tiles::TB && T <= 32768;
}

size_t tiles_f32_workspace(int64_t n, int64_t d, int64_t k) {
  return tiles_layout_f32(nullptr, 0, n, d, k).bytes;
}

int launch_pool_f32_lists(const float *xs, int64_t np, int d, int S, int vec4,
                          const int32_t *tlist, const int32_t *tlen, int64_t tstride,
                          const int32_t *perm, uint64_t *keys, cudaStream_t stream);

// The pruned F32 pool: every row's S best approximate keys in keys (n x S,
// original order, original ids), for pool_simt.cu's rerank + fallback.
struct FbTiles {  // pool_simt.cu: the exact rescan's view of the pass-2 lists
  const int32_t *lists, *lens;
  int64_t stride;
  const int32_t *perm, *ipos;
  const float *xs;
};

namespace tiles {
// original id -> tile-sorted position
__global__ void inverse_perm_kernel(const int32_t *__restrict__ perm, int64_t np,
                                    int32_t *__restrict__ ipos) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < np;
       p += (int64_t)gridDim.x * blockDim.x)
    if (perm[p] >= 0) ipos[perm[p]] = (int32_t)p;
}
}  // namespace tiles

int launch_pool_tiles_f32(const float *X, int64_t n, int d, int K, int S, uint64_t *keys,
                          void *tws, size_t tws_bytes, cudaStream_t stream, bool *handled,
                          bool *lb_keys, FbTiles *ft) {
  using namespace tiles;
  *handled = false;
  *lb_keys = false;
  if (!tiles_f32_supported(n, d, K)) return PGK_OK;
  LayoutF32 L = tiles_layout_f32(tws, tws_bytes, n, d, K);
  if (L.bytes > tws_bytes) {
    set_error("F32 tile workspace too small");
    return PGK_ERR_NOMEM;
  }
  const int sms = num_sms();
  const int64_t C = L.C, NP = L.NPmax, T = L.Tmax;
  const unsigned g = (unsigned)sms * 8;
  const int da = d < DA ? d : DA;
  // 1. approximate nearest center on quantised leading dimensions (tcgen05)
  const uint32_t mm0[2] = {0xffffffffu, 0u};
  PGK_CUDA(cudaMemcpyAsync(L.mm, mm0, sizeof(mm0), cudaMemcpyHostToDevice, stream));
  minmax_kernel<<<g, 256, 0, stream>>>(X, n, d, da, L.mm);
  PGK_CHECK_LAUNCH("minmax_kernel");
  dbg_stage("minmax_kernel", stream);
  quantize_kernel<<<g, 256, 0, stream>>>(X, n, 1, d, da, L.mm, L.xq);
  PGK_CHECK_LAUNCH("quantize_kernel");
  dbg_stage("quantize_kernel", stream);
  quantize_kernel<<<g, 256, 0, stream>>>(X, C, CSTRIDE_F, d, da, L.mm, L.cen_q);
  PGK_CHECK_LAUNCH("quantize_kernel");
  dbg_stage("quantize_kernel", stream);
  int rc = launch_norms_u8(L.cen_q, C, da, L.cnorm, stream);
  if (rc) return rc;
  rc = launch_norms_u8(L.xq, n, da, L.xnorm, stream);
  if (rc) return rc;
  bool h = false;
  rc = launch_pool_tc_u8_lists(L.cen_q, C, da, L.xq, n, 0, L.cnorm, L.xnorm, 1, L.akeys,
                               L.sub_ws, L.sub_bytes, stream, nullptr, nullptr, nullptr, 0,
                               nullptr, &h);
  if (rc) return rc;
  dbg_stage("assign tc", stream);
  if (!h) return PGK_OK;
  // 2. counting sort by center, runs padded to whole tiles
  PGK_CUDA(cudaMemsetAsync(L.hist, 0, C * 4, stream));
  PGK_CUDA(cudaMemsetAsync(L.cursor, 0, C * 4, stream));
  assign_hist_kernel<<<g, 256, 0, stream>>>(L.akeys, n, L.hist, L.assign);
  PGK_CHECK_LAUNCH("assign_hist_kernel");
  dbg_stage("assign_hist_kernel", stream);
  padded_len_kernel<<<g, 256, 0, stream>>>(L.hist, C, L.off);
  PGK_CHECK_LAUNCH("padded_len_kernel");
  dbg_stage("padded_len_kernel", stream);
  rc = exclusive_scan(L.off, L.off, C + 1, L.scan_tmp, stream);
  if (rc) return rc;
  fill_i32_kernel<<<g, 256, 0, stream>>>(L.perm, NP, -1);
  PGK_CHECK_LAUNCH("fill_i32_kernel");
  assign_scatter_kernel<<<g, 256, 0, stream>>>(L.assign, n, L.off, L.cursor, L.perm);
  PGK_CHECK_LAUNCH("assign_scatter_kernel");
  dbg_stage("assign_scatter_kernel", stream);
  // 3. sorted rows, tile summaries (float64), centroid distances
  gather_sorted_f32_kernel<<<g, 256, 0, stream>>>(X, d, L.perm, NP, L.xs);
  PGK_CHECK_LAUNCH("gather_sorted_f32_kernel");
  tile_stats_f32_kernel<<<g, 256, 0, stream>>>(L.xs, L.perm, d, T, L.cent, L.rad, L.size);
  PGK_CHECK_LAUNCH("tile_stats_f32_kernel");
  PGK_CUDA(cudaMemsetAsync(L.total, 0, 4 * sizeof(unsigned long long), stream));
  tile_dist_kernel<false><<<dim3((unsigned)((T + DB - 1) / DB), (unsigned)((T + DB - 1) / DB)),
                            256, 0, stream>>>(L.cent, T, d, L.dcm, nullptr);
  PGK_CHECK_LAUNCH("tile_dist_kernel");
  dbg_stage("tile_dist_kernel", stream);
  // 4. pass 1: top-K over each query tile's nearest tiles -> U_Q
  const int vec4 = (d % 4 == 0);
  tile_nearest_kernel<<<g, 256, 0, stream>>>(L.dcm, L.size, T, K, L.lists, L.lens, L.total + 1);
  PGK_CHECK_LAUNCH("tile_nearest_kernel");
  dbg_stage("tile_nearest_kernel", stream);
  // float pools on the tensor cores (pool_tc_f32.cu): centred bf16 operands,
  // proven bounds.  PGK_F32_TC=1: pass 2 only (SIMT pass 1), 2 (default): both
  static int tc_mode = -1;
  if (tc_mode < 0) {
    const char *e = getenv("PGK_F32_TC");
    tc_mode = e ? atoi(e) : 2;
  }
  const bool use_tc = L.tcf_ws != nullptr && tc_mode > 0;
  if (use_tc) {
    rc = tcf32_prepare(L.xs, L.perm, L.cent, L.rad, L.size, NP, T, d, L.tcf_ws, L.tcf_bytes, stream);
    if (rc) return rc;
    dbg_stage("tcf32_prepare", stream);
  }
  const double gamma = (double)(d + 2) * 5.9604644775390625e-08 * 1.001 + 1e-12;
  if (use_tc && tc_mode >= 2) {
    rc = tcf32_pass(L.xs, NP, T, d, L.perm, L.lists, L.lens, T, K, 1, L.U, nullptr, L.tcf_ws,
                    L.tcf_bytes, stream);
    if (rc) return rc;
    dbg_stage("tcf32 pass 1", stream);
  } else {
    rc = launch_pool_f32_lists(L.xs, NP, d, K, vec4, L.lists, L.lens, T, L.perm, L.keys1, stream);
    if (rc) return rc;
    tile_ubound_kernel<<<g, 256, 0, stream>>>(L.keys1, K, L.perm, T, L.U, 1.0 / (1.0 - gamma));
    PGK_CHECK_LAUNCH("tile_ubound_kernel");
    dbg_stage("tile_ubound_kernel", stream);
    if (use_tc) {
      rc = tcf32_tau_from_keys(L.keys1, K, L.perm, NP, T, d, 1.0 / (1.0 - gamma), L.tcf_ws,
                               L.tcf_bytes, stream);
      if (rc) return rc;
    }
  }
  // 5. pass 2: every tile that can hold a pool member; S approximate survivors
  const double dc_margin = std::max(DC_MARGIN, 2.0 * gamma);
  tile_filter_kernel<<<g, 256, 0, stream>>>(L.dcm, L.rad, L.size, L.U, T, L.lists, L.lens,
                                            L.total, dc_margin);
  PGK_CHECK_LAUNCH("tile_filter_kernel");
  dbg_stage("tile_filter_kernel", stream);
  if (use_tc) {
    rc = tcf32_pass(L.xs, NP, T, d, L.perm, L.lists, L.lens, T, S, 0, nullptr, keys, L.tcf_ws,
                    L.tcf_bytes, stream);
    if (rc) return rc;
    *lb_keys = true;
    dbg_stage("tcf32 pass 2", stream);
  } else {
    rc = launch_pool_f32_lists(L.xs, NP, d, S, vec4, L.lists, L.lens, T, L.perm, keys, stream);
    if (rc) return rc;
  }
  const char *se = getenv("PGK_TILES_STATS");
  if (se && se[0] == '1') {
    unsigned long long tot[2] = {0, 0};
    PGK_CUDA(cudaMemcpyAsync(tot, L.total, sizeof(tot), cudaMemcpyDeviceToHost, stream));
    std::vector<double> hr(T), hu(T);
    std::vector<int32_t> hs(T);
    PGK_CUDA(cudaMemcpyAsync(hr.data(), L.rad, T * 8, cudaMemcpyDeviceToHost, stream));
    PGK_CUDA(cudaMemcpyAsync(hu.data(), L.U, T * 8, cudaMemcpyDeviceToHost, stream));
    PGK_CUDA(cudaMemcpyAsync(hs.data(), L.size, T * 4, cudaMemcpyDeviceToHost, stream));
    PGK_CUDA(cudaStreamSynchronize(stream));
    std::vector<double> r2, u2;
    for (int64_t t = 0; t < T; ++t)
      if (hs[t] > 0) { r2.push_back(hr[t]); u2.push_back(hu[t]); }
    auto q = [](std::vector<double> v, double f) {
      std::sort(v.begin(), v.end());
      return v.empty() ? 0.0 : v[(size_t)(f * (v.size() - 1))];
    };
    const double real = (double)r2.size();
    fprintf(stderr,
            "[tiles f32] %.0f tiles; pass-1 pairs %llu, pass-2 pairs %llu = %.3f%% of all, mean "
            "list %.1f | radius p50/p90 %.3g %.3g | U_Q p50/p90 %.3g %.3g\n",
            real, tot[1], tot[0], 100.0 * tot[0] / (real * real), tot[0] / real, q(r2, .5),
            q(r2, .9), q(u2, .5), q(u2, .9));
  }
  {  // work record: [2] assignment (center) pairs, [3] done
    const unsigned long long rec[2] = {
        (unsigned long long)((n + TB - 1) / TB) * (unsigned long long)((C + TB - 1) / TB), 1ull};
    PGK_CUDA(cudaMemcpyAsync(L.total + 2, rec, sizeof(rec), cudaMemcpyHostToDevice, stream));
  }
  // the exact rescan of rows whose proof fails reads only their pass-2 tiles
  // (assign is free after the counting sort: it takes the inverse permutation)
  inverse_perm_kernel<<<g, 256, 0, stream>>>(L.perm, NP, L.assign);
  PGK_CHECK_LAUNCH("inverse_perm_kernel");
  *ft = FbTiles{L.lists, L.lens, T, L.perm, L.assign, L.xs};
  *handled = true;
  return PGK_OK;
}

// Locality order of the last pruned launch: the real rows of the tile
// permutation, tile by tile (identity when the pruned path did not run).
__global__ void order_scan_kernel(const int32_t *__restrict__ size, int64_t T,
                                  int64_t *__restrict__ toff) {
  // single block: per-thread serial chunk + block scan of chunk sums
  __shared__ int64_t part[1024];
  const int64_t per = (T + 1023) / 1024;
  const int64_t lo = threadIdx.x * per, hi = min(T, lo + per);
  int64_t sum = 0;
  for (int64_t t = lo; t < hi; ++t) sum += size[t];
  part[threadIdx.x] = sum;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int64_t v = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int64_t run = part[threadIdx.x] - sum;
  for (int64_t t = lo; t < hi; ++t) {
    toff[t] = run;
    run += size[t];
  }
}

__global__ void order_emit_kernel(const int32_t *__restrict__ perm, const int64_t *__restrict__ toff,
                                  int64_t T, int64_t n,
                                  const unsigned long long *__restrict__ work,
                                  int32_t *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const bool pruned = work[3] != 0;
  if (!pruned) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
      out[i] = (int32_t)i;
    return;
  }
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < T;
       t += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int64_t o = toff[t];
    for (int r0 = 0; r0 < tiles::TB; r0 += 32) {
      const int32_t v = perm[t * tiles::TB + r0 + lane];
      const unsigned b = __ballot_sync(0xffffffffu, v >= 0);
      if (v >= 0) out[o + __popc(b & lanemask_lt())] = v;
      o += __popc(b);
    }
  }
}

static int tiles_order_ptrs(const int32_t *size, const int32_t *perm, int64_t T, int64_t n,
                            const unsigned long long *total, int64_t *toff, int32_t *out,
                            cudaStream_t stream) {
  order_scan_kernel<<<1, 1024, 0, stream>>>(size, T, toff);
  PGK_CHECK_LAUNCH("order_scan_kernel");
  order_emit_kernel<<<(unsigned)num_sms() * 4, 256, 0, stream>>>(perm, toff, T, n, total, out);
  PGK_CHECK_LAUNCH("order_emit_kernel");
  return PGK_OK;
}

int tiles_order(void *tws, int64_t n, int64_t d, int32_t *out, cudaStream_t stream) {
  tiles::Layout L = tiles_layout(tws, ~size_t(0), n, d);
  // toff reuses the assignment-key scratch (n >= T entries, free after the sort)
  return tiles_order_ptrs(L.size, L.perm, L.Tmax, n, L.total,
                          reinterpret_cast<int64_t *>(L.akeys), out, stream);
}

int tiles_f32_order(void *tws, int64_t n, int64_t d, int64_t k, int32_t *out,
                    cudaStream_t stream) {
  tiles::LayoutF32 L = tiles_layout_f32(tws, ~size_t(0), n, d, k);
  return tiles_order_ptrs(L.size, L.perm, L.Tmax, n, L.total,
                          reinterpret_cast<int64_t *>(L.akeys), out, stream);
}

// Work record of the last pruned launch on `tws` (blocking read):
// out[0] pass-2 tile pairs, out[1] pass-1, out[2] assignment, out[3] = 1 if
// the pruned path ran.
int tiles_work(const void *tws, int64_t n, int64_t d, unsigned long long out[4],
               cudaStream_t stream) {
  tiles::Layout L = tiles_layout(const_cast<void *>(tws), ~size_t(0), n, d);
  PGK_CUDA(cudaMemcpyAsync(out, L.total, 4 * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, stream));
  PGK_CUDA(cudaStreamSynchronize(stream));
  return PGK_OK;
}

int tiles_f32_work(const void *tws, int64_t n, int64_t d, int64_t k, unsigned long long out[4],
                   cudaStream_t stream) {
  tiles::LayoutF32 L = tiles_layout_f32(const_cast<void *>(tws), ~size_t(0), n, d, k);
  PGK_CUDA(cudaMemcpyAsync(out, L.total, 4 * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, stream));
  PGK_CUDA(cudaStreamSynchronize(stream));
  return PGK_OK;
}

}  // namespace pgk
