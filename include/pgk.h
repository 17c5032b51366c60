/*
 * pgk.h -- C ABI of the B200 (sm_100a) RNG index-construction hot path.
 *
 * The reference (pgann, Python + numba) has no FFI of its own: its hot loops are
 * numba kernels called from prune.py / oracle.py with plain numpy arrays and
 * caller-allocated out-params.  Each entry point below replaces one of those
 * call sites (cited per function) and keeps its array conventions:
 *   data      float32 (n, d) row-major, row i == id i        (core.py:18-47)
 *   offsets   int64, counts int32, ids int32 (-1 = EMPTY), dists float32
 *   strategy  0 = "rng", 1 = "alpha"; cos_alpha float64      (prune.py:24-56)
 *             2 = "slack" (extension, no reference equivalent: s^2 * dwv < dv,
 *             with s^2 >= 1 passed in the cos_alpha argument)
 *
 * Conventions of this ABI:
 *   - every pointer argument is a DEVICE pointer unless the name says _host;
 *   - `stream` is a cudaStream_t passed as void*; work is enqueued
 *     asynchronously on it (no host synchronisation unless stated);
 *   - no hidden allocations: scratch comes from the caller as (ws, ws_bytes),
 *     sized by the matching *_workspace() query;
 *   - no global mutable state; return PGK_OK (0) or an error code, with a
 *     message from pgk_last_error() (thread-local).  Nothing throws across
 *     the ABI.
 *   - outputs are written in full, padding included (-1 ids / +inf dists), so
 *     the caller need not pre-fill them the way prune.py:117-120 does.
 */
#ifndef PGK_H_
#define PGK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PGK_OK 0
#define PGK_ERR_INVALID 1     /* bad argument (shim raises ValueError)      */
#define PGK_ERR_CUDA 2        /* CUDA launch / runtime error (RuntimeError) */
#define PGK_ERR_NOMEM 3       /* workspace too small (MemoryError)          */
#define PGK_ERR_UNSUPPORTED 4 /* shape outside the supported range          */

/* Distance mode of the exact-kNN pool kernel. */
#define PGK_POOL_AUTO 0 /* detect (one small device->host read)              */
#define PGK_POOL_U8 1   /* every value an integer in [0,255], d <= 258: exact */
#define PGK_POOL_F32 2  /* general fp32 data: approximate pass + fp64 rerank  */
/* OR-ed into a mode (same value for the workspace query and the call): skip
 * the exact tile pruning and scan every pair (the brute-force kernels) --
 * the reference result by a second route, for verification. */
#define PGK_POOL_NO_PRUNE 0x10

const char *pgk_version(void);
const char *pgk_last_error(void);

/* Number of SMs / device sanity check; returns PGK_OK when an sm_100 device is
 * current. */
int pgk_device_check(int *sm_count_host);

/* ---------------------------------------------------------------------------
 * Phase A edge selection.  Replaces _kernels.prune_batch (_kernels.py:412-427,
 * called at prune.py:123-125) / _prune_row (_kernels.py:364-409).
 * For every u: greedy occlusion / alpha-angle scan of the ascending (dist, id)
 * slice cand_ids[cand_off[u] .. cand_off[u]+cand_counts[u]), kept <= M.
 * out rows have stride `width` (>= M); dist_evals / angle_evals are per-node
 * counters, identical to the reference's.  Bit-exact with the reference
 * (fp32 sequential squared L2, fp64 law-of-cosines angle).
 * ------------------------------------------------------------------------- */
int pgk_prune_batch(const float *data, int64_t n, int64_t d,
                    const int64_t *cand_off, const int32_t *cand_counts,
                    const int32_t *cand_ids, const float *cand_dists,
                    int strategy, double cos_alpha, int64_t M, int64_t width,
                    int32_t *out_ids, float *out_dists, int32_t *out_counts,
                    int64_t *dist_evals, int64_t *angle_evals, void *stream);

/* Same scan for an arbitrary set of rows: row r holds the candidates of node
 * row_node[r] (self-skip uses that id).  prune_row_single (_kernels.py:948-958)
 * is the one-row case; pgk_prune_batch is row_node == NULL (row r == node r). */
int pgk_prune_rows(const float *data, int64_t n, int64_t d, int64_t n_rows,
                   const int32_t *row_node, const int64_t *cand_off,
                   const int32_t *cand_counts, const int32_t *cand_ids,
                   const float *cand_dists, int strategy, double cos_alpha,
                   int64_t M, int64_t width, int32_t *out_ids, float *out_dists,
                   int32_t *out_counts, int64_t *dist_evals, int64_t *angle_evals,
                   void *stream);

/* Exact-integer variants.  When every value of `data` is an integer in
 * [0,255] and d <= 128 (pgk_detect_u8), the reference's sequential fp32
 * squared_l2 never leaves the exact-integer range (all partial sums < 2^24),
 * so the kernels may compute it as |w|^2 + |v|^2 - 2 w.v on a u8 copy of the
 * rows: bit-identical results, 4x fewer bytes.  pgk_make_u8 builds that copy
 * (rows of 128 bytes, zero padded; int32 squared norms).  data_u8 == NULL
 * selects the fp32 path (then these equal pgk_prune_rows).  row_order
 * (optional, a permutation of 0..n_rows-1) is only the processing order --
 * e.g. pgk_knn_order's locality order; results do not depend on it. */
int pgk_make_u8(const float *data, int64_t n, int64_t d, uint8_t *out_u8,
                int32_t *out_norms, void *stream);
int pgk_prune_rows_ex(const float *data, const uint8_t *data_u8,
                      const int32_t *norms_u8, int64_t n, int64_t d, int64_t n_rows,
                      const int32_t *row_node, const int32_t *row_order,
                      const int64_t *cand_off,
                      const int32_t *cand_counts, const int32_t *cand_ids,
                      const float *cand_dists, int strategy, double cos_alpha,
                      int64_t M, int64_t width, int32_t *out_ids, float *out_dists,
                      int32_t *out_counts, int64_t *dist_evals,
                      int64_t *angle_evals, void *ws, size_t ws_bytes, void *stream);
/* Workspace of pgk_prune_rows_ex's exact-integer path: with it (and data_u8),
 * rows of <= 128 candidates run through the tensor-core C x C Gram kernel
 * (one tcgen05 kind::i8 MMA per point); without it, the per-warp kernel. */
int pgk_prune_workspace(int64_t n_rows, size_t *ws_bytes_host);

/* ---------------------------------------------------------------------------
 * Phase B: reverse-edge insertion + re-prune.  Replaces
 * prune.add_reverse_and_prune (prune.py:129-151) = np.bincount/cumsum +
 * _kernels.scatter_reverse (_kernels.py:530-541) + merge_with_reverse
 * (_kernels.py:544-588) + prune_all.  a_* is the phase-A adjacency
 * (n, a_width); outputs as pgk_prune_batch with stride out_width (>= M).
 * ------------------------------------------------------------------------- */
int pgk_reverse_workspace(int64_t n, int64_t a_width, size_t *ws_bytes_host);
int pgk_add_reverse_and_prune(const float *data, int64_t n, int64_t d,
                              const int32_t *a_ids, const float *a_dists,
                              const int32_t *a_counts, int64_t a_width,
                              int strategy, double cos_alpha, int64_t M,
                              int64_t out_width, int32_t *out_ids,
                              float *out_dists, int32_t *out_counts,
                              int64_t *dist_evals, int64_t *angle_evals,
                              void *ws, size_t ws_bytes, void *stream);
/* exact-integer variant (see pgk_prune_rows_ex) */
int pgk_add_reverse_and_prune_ex(const float *data, const uint8_t *data_u8,
                                 const int32_t *norms_u8, const int32_t *row_order,
                                 int64_t n, int64_t d,
                                 const int32_t *a_ids, const float *a_dists,
                                 const int32_t *a_counts, int64_t a_width,
                                 int strategy, double cos_alpha, int64_t M,
                                 int64_t out_width, int32_t *out_ids,
                                 float *out_dists, int32_t *out_counts,
                                 int64_t *dist_evals, int64_t *angle_evals,
                                 void *ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * Exact k-NN candidate pools.  Replaces oracle.ground_truth_table
 * (oracle.py:31-65; queries = data rows, exclude_self) composed with the fp32
 * list distances _kernels.squared_l2 (_kernels.py:17-24) and the (dist, id)
 * re-sort sort_pairs (_kernels.py:298-324) that the reference's tests use to
 * feed prune_all (test_nsg.py:16-24, test_prune.py:35-41).
 *   queries == NULL  -> queries are the data rows (nq == n);
 *   gt_ids (optional, may be NULL): (nq, k) ids in (float64 dist, id) order,
 *                     i.e. ground_truth_table's output;
 *   pool_ids / pool_dists: (nq, k) ids + fp32 squared_l2 dists, rows ascending
 *                     by (fp32 dist, id).
 * mode: PGK_POOL_*; AUTO performs a single blocking 4-byte read.
 * ------------------------------------------------------------------------- */
int pgk_detect_u8(const float *data, int64_t n, int64_t d, int *is_u8_host,
                  void *ws, size_t ws_bytes, void *stream);
int pgk_knn_workspace(int64_t n, int64_t nq, int64_t d, int64_t k, int mode,
                      size_t *ws_bytes_host);
int pgk_knn_pools(const float *data, int64_t n, int64_t d,
                  const float *queries, int64_t nq, int64_t k, int exclude_self,
                  int mode, int32_t *gt_ids, int32_t *pool_ids,
                  float *pool_dists, void *ws, size_t ws_bytes, void *stream);

/* pgk_knn_pools for the self pool (queries == data, exclude_self, mode
 * PGK_POOL_U8) from the caller's exact-integer copy: data_u8 (n rows of 128
 * bytes) and norms (int32 squared norms), as pgk_make_u8 writes them, so the
 * pool does not convert `data` again.  The caller guarantees (e.g. by
 * pgk_detect_u8) that every value of `data` is an integer in [0, 255] and d <= 128. */
int pgk_knn_pools_u8(const float *data, const uint8_t *data_u8, const int32_t *norms, int64_t n,
                     int64_t d, int64_t k, int assigned, int32_t *gt_ids, int32_t *pool_ids,
                     float *pool_dists, void *ws, size_t ws_bytes, void *stream);

/* Host-data pipeline pieces (package: RngBuilder.build_host): the rows of a
 * pinned host array reach the device in chunks, and the tile pruning's
 * center assignment runs per chunk as it lands instead of after the whole
 * copy.  pgk_tiles_u8_prepare takes the centers (rows 0, s, 2s, ... of the
 * data, s = pgk_tiles_center_stride(), fp32 on the device, e.g. by
 * pgk_copy_rows_h2d with a pitch of s rows); pgk_tiles_u8_assign then assigns
 * rows [row0, row0 + nrows) from their pgk_make_u8 rows and norms; a final
 * pgk_knn_pools_u8(..., assigned = 1, ...) on the same workspace continues
 * from there.  pgk_detect_u8_async clears *flag (device int, caller sets it to
 * 1) when a value of the rows is not an integer in [0, 255]. */
int64_t pgk_tiles_center_stride(void);
/* 1 when the exact tile-pruned pool (and so this pipeline) applies to the
 * shape (n, d, k) in this process (d <= 128, k <= 256, enough rows, the tile
 * count within its limit, PGK_DISABLE_PRUNE unset), else 0: callers take
 * pgk_knn_pools_u8 without `assigned` (or pgk_knn_pools) then. */
int pgk_tiles_supported(int64_t n, int64_t d, int64_t k);
int pgk_tiles_u8_prepare(void *ws, size_t ws_bytes, int64_t n, int64_t d, int64_t k,
                         const float *centers, void *stream);
int pgk_tiles_u8_assign(void *ws, size_t ws_bytes, int64_t n, int64_t d, int64_t k,
                        const uint8_t *rows_u8, const int32_t *norms, int64_t row0, int64_t nrows,
                        void *stream);
int pgk_detect_u8_async(const float *data, int64_t n, int64_t d, int *flag, void *stream);
int pgk_copy_rows_h2d(void *dst, const void *src_host, int64_t rows, int64_t row_bytes,
                      int64_t src_pitch, void *stream);

/* Number of query rows that needed the exact float64 fallback scan in the most
 * recent pgk_knn_pools call on this workspace (device int32 inside ws; this
 * helper performs a blocking read). */
int pgk_knn_fallback_rows(const void *ws, int *rows_host, void *stream);

/* Work record of the most recent pgk_knn_pools call on this workspace
 * (blocking read; same n, nq, d, k, mode as the workspace query):
 * work_host[0] = pass-2 128x128 tile pairs, [1] = pass-1 pairs,
 * [2] = center-assignment pairs, [3] = 1 when the exact tile-pruned tcgen05
 * path ran (all zero otherwise: the brute-force kernels ran). */
int pgk_knn_work(const void *ws, int64_t n, int64_t nq, int64_t d, int64_t k,
                 int mode, uint64_t *work_host, void *stream);

/* A locality-friendly processing order (permutation of 0..n-1, written to
 * `order`, device int32[n]) for the selection passes: the exact-pruned pool's
 * spatial tile order, identity when the pruned path did not run.  Enqueued
 * on the stream, no host sync. */
int pgk_knn_order(const void *ws, int64_t n, int64_t d, int64_t k, int mode,
                  int32_t *order, void *stream);

/* ---- beam search and phase C ----------------------
 * Replaces the numba search core the reference binds from Python:
 * _kernels.search_one / search_many (_kernels.py:209-245, called by
 * search.kann_search / search_batch, search.py:43-94, and by prune._connect /
 * entry_point, prune.py:154-199) and graph.reachable_from (graph.py:112-123).
 *
 * pgk_beam_search: per query (rows of `queries`, device f32[nq*d]) a beam
 * search with pool width L (<= 256) from `ep` (or eps[qi] when eps != NULL)
 * over the adjacency adj (device int32[n*width], -1 padded) with `counts`;
 * writes the first k pool entries skipping `exclude` (out_ids / out_dists
 * [nq*k], -1 / +inf padded) and, when non-NULL, dist_counts / n_expanded
 * [nq] (int64).  exclude == -2 skips each query's own index (query row i is
 * node i: _kernels.batch_self_search, _kernels.py:252-281).
 * ws: pgk_search_workspace(n, nq) bytes. */
int pgk_search_workspace(int64_t n, int64_t nq, size_t *ws_bytes_host);
int pgk_beam_search(const float *data, int64_t n, int64_t d, const int32_t *adj,
                    int64_t width, const int32_t *counts, const float *queries, int64_t nq,
                    int64_t k, int64_t L, const int32_t *eps, int32_t ep, int32_t exclude,
                    int32_t *out_ids, float *out_dists, int64_t *dist_counts,
                    int64_t *n_expanded, void *ws, size_t ws_bytes, void *stream);

/* pgk_beam_search plus the expansion order of every query: expansions
 * (device int32[nq*exp_cap]) receives the first exp_cap expanded nodes in
 * order (n_expanded tells how many there were) and exp_worst (device
 * uint64[nq*exp_cap], optional) the pool's admission bound -- its last
 * packed (dist, id) key, or ~0 while not full -- right after each expansion.
 * pgk_pair_dists: out[i] = squared_l2(data[a[i]], data[b[i]]) (fp32,
 * _kernels.py:17-24). */
int pgk_beam_search_ex(const float *data, int64_t n, int64_t d, const int32_t *adj,
                       int64_t width, const int32_t *counts, const float *queries, int64_t nq,
                       int64_t k, int64_t L, const int32_t *eps, int32_t ep, int32_t exclude,
                       int32_t *out_ids, float *out_dists, int64_t *dist_counts,
                       int64_t *n_expanded, int32_t *expansions, uint64_t *exp_worst,
                       int64_t exp_cap, void *ws, size_t ws_bytes, void *stream);
int pgk_pair_dists(const float *data, int64_t d, const int32_t *a, const int32_t *b, int64_t m,
                   float *out, void *stream);

/* Reachability bitmap seen (device uint32[(n+31)/32], bit v = node v):
 * pgk_mark_reachable adds every node reachable from `start` through nodes not
 * yet marked (start included; one-CTA BFS enqueued on the stream).
 * pgk_first_unseen writes the smallest unmarked id, or -1 (blocking).
 * ws: pgk_reach_workspace(n) bytes. */
int pgk_reach_workspace(int64_t n, size_t *ws_bytes_host);
int pgk_mark_reachable(const int32_t *adj, int64_t width, const int32_t *counts, int64_t n,
                       int32_t start, uint32_t *seen, void *ws, size_t ws_bytes, void *stream);
int pgk_first_unseen(const uint32_t *seen, int64_t n, int32_t *out_host, void *ws,
                     void *stream);
/* Phase C's component heads, in order (prune.py:174-199: the first unreached
 * id, all it reaches, the next first unreached id, ...) into heads (device
 * int32[n]); marks them in seen; *n_heads_host = count (blocking). */
int pgk_component_heads(const int32_t *adj, int64_t width, const int32_t *counts, int64_t n,
                        uint32_t *seen, int32_t *heads, int32_t *n_heads_host, void *ws,
                        size_t ws_bytes, void *stream);

/* ---- NN-Descent and FastNSG bookkeeping ---------------
 * pgk_knng_init: knng.knng_init_random's row fill (_kernels.knng_init_rows,
 * _kernels.py:764-798): draws (device int64[n*D], the host rng's draws) ->
 * ids / dists (n*k0, sorted by (dist, id)); shortfall[u] > 0 marks rows
 * with fewer than k0 distinct draws (the caller repairs them and re-sorts
 * them with pgk_knng_sort_rows, which sorts the listed rows' given ids).
 * pgk_knng_round: one NN-Descent round (knng.knng_descent_iterate,
 * knng.py:64-101 with _kernels cap_reverse / _select_join / knng_join_round)
 * from ids / dists / flags (uint8, n*k0) into the out arrays, with per-node
 * accepted-update and distance counts.  ws: pgk_knng_round_workspace bytes.
 * pgk_mark_fresh: fresh[u*cw+j] = cand[u*cw+j] absent from prev row u
 * (_kernels.mark_fresh, _kernels.py:722-733). */
int pgk_knng_init(const float *data, int64_t n, int64_t d, const int64_t *draws, int64_t D,
                  int64_t k0, int32_t *ids, float *dists, int32_t *shortfall, void *stream);
int pgk_knng_sort_rows(const float *data, int64_t d, const int32_t *rows, int64_t nrows,
                       int64_t k0, int32_t *ids, float *dists, void *stream);
int pgk_knng_round_workspace(int64_t n, int64_t k0, int64_t cap, size_t *ws_bytes_host);
int pgk_knng_round(const float *data, int64_t n, int64_t d, int64_t k0, const int32_t *ids,
                   const float *dists, const uint8_t *flags, int64_t cap_new, int64_t cap_old,
                   int32_t *out_ids, float *out_dists, uint8_t *out_flags, int64_t *upd_counts,
                   int64_t *dist_evals, void *ws, size_t ws_bytes, void *stream);
int pgk_mark_fresh(const int32_t *cand, int64_t cw, const int32_t *ccnt, const int32_t *prev,
                   int64_t pw, const int32_t *pcnt, int64_t n, uint8_t *fresh, void *stream);

/* core.centroid (core.py:153-155): float64 column means, written as f32[d]
 * (deterministic two-level sum).  ws: pgk_centroid_workspace(n, d) bytes. */
int pgk_centroid_workspace(int64_t n, int64_t d, size_t *ws_bytes_host);
int pgk_centroid(const float *data, int64_t n, int64_t d, float *out, void *ws,
                 size_t ws_bytes, void *stream);

/* Cumulative number of kernel launches this library has issued since it was
 * loaded (process-wide; the bench reports the difference around its timed
 * region as gpu_launches). */
int64_t pgk_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* PGK_H_ */
