// api.cu -- the extern "C" boundary (include/pgk.h).  Validates arguments,
// maps errors to codes + a thread-local message, forwards to the kernels.
#include <cstdarg>
#include <map>
#include <mutex>

#include "common.cuh"

namespace pgk {

static thread_local char g_err[512] = "";
std::atomic<int64_t> g_launches{0};

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// Per-device caches (one process may drive several GPUs from several threads).
static constexpr int kMaxDevices = 64;
static std::atomic<int> g_sms[kMaxDevices];

int num_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) dev = 0;
  int v = g_sms[dev].load(std::memory_order_relaxed);
  if (!v) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
    g_sms[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

cudaError_t ensure_smem(const void *fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void *, int>, size_t> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find({fn, dev});
  if (it != done.end() && it->second >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) done[{fn, dev}] = bytes;
  return e;
}

size_t prune_workspace(int64_t n_rows);
size_t search_workspace(int64_t n, int64_t nq);
int beam_search(const float *, int64_t, int64_t, const int32_t *, int64_t, const int32_t *,
                const float *, int64_t, int64_t, int64_t, const int32_t *, int32_t, int32_t,
                int32_t *, float *, int64_t *, int64_t *, void *, size_t, cudaStream_t,
                int32_t *, int64_t, uint64_t *);
int pair_dists(const float *, int64_t, const int32_t *, const int32_t *, int64_t, float *,
               cudaStream_t);
int component_heads(const int32_t *, int64_t, const int32_t *, int64_t, uint32_t *, int32_t *,
                    int32_t *, void *, size_t, cudaStream_t);
size_t reach_workspace(int64_t n);
int mark_reachable(const int32_t *, int64_t, const int32_t *, int64_t, int32_t, uint32_t *,
                   void *, size_t, cudaStream_t);
int first_unseen(const uint32_t *, int64_t, int32_t *, void *, cudaStream_t);
size_t centroid_workspace(int64_t n, int64_t d);
int knng_init(const float *, int64_t, int64_t, const int64_t *, int64_t, int64_t, int32_t *,
              float *, int32_t *, cudaStream_t);
int knng_sort_rows(const float *, int64_t, const int32_t *, int64_t, int64_t, int32_t *, float *,
                   cudaStream_t);
size_t knng_round_workspace(int64_t n, int64_t k0, int64_t cap);
int knng_round(const float *, int64_t, int64_t, int64_t, const int32_t *, const float *,
               const uint8_t *, int64_t, int64_t, int32_t *, float *, uint8_t *, int64_t *,
               int64_t *, void *, size_t, cudaStream_t);
int mark_fresh(const int32_t *, int64_t, const int32_t *, const int32_t *, int64_t,
               const int32_t *, int64_t, uint8_t *, cudaStream_t);
int centroid(const float *, int64_t, int64_t, float *, void *, size_t, cudaStream_t);
int launch_prune(const float *, const uint8_t *, const int32_t *, int64_t, int64_t,
                 const int32_t *, const int32_t *, void *, size_t, const int64_t *,
                 const int32_t *, const int32_t *,
                 const float *, int, double, int64_t, int64_t, int32_t *, float *, int32_t *,
                 int64_t *, int64_t *, cudaStream_t, bool short_rows = false);
int make_u8(const float *, int64_t, int64_t, uint8_t *, int32_t *, cudaStream_t);
int reverse_workspace(int64_t n, int64_t width, size_t *bytes);
int add_reverse_and_prune(const float *, const uint8_t *, const int32_t *, const int32_t *,
                          int64_t, int64_t,
                          const int32_t *, const float *,
                          const int32_t *, int64_t, int, double, int64_t, int64_t,
                          int32_t *, float *, int32_t *, int64_t *, int64_t *, void *,
                          size_t, cudaStream_t);
int knn_workspace(int64_t, int64_t, int64_t, int64_t, int, size_t *);
int knn_pools(const float *, int64_t, int64_t, const float *, int64_t, int64_t, int, int,
              int32_t *, int32_t *, float *, void *, size_t, cudaStream_t,
              const uint8_t *xu8_in = nullptr, const int32_t *norms_in = nullptr,
              bool assigned = false);
int knn_tiles_prepare(void *, size_t, int64_t, int64_t, int64_t, const float *, cudaStream_t);
int knn_tiles_assign(void *, size_t, int64_t, int64_t, int64_t, const uint8_t *, const int32_t *,
                     int64_t, int64_t, cudaStream_t);
int detect_u8_async(const float *, int64_t, int64_t, int *, cudaStream_t);
int64_t tiles_center_stride();
bool tiles_supported(int64_t n, int64_t d, int64_t k);
int detect_u8(const float *, int64_t, int64_t, int *, void *, size_t, cudaStream_t);
int fallback_rows(const void *, int *, cudaStream_t);
int knn_work(const void *, int64_t, int64_t, int64_t, int64_t, int, unsigned long long *,
             cudaStream_t);
int knn_order(const void *, int64_t, int64_t, int64_t, int64_t, int, int32_t *, cudaStream_t);

}  // namespace pgk

using namespace pgk;

static int check_prune_args(const float *data, int64_t n, int64_t d, int strategy,
                            int64_t M, int64_t width) {
  PGK_REQUIRE(n >= 0 && d >= 1, "bad shape n=%lld d=%lld", (long long)n, (long long)d);
  PGK_REQUIRE(n == 0 || data, "data is NULL");
  PGK_REQUIRE(strategy == 0 || strategy == 1 || strategy == 2,
              "strategy must be 0 (rng), 1 (alpha) or 2 (slack)");
  PGK_REQUIRE(M >= 1, "M must be >= 1");
  PGK_REQUIRE(width >= M, "row width %lld < M %lld", (long long)width, (long long)M);
  PGK_REQUIRE(n < 0x7fffffffLL && width < 0x7fffffffLL, "n / width exceed int32 ids");
  return PGK_OK;
}

extern "C" {

const char *pgk_version(void) { return "pgk 0.1 (sm_100a)"; }
const char *pgk_last_error(void) { return g_err; }
int64_t pgk_launch_count(void) { return g_launches.load(); }

int pgk_device_check(int *sm_count_host) {
  int dev = 0;
  PGK_CUDA(cudaGetDevice(&dev));
  cudaDeviceProp p;
  PGK_CUDA(cudaGetDeviceProperties(&p, dev));
  if (sm_count_host) *sm_count_host = p.multiProcessorCount;
  if (p.major != 10) {
    set_error("device %s is sm_%d%d; this library is built for sm_100a", p.name, p.major,
              p.minor);
    return PGK_ERR_UNSUPPORTED;
  }
  return PGK_OK;
}

int pgk_prune_batch(const float *data, int64_t n, int64_t d, const int64_t *cand_off,
                    const int32_t *cand_counts, const int32_t *cand_ids,
                    const float *cand_dists, int strategy, double cos_alpha, int64_t M,
                    int64_t width, int32_t *out_ids, float *out_dists, int32_t *out_counts,
                    int64_t *dist_evals, int64_t *angle_evals, void *stream) {
  int rc = check_prune_args(data, n, d, strategy, M, width);
  if (rc) return rc;
  return launch_prune(data, nullptr, nullptr, n, d, nullptr, nullptr, nullptr, 0, cand_off,
                      cand_counts, cand_ids, cand_dists, strategy,
                      cos_alpha, M, width, out_ids, out_dists, out_counts, dist_evals,
                      angle_evals, (cudaStream_t)stream);
}

int pgk_prune_rows(const float *data, int64_t n, int64_t d, int64_t n_rows,
                   const int32_t *row_node, const int64_t *cand_off,
                   const int32_t *cand_counts, const int32_t *cand_ids,
                   const float *cand_dists, int strategy, double cos_alpha, int64_t M,
                   int64_t width, int32_t *out_ids, float *out_dists, int32_t *out_counts,
                   int64_t *dist_evals, int64_t *angle_evals, void *stream) {
  return pgk_prune_rows_ex(data, nullptr, nullptr, n, d, n_rows, row_node, nullptr, cand_off,
                           cand_counts, cand_ids, cand_dists, strategy, cos_alpha, M, width,
                           out_ids, out_dists, out_counts, dist_evals, angle_evals, nullptr, 0,
                           stream);
}

int pgk_prune_rows_ex(const float *data, const uint8_t *data_u8, const int32_t *norms_u8,
                      int64_t n, int64_t d, int64_t n_rows, const int32_t *row_node,
                      const int32_t *row_order,
                      const int64_t *cand_off, const int32_t *cand_counts,
                      const int32_t *cand_ids, const float *cand_dists, int strategy,
                      double cos_alpha, int64_t M, int64_t width, int32_t *out_ids,
                      float *out_dists, int32_t *out_counts, int64_t *dist_evals,
                      int64_t *angle_evals, void *ws, size_t ws_bytes, void *stream) {
  int rc = check_prune_args(data, n, d, strategy, M, width);
  if (rc) return rc;
  PGK_REQUIRE(n_rows >= 0, "n_rows must be >= 0");
  PGK_REQUIRE(!data_u8 || (norms_u8 && d <= 128), "u8 rows need norms and d <= 128");
  return launch_prune(data, data_u8, norms_u8, n_rows, d, row_node, row_order, ws, ws_bytes,
                      cand_off,
                      cand_counts, cand_ids, cand_dists, strategy, cos_alpha, M, width, out_ids,
                      out_dists, out_counts, dist_evals, angle_evals, (cudaStream_t)stream);
}

int pgk_prune_workspace(int64_t n_rows, size_t *ws_bytes_host) {
  PGK_REQUIRE(ws_bytes_host, "ws_bytes_host is NULL");
  *ws_bytes_host = prune_workspace(n_rows);
  return PGK_OK;
}

int pgk_make_u8(const float *data, int64_t n, int64_t d, uint8_t *out_u8, int32_t *out_norms,
                void *stream) {
  PGK_REQUIRE(data && out_u8 && out_norms, "NULL argument");
  return make_u8(data, n, d, out_u8, out_norms, (cudaStream_t)stream);
}

int pgk_reverse_workspace(int64_t n, int64_t a_width, size_t *ws_bytes_host) {
  PGK_REQUIRE(ws_bytes_host, "ws_bytes_host is NULL");
  return reverse_workspace(n, a_width, ws_bytes_host);
}

int pgk_add_reverse_and_prune(const float *data, int64_t n, int64_t d, const int32_t *a_ids,
                              const float *a_dists, const int32_t *a_counts,
                              int64_t a_width, int strategy, double cos_alpha, int64_t M,
                              int64_t out_width, int32_t *out_ids, float *out_dists,
                              int32_t *out_counts, int64_t *dist_evals,
                              int64_t *angle_evals, void *ws, size_t ws_bytes,
                              void *stream) {
  return pgk_add_reverse_and_prune_ex(data, nullptr, nullptr, nullptr, n, d, a_ids, a_dists,
                                      a_counts,
                                      a_width, strategy, cos_alpha, M, out_width, out_ids,
                                      out_dists, out_counts, dist_evals, angle_evals, ws,
                                      ws_bytes, stream);
}

int pgk_add_reverse_and_prune_ex(const float *data, const uint8_t *data_u8,
                                 const int32_t *norms_u8, const int32_t *row_order,
                                 int64_t n, int64_t d,
                                 const int32_t *a_ids, const float *a_dists,
                                 const int32_t *a_counts, int64_t a_width, int strategy,
                                 double cos_alpha, int64_t M, int64_t out_width,
                                 int32_t *out_ids, float *out_dists, int32_t *out_counts,
                                 int64_t *dist_evals, int64_t *angle_evals, void *ws,
                                 size_t ws_bytes, void *stream) {
  int rc = check_prune_args(data, n, d, strategy, M, out_width);
  if (rc) return rc;
  PGK_REQUIRE(a_width >= 1, "phase-A width must be >= 1");
  PGK_REQUIRE(!data_u8 || (norms_u8 && d <= 128), "u8 rows need norms and d <= 128");
  return add_reverse_and_prune(data, data_u8, norms_u8, row_order, n, d, a_ids, a_dists,
                               a_counts, a_width,
                               strategy, cos_alpha, M, out_width, out_ids, out_dists, out_counts,
                               dist_evals, angle_evals, ws, ws_bytes, (cudaStream_t)stream);
}

int pgk_detect_u8(const float *data, int64_t n, int64_t d, int *is_u8_host, void *ws,
                  size_t ws_bytes, void *stream) {
  PGK_REQUIRE(data && is_u8_host, "NULL argument");
  return detect_u8(data, n, d, is_u8_host, ws, ws_bytes, (cudaStream_t)stream);
}

int pgk_knn_workspace(int64_t n, int64_t nq, int64_t d, int64_t k, int mode,
                      size_t *ws_bytes_host) {
  PGK_REQUIRE(ws_bytes_host, "ws_bytes_host is NULL");
  return knn_workspace(n, nq <= 0 ? n : nq, d, k, mode, ws_bytes_host);
}

int pgk_knn_pools(const float *data, int64_t n, int64_t d, const float *queries, int64_t nq,
                  int64_t k, int exclude_self, int mode, int32_t *gt_ids, int32_t *pool_ids,
                  float *pool_dists, void *ws, size_t ws_bytes, void *stream) {
  PGK_REQUIRE(data && pool_ids && pool_dists && ws, "NULL argument");
  return knn_pools(data, n, d, queries, nq, k, exclude_self, mode, gt_ids, pool_ids,
                   pool_dists, ws, ws_bytes, (cudaStream_t)stream);
}

int pgk_knn_pools_u8(const float *data, const uint8_t *data_u8, const int32_t *norms, int64_t n,
                     int64_t d, int64_t k, int assigned, int32_t *gt_ids, int32_t *pool_ids,
                     float *pool_dists, void *ws, size_t ws_bytes, void *stream) {
  PGK_REQUIRE(data && data_u8 && norms && pool_ids && pool_dists && ws, "NULL argument");
  PGK_REQUIRE(d <= 128, "exact-integer rows need d <= 128");
  return knn_pools(data, n, d, nullptr, n, k, 1, PGK_POOL_U8, gt_ids, pool_ids, pool_dists, ws,
                   ws_bytes, (cudaStream_t)stream, data_u8, norms, assigned != 0);
}

int64_t pgk_tiles_center_stride(void) { return tiles_center_stride(); }
int pgk_tiles_supported(int64_t n, int64_t d, int64_t k) {
  return n > 0 && d >= 1 && k >= 1 && tiles_supported(n, d, k) ? 1 : 0;
}

int pgk_tiles_u8_prepare(void *ws, size_t ws_bytes, int64_t n, int64_t d, int64_t k,
                         const float *centers, void *stream) {
  PGK_REQUIRE(ws && centers, "NULL argument");
  return knn_tiles_prepare(ws, ws_bytes, n, d, k, centers, (cudaStream_t)stream);
}

int pgk_tiles_u8_assign(void *ws, size_t ws_bytes, int64_t n, int64_t d, int64_t k,
                        const uint8_t *rows_u8, const int32_t *norms, int64_t row0, int64_t nrows,
                        void *stream) {
  PGK_REQUIRE(ws && rows_u8 && norms, "NULL argument");
  return knn_tiles_assign(ws, ws_bytes, n, d, k, rows_u8, norms, row0, nrows,
                          (cudaStream_t)stream);
}

int pgk_detect_u8_async(const float *data, int64_t n, int64_t d, int *flag, void *stream) {
  PGK_REQUIRE(data && flag, "NULL argument");
  return detect_u8_async(data, n, d, flag, (cudaStream_t)stream);
}

int pgk_copy_rows_h2d(void *dst, const void *src_host, int64_t rows, int64_t row_bytes,
                      int64_t src_pitch, void *stream) {
  PGK_REQUIRE(dst && src_host && rows >= 0 && row_bytes > 0 && src_pitch >= row_bytes,
              "bad strided copy");
  if (rows == 0) return PGK_OK;
  PGK_CUDA(cudaMemcpy2DAsync(dst, (size_t)row_bytes, src_host, (size_t)src_pitch,
                             (size_t)row_bytes, (size_t)rows, cudaMemcpyHostToDevice,
                             (cudaStream_t)stream));
  return PGK_OK;
}

int pgk_knn_work(const void *ws, int64_t n, int64_t nq, int64_t d, int64_t k, int mode,
                 uint64_t *work_host, void *stream) {
  PGK_REQUIRE(ws && work_host, "NULL argument");
  return knn_work(ws, n, nq <= 0 ? n : nq, d, k, mode,
                  reinterpret_cast<unsigned long long *>(work_host), (cudaStream_t)stream);
}

int pgk_knn_order(const void *ws, int64_t n, int64_t d, int64_t k, int mode, int32_t *order,
                  void *stream) {
  PGK_REQUIRE(ws && order, "NULL argument");
  return knn_order(ws, n, n, d, k, mode, order, (cudaStream_t)stream);
}

int pgk_knn_fallback_rows(const void *ws, int *rows_host, void *stream) {
  PGK_REQUIRE(ws && rows_host, "NULL argument");
  return fallback_rows(ws, rows_host, (cudaStream_t)stream);
}

int pgk_search_workspace(int64_t n, int64_t nq, size_t *ws_bytes_host) {
  PGK_REQUIRE(ws_bytes_host, "NULL argument");
  *ws_bytes_host = search_workspace(n, nq);
  return PGK_OK;
}

int pgk_beam_search(const float *data, int64_t n, int64_t d, const int32_t *adj,
                    int64_t width, const int32_t *counts, const float *queries, int64_t nq,
                    int64_t k, int64_t L, const int32_t *eps, int32_t ep, int32_t exclude,
                    int32_t *out_ids, float *out_dists, int64_t *dist_counts,
                    int64_t *n_expanded, void *ws, size_t ws_bytes, void *stream) {
  PGK_REQUIRE(data && adj && counts && out_ids && out_dists && ws, "NULL argument");
  PGK_REQUIRE(nq == 0 || queries, "NULL queries");
  return beam_search(data, n, d, adj, width, counts, queries, nq, k, L, eps, ep, exclude,
                     out_ids, out_dists, dist_counts, n_expanded, ws, ws_bytes,
                     (cudaStream_t)stream, nullptr, 0, nullptr);
}

int pgk_beam_search_ex(const float *data, int64_t n, int64_t d, const int32_t *adj,
                       int64_t width, const int32_t *counts, const float *queries, int64_t nq,
                       int64_t k, int64_t L, const int32_t *eps, int32_t ep, int32_t exclude,
                       int32_t *out_ids, float *out_dists, int64_t *dist_counts,
                       int64_t *n_expanded, int32_t *expansions, uint64_t *exp_worst,
                       int64_t exp_cap, void *ws, size_t ws_bytes, void *stream) {
  PGK_REQUIRE(data && adj && counts && out_ids && out_dists && ws, "NULL argument");
  PGK_REQUIRE(nq == 0 || queries, "NULL queries");
  PGK_REQUIRE((!expansions && !exp_worst) || exp_cap >= 1, "exp_cap must be >= 1");
  return beam_search(data, n, d, adj, width, counts, queries, nq, k, L, eps, ep, exclude,
                     out_ids, out_dists, dist_counts, n_expanded, ws, ws_bytes,
                     (cudaStream_t)stream, expansions, exp_cap, exp_worst);
}

int pgk_pair_dists(const float *data, int64_t d, const int32_t *a, const int32_t *b, int64_t m,
                   float *out, void *stream) {
  PGK_REQUIRE(data && out && (m == 0 || (a && b)), "NULL argument");
  return pair_dists(data, d, a, b, m, out, (cudaStream_t)stream);
}

int pgk_component_heads(const int32_t *adj, int64_t width, const int32_t *counts, int64_t n,
                        uint32_t *seen, int32_t *heads, int32_t *n_heads_host, void *ws,
                        size_t ws_bytes, void *stream) {
  PGK_REQUIRE(adj && counts && seen && heads && n_heads_host && ws, "NULL argument");
  return component_heads(adj, width, counts, n, seen, heads, n_heads_host, ws, ws_bytes,
                         (cudaStream_t)stream);
}

int pgk_reach_workspace(int64_t n, size_t *ws_bytes_host) {
  PGK_REQUIRE(ws_bytes_host, "NULL argument");
  *ws_bytes_host = reach_workspace(n);
  return PGK_OK;
}

int pgk_mark_reachable(const int32_t *adj, int64_t width, const int32_t *counts, int64_t n,
                       int32_t start, uint32_t *seen, void *ws, size_t ws_bytes, void *stream) {
  PGK_REQUIRE(adj && counts && seen && ws, "NULL argument");
  return mark_reachable(adj, width, counts, n, start, seen, ws, ws_bytes, (cudaStream_t)stream);
}

int pgk_first_unseen(const uint32_t *seen, int64_t n, int32_t *out_host, void *ws,
                     void *stream) {
  PGK_REQUIRE(seen && out_host && ws, "NULL argument");
  return first_unseen(seen, n, out_host, ws, (cudaStream_t)stream);
}

int pgk_knng_init(const float *data, int64_t n, int64_t d, const int64_t *draws, int64_t D,
                  int64_t k0, int32_t *ids, float *dists, int32_t *shortfall, void *stream) {
  PGK_REQUIRE(data && draws && ids && dists && shortfall, "NULL argument");
  return knng_init(data, n, d, draws, D, k0, ids, dists, shortfall, (cudaStream_t)stream);
}

int pgk_knng_sort_rows(const float *data, int64_t d, const int32_t *rows, int64_t nrows,
                       int64_t k0, int32_t *ids, float *dists, void *stream) {
  PGK_REQUIRE(data && ids && dists && (nrows == 0 || rows), "NULL argument");
  return knng_sort_rows(data, d, rows, nrows, k0, ids, dists, (cudaStream_t)stream);
}

int pgk_knng_round_workspace(int64_t n, int64_t k0, int64_t cap, size_t *ws_bytes_host) {
  PGK_REQUIRE(ws_bytes_host, "NULL argument");
  *ws_bytes_host = knng_round_workspace(n, k0, cap);
  return PGK_OK;
}

int pgk_knng_round(const float *data, int64_t n, int64_t d, int64_t k0, const int32_t *ids,
                   const float *dists, const uint8_t *flags, int64_t cap_new, int64_t cap_old,
                   int32_t *out_ids, float *out_dists, uint8_t *out_flags, int64_t *upd_counts,
                   int64_t *dist_evals, void *ws, size_t ws_bytes, void *stream) {
  PGK_REQUIRE(data && ids && dists && flags && out_ids && out_dists && out_flags && upd_counts &&
                  dist_evals && ws,
              "NULL argument");
  PGK_REQUIRE(cap_new >= 1 && cap_old >= 1, "caps must be >= 1");
  return knng_round(data, n, d, k0, ids, dists, flags, cap_new, cap_old, out_ids, out_dists,
                    out_flags, upd_counts, dist_evals, ws, ws_bytes, (cudaStream_t)stream);
}

int pgk_mark_fresh(const int32_t *cand, int64_t cw, const int32_t *ccnt, const int32_t *prev,
                   int64_t pw, const int32_t *pcnt, int64_t n, uint8_t *fresh, void *stream) {
  PGK_REQUIRE(cand && ccnt && prev && pcnt && fresh, "NULL argument");
  return mark_fresh(cand, cw, ccnt, prev, pw, pcnt, n, fresh, (cudaStream_t)stream);
}

int pgk_centroid_workspace(int64_t n, int64_t d, size_t *ws_bytes_host) {
  PGK_REQUIRE(ws_bytes_host, "NULL argument");
  *ws_bytes_host = centroid_workspace(n, d);
  return PGK_OK;
}

int pgk_centroid(const float *data, int64_t n, int64_t d, float *out, void *ws,
                 size_t ws_bytes, void *stream) {
  PGK_REQUIRE(data && out && ws, "NULL argument");
  return centroid(data, n, d, out, ws, ws_bytes, (cudaStream_t)stream);
}

}  // extern "C"
