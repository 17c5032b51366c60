// pool_tc.cu -- tensor-core (tcgen05, kind::i8) exact k-NN pool for
// integer-valued data.  (placeholder: returns handled=false until the kernel
// lands; the SIMT U8 tile kernel is used meanwhile.)
#include "common.cuh"

namespace pgk {

int launch_pool_tc_u8(const float *X, int64_t n, int d, const float *Q, int64_t nq,
                      int exclude_self, const int32_t *xnorm, const int32_t *qnorm, int K,
                      uint64_t *keys, cudaStream_t stream, bool *handled) {
  (void)X; (void)n; (void)d; (void)Q; (void)nq; (void)exclude_self; (void)xnorm;
  (void)qnorm; (void)K; (void)keys; (void)stream;
  *handled = false;
  return PGK_OK;
}

}  // namespace pgk
