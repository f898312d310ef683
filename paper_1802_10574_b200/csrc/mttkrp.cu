// mttkrp.cu — placeholder until the MTTKRP kernels land (returns an error).
#include "runtime.h"
using namespace stamrt;
extern "C" int stam_cuda_mttkrp_dense(stam_cuda_ctx*, const stam_csf3_view*, const stam_dense_view*,
                                      const stam_dense_view*, const stam_options*,
                                      stam_dense_result*, stam_stats*) {
  return guarded([&] { fail(STAM_ERR_UNSUPPORTED_MERGE, "mttkrp not built yet"); });
}
extern "C" int stam_cuda_mttkrp_sparse(stam_cuda_ctx*, const stam_csf3_view*, const stam_csr_view*,
                                       const stam_csr_view*, const stam_options*,
                                       stam_csr_result*, stam_stats*) {
  return guarded([&] { fail(STAM_ERR_UNSUPPORTED_MERGE, "mttkrp not built yet"); });
}
