// spgemm.cu — placeholder until the Gustavson kernels land (returns an error).
#include "runtime.h"
using namespace stamrt;
extern "C" int stam_cuda_spgemm(stam_cuda_ctx*, const stam_csr_view*, const stam_csr_view*,
                                const stam_options*, stam_csr_result*, stam_stats*) {
  return guarded([&] { fail(STAM_ERR_UNSUPPORTED_MERGE, "spgemm not built yet"); });
}
