// index.cu — device code shared by the COMPUTE-mode entry points (index.cuh).
#include "index.cuh"

namespace stamgpu {

__global__ void index_local_positions_kernel(const int64_t* ipos, int64_t m, int64_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); i < m;
       i += (int64_t)gridDim.x * (blockDim.x / 32)) {
    const int64_t b = ipos[i], e = ipos[i + 1];
    for (int64_t t = b + lane_id(); t < e; t += 32) out[t] = t - b;
  }
}

}  // namespace stamgpu
