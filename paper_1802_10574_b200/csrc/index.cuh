// index.cuh — lookups into a pre-assembled CSR index (COMPUTE mode, SPEC
// run_compute_after_assemble): binary search over a row's sorted columns; an
// unsorted index (sort = false) is searched through a per-row sorted copy and
// the permutation back to the caller's positions.
#pragma once

#include <cub/device/device_segmented_sort.cuh>
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "runtime.h"

namespace stamgpu {

// Position (in the caller's index) of column col in row [c0, c0+cn), or -1.
__device__ __forceinline__ int64_t index_lookup(const int64_t* skey, const int64_t* perm,
                                               int64_t c0, int64_t cn, int64_t col) {
  int64_t lo = 0, len = cn;  // first index with skey >= col
  while (len > 0) {
    const int64_t h = len >> 1;
    if (skey[c0 + lo + h] < col) {
      lo += h + 1;
      len -= h + 1;
    } else {
      len = h;
    }
  }
  if (lo < cn && skey[c0 + lo] == col) return c0 + (perm ? perm[c0 + lo] : lo);
  return -1;
}

// Row-local positions 0..len-1 of every index entry.
__global__ void index_local_positions_kernel(const int64_t* ipos, int64_t m, int64_t* out);

// Search structure of an index: sorted rows are used as they are (perm =
// nullptr); unsorted rows are sorted per row with their positions carried.
struct IndexSearch {
  const int64_t* skey;
  const int64_t* perm;
};

inline IndexSearch make_index_search(stamrt::Call& call, const int64_t* ipos, const int64_t* iidx,
                                     int64_t m, int64_t nnz, bool sorted) {
  if (sorted || nnz == 0) return {iidx, nullptr};
  auto* keys_out = call.scratch_n<int64_t>((size_t)nnz);
  auto* pos_in = call.scratch_n<int64_t>((size_t)nnz);
  auto* pos_out = call.scratch_n<int64_t>((size_t)nnz);
  call.before_launch("index_positions");
  index_local_positions_kernel<<<(unsigned)std::min<int64_t>(stamrt::ceil_div(m, 8),
                                                             (int64_t)call.ctx()->num_sms * 16),
                                 256, 0, call.stream()>>>(ipos, m, pos_in);
  call.after_launch();
  size_t tb = 0;
  STAM_CUDA_CHECK(cub::DeviceSegmentedSort::SortPairs(nullptr, tb, iidx, keys_out, pos_in, pos_out,
                                                      nnz, m, ipos, ipos + 1, call.stream()));
  void* tmp = call.scratch(tb);
  call.before_launch("index_sort");
  STAM_CUDA_CHECK(cub::DeviceSegmentedSort::SortPairs(tmp, tb, iidx, keys_out, pos_in, pos_out,
                                                      nnz, m, ipos, ipos + 1, call.stream()));
  call.after_launch();
  return {keys_out, pos_out};
}

}  // namespace stamgpu
