// mttkrp.cu — CSF MTTKRP, dense and sparse result.
//
// Dense (golden CIN test_transform.cpp:166-173 in paper
// letters, written B*D*C so the workspace hoists):
//   forall(i,j) ((forall(r) A(i,r) += w0(r)*C(j,r)) where
//                (forall(k,r) w0(r) += B(i,j,k)*D(k,r)))
// Sparse (test_transform.cpp:175-184), w0 consumed at C's stored
// coordinates with a presence check (Workspace::present, workspace.h:35):
//   forall(i) ((forall(r) A(i,r) = w1(r)) where (forall(j) ((forall(r)
//     w1(r) += w0(r)*C(j,r)) where (forall(k,r) w0(r) += B(i,j,k)*D(k,r)))))
//
// B200 design:
//  dense  — the nonzeros are cut into fiber-aligned chunks of ~equal nnz (so
//           the power-law i-slices, one holding 38% of the nnz, spread over
//           the whole GPU); a warp walks a chunk's fibers; the w0 row lives in
//           registers, two half-warps take alternate nonzeros and read D rows
//           with 128-bit loads (R = 32: one row = 16 lanes x double2); at the
//           fiber end w0 * C(j,:) is accumulated per slice.  Slices inside a
//           chunk are stored directly; slices cut by chunk boundaries leave
//           per-chunk partials that a second kernel sums in chunk order
//           (deterministic; no atomics on the heavy slices).
//  sparse — one pass: ordered tiles of slices with decoupled look-back; a warp
//           per slice, lanes over fibers; per fiber, w0 is evaluated only at
//           C_j's stored coordinates (presence-checked lookups into the sorted
//           D rows); w1 is a dense R-wide shared-memory workspace with a
//           presence bitmap, drained sorted by ballot/popcount compaction.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "common.cuh"
#include "runtime.h"

namespace stamgpu {
namespace {

// ===========================================================================
// dense
// ===========================================================================
struct DenseParams {
  int64_t I, J, K, R;
  int64_t nfibers, nnz;
  const int64_t* pos1;
  const int64_t* idx1;
  const int64_t* pos2;
  const int64_t* idx2;
  const double* vals;
  const double* C;  // J x R
  const double* D;  // K x R
  double* A;        // I x R (zeroed)
  int64_t chunk_nnz;
  int64_t nchunks;
  double* part;       // [ncb][nchunks][2][32] partials (head, tail)
  int64_t* part_slice;  // [nchunks][2]: head slice (-1 none, -2 empty chunk), tail slice
};

__device__ __forceinline__ int64_t lower_bound_g(const int64_t* a, int64_t n, int64_t x) {
  int64_t lo = 0;
  while (n > 0) {
    const int64_t h = n >> 1;
    if (a[lo + h] < x) {
      lo += h + 1;
      n -= h + 1;
    } else {
      n = h;
    }
  }
  return lo;
}

// Slice containing fiber f: last i with pos1[i] <= f (pos1 has I+1 entries).
__device__ __forceinline__ int64_t slice_of(const int64_t* pos1, int64_t I, int64_t f) {
  int64_t lo = 0, hi = I;  // pos1[lo] <= f < pos1[hi]
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (pos1[mid] <= f) lo = mid; else hi = mid;
  }
  return lo;
}

// Column-block pass of 32 columns starting at cb.  kVec: lanes hold double2
// (half-warp per nonzero, two nonzeros per step) when R is even and the rows
// are 16-byte aligned; otherwise a full warp per nonzero, one double per lane.
template <bool kVec>
struct Lanes {
  static constexpr int kPerStep = kVec ? 2 : 1;
};

template <bool kVec>
__global__ void __launch_bounds__(256) mttkrp_dense_kernel(const DenseParams P) {
  const int lane = (int)lane_id();
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t ncb = (P.R + 31) / 32;
  // lane geometry
  const int half = kVec ? (lane >> 4) : 0;
  const int hl = kVec ? (lane & 15) : lane;
  for (int64_t task = gwarp; task < P.nchunks * ncb; task += nwarps) {
    const int64_t c = task % P.nchunks;
    const int64_t cbi = task / P.nchunks;
    const int64_t cb = cbi * 32;
    // columns held by this lane: kVec -> cb + 2*hl, +1 ; else cb + hl
    const int64_t col = kVec ? cb + 2 * hl : cb + hl;
    const bool col_ok = col < P.R;
    // fiber range of the chunk: fibers whose first nonzero lies in it
    const int64_t fa = lower_bound_g(P.pos2, P.nfibers, c * P.chunk_nnz);
    const int64_t fb = lower_bound_g(P.pos2, P.nfibers, (c + 1) * P.chunk_nnz);
    double* part = P.part + ((cbi * P.nchunks + c) * 2) * 32;
    if (fa >= fb) {
      if (lane == 0 && cbi == 0) {
        P.part_slice[2 * c] = -2;
        P.part_slice[2 * c + 1] = -1;
      }
      continue;
    }
    int64_t s = slice_of(P.pos1, P.I, fa);
    int64_t s_end = P.pos1[s + 1];
    const int64_t head_slice = s;
    bool head_open = P.pos1[s] < fa;  // first slice began in an earlier chunk
    bool wrote_head = false;
    double acc0 = 0.0, acc1 = 0.0;
    auto flush = [&](int64_t sl, bool started_here, bool ends_here) {
      // combine halves: both halves accumulated the same w0*C, only half 0 writes
      if (started_here && ends_here) {
        if (col_ok && half == 0) {
          if (kVec) {
            reinterpret_cast<double2*>(P.A + sl * P.R + col)[0] = make_double2(acc0, acc1);
          } else {
            P.A[sl * P.R + col] = acc0;
          }
        }
      } else {
        // partial: head (slot 0) if it began before this chunk, else tail (slot 1)
        const int slot = started_here ? 1 : 0;
        if (half == 0) {
          if (kVec) {
            part[slot * 32 + 2 * hl] = acc0;
            part[slot * 32 + 2 * hl + 1] = acc1;
          } else {
            part[slot * 32 + hl] = acc0;
          }
        }
        if (lane == 0 && cbi == 0) P.part_slice[2 * c + slot] = sl;
        if (slot == 0) wrote_head = true;
      }
      acc0 = 0.0;
      acc1 = 0.0;
    };
    for (int64_t f = fa; f < fb; f++) {
      while (f >= s_end) {  // next non-empty slice
        s++;
        s_end = P.pos1[s + 1];
        head_open = false;
      }
      const int64_t j = P.idx1[f];
      const int64_t z0 = P.pos2[f], z1 = P.pos2[f + 1];
      double w0 = 0.0, w1 = 0.0;
      for (int64_t zb = z0; zb < z1; zb += 32) {
        const int n = (int)min((int64_t)32, z1 - zb);
        int kz = 0;
        double bz = 0.0;
        if (lane < n) {
          kz = (int)P.idx2[zb + lane];
          bz = P.vals[zb + lane];
        }
        const int steps = (n + Lanes<kVec>::kPerStep - 1) / Lanes<kVec>::kPerStep;
#pragma unroll 4
        for (int t = 0; t < steps; t++) {
          const int src = t * Lanes<kVec>::kPerStep + half;
          const int k = __shfl_sync(kFull, kz, src & 31);
          double b = __shfl_sync(kFull, bz, src & 31);
          if (src >= n) b = 0.0;
          if (col_ok) {
            if (kVec) {
              const double2 d = __ldg(reinterpret_cast<const double2*>(P.D + (int64_t)k * P.R + col));
              w0 = fma(b, d.x, w0);
              w1 = fma(b, d.y, w1);
            } else {
              w0 = fma(b, __ldg(P.D + (int64_t)k * P.R + col), w0);
            }
          }
        }
      }
      if (kVec) {
        w0 += __shfl_xor_sync(kFull, w0, 16);
        w1 += __shfl_xor_sync(kFull, w1, 16);
      }
      if (col_ok) {
        if (kVec) {
          const double2 cj = __ldg(reinterpret_cast<const double2*>(P.C + j * P.R + col));
          acc0 = fma(w0, cj.x, acc0);
          acc1 = fma(w1, cj.y, acc1);
        } else {
          acc0 = fma(w0, __ldg(P.C + j * P.R + col), acc0);
        }
      }
      // slice ends inside this chunk?
      if (f + 1 == s_end) flush(s, !head_open, true);
    }
    // the last slice continues past the chunk
    if (fb < s_end) flush(s, !head_open, false);
    if (lane == 0 && cbi == 0) {
      if (!wrote_head) P.part_slice[2 * c] = -1;
      // tail slot written only when the last slice started here and continues
      if (!(fb < s_end && !head_open)) P.part_slice[2 * c + 1] = -1;
    }
    (void)head_slice;
  }
}

// Sums the partials of every slice cut by chunk boundaries, in chunk order.
__global__ void mttkrp_dense_fixup_kernel(const DenseParams P) {
  const int lane = (int)lane_id();
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t ncb = (P.R + 31) / 32;
  for (int64_t task = gwarp; task < P.nchunks * ncb; task += nwarps) {
    const int64_t c = task % P.nchunks;
    const int64_t cbi = task / P.nchunks;
    const int64_t s = P.part_slice[2 * c + 1];
    if (s < 0) continue;  // this chunk does not start a cut slice
    const int64_t col = cbi * 32 + lane;
    const double* base = P.part + cbi * P.nchunks * 64;
    double sum = base[(c * 2 + 1) * 32 + lane];
    for (int64_t c2 = c + 1; c2 < P.nchunks; c2++) {
      const int64_t h = P.part_slice[2 * c2];
      if (h == -2) continue;  // empty chunk (inside a long fiber)
      if (h != s) break;
      sum += base[(c2 * 2) * 32 + lane];
    }
    if (col < P.R) P.A[s * P.R + col] = sum;
  }
}

// ===========================================================================
// sparse
// ===========================================================================
constexpr int kSpWarps = 8;
constexpr int kSpSlicesPerWarp = 2;
constexpr int kSpTile = kSpWarps * kSpSlicesPerWarp;

struct SparseParams {
  int64_t I, R;
  int64_t nfibers, nnz;
  const int64_t* pos1;
  const int64_t* idx1;
  const int64_t* pos2;
  const int64_t* idx2;
  const double* vals;
  const int64_t* cpos;
  const int64_t* cidx;
  const double* cvals;
  const int64_t* dpos;
  const int64_t* didx;
  const double* dvals;
  int64_t ntiles;
  int64_t* out_pos;
  int64_t* out_idx;
  double* out_vals;
  uint64_t* tile_status;
  unsigned long long* tile_counter;
  int64_t* total_nnz;
};

__device__ __forceinline__ int64_t locate(const int64_t* a, int64_t n, int64_t x) {
  int64_t lo = 0, len = n;
  while (len > 0) {
    const int64_t h = len >> 1;
    if (a[lo + h] < x) {
      lo += h + 1;
      len -= h + 1;
    } else {
      len = h;
    }
  }
  return (lo < n && a[lo] == x) ? lo : -1;
}

// Evaluates slice i into the warp's workspace (vals[R], bits[R/32]).
__device__ void sparse_slice(const SparseParams& P, int64_t i, double* wv, uint32_t* wb) {
  const int lane = (int)lane_id();
  const int64_t f0 = P.pos1[i], f1 = P.pos1[i + 1];
  for (int64_t f = f0 + lane; f < f1; f += 32) {
    const int64_t j = P.idx1[f];
    const int64_t z0 = P.pos2[f], z1 = P.pos2[f + 1];
    const int64_t c0 = P.cpos[j], c1 = P.cpos[j + 1];
    if (z1 - z0 == 1) {
      // single nonzero: intersect C_j with D_k by merging the sorted rows
      const int64_t k = P.idx2[z0];
      const double b = P.vals[z0];
      int64_t d = P.dpos[k];
      const int64_t d1 = P.dpos[k + 1];
      int64_t q = c0;
      while (q < c1 && d < d1) {
        const int64_t rc = P.cidx[q], rd = P.didx[d];
        if (rc < rd) {
          q++;
        } else if (rd < rc) {
          d++;
        } else {
          // w0(r) = 0 + b*D(k,r);  w1(r) += w0(r)*C(j,r)
          const double w0 = add_rn(0.0, mul_rn(b, P.dvals[d]));
          atomicAdd(&wv[rc], mul_rn(w0, P.cvals[q]));
          atomicOr(&wb[rc >> 5], 1u << (rc & 31));
          q++;
          d++;
        }
      }
    } else {
      // general fiber: w0 at each of C_j's coordinates, accumulated over k
      for (int64_t q = c0; q < c1; q++) {
        const int64_t r = P.cidx[q];
        double w0 = 0.0;
        bool present = false;
        for (int64_t z = z0; z < z1; z++) {
          const int64_t k = P.idx2[z];
          const int64_t d0 = P.dpos[k];
          const int64_t at = locate(P.didx + d0, P.dpos[k + 1] - d0, r);
          if (at >= 0) {
            w0 = add_rn(w0, mul_rn(P.vals[z], P.dvals[d0 + at]));
            present = true;
          }
        }
        if (present) {
          atomicAdd(&wv[r], mul_rn(w0, P.cvals[q]));
          atomicOr(&wb[r >> 5], 1u << (r & 31));
        }
      }
    }
  }
}

__global__ void __launch_bounds__(kSpWarps * 32) mttkrp_sparse_kernel(const SparseParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int64_t tile_sh;
  __shared__ int64_t cnt_sh[kSpTile];
  __shared__ int64_t dst_sh[kSpTile];
  const int lane = (int)lane_id();
  const int warp = threadIdx.x >> 5;
  const int64_t R = P.R;
  const int nwords = (int)((R + 31) / 32);
  // per warp: kSpSlicesPerWarp workspaces of R doubles + nwords bitmap words
  const size_t ws_bytes = (size_t)R * 8 + (size_t)nwords * 4;
  unsigned char* wbase = smem_raw + (size_t)warp * kSpSlicesPerWarp * ((ws_bytes + 15) & ~(size_t)15);
  if (threadIdx.x == 0) tile_sh = (int64_t)atomicAdd(P.tile_counter, 1ull);
  __syncthreads();
  const int64_t tile = tile_sh;
  const int64_t i0 = tile * kSpTile;
  for (int k = 0; k < kSpSlicesPerWarp; k++) {
    const int t = warp * kSpSlicesPerWarp + k;
    const int64_t i = i0 + t;
    double* wv = reinterpret_cast<double*>(wbase + k * ((ws_bytes + 15) & ~(size_t)15));
    uint32_t* wb = reinterpret_cast<uint32_t*>(wv + R);
    for (int64_t r = lane; r < R; r += 32) wv[r] = 0.0;
    for (int w = lane; w < nwords; w += 32) wb[w] = 0u;
    __syncwarp();
    int64_t cnt = 0;
    if (i < P.I) {
      sparse_slice(P, i, wv, wb);
      __syncwarp();
      for (int w = lane; w < nwords; w += 32) cnt += __popc(wb[w]);
      cnt = warp_sum(cnt);
    }
    if (lane == 0) cnt_sh[t] = cnt;
  }
  __syncthreads();
  if (warp == 0) {
    const int64_t c = lane < kSpTile ? cnt_sh[lane] : 0;
    const int64_t inc = warp_inclusive_scan(c);
    const int64_t agg = __shfl_sync(kFull, inc, 31);
    const int64_t base = lookback_exclusive(P.tile_status, tile, agg);
    if (lane < kSpTile) {
      dst_sh[lane] = base + inc - c;
      if (i0 + lane < P.I) P.out_pos[i0 + lane + 1] = base + inc;
    }
    if (lane == 0) {
      if (tile == 0) P.out_pos[0] = 0;
      if (tile == P.ntiles - 1) *P.total_nnz = base + agg;
    }
  }
  __syncthreads();
  // drain: sorted by ballot/popcount over the presence bitmap
  for (int k = 0; k < kSpSlicesPerWarp; k++) {
    const int t = warp * kSpSlicesPerWarp + k;
    if (i0 + t >= P.I) continue;
    const double* wv = reinterpret_cast<double*>(wbase + k * ((ws_bytes + 15) & ~(size_t)15));
    const uint32_t* wb = reinterpret_cast<const uint32_t*>(wv + R);
    int64_t out = dst_sh[t];
    for (int w = 0; w < nwords; w++) {
      const uint32_t bits = wb[w];
      if (bits == 0) continue;
      const bool mine = (bits >> lane) & 1u;
      if (mine) {
        const int rank = __popc(bits & ((1u << lane) - 1u));
        const int64_t r = (int64_t)w * 32 + lane;
        P.out_idx[out + rank] = r;
        P.out_vals[out + rank] = wv[r];
      }
      out += __popc(bits);
    }
  }
}

}  // namespace
}  // namespace stamgpu

using namespace stamrt;

extern "C" int stam_cuda_mttkrp_dense(stam_cuda_ctx* ctx, const stam_csf3_view* B,
                                      const stam_dense_view* Cm, const stam_dense_view* Dm,
                                      const stam_options* opts, stam_dense_result* A,
                                      stam_stats* stats) {
  using namespace stamgpu;
  return guarded([&] {
    Call call(reinterpret_cast<Ctx*>(ctx), opts, stats);
    check_csf3_view(B, "mttkrp B");
    check_dense_view(Cm, "mttkrp C");
    check_dense_view(Dm, "mttkrp D");
    if (Cm->nrows != B->dims[1] || Dm->nrows != B->dims[2])
      fail(STAM_ERR_DIMENSION_MISMATCH, "mttkrp: C rows != dim 1 or D rows != dim 2");
    if (Cm->ncols != Dm->ncols) fail(STAM_ERR_DIMENSION_MISMATCH, "mttkrp: C and D ranks differ");
    if (B->dims[2] >= (int64_t)INT32_MAX)
      fail(STAM_ERR_UNSUPPORTED_MERGE, "mttkrp: dimension 2 must be below 2^31");
    const int64_t I = B->dims[0], R = Cm->ncols;
    DenseParams P{};
    P.I = I;
    P.J = B->dims[1];
    P.K = B->dims[2];
    P.R = R;
    P.nfibers = B->nfibers;
    P.nnz = B->nnz;
    P.pos1 = call.device_input(B->pos1, (size_t)I + 1, B->mem);
    P.idx1 = call.device_input(B->idx1, (size_t)B->nfibers, B->mem);
    P.pos2 = call.device_input(B->pos2, (size_t)B->nfibers + 1, B->mem);
    P.idx2 = call.device_input(B->idx2, (size_t)B->nnz, B->mem);
    P.vals = call.device_input(B->vals, (size_t)B->nnz, B->mem);
    P.C = call.device_input(Cm->vals, (size_t)(Cm->nrows * R), Cm->mem);
    P.D = call.device_input(Dm->vals, (size_t)(Dm->nrows * R), Dm->mem);
    call.alloc_dense_result(A, I, R);
    P.A = A->vals;
    STAM_CUDA_CHECK(cudaMemsetAsync(P.A, 0, sizeof(double) * (size_t)(I * R), call.stream()));
    const int sms = call.ctx()->num_sms;
    const int64_t warps = (int64_t)sms * 64;
    const int64_t ncb = (R + 31) / 32;
    P.chunk_nnz = std::max<int64_t>(256, ceil_div(std::max<int64_t>(B->nnz, 1), warps * 2));
    P.nchunks = std::max<int64_t>(1, ceil_div(B->nnz, P.chunk_nnz));
    P.part = call.scratch_n<double>((size_t)(ncb * P.nchunks * 64));
    P.part_slice = call.scratch_n<int64_t>((size_t)(2 * P.nchunks));
    const bool vec = (R % 2 == 0) && ((uintptr_t)P.C % 16 == 0) && ((uintptr_t)P.D % 16 == 0);
    const int64_t tasks = P.nchunks * ncb;
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(tasks, 8), (int64_t)sms * 8);
    if (B->nfibers > 0) {
      call.before_launch("mttkrp_dense");
      if (vec)
        mttkrp_dense_kernel<true><<<grid, 256, 0, call.stream()>>>(P);
      else
        mttkrp_dense_kernel<false><<<grid, 256, 0, call.stream()>>>(P);
      call.after_launch();
      call.before_launch("mttkrp_dense_fixup");
      mttkrp_dense_fixup_kernel<<<grid, 256, 0, call.stream()>>>(P);
      call.after_launch();
    }
    call.finish_dense_result(A);
    call.finish();
    stam_stats* st = call.stats();
    st->mults = (B->nnz + B->nfibers) * R;  // SPEC.md:416 hoisted count
    st->adds = st->mults;
    st->ws_resets = B->nfibers;
  });
}

extern "C" int stam_cuda_mttkrp_sparse(stam_cuda_ctx* ctx, const stam_csf3_view* B,
                                       const stam_csr_view* Cv, const stam_csr_view* Dv,
                                       const stam_options* opts, stam_csr_result* A,
                                       stam_stats* stats) {
  using namespace stamgpu;
  return guarded([&] {
    Call call(reinterpret_cast<Ctx*>(ctx), opts, stats);
    check_csf3_view(B, "mttkrp B");
    check_csr_view(Cv, "mttkrp C");
    check_csr_view(Dv, "mttkrp D");
    if (Cv->nrows != B->dims[1] || Dv->nrows != B->dims[2])
      fail(STAM_ERR_DIMENSION_MISMATCH, "mttkrp: C rows != dim 1 or D rows != dim 2");
    if (Cv->ncols != Dv->ncols) fail(STAM_ERR_DIMENSION_MISMATCH, "mttkrp: C and D ranks differ");
    const int64_t I = B->dims[0], R = Cv->ncols;
    const size_t ws_bytes = (((size_t)R * 8 + (size_t)((R + 31) / 32) * 4) + 15) & ~(size_t)15;
    const size_t smem = ws_bytes * kSpSlicesPerWarp * kSpWarps;
    if (smem > call.ctx()->smem_optin)
      fail(STAM_ERR_UNSUPPORTED_MERGE, "sparse mttkrp: rank too large for the shared-memory "
                                       "row workspace in ABI v1 (R <= ~1700)");
    SparseParams P{};
    P.I = I;
    P.R = R;
    P.nfibers = B->nfibers;
    P.nnz = B->nnz;
    P.pos1 = call.device_input(B->pos1, (size_t)I + 1, B->mem);
    P.idx1 = call.device_input(B->idx1, (size_t)B->nfibers, B->mem);
    P.pos2 = call.device_input(B->pos2, (size_t)B->nfibers + 1, B->mem);
    P.idx2 = call.device_input(B->idx2, (size_t)B->nnz, B->mem);
    P.vals = call.device_input(B->vals, (size_t)B->nnz, B->mem);
    P.cpos = call.device_input(Cv->pos, (size_t)Cv->nrows + 1, Cv->mem);
    P.cidx = call.device_input(Cv->idx, (size_t)Cv->nnz, Cv->mem);
    P.cvals = call.device_input(Cv->vals, (size_t)Cv->nnz, Cv->mem);
    P.dpos = call.device_input(Dv->pos, (size_t)Dv->nrows + 1, Dv->mem);
    P.didx = call.device_input(Dv->idx, (size_t)Dv->nnz, Dv->mem);
    P.dvals = call.device_input(Dv->vals, (size_t)Dv->nnz, Dv->mem);
    P.ntiles = ceil_div(I, kSpTile);
    // a row of A has at most R entries: I*R bounds the output (no counting pass)
    const int64_t bound = I * R;
    call.alloc_csr_result(A, I, R, std::min<int64_t>(bound, (int64_t)1 << 40));
    P.out_pos = A->pos;
    P.out_idx = A->idx;
    P.out_vals = A->vals;
    auto* ctl = static_cast<uint64_t*>(call.scratch_zero((4 + (size_t)P.ntiles) * 8));
    P.tile_counter = reinterpret_cast<unsigned long long*>(ctl);
    P.total_nnz = reinterpret_cast<int64_t*>(ctl + 2);
    P.tile_status = ctl + 4;
    STAM_CUDA_CHECK(cudaFuncSetAttribute(mttkrp_sparse_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    call.before_launch("mttkrp_sparse");
    mttkrp_sparse_kernel<<<(unsigned)P.ntiles, kSpWarps * 32, smem, call.stream()>>>(P);
    call.after_launch();
    const int64_t nnz = call.read_scalar(P.total_nnz);
    call.finish_csr_result(A, nnz);
    call.finish();
    stam_stats* st = call.stats();
    st->ws_resets = B->nfibers + I;
    st->appends = nnz;
  });
}
