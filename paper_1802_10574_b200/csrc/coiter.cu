// coiter.cu — the SPEC kernels outside the workspace plans:
// TTV, row-dot (two-way intersection co-iteration) and the merge-based SpAdd
// baseline (pairwise two-way union co-iteration) the paper compares the
// workspace plan against.
//
// Every value is the reference's sequential sum in coordinate order
// (bit-identical to oracle/stam_oracle.c); merge_compares counts the
// two-pointer loop iterations the CPU co-iteration performs,
// computed per row from the merged positions rather than by walking (an
// intersection stops at the first exhausted row; a union runs to the end of
// both, one iteration per union coordinate).
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "runtime.h"

namespace stamgpu {
namespace {

// number of elements < x (lower) or <= x (upper) in sorted s[0, n)
__device__ __forceinline__ int64_t lower_g(const int64_t* s, int64_t n, int64_t x) {
  int64_t lo = 0;
  while (n > 0) {
    const int64_t h = n >> 1;
    if (s[lo + h] < x) {
      lo += h + 1;
      n -= h + 1;
    } else {
      n = h;
    }
  }
  return lo;
}
__device__ __forceinline__ int64_t upper_g(const int64_t* s, int64_t n, int64_t x) {
  int64_t lo = 0;
  while (n > 0) {
    const int64_t h = n >> 1;
    if (s[lo + h] <= x) {
      lo += h + 1;
      n -= h + 1;
    } else {
      n = h;
    }
  }
  return lo;
}

// Intersection loop iterations over sorted rows of lengths nx, ny with m
// coinciding entries: every iteration consumes one element (two on a match)
// until one row is exhausted.  (The union loop runs until both are exhausted:
// one iteration per union coordinate.)
__device__ __forceinline__ int64_t two_pointer_steps(const int64_t* x, int64_t nx, const int64_t* y,
                                                     int64_t ny, int64_t m) {
  if (nx == 0 || ny == 0) return 0;
  const int64_t xl = x[nx - 1], yl = y[ny - 1];
  int64_t cx, cy;
  if (xl < yl) {
    cx = nx;
    cy = upper_g(y, ny, xl);
  } else if (yl < xl) {
    cy = ny;
    cx = upper_g(x, nx, yl);
  } else {
    cx = nx;
    cy = ny;
  }
  return cx + cy - m;
}

// ---------------------------------------------------------------------------
// TTV: A(i,j) = sum_k B(i,j,k) c(k); one thread per fiber, k in order.
__global__ void ttv_kernel(int64_t nfibers, const int64_t* pos2, const int64_t* idx2,
                           const double* vals, const double* c, double* out) {
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < nfibers;
       f += (int64_t)gridDim.x * blockDim.x) {
    double w = 0.0;
    for (int64_t p = pos2[f]; p < pos2[f + 1]; p++) w = add_rn(w, mul_rn(vals[p], __ldg(c + idx2[p])));
    out[f] = w;
  }
}

// ---------------------------------------------------------------------------
// row-dot: a(i) = sum_j B(i,j) C(i,j) over the intersection, j ascending.  A
// warp per row; lanes take B's entries and locate them in C; matches are
// accumulated in lane (= j) order.
__global__ void rowdot_kernel(int64_t nrows, const int64_t* bpos, const int64_t* bidx,
                              const double* bval, const int64_t* cpos, const int64_t* cidx,
                              const double* cval, double* a, unsigned long long* counters) {
  const int lane = (int)lane_id();
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long steps = 0, mults = 0;
  for (int64_t i = warp; i < nrows; i += nwarps) {
    const int64_t b0 = bpos[i], nb = bpos[i + 1] - b0;
    const int64_t c0 = cpos[i], nc = cpos[i + 1] - c0;
    double w = 0.0;
    int64_t matches = 0;
    for (int64_t t0 = 0; t0 < nb; t0 += 32) {
      const int64_t t = t0 + lane;
      double prod = 0.0;
      bool hit = false;
      if (t < nb && nc > 0) {
        const int64_t x = bidx[b0 + t];
        const int64_t r = lower_g(cidx + c0, nc, x);
        if (r < nc && cidx[c0 + r] == x) {
          hit = true;
          prod = mul_rn(bval[b0 + t], cval[c0 + r]);
        }
      }
      unsigned m = __ballot_sync(kFull, hit);
      matches += __popc(m);
      while (m) {  // ascending j
        const int src = __ffs(m) - 1;
        w = add_rn(w, __shfl_sync(kFull, prod, src));
        m &= m - 1;
      }
    }
    if (lane == 0) {
      a[i] = w;
      steps += (unsigned long long)two_pointer_steps(bidx + b0, nb, cidx + c0, nc, matches);
      mults += (unsigned long long)matches;
    }
  }
  if (lane == 0) {
    atomicAdd(&counters[0], steps);
    atomicAdd(&counters[1], mults);
  }
}

// ---------------------------------------------------------------------------
// Merge-based SpAdd: one two-pointer union D = X + Y per stage.  Pass 1
// counts each row's union (and the loop's iterations); pass 2 places every
// entry at (own index) + (other row's entries below it) - (matches before
// it): coinciding entries add, lone entries are copied.
struct Csr2 {
  const int64_t* pos;
  const int64_t* idx;
  const double* val;
};

__global__ void union_count_kernel(int64_t nrows, Csr2 X, Csr2 Y, int64_t* cnt,
                                   unsigned long long* counters) {
  const int lane = (int)lane_id();
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long steps = 0, adds = 0;
  for (int64_t i = warp; i < nrows; i += nwarps) {
    const int64_t x0 = X.pos[i], nx = X.pos[i + 1] - x0;
    const int64_t y0 = Y.pos[i], ny = Y.pos[i + 1] - y0;
    int64_t m = 0;
    for (int64_t t0 = 0; t0 < nx; t0 += 32) {
      const int64_t t = t0 + lane;
      bool hit = false;
      if (t < nx && ny > 0) {
        const int64_t v = X.idx[x0 + t];
        const int64_t r = lower_g(Y.idx + y0, ny, v);
        hit = r < ny && Y.idx[y0 + r] == v;
      }
      m += __popc(__ballot_sync(kFull, hit));
    }
    if (lane == 0) {
      cnt[i] = nx + ny - m;
      steps += (unsigned long long)(nx + ny - m);  // one iteration per union coordinate
      adds += (unsigned long long)m;
    }
  }
  if (lane == 0) {
    atomicAdd(&counters[0], steps);
    atomicAdd(&counters[1], adds);
  }
}

__global__ void union_write_kernel(int64_t nrows, Csr2 X, Csr2 Y, const int64_t* dpos,
                                   int64_t* didx, double* dval) {
  const int lane = (int)lane_id();
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned lt = lanemask_lt();
  for (int64_t i = warp; i < nrows; i += nwarps) {
    const int64_t x0 = X.pos[i], nx = X.pos[i + 1] - x0;
    const int64_t y0 = Y.pos[i], ny = Y.pos[i + 1] - y0;
    const int64_t d0 = dpos[i];
    // X's entries (with their partner in Y when they coincide)
    int64_t before = 0;  // matches among X's earlier entries
    for (int64_t t0 = 0; t0 < nx; t0 += 32) {
      const int64_t t = t0 + lane;
      bool hit = false;
      int64_t v = 0, r = 0;
      if (t < nx) {
        v = X.idx[x0 + t];
        r = ny > 0 ? lower_g(Y.idx + y0, ny, v) : 0;
        hit = r < ny && Y.idx[y0 + r] == v;
      }
      const unsigned m = __ballot_sync(kFull, hit);
      if (t < nx) {
        const int64_t o = d0 + t + r - (before + __popc(m & lt));
        didx[o] = v;
        dval[o] = hit ? add_rn(X.val[x0 + t], Y.val[y0 + r]) : X.val[x0 + t];
      }
      before += __popc(m);
    }
    // Y's entries without a partner
    before = 0;
    for (int64_t t0 = 0; t0 < ny; t0 += 32) {
      const int64_t t = t0 + lane;
      bool hit = false;
      int64_t v = 0, r = 0;
      if (t < ny) {
        v = Y.idx[y0 + t];
        r = nx > 0 ? lower_g(X.idx + x0, nx, v) : 0;
        hit = r < nx && X.idx[x0 + r] == v;
      }
      const unsigned m = __ballot_sync(kFull, hit);
      if (t < ny && !hit) {
        const int64_t o = d0 + t + r - (before + __popc(m & lt));
        didx[o] = v;
        dval[o] = Y.val[y0 + t];
      }
      before += __popc(m);
    }
  }
}

unsigned grid_warps(int64_t rows, int sms) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(stamrt::ceil_div(rows, 8), (int64_t)sms * 16));
}

}  // namespace
}  // namespace stamgpu

using namespace stamrt;

extern "C" int stam_cuda_ttv(stam_cuda_ctx* ctx, const stam_csf3_view* B, const stam_dense_view* c,
                             const stam_options* opts, stam_csr_result* A, stam_stats* stats) {
  using namespace stamgpu;
  return guarded([&] {
    Call call(reinterpret_cast<Ctx*>(ctx), opts, stats);
    check_csf3_view(B, "ttv B");
    check_dense_view(c, "ttv c");
    if (c->nrows * c->ncols != B->dims[2])
      fail(STAM_ERR_DIMENSION_MISMATCH, "ttv: c must hold dims[2] values");
    const int64_t I = B->dims[0], F = B->nfibers;
    const int64_t* pos1 = call.device_input(B->pos1, (size_t)I + 1, B->mem);
    const int64_t* idx1 = call.device_input(B->idx1, (size_t)F, B->mem);
    const int64_t* pos2 = call.device_input(B->pos2, (size_t)F + 1, B->mem);
    const int64_t* idx2 = call.device_input(B->idx2, (size_t)B->nnz, B->mem);
    const double* vals = call.device_input(B->vals, (size_t)B->nnz, B->mem);
    const double* cv = call.device_input(c->vals, (size_t)B->dims[2], c->mem);
    call.alloc_csr_result(A, I, B->dims[1], F);
    STAM_CUDA_CHECK(cudaMemcpyAsync(A->pos, pos1, sizeof(int64_t) * ((size_t)I + 1),
                                    cudaMemcpyDeviceToDevice, call.stream()));
    if (F > 0) {
      STAM_CUDA_CHECK(cudaMemcpyAsync(A->idx, idx1, sizeof(int64_t) * (size_t)F,
                                      cudaMemcpyDeviceToDevice, call.stream()));
      call.before_launch("ttv");
      ttv_kernel<<<(unsigned)std::min<int64_t>(ceil_div(F, 256), (int64_t)call.ctx()->num_sms * 16),
                   256, 0, call.stream()>>>(F, pos2, idx2, vals, cv, A->vals);
      call.after_launch();
    }
    call.finish_csr_result(A, F);
    call.finish();
    stam_stats* st = call.stats();
    st->mults = B->nnz;
    st->adds = B->nnz;
    st->appends = F;
  });
}

extern "C" int stam_cuda_rowdot(stam_cuda_ctx* ctx, const stam_csr_view* B, const stam_csr_view* C,
                                const stam_options* opts, stam_dense_result* a, stam_stats* stats) {
  using namespace stamgpu;
  return guarded([&] {
    Call call(reinterpret_cast<Ctx*>(ctx), opts, stats);
    check_csr_view(B, "rowdot B");
    check_csr_view(C, "rowdot C");
    if (B->nrows != C->nrows || B->ncols != C->ncols)
      fail(STAM_ERR_DIMENSION_MISMATCH, "rowdot: B and C must have equal dimensions");
    const int64_t n = B->nrows;
    const int64_t* bpos = call.device_input(B->pos, (size_t)n + 1, B->mem);
    const int64_t* bidx = call.device_input(B->idx, (size_t)B->nnz, B->mem);
    const double* bval = call.device_input(B->vals, (size_t)B->nnz, B->mem);
    const int64_t* cpos = call.device_input(C->pos, (size_t)n + 1, C->mem);
    const int64_t* cidx = call.device_input(C->idx, (size_t)C->nnz, C->mem);
    const double* cval = call.device_input(C->vals, (size_t)C->nnz, C->mem);
    call.alloc_dense_result(a, n, 1);
    auto* counters = static_cast<unsigned long long*>(call.scratch_zero(sizeof(int64_t) * 2));
    call.before_launch("rowdot");
    rowdot_kernel<<<grid_warps(n, call.ctx()->num_sms), 256, 0, call.stream()>>>(
        n, bpos, bidx, bval, cpos, cidx, cval, a->vals, counters);
    call.after_launch();
    int64_t cnt[2];
    call.read_scalars(reinterpret_cast<const int64_t*>(counters), 2, cnt);
    call.finish_dense_result(a);
    call.finish();
    stam_stats* st = call.stats();
    st->merge_compares = cnt[0];
    st->mults = cnt[1];
    st->adds = cnt[1];
  });
}

extern "C" int stam_cuda_spadd_merge(stam_cuda_ctx* ctx, int32_t nops, const stam_csr_view* ops,
                                     const stam_options* opts, stam_csr_result* D,
                                     stam_stats* stats) {
  using namespace stamgpu;
  return guarded([&] {
    Call call(reinterpret_cast<Ctx*>(ctx), opts, stats);
    if (!ops) fail(STAM_ERR_PRECONDITION_VIOLATED, "null operand array");
    if (nops < 2) fail(STAM_ERR_ARITY_MISMATCH, "spadd needs at least two operands");
    for (int p = 0; p < nops; p++) {
      check_csr_view(&ops[p], "spadd operand");
      if (ops[p].nrows != ops[0].nrows || ops[p].ncols != ops[0].ncols)
        fail(STAM_ERR_DIMENSION_MISMATCH, "spadd operands must have equal dimensions");
    }
    const int64_t n = ops[0].nrows;
    auto dev = [&](const stam_csr_view& v) {
      return Csr2{call.device_input(v.pos, (size_t)n + 1, v.mem),
                  call.device_input(v.idx, (size_t)v.nnz, v.mem),
                  call.device_input(v.vals, (size_t)v.nnz, v.mem)};
    };
    auto* counters = static_cast<unsigned long long*>(call.scratch_zero(sizeof(int64_t) * 2));
    auto* cnt = call.scratch_n<int64_t>((size_t)n + 1);
    size_t sb = 0;
    STAM_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, sb, cnt, cnt, n + 1, call.stream()));
    void* stmp = call.scratch(sb);
    const unsigned grid = grid_warps(n, call.ctx()->num_sms);
    Csr2 X = dev(ops[0]);
    int64_t nnz = 0;
    for (int p = 1; p < nops; p++) {
      const Csr2 Y = dev(ops[p]);
      STAM_CUDA_CHECK(cudaMemsetAsync(cnt + n, 0, sizeof(int64_t), call.stream()));
      call.before_launch("spadd_merge_count");
      union_count_kernel<<<grid, 256, 0, call.stream()>>>(n, X, Y, cnt, counters);
      call.after_launch();
      call.before_launch("spadd_merge_scan");
      STAM_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(stmp, sb, cnt, cnt, n + 1, call.stream()));
      call.after_launch();
      nnz = call.read_scalar(cnt + n);
      int64_t* dpos;
      int64_t* didx;
      double* dval;
      if (p == nops - 1) {
        call.alloc_csr_result(D, n, ops[0].ncols, nnz);
        dpos = D->pos;
        didx = D->idx;
        dval = D->vals;
      } else {  // intermediate sum, freed with the call
        dpos = call.scratch_n<int64_t>((size_t)n + 1);
        didx = call.scratch_n<int64_t>((size_t)std::max<int64_t>(nnz, 1));
        dval = call.scratch_n<double>((size_t)std::max<int64_t>(nnz, 1));
      }
      STAM_CUDA_CHECK(cudaMemcpyAsync(dpos, cnt, sizeof(int64_t) * ((size_t)n + 1),
                                      cudaMemcpyDeviceToDevice, call.stream()));
      call.before_launch("spadd_merge_write");
      union_write_kernel<<<grid, 256, 0, call.stream()>>>(n, X, Y, dpos, didx, dval);
      call.after_launch();
      X = Csr2{dpos, didx, dval};
    }
    int64_t c2[2];
    call.read_scalars(reinterpret_cast<const int64_t*>(counters), 2, c2);
    call.finish_csr_result(D, nnz);
    call.finish();
    stam_stats* st = call.stats();
    st->merge_compares = c2[0];
    st->adds = c2[1];
    st->appends = nnz;
  });
}
