// kernels.cpp — stam::spgemm / spadd / mttkrp over the C ABI (stam_cuda.h).
//
// Inputs are the caller's host TensorStorage arrays (staged to the GPU inside
// the call); results come back into host memory and are adopted in bulk by
// TensorStorage::fromArrays.  Status codes map back to stam::Error.
#include "stam/kernels.h"

#include <cstring>
#include <map>
#include <vector>

#include "stam/error.h"
#include "stam_cuda.h"

namespace stam {

namespace {

[[noreturn]] void rethrow(int status) {
  const std::string msg = stam_cuda_last_error();
  if (status >= 1 && status <= 1 + (int)ErrorCode::Internal)
    throw Error(static_cast<ErrorCode>(status - 1), msg);
  throw Error(ErrorCode::Internal, "device error " + std::to_string(status) + ": " + msg);
}

void check(int status) {
  if (status != STAM_OK) rethrow(status);
}

stam_cuda_ctx* context(int device) {
  struct Holder {
    std::map<int, stam_cuda_ctx*> ctx;
    ~Holder() {
      for (auto& [d, c] : ctx) stam_cuda_ctx_destroy(c);
    }
  };
  thread_local Holder holder;  // one context per host thread (stam_cuda.h threading rule)
  auto it = holder.ctx.find(device);
  if (it != holder.ctx.end()) return it->second;
  stam_cuda_ctx* c = nullptr;
  check(stam_cuda_ctx_create(device, &c));
  holder.ctx[device] = c;
  return c;
}

void require(const TensorStorage& t, const TensorFormat& f, const char* what) {
  if (!(t.format() == f))
    fail(ErrorCode::OrderMismatch, std::string(what) + " must be stored as " + f.str() +
                                       ", got " + t.format().str());
}

stam_csr_view csrView(const TensorStorage& t) {
  stam_csr_view v{};
  v.nrows = t.dimensions()[0];
  v.ncols = t.dimensions()[1];
  v.nnz = t.storedCount();
  v.pos = t.level(1).pos.data();
  v.idx = t.level(1).idx.data();
  v.vals = t.vals().data();
  v.mem = STAM_MEM_HOST;
  return v;
}

stam_options options(const KernelOptions& o) {
  stam_options opts;
  stam_cuda_default_options(&opts);
  opts.sort = o.sort ? 1 : 0;
  opts.mode = o.mode == ExecutionMode::Fused ? STAM_MODE_FUSED
              : o.mode == ExecutionMode::Assemble ? STAM_MODE_ASSEMBLE
                                                  : STAM_MODE_COMPUTE;
  opts.result_mem = STAM_MEM_HOST;
  opts.timing = 1;
  return opts;
}

void report(const stam_stats& s, ExecutionStats* out) {
  if (!out) return;
  out->mults = s.mults;
  out->adds = s.adds;
  out->merge_compares = s.merge_compares;
  out->sparse_inserts = s.sparse_inserts;
  out->appends = s.appends;
  out->ws_inserts = s.ws_inserts;
  out->ws_resets = s.ws_resets;
  out->bytes_allocated = s.bytes_allocated;
  out->kernel_launches = s.kernel_launches;
  out->kernel_ms = s.total_kernel_ms;
  out->main_kernel = s.main_kernel;
}

TensorStorage adoptCsr(stam_cuda_ctx* ctx, stam_csr_result& r, bool sorted = true) {
  TensorStorage::Level l0, l1;
  l1.pos.assign(r.pos, r.pos + r.nrows + 1);
  l1.idx.assign(r.idx, r.idx + r.nnz);
  std::vector<double> vals(r.vals, r.vals + r.nnz);
  const std::vector<int64_t> dims = {r.nrows, r.ncols};
  check(stam_cuda_release(ctx, r.handle));
  std::vector<TensorStorage::Level> levels;
  levels.push_back(std::move(l0));
  levels.push_back(std::move(l1));
  // the kernels produce valid CSR; skip the O(nnz) validation
  const TensorFormat fmt = sorted ? csr() : TensorFormat({dense(), compressed(false)});
  return TensorStorage::fromArrays(dims, fmt, std::move(levels), std::move(vals), false);
}

}  // namespace

TensorStorage spgemm(const TensorStorage& A, const TensorStorage& B, const KernelOptions& o,
                     ExecutionStats* stats) {
  require(A, csr(), "spgemm A");
  require(B, csr(), "spgemm B");
  if (A.dimensions()[1] != B.dimensions()[0])
    fail(ErrorCode::DimensionMismatch, "spgemm: A columns != B rows");
  stam_cuda_ctx* ctx = context(o.device);
  const stam_csr_view a = csrView(A), b = csrView(B);
  const stam_options opts = options(o);
  stam_csr_result r{};
  stam_stats st{};
  if (o.mode == ExecutionMode::Compute)
    fail(ErrorCode::PreconditionViolated,
         "spgemm: compute mode needs the pre-assembled index (spgemmCompute)");
  check(stam_cuda_spgemm(ctx, &a, &b, &opts, &r, &st));
  report(st, stats);
  return adoptCsr(ctx, r, o.sort);
}

TensorStorage spgemmCompute(const TensorStorage& A, const TensorStorage& B,
                            const TensorStorage& assembled, const KernelOptions& o,
                            ExecutionStats* stats) {
  require(A, csr(), "spgemm A");
  require(B, csr(), "spgemm B");
  if (assembled.format().order() != 2 || assembled.format().levelFormat(1).kind != ModeKind::Compressed)
    fail(ErrorCode::PreconditionViolated, "spgemmCompute: the assembled index must be CSR");
  if (A.dimensions()[1] != B.dimensions()[0])
    fail(ErrorCode::DimensionMismatch, "spgemm: A columns != B rows");
  stam_cuda_ctx* ctx = context(o.device);
  const stam_csr_view a = csrView(A), b = csrView(B), c = csrView(assembled);
  stam_options opts = options(o);
  opts.mode = STAM_MODE_COMPUTE;
  opts.sort = assembled.format().levelFormat(1).ordered ? 1 : 0;
  stam_csr_result r{};
  stam_stats st{};
  check(stam_cuda_spgemm_compute(ctx, &a, &b, &c, &opts, &r, &st));
  report(st, stats);
  return adoptCsr(ctx, r, opts.sort != 0);
}

TensorStorage spadd(std::span<const TensorStorage* const> ops, const KernelOptions& o,
                    ExecutionStats* stats) {
  if (ops.size() < 2) fail(ErrorCode::ArityMismatch, "spadd needs at least two operands");
  std::vector<stam_csr_view> views;
  for (const TensorStorage* t : ops) {
    require(*t, csr(), "spadd operand");
    if (t->dimensions() != ops[0]->dimensions())
      fail(ErrorCode::DimensionMismatch, "spadd operands must have equal dimensions");
    views.push_back(csrView(*t));
  }
  if (o.mode == ExecutionMode::Compute)
    fail(ErrorCode::PreconditionViolated,
         "spadd: compute mode needs the pre-assembled index (spaddCompute)");
  stam_cuda_ctx* ctx = context(o.device);
  const stam_options opts = options(o);
  stam_csr_result r{};
  stam_stats st{};
  check(stam_cuda_spadd(ctx, (int32_t)views.size(), views.data(), &opts, &r, &st));
  report(st, stats);
  return adoptCsr(ctx, r);
}

TensorStorage spaddCompute(std::span<const TensorStorage* const> ops,
                           const TensorStorage& assembled, const KernelOptions& o,
                           ExecutionStats* stats) {
  if (ops.size() < 2) fail(ErrorCode::ArityMismatch, "spadd needs at least two operands");
  std::vector<stam_csr_view> views;
  for (const TensorStorage* t : ops) {
    require(*t, csr(), "spadd operand");
    if (t->dimensions() != ops[0]->dimensions())
      fail(ErrorCode::DimensionMismatch, "spadd operands must have equal dimensions");
    views.push_back(csrView(*t));
  }
  if (assembled.format().order() != 2 || assembled.format().levelFormat(1).kind != ModeKind::Compressed)
    fail(ErrorCode::PreconditionViolated, "spaddCompute: the assembled index must be CSR");
  stam_cuda_ctx* ctx = context(o.device);
  const stam_csr_view idx = csrView(assembled);
  stam_options opts = options(o);
  opts.mode = STAM_MODE_COMPUTE;
  opts.sort = assembled.format().levelFormat(1).ordered ? 1 : 0;
  stam_csr_result r{};
  stam_stats st{};
  check(stam_cuda_spadd_compute(ctx, (int32_t)views.size(), views.data(), &idx, &opts, &r, &st));
  report(st, stats);
  return adoptCsr(ctx, r, opts.sort != 0);
}

TensorStorage mttkrp(const TensorStorage& B, const TensorStorage& C, const TensorStorage& D,
                     const KernelOptions& o, ExecutionStats* stats) {
  require(B, csf(3), "mttkrp B");
  stam_csf3_view b{};
  for (int d = 0; d < 3; d++) b.dims[d] = B.dimensions()[(size_t)d];
  b.nfibers = (int64_t)B.level(1).idx.size();
  b.nnz = B.storedCount();
  b.pos1 = B.level(1).pos.data();
  b.idx1 = B.level(1).idx.data();
  b.pos2 = B.level(2).pos.data();
  b.idx2 = B.level(2).idx.data();
  b.vals = B.vals().data();
  b.mem = STAM_MEM_HOST;
  stam_cuda_ctx* ctx = context(o.device);
  const stam_options opts = options(o);
  stam_stats st{};
  if (C.format() == denseFormat(2) && D.format() == denseFormat(2)) {
    stam_dense_view c{C.dimensions()[0], C.dimensions()[1], C.vals().data(), STAM_MEM_HOST, 0};
    stam_dense_view d{D.dimensions()[0], D.dimensions()[1], D.vals().data(), STAM_MEM_HOST, 0};
    stam_dense_result r{};
    check(stam_cuda_mttkrp_dense(ctx, &b, &c, &d, &opts, &r, &st));
    report(st, stats);
    TensorStorage out({r.nrows, r.ncols}, denseFormat(2));
    std::memcpy(out.vals().data(), r.vals, sizeof(double) * (size_t)(r.nrows * r.ncols));
    check(stam_cuda_release(ctx, r.handle));
    return out;
  }
  require(C, csr(), "mttkrp C");
  require(D, csr(), "mttkrp D");
  const stam_csr_view c = csrView(C), d = csrView(D);
  stam_csr_result r{};
  check(stam_cuda_mttkrp_sparse(ctx, &b, &c, &d, &opts, &r, &st));
  report(st, stats);
  return adoptCsr(ctx, r);
}

namespace {
stam_csf3_view csfView(const TensorStorage& B) {
  stam_csf3_view b{};
  for (int d = 0; d < 3; d++) b.dims[d] = B.dimensions()[(size_t)d];
  b.nfibers = (int64_t)B.level(1).idx.size();
  b.nnz = B.storedCount();
  b.pos1 = B.level(1).pos.data();
  b.idx1 = B.level(1).idx.data();
  b.pos2 = B.level(2).pos.data();
  b.idx2 = B.level(2).idx.data();
  b.vals = B.vals().data();
  b.mem = STAM_MEM_HOST;
  return b;
}
}  // namespace

TensorStorage ttv(const TensorStorage& B, const TensorStorage& c, const KernelOptions& o,
                  ExecutionStats* stats) {
  require(B, csf(3), "ttv B");
  if (!c.format().allDense()) fail(ErrorCode::PreconditionViolated, "ttv: c must be dense");
  if (c.storedCount() != B.dimensions()[2])
    fail(ErrorCode::DimensionMismatch, "ttv: c must hold dims[2] values");
  const stam_csf3_view b = csfView(B);
  const stam_dense_view cv{c.storedCount(), 1, c.vals().data(), STAM_MEM_HOST, 0};
  stam_cuda_ctx* ctx = context(o.device);
  const stam_options opts = options(o);
  stam_csr_result r{};
  stam_stats st{};
  check(stam_cuda_ttv(ctx, &b, &cv, &opts, &r, &st));
  report(st, stats);
  return adoptCsr(ctx, r);
}

TensorStorage rowdot(const TensorStorage& B, const TensorStorage& C, const KernelOptions& o,
                     ExecutionStats* stats) {
  require(B, csr(), "rowdot B");
  require(C, csr(), "rowdot C");
  if (B.dimensions() != C.dimensions())
    fail(ErrorCode::DimensionMismatch, "rowdot: B and C must have equal dimensions");
  const stam_csr_view b = csrView(B), c = csrView(C);
  stam_cuda_ctx* ctx = context(o.device);
  const stam_options opts = options(o);
  stam_dense_result r{};
  stam_stats st{};
  check(stam_cuda_rowdot(ctx, &b, &c, &opts, &r, &st));
  report(st, stats);
  TensorStorage out({r.nrows}, denseFormat(1));
  std::memcpy(out.vals().data(), r.vals, sizeof(double) * (size_t)r.nrows);
  check(stam_cuda_release(ctx, r.handle));
  return out;
}

TensorStorage spaddMerge(std::span<const TensorStorage* const> ops, const KernelOptions& o,
                         ExecutionStats* stats) {
  if (ops.size() < 2) fail(ErrorCode::ArityMismatch, "spadd needs at least two operands");
  std::vector<stam_csr_view> views;
  for (const TensorStorage* t : ops) {
    require(*t, csr(), "spadd operand");
    if (t->dimensions() != ops[0]->dimensions())
      fail(ErrorCode::DimensionMismatch, "spadd operands must have equal dimensions");
    views.push_back(csrView(*t));
  }
  stam_cuda_ctx* ctx = context(o.device);
  const stam_options opts = options(o);
  stam_csr_result r{};
  stam_stats st{};
  check(stam_cuda_spadd_merge(ctx, (int32_t)views.size(), views.data(), &opts, &r, &st));
  report(st, stats);
  return adoptCsr(ctx, r);
}

}  // namespace stam
