// stam/kernels.h — the B200 engine entry points for the workspace kernels.
//
// The reference leaves its engine empty (src/engine.cpp:1; SPEC execute(),
// SPEC.md:377-385).  These are the fixed-plan instances of execute() for the
// three loop nests schedule() emits (golden CIN, tests/test_transform.cpp:
// 141-147 SpGEMM, 166-184 MTTKRP, 275-284 SpAdd), over the reference's
// TensorStorage types.  Each call goes through the C ABI (stam_cuda.h) to the
// sm_100a kernels; failures throw stam::Error with the reference ErrorCode.
#pragma once

#include <cstdint>
#include <span>
#include <string>

#include "stam/storage.h"

namespace stam {

enum class ExecutionMode { Compute, Assemble, Fused };

struct KernelOptions {
  bool sort = true;
  ExecutionMode mode = ExecutionMode::Fused;
  int device = 0;
};

/// SPEC.md:368-371 counters, plus device timings.
struct ExecutionStats {
  int64_t mults = 0, adds = 0, merge_compares = 0, sparse_inserts = 0, appends = 0;
  int64_t ws_inserts = 0, ws_resets = 0, bytes_allocated = 0, kernel_launches = 0;
  double kernel_ms = 0.0;
  std::string main_kernel;
};

/// C = A·B; A, B csr(); C csr() with sorted columns (o.sort = false: each
/// row's columns in workspace order, format {dense, compressed(unordered)}).
/// o.mode: Fused (index + values) or Assemble (exact index, zero values).
TensorStorage spgemm(const TensorStorage& A, const TensorStorage& B, const KernelOptions& = {},
                     ExecutionStats* = nullptr);

/// Compute mode (SPEC run_compute_after_assemble): the values of A·B written
/// into `assembled`'s index, which is returned unchanged with the values;
/// bit-identical to the CPU workspace.  Throws MissingSlot when a product's
/// column is absent from its row.
TensorStorage spgemmCompute(const TensorStorage& A, const TensorStorage& B,
                            const TensorStorage& assembled, const KernelOptions& = {},
                            ExecutionStats* = nullptr);

/// D = ops[0] + ops[1] + ...; all csr() of equal dimensions.  o.mode: Fused
/// or Assemble (exact union index, zero values).
TensorStorage spadd(std::span<const TensorStorage* const> ops, const KernelOptions& = {},
                    ExecutionStats* = nullptr);

/// Compute mode: the operands' values written into `assembled`'s index in
/// operand order (bit-identical to the workspace); MissingSlot when an
/// operand column is absent from its row.
TensorStorage spaddCompute(std::span<const TensorStorage* const> ops,
                           const TensorStorage& assembled, const KernelOptions& = {},
                           ExecutionStats* = nullptr);

/// A(i,r) = sum_{j,k} B(i,j,k) D(k,r) C(j,r); B csf(3).  Dense factors
/// (denseFormat(2)) give a dense A; csr() factors give a csr() A.
TensorStorage mttkrp(const TensorStorage& B, const TensorStorage& C, const TensorStorage& D,
                     const KernelOptions& = {}, ExecutionStats* = nullptr);

/// TTV (SPEC Fig. ttv): A(i,j) = sum_k B(i,j,k) c(k); B csf(3), c a dense
/// vector (denseFormat(1) or (2)) of dims[2] values; A csr() over B's fibers.
TensorStorage ttv(const TensorStorage& B, const TensorStorage& c, const KernelOptions& = {},
                  ExecutionStats* = nullptr);

/// row-dot: a(i) = sum_j B(i,j) C(i,j) by intersection; csr()
/// inputs, denseFormat(1) result; stats->merge_compares = loop iterations.
TensorStorage rowdot(const TensorStorage& B, const TensorStorage& C, const KernelOptions& = {},
                     ExecutionStats* = nullptr);

/// Merge-based SpAdd baseline: pairwise two-way unions.
TensorStorage spaddMerge(std::span<const TensorStorage* const> ops, const KernelOptions& = {},
                         ExecutionStats* = nullptr);

}  // namespace stam
