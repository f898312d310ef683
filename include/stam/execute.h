// stam/execute.h — CIN-driven dispatch: the engine's
// execute(plan, inputs, mode) (the reference's
// src/engine.cpp is a placeholder) for the concrete index notation that
// schedule() prints.  The statement is parsed (forall / where / sequences /
// assignments over products of accesses), matched structurally — any tensor
// and index-variable names — against the plans the GPU kernels implement,
// and run on them:
//
//   forall(i) ((forall(j) C(i,j) = w(j)) where (forall(k,j) w(j) += A(i,k)*B(k,j)))
//       SpGEMM (golden CIN tests/test_transform.cpp:141-147)
//   forall(i) ((forall(j) D(i,j) = w(j)) where ((forall(j) w(j) = X1(i,j) ;
//                                                forall(j) w(j) += X2(i,j) ; ...)))
//       SpAdd, k operands (test_transform.cpp:275-284)
//   forall(i,k) ((forall(j) A(i,j) += w(j)*D(k,j)) where (forall(l,j) w(j) += B(i,k,l)*C(l,j)))
//       MTTKRP, dense factors and result (test_transform.cpp:166-173)
//   forall(i) ((forall(j) A(i,j) = v(j)) where (forall(k) ((forall(j) v(j) += w(j)*D(k,j))
//       where (forall(l,j) w(j) += B(i,k,l)*C(l,j)))))
//       MTTKRP, sparse factors and result (test_transform.cpp:175-184)
//   forall(i,j,k) A(i,j) += B(i,j,k)*c(k)     TTV (SPEC Fig. ttv)
//   forall(i,j) a(i) += B(i,j)*C(i,j)         row-dot, intersection
//   forall(i,j) A(i,j) = B(i,j) + C(i,j)      two-way union merge
//
// Statements outside these plans throw Error(UnsupportedMerge) (e.g. a 3-way
// sparse merge without a workspace: SPEC's graph design decision) or
// Error(UnplannableResult) (a sparse result written by scattered inserts,
// e.g. `forall(i,k,j) A(i,j) += B(i,k)*C(k,j)`); syntax errors throw
// Error(Parse).
#pragma once

#include <map>
#include <string>

#include "stam/kernels.h"
#include "stam/storage.h"

namespace stam {

struct ExecuteResult {
  std::string tensor;    // name of the result tensor in the statement
  std::string plan;      // "spgemm", "spadd", "mttkrp_dense", "mttkrp_sparse", "ttv",
                         // "rowdot", "spadd_merge"
  TensorStorage result;
  ExecutionStats stats;
};

/// Runs `cin` with its input tensors bound by name.  Dense vectors (TTV's c)
/// and dense factors are denseFormat storages; sparse operands csr()/csf(3).
ExecuteResult execute(const std::string& cin,
                      const std::map<std::string, const TensorStorage*>& inputs,
                      const KernelOptions& options = {});

}  // namespace stam
