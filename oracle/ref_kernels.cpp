// ref_kernels.cpp — the hot-path loop nests driven through the REFERENCE's own
// stam::Workspace and stam::TensorBuilder (TEST INFRASTRUCTURE ONLY).
//
// oracle/Makefile compiles this file together with the reference sources
// /root/reference/proj/src/{storage,workspace,format,error}.cpp, unmodified,
// into oracle/_ref/libstamref.so.  The reference has no engine (src/engine.cpp:1
// is a placeholder), so the loop nests here follow the golden CIN that the
// reference's schedule() emits (tests/test_transform.cpp:141-147, 166-184,
// 275-284) and SPEC's engine loop; every
// workspace operation (insert/accumulate, insert/assign, present, drain(sort),
// reset) and every output append is the reference's own code.
//
// Used to (1) pin oracle/stam_oracle.c bit-for-bit on seeded inputs and
// generate tests/golden/, and (2) time the reference CPU path for bench.py
// --impl reference (rows split over host threads, each thread with its own
// Workspace and TensorBuilder: distinct invocations).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "stam/error.h"
#include "stam/format.h"
#include "stam/storage.h"
#include "stam/workspace.h"

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_err;

struct CsrIn {
  int64_t nrows, ncols, nnz;
  const int64_t* pos;
  const int64_t* idx;
  const double* vals;
};

struct Csf3In {
  int64_t dims[3];
  int64_t nfibers, nnz;
  const int64_t* pos1;
  const int64_t* idx1;
  const int64_t* pos2;
  const int64_t* idx2;
  const double* vals;
};

// Output owned by this library (freed by ref_free).
struct CsrOut {
  int64_t nrows, ncols, nnz;
  int64_t* pos;
  int64_t* idx;
  double* vals;
};

// Runs body(r0, r1, builder) per thread over row blocks and concatenates
// the finalized TensorStorage blocks into `out`.
template <typename Body>
int run_blocks(int64_t nrows, int64_t ncols, int nthreads, Body body, CsrOut* out) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > nrows) nthreads = (int)std::max<int64_t>(1, nrows);
  std::vector<stam::TensorStorage> parts(nthreads);
  std::vector<std::string> errs(nthreads);
  auto work = [&](int b) {
    try {
      const int64_t r0 = nrows * b / nthreads, r1 = nrows * (b + 1) / nthreads;
      stam::TensorBuilder builder({std::max<int64_t>(1, r1 - r0), ncols}, stam::csr());
      body(r0, r1, builder);
      parts[b] = builder.finalize();
    } catch (const std::exception& e) {
      errs[b] = e.what();
    }
  };
  std::vector<std::thread> th;
  for (int b = 1; b < nthreads; b++) th.emplace_back(work, b);
  work(0);
  for (auto& t : th) t.join();
  for (auto& e : errs)
    if (!e.empty()) {
      g_err = e;
      return -1;
    }
  int64_t nnz = 0;
  for (auto& p : parts) nnz += p.storedCount();
  out->nrows = nrows;
  out->ncols = ncols;
  out->nnz = nnz;
  out->pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nrows + 1));
  out->idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)std::max<int64_t>(1, nnz));
  out->vals = (double*)malloc(sizeof(double) * (size_t)std::max<int64_t>(1, nnz));
  out->pos[0] = 0;
  std::vector<int64_t> offs(nthreads + 1, 0);
  for (int b = 0; b < nthreads; b++) offs[b + 1] = offs[b] + parts[b].storedCount();
  auto copy = [&](int b) {
    const int64_t r0 = nrows * b / nthreads, r1 = nrows * (b + 1) / nthreads;
    const auto& lv = parts[b].level(1);
    const int64_t off = offs[b];
    for (int64_t r = r0; r < r1; r++) out->pos[r + 1] = off + lv.pos[r - r0 + 1];
    const int64_t n = parts[b].storedCount();
    if (n) {
      std::memcpy(out->idx + off, lv.idx.data(), sizeof(int64_t) * (size_t)n);
      std::memcpy(out->vals + off, parts[b].vals().data(), sizeof(double) * (size_t)n);
    }
  };
  std::vector<std::thread> cth;
  for (int b = 1; b < nthreads; b++) cth.emplace_back(copy, b);
  copy(0);
  for (auto& t : cth) t.join();
  return 0;
}

}  // namespace

REF_API const char* ref_last_error() { return g_err.c_str(); }

REF_API void ref_free(CsrOut* m) {
  if (!m) return;
  free(m->pos);
  free(m->idx);
  free(m->vals);
  m->pos = m->idx = nullptr;
  m->vals = nullptr;
}

// C = A*B:  forall(i) ((forall(j) C(i,j) = w0(j)) where
//                      (forall(k,j) w0(j) += A(i,k)*B(k,j)))
REF_API int ref_spgemm(const CsrIn* A, const CsrIn* B, int nthreads, CsrOut* C) {
  auto body = [&](int64_t r0, int64_t r1, stam::TensorBuilder& out) {
    stam::Workspace w0({B->ncols});
    for (int64_t i = r0; i < r1; i++) {
      for (int64_t p = A->pos[i]; p < A->pos[i + 1]; p++) {
        const int64_t k = A->idx[p];
        const double a = A->vals[p];
        for (int64_t q = B->pos[k]; q < B->pos[k + 1]; q++)
          w0.insert(B->idx[q], a * B->vals[q], /*accumulate=*/true);
      }
      out.appendRow({i - r0}, w0.drain(/*sort=*/true));
    }
  };
  return run_blocks(A->nrows, B->ncols, nthreads, body, C);
}

// D = ops[0] + ops[1] + ...:  w0 = ops[0] ; w0 += ops[1] ; ...
REF_API int ref_spadd(int nops, const CsrIn* ops, int nthreads, CsrOut* D) {
  auto body = [&](int64_t r0, int64_t r1, stam::TensorBuilder& out) {
    stam::Workspace w0({ops[0].ncols});
    for (int64_t i = r0; i < r1; i++) {
      for (int o = 0; o < nops; o++)
        for (int64_t q = ops[o].pos[i]; q < ops[o].pos[i + 1]; q++)
          w0.insert(ops[o].idx[q], ops[o].vals[q], /*accumulate=*/o > 0);
      out.appendRow({i - r0}, w0.drain(/*sort=*/true));
    }
  };
  return run_blocks(ops[0].nrows, ops[0].ncols, nthreads, body, D);
}

// Dense MTTKRP into A (caller-allocated dims[0]*R, zeroed here):
//   forall(i,j) ((forall(r) A(i,r) += w0(r)*C(j,r)) where
//                (forall(k,r) w0(r) += B(i,j,k)*D(k,r)))
REF_API int ref_mttkrp_dense(const Csf3In* B, const double* C, const double* D, int64_t R,
                             int nthreads, double* A) {
  try {
    const int64_t I = B->dims[0];
    std::memset(A, 0, sizeof(double) * (size_t)(I * R));
    if (nthreads < 1) nthreads = 1;
    std::vector<std::string> errs(nthreads);
    auto work = [&](int b) {
      try {
        stam::Workspace w0({R});
        const int64_t i0 = I * b / nthreads, i1 = I * (b + 1) / nthreads;
        for (int64_t i = i0; i < i1; i++) {
          for (int64_t f = B->pos1[i]; f < B->pos1[i + 1]; f++) {
            const int64_t j = B->idx1[f];
            for (int64_t p = B->pos2[f]; p < B->pos2[f + 1]; p++) {
              const int64_t k = B->idx2[p];
              const double bv = B->vals[p];
              for (int64_t r = 0; r < R; r++) w0.insert(r, bv * D[k * R + r], true);
            }
            for (int64_t r = 0; r < R; r++) A[i * R + r] += w0.value(r) * C[j * R + r];
            w0.reset();
          }
        }
      } catch (const std::exception& e) {
        errs[b] = e.what();
      }
    };
    std::vector<std::thread> th;
    for (int b = 1; b < nthreads; b++) th.emplace_back(work, b);
    work(0);
    for (auto& t : th) t.join();
    for (auto& e : errs)
      if (!e.empty()) {
        g_err = e;
        return -1;
      }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Sparse MTTKRP, presence-checked w0:
//   forall(i) ((forall(r) A(i,r) = w1(r)) where (forall(j) ((forall(r)
//     w1(r) += w0(r)*C(j,r)) where (forall(k,r) w0(r) += B(i,j,k)*D(k,r)))))
REF_API int ref_mttkrp_sparse(const Csf3In* B, const CsrIn* C, const CsrIn* D, int nthreads,
                              CsrOut* A) {
  const int64_t R = C->ncols;
  auto body = [&](int64_t r0, int64_t r1, stam::TensorBuilder& out) {
    stam::Workspace w0({R}), w1({R});
    for (int64_t i = r0; i < r1; i++) {
      for (int64_t f = B->pos1[i]; f < B->pos1[i + 1]; f++) {
        const int64_t j = B->idx1[f];
        for (int64_t p = B->pos2[f]; p < B->pos2[f + 1]; p++) {
          const int64_t k = B->idx2[p];
          const double bv = B->vals[p];
          for (int64_t q = D->pos[k]; q < D->pos[k + 1]; q++)
            w0.insert(D->idx[q], bv * D->vals[q], true);
        }
        for (int64_t q = C->pos[j]; q < C->pos[j + 1]; q++) {
          const int64_t r = C->idx[q];
          if (w0.present(r)) w1.insert(r, w0.value(r) * C->vals[q], true);
        }
        w0.reset();
      }
      out.appendRow({i - r0}, w1.drain(/*sort=*/true));
    }
  };
  return run_blocks(B->dims[0], R, nthreads, body, A);
}
