/*
 * stam_oracle.h — CPU restatement of the reference algorithms for the hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker and the CPU
 * baseline leg of bench.py; only tests/, __graft_entry__.smoke() and bench.py
 * (cpu_baseline / --impl reference) may load it.  The product path
 * (paper_1802_10574_b200, libstam_cuda.so) never calls it and has no CPU
 * fallback.
 *
 * Each kernel restates the loop nest `schedule()` emits for it (golden CIN in
 * /root/reference/proj/tests/test_transform.cpp) over the reference's
 * workspace semantics (src/workspace.cpp:34-80): a dense value array, a guard
 * flag per coordinate and a coordinate list; `insert(accumulate)` adds the
 * already-rounded product into the value, `insert(assign)` overwrites it, a
 * sorted drain sorts the coordinate list then resets.  Build with
 * -ffp-contract=off so `w += a*b` rounds the product first, as the reference
 * does (the product is computed by the caller of Workspace::insert).
 *
 * Every function also produces the absolute-value twin s = sum |terms| per
 * output entry, for the scaled parity criterion
 *     |x_gpu - x_ref| <= 1e-12 * max(|x_ref|, s_ref).
 *
 * Parity pin: tests/golden/ holds outputs of the reference's own
 * stam::Workspace / stam::TensorBuilder (compiled from /root/reference by
 * oracle/Makefile into oracle/_ref/) on seeded inputs; tests check this
 * restatement against them bit-for-bit.
 */
#ifndef STAM_ORACLE_H_
#define STAM_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_csr {
  int64_t nrows, ncols, nnz;
  int64_t* pos;  /* [nrows+1] */
  int64_t* idx;  /* [nnz] */
  double* vals;  /* [nnz] */
  double* absv;  /* [nnz] sum of |terms| per entry */
} oracle_csr;

typedef struct oracle_csf3 {
  int64_t dims[3];
  int64_t nfibers, nnz;
  const int64_t* pos1;
  const int64_t* idx1;
  const int64_t* pos2;
  const int64_t* idx2;
  const double* vals;
} oracle_csf3;

typedef struct oracle_csr_in {
  int64_t nrows, ncols, nnz;
  const int64_t* pos;
  const int64_t* idx;
  const double* vals;
} oracle_csr_in;

/* C = A*B: forall(i) ((forall(j) C(i,j) = w0(j)) where
 *          (forall(k,j) w0(j) += A(i,k)*B(k,j)))  (test_transform.cpp:141-147) */
int oracle_spgemm(const oracle_csr_in* A, const oracle_csr_in* B, int nthreads, oracle_csr* C);

/* D = ops[0] + ... : w0 = ops[0]; w0 += ops[1]; ...  (test_transform.cpp:275-284) */
int oracle_spadd(int nops, const oracle_csr_in* ops, int nthreads, oracle_csr* D);

/* A(i,r) = sum_j C(j,r) * (sum_k B(i,j,k) D(k,r)), dense R-wide factors
 * (SURVEY §8a-7).  A and Aabs are caller-allocated dims[0]*R. */
int oracle_mttkrp_dense(const oracle_csf3* B, const double* C, const double* D, int64_t R,
                        int nthreads, double* A, double* Aabs);

/* Sparse factors, CSR result, presence-checked w0. */
int oracle_mttkrp_sparse(const oracle_csf3* B, const oracle_csr_in* C, const oracle_csr_in* D,
                         int nthreads, oracle_csr* A);

void oracle_free(oracle_csr* m);

/* counters of SPEC.md:414-418 for the last call on this thread */
typedef struct oracle_counters {
  int64_t mults, adds, ws_inserts, ws_resets, appends;
  int64_t merge_compares; /* co-iteration loop iterations */
} oracle_counters;

/* TTV (SPEC Fig. ttv; forall(i,j,k) A(i,j) += B(i,j,k)*c(k)): A has B's
 * (i,j) fibers as its CSR pattern; A(i,j) = ((0 + b1*c(k1)) + b2*c(k2)) + ...
 * in k order. */
int oracle_ttv(const oracle_csf3* B, const double* c, oracle_csr* A);

/* row-dot (a(i) = sum(j) B(i,j)*C(i,j), both CSR, no
 * workspace): two-pointer intersection of the sorted rows, products summed
 * in j order from 0; one merge_compare per loop iteration. */
int oracle_rowdot(const oracle_csr_in* B, const oracle_csr_in* C, double* a, double* aabs);

/* Merge-based SpAdd baseline (the paper's comparison to the
 * workspace plan): D = ((ops[0] + ops[1]) + ops[2]) + ...; each step is a
 * union co-iteration of two sorted rows while either has entries left
 * (coinciding entries add, lone entries are copied); one merge_compare per
 * loop iteration, i.e. per union coordinate. */
int oracle_spadd_merge(int nops, const oracle_csr_in* ops, oracle_csr* D);
void oracle_last_counters(oracle_counters* out);

#ifdef __cplusplus
}
#endif

#endif
