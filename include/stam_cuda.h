/*
 * stam_cuda.h — C ABI of the B200 (sm_100a) workspace sparse kernels.
 *
 * This is the drop-in boundary for the engine slot of the reference `stam`
 * library.  The reference ships no kernel entry points: `src/engine.cpp:1` is a
 * placeholder and SPEC's intended call is
 *     execute(plan, inputs, mode) -> (TensorStorage, ExecutionStats)
 * (`SPEC.md:377-385`).  Each call below is one fixed instance of that call for
 * the loop nest `schedule()` emits for the kernel (golden CIN in
 * `tests/test_transform.cpp:141-147,166-184,275-284`), taking plain pointer
 * views of the reference's storage layout (`include/stam/storage.h:17-72`):
 *
 *   CSR  = format csr()        {dense, compressed}           (format.cpp:83)
 *   CSF3 = format csf(3)       {dense, compressed, compressed} (format.cpp:91-95)
 *   dense= format denseFormat(2), row-major p = i*cols + r   (format.cpp:79-81,
 *                                                              storage.cpp:69-70)
 *
 * Index arrays are int64 and values fp64, exactly the reference widths
 * (`storage.h:21-22,71`).  There is no CPU fallback: every call runs sm_100a
 * kernels or returns an error.
 *
 * Ownership: inputs are borrowed for the duration of the call.  Results are
 * library-allocated (device memory or pinned host memory, per
 * stam_options.result_mem) and released with stam_cuda_release().
 *
 * Errors: every call returns 0 on success, otherwise a stam_status code.
 * Codes 1..21 are 1 + (int)stam::ErrorCode (`include/stam/error.h:9-31`), so
 * the C++ wrapper rethrows stam::Error with the same code.  The message of the
 * last failure on the calling thread is stam_cuda_last_error().  No C++
 * exception crosses this boundary.
 *
 * Threading: a context is single-owner (like the reference's builders and
 * workspaces); calls on distinct contexts may run concurrently
 * (SPEC.md:425-426).  Calls are synchronous on return.
 */
#ifndef STAM_CUDA_H_
#define STAM_CUDA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define STAM_CUDA_API __attribute__((visibility("default")))
#else
#define STAM_CUDA_API
#endif

#define STAM_CUDA_ABI_VERSION 1

/* ---- status codes --------------------------------------------------------*/
enum stam_status {
  STAM_OK = 0,
  /* 1 + (int)stam::ErrorCode, error.h:9-31 */
  STAM_ERR_PARSE = 1,
  STAM_ERR_ARITY_MISMATCH = 2,
  STAM_ERR_DIMENSION_MISMATCH = 3,
  STAM_ERR_ORDER_MISMATCH = 4,
  STAM_ERR_OUT_OF_RANGE = 5,
  STAM_ERR_APPEND_OUT_OF_ORDER = 6,
  STAM_ERR_ILL_FORMED = 7,
  STAM_ERR_PRECONDITION_VIOLATED = 8,
  STAM_ERR_UNSUPPORTED_MERGE = 15,
  STAM_ERR_MISSING_SLOT = 18,
  STAM_ERR_CHECK_FAILED = 19,
  STAM_ERR_INTERNAL = 21,
  /* device-side failures (no reference equivalent) */
  STAM_ERR_CUDA = 64,
  STAM_ERR_OUT_OF_MEMORY = 65,
  STAM_ERR_NO_DEVICE = 66
};

enum stam_mem { STAM_MEM_HOST = 0, STAM_MEM_DEVICE = 1 };

/* Execution modes of SPEC.md:372-374 (ExecutionMode) */
enum stam_mode { STAM_MODE_FUSED = 0, STAM_MODE_ASSEMBLE = 1, STAM_MODE_COMPUTE = 2 };

/* ---- views (borrowed) ----------------------------------------------------*/

/* CSR: level(1).pos [nrows+1], level(1).idx [nnz] strictly increasing per
 * row, vals [nnz] (storage.h:19-23,71; validate() storage.cpp:103-147). */
typedef struct stam_csr_view {
  int64_t nrows;
  int64_t ncols;
  int64_t nnz;
  const int64_t* pos;
  const int64_t* idx;
  const double* vals;
  int32_t mem; /* enum stam_mem */
  int32_t _pad;
} stam_csr_view;

/* CSF(3), mode order (i,j,k): level(1).pos [dims[0]+1], level(1).idx
 * [nfibers], level(2).pos [nfibers+1], level(2).idx [nnz], vals [nnz]. */
typedef struct stam_csf3_view {
  int64_t dims[3];
  int64_t nfibers;
  int64_t nnz;
  const int64_t* pos1;
  const int64_t* idx1;
  const int64_t* pos2;
  const int64_t* idx2;
  const double* vals;
  int32_t mem;
  int32_t _pad;
} stam_csf3_view;

/* Dense row-major matrix (denseFormat(2)). */
typedef struct stam_dense_view {
  int64_t nrows;
  int64_t ncols;
  const double* vals;
  int32_t mem;
  int32_t _pad;
} stam_dense_view;

/* ---- results (library-owned) ---------------------------------------------*/
typedef struct stam_csr_result {
  int64_t nrows;
  int64_t ncols;
  int64_t nnz;
  int64_t* pos;
  int64_t* idx;
  double* vals;
  int32_t mem;
  int32_t _pad;
  void* handle; /* release with stam_cuda_release */
} stam_csr_result;

typedef struct stam_dense_result {
  int64_t nrows;
  int64_t ncols;
  double* vals;
  int32_t mem;
  int32_t _pad;
  void* handle;
} stam_dense_result;

/* ---- options and counters ------------------------------------------------*/
typedef struct stam_options {
  int32_t sort;       /* 1 (default): sorted coordinates per row */
  int32_t mode;       /* enum stam_mode: FUSED / ASSEMBLE (SpGEMM, SpAdd); COMPUTE via *_compute */
  int32_t result_mem; /* enum stam_mem for the result buffers */
  int32_t timing;     /* 1: record CUDA events around each kernel (stats) */
} stam_options;

/* SPEC.md:368-371 ExecutionStats, plus device timings. */
typedef struct stam_stats {
  int64_t mults;
  int64_t adds;
  int64_t merge_compares;
  int64_t sparse_inserts;
  int64_t appends;
  int64_t ws_inserts;
  int64_t ws_resets;
  int64_t bytes_allocated;
  int64_t kernel_launches;  /* kernels this call launched */
  float main_kernel_ms;     /* duration of the dominant kernel (timing=1) */
  float total_kernel_ms;    /* sum over this call's kernels (timing=1) */
  float h2d_ms;             /* input staging when views are host memory */
  float d2h_ms;             /* result copy when result_mem is host */
  char main_kernel[48];     /* name of the dominant kernel */
} stam_stats;

typedef struct stam_cuda_ctx stam_cuda_ctx;

/* ---- context -------------------------------------------------------------*/
STAM_CUDA_API int stam_cuda_abi_version(void);
STAM_CUDA_API const char* stam_cuda_last_error(void);
STAM_CUDA_API void stam_cuda_default_options(stam_options* opts);

/* Creates a context on `device`: a non-blocking stream and a stream-ordered
 * memory pool for scratch and results. */
STAM_CUDA_API int stam_cuda_ctx_create(int device, stam_cuda_ctx** out);
STAM_CUDA_API int stam_cuda_ctx_destroy(stam_cuda_ctx* ctx);
/* Runs subsequent calls on the caller's stream (a cudaStream_t); NULL
 * restores the context's own stream. */
STAM_CUDA_API int stam_cuda_ctx_set_stream(stam_cuda_ctx* ctx, void* stream);
STAM_CUDA_API int stam_cuda_ctx_device(const stam_cuda_ctx* ctx);
STAM_CUDA_API int stam_cuda_synchronize(stam_cuda_ctx* ctx);

/* Frees a result's buffers (device memory back to the pool, pinned host
 * memory back to the context cache). */
STAM_CUDA_API int stam_cuda_release(stam_cuda_ctx* ctx, void* handle);

/* ---- kernels -------------------------------------------------------------*/

/* C = A·B, Gustavson row-wise with a per-row workspace:
 *   forall(i) ((forall(j) C(i,j) = w0(j)) where (forall(k,j) w0(j) += A(i,k)*B(k,j)))
 * (test_transform.cpp:141-147).  CSR x CSR -> CSR, sorted columns.  Rows are
 * binned by their product count; symbolic pass, scan, numeric pass. */
STAM_CUDA_API int stam_cuda_spgemm(stam_cuda_ctx* ctx, const stam_csr_view* A,
                                   const stam_csr_view* B,
                                   const stam_options* opts,
                                   stam_csr_result* C, stam_stats* stats);

/* opts->mode: FUSED (default) computes index and values; ASSEMBLE computes
 * the exact index only (values zero; the symbolic / assembly phase,
 * PAPER.md:1116-1146); COMPUTE is stam_cuda_spgemm_compute.  opts->sort = 0
 * leaves each row's columns in workspace order (same set per row). */

/* COMPUTE mode (SPEC run_compute_after_assemble): the
 * values of A·B written into the pre-assembled index `Cidx` (pos/idx, e.g. an
 * ASSEMBLE result; rows sorted unless opts->sort = 0; values ignored).  The
 * result carries Cidx's pos/idx unchanged and every value is the canonical
 * sequential sum (bit-identical to the CPU reference).  A product whose
 * column is absent from its row fails with STAM_ERR_MISSING_SLOT. */
STAM_CUDA_API int stam_cuda_spgemm_compute(stam_cuda_ctx* ctx, const stam_csr_view* A,
                                           const stam_csr_view* B, const stam_csr_view* Cidx,
                                           const stam_options* opts,
                                           stam_csr_result* C, stam_stats* stats);

/* D = ops[0] + ops[1] + ... , every operand row scattered into one row
 * workspace in operand order, no pairwise merge:
 *   forall(i) ((forall(j) D(i,j) = w0(j)) where ((forall(j) w0(j) = B(i,j) ;
 *                forall(j) w0(j) += C(i,j) ; ...)))   (test_transform.cpp:275-284)
 * nops >= 2, all operands of equal dimensions; any count (beyond 16 the
 * workspace sequence continues across kernel calls with the partial sum as
 * operand 0 — bit-identical to one pass). */
STAM_CUDA_API int stam_cuda_spadd(stam_cuda_ctx* ctx, int32_t nops,
                                  const stam_csr_view* ops,
                                  const stam_options* opts, stam_csr_result* D,
                                  stam_stats* stats);

/* opts->mode: FUSED or ASSEMBLE (exact union index, zero values; no value
 * traffic).  Rows come out sorted either way (a valid sort = 0 order). */

/* COMPUTE mode for SpAdd: operand values written into the pre-assembled
 * index `Didx` (sorted rows unless opts->sort = 0) in operand order (operand 0
 * assigns, later operands accumulate) — bit-identical to the workspace.  An
 * operand column absent from its row fails with STAM_ERR_MISSING_SLOT. */
STAM_CUDA_API int stam_cuda_spadd_compute(stam_cuda_ctx* ctx, int32_t nops,
                                          const stam_csr_view* ops, const stam_csr_view* Didx,
                                          const stam_options* opts, stam_csr_result* D,
                                          stam_stats* stats);

/* A(i,r) = sum_{j,k} B(i,j,k)·D(k,r)·C(j,r), dense factors, dense A:
 *   forall(i,j) ((forall(r) A(i,r) += w0(r)*C(j,r)) where
 *                (forall(k,r) w0(r) += B(i,j,k)*D(k,r)))
 * (paper letters test_transform.cpp:166-173).  C is
 * dims[1] x R, D is dims[2] x R, A is dims[0] x R. */
STAM_CUDA_API int stam_cuda_mttkrp_dense(stam_cuda_ctx* ctx,
                                         const stam_csf3_view* B,
                                         const stam_dense_view* C,
                                         const stam_dense_view* D,
                                         const stam_options* opts,
                                         stam_dense_result* A, stam_stats* stats);

/* Same contraction with CSR factors and a CSR result built by compacting the
 * rank-R row workspace w1; w0 is consumed with a presence check
 * (Workspace::present, workspace.h:35):
 *   forall(i) ((forall(r) A(i,r) = w1(r)) where (forall(j) ((forall(r)
 *     w1(r) += w0(r)*C(j,r)) where (forall(k,r) w0(r) += B(i,j,k)*D(k,r)))))
 * (paper letters test_transform.cpp:175-184). */
STAM_CUDA_API int stam_cuda_mttkrp_sparse(stam_cuda_ctx* ctx,
                                          const stam_csf3_view* B,
                                          const stam_csr_view* C,
                                          const stam_csr_view* D,
                                          const stam_options* opts,
                                          stam_csr_result* A, stam_stats* stats);

/* ---- SPEC kernels outside the workspace plans ------------*/

/* TTV (SPEC Fig. ttv: forall(i,j,k) A(i,j) += B(i,j,k)*c(k)): CSR result over
 * B's (i,j) fibers, each value summed over k in order.  c holds dims[2]
 * values (any dense shape). */
STAM_CUDA_API int stam_cuda_ttv(stam_cuda_ctx* ctx, const stam_csf3_view* B,
                                const stam_dense_view* c, const stam_options* opts,
                                stam_csr_result* A, stam_stats* stats);

/* row-dot (a(i) = sum(j) B(i,j)*C(i,j), no workspace):
 * intersection of the sorted rows, summed in j order; a is nrows x 1.
 * stats->merge_compares = the two-pointer loop iterations. */
STAM_CUDA_API int stam_cuda_rowdot(stam_cuda_ctx* ctx, const stam_csr_view* B,
                                   const stam_csr_view* C, const stam_options* opts,
                                   stam_dense_result* a, stam_stats* stats);

/* Merge-based SpAdd baseline: D = ((ops[0] + ops[1]) +
 * ops[2]) + ..., each step a two-way union co-iteration (coinciding entries
 * add, lone entries are copied); stats->merge_compares counts the loop
 * iterations (one per union coordinate).  The workspace plan is
 * stam_cuda_spadd (merge_compares == 0). */
STAM_CUDA_API int stam_cuda_spadd_merge(stam_cuda_ctx* ctx, int32_t nops,
                                        const stam_csr_view* ops, const stam_options* opts,
                                        stam_csr_result* D, stam_stats* stats);

#ifdef __cplusplus
}
#endif

#endif /* STAM_CUDA_H_ */
