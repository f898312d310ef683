/*
 * stam_oracle.c — CPU restatement of the workspace kernels (test infrastructure).
 * See stam_oracle.h for the contract; build with -O2 -ffp-contract=off.
 *
 * Reference anchors:
 *   Workspace::insert / mark / drain / reset     src/workspace.cpp:34-80
 *   TensorBuilder append order + assembly        src/storage.cpp:242-375
 *   SpGEMM CIN   tests/test_transform.cpp:141-147 (+ SURVEY probe A.1)
 *   SpAdd CIN    tests/test_transform.cpp:275-284
 *   MTTKRP CIN   tests/test_transform.cpp:166-184 (+ SURVEY probe A.1, P1)
 *   engine loop  SPEC.md:377-410, counters SPEC.md:414-418
 *
 * Rows (slices) are independent, so `nthreads` > 1 splits them into
 * contiguous blocks, each with its own workspace (the reference's concurrency
 * model: distinct invocations may run concurrently); the
 * per-block results are concatenated.  Results do not depend on nthreads.
 */
#include "stam_oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <pthread.h>

/* Runs fn(b, arg) for b in [0, n) on n threads (b = 0 on the caller). */
typedef void (*par_fn)(int b, void* arg);
typedef struct par_job {
  par_fn fn;
  void* arg;
  int b;
} par_job;
static void* par_tramp(void* p) {
  par_job* j = (par_job*)p;
  j->fn(j->b, j->arg);
  return NULL;
}
static void par_run(int n, par_fn fn, void* arg) {
  if (n <= 1) {
    fn(0, arg);
    return;
  }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n);
  par_job* jobs = (par_job*)malloc(sizeof(par_job) * (size_t)n);
  int* ok = (int*)calloc((size_t)n, sizeof(int));
  for (int b = 1; b < n; b++) {
    jobs[b].fn = fn;
    jobs[b].arg = arg;
    jobs[b].b = b;
    ok[b] = pthread_create(&th[b], NULL, par_tramp, &jobs[b]) == 0;
    if (!ok[b]) fn(b, arg);
  }
  fn(0, arg);
  for (int b = 1; b < n; b++)
    if (ok[b]) pthread_join(th[b], NULL);
  free(th);
  free(jobs);
  free(ok);
}

static __thread oracle_counters g_counters;

void oracle_last_counters(oracle_counters* out) { *out = g_counters; }

/* ------------------------------------------------------------------------ */
/* dense workspace: vals + guard flags + coordinate list (workspace.h:55-59) */
typedef struct ws_t {
  int64_t size;
  double* vals;
  double* absv;
  unsigned char* flag;
  int64_t* list;
  int64_t n;
} ws_t;

static int ws_init(ws_t* w, int64_t size) {
  w->size = size;
  w->n = 0;
  w->vals = (double*)calloc((size_t)size, sizeof(double));
  w->absv = (double*)calloc((size_t)size, sizeof(double));
  w->flag = (unsigned char*)calloc((size_t)size, 1);
  w->list = (int64_t*)malloc((size_t)size * sizeof(int64_t));
  return (w->vals && w->absv && w->flag && w->list) ? 0 : -1;
}

static void ws_destroy(ws_t* w) {
  free(w->vals);
  free(w->absv);
  free(w->flag);
  free(w->list);
}

/* insert(coord, v, accumulate) — workspace.cpp:34-46 */
static inline void ws_insert(ws_t* w, int64_t c, double v, double av, int accumulate) {
  if (accumulate) {
    w->vals[c] += v;
    w->absv[c] += av;
  } else {
    w->vals[c] = v;
    w->absv[c] = av;
  }
  if (!w->flag[c]) {
    w->flag[c] = 1;
    w->list[w->n++] = c;
  }
}

/* in-place ascending sort of int64 keys (introsort-free quicksort + insertion) */
static void sort_i64(int64_t* a, int64_t n) {
  while (n > 24) {
    int64_t p = a[n / 2], i = 0, j = n - 1;
    int64_t x = a[0], y = a[n - 1];
    /* median of three */
    if ((x < p) != (x < y)) p = x;
    else if ((y < p) != (y < x)) p = y;
    while (i <= j) {
      while (a[i] < p) i++;
      while (a[j] > p) j--;
      if (i <= j) {
        int64_t t = a[i];
        a[i] = a[j];
        a[j] = t;
        i++;
        j--;
      }
    }
    /* recurse on the smaller side */
    if (j + 1 < n - i) {
      sort_i64(a, j + 1);
      a += i;
      n -= i;
    } else {
      sort_i64(a + i, n - i);
      n = j + 1;
    }
  }
  for (int64_t i = 1; i < n; i++) {
    int64_t v = a[i], k = i - 1;
    while (k >= 0 && a[k] > v) {
      a[k + 1] = a[k];
      k--;
    }
    a[k + 1] = v;
  }
}

/* growable row-block output (the builder's doubling, storage.cpp:223-240) */
typedef struct blk_t {
  int64_t n, cap;
  int64_t* idx;
  double* vals;
  double* absv;
} blk_t;

static int blk_reserve(blk_t* b, int64_t need) {
  if (need <= b->cap) return 0;
  int64_t cap = b->cap ? b->cap : 1024;
  while (cap < need) cap *= 2;
  int64_t* ni = (int64_t*)realloc(b->idx, (size_t)cap * sizeof(int64_t));
  if (!ni) return -1;
  b->idx = ni;
  double* nv = (double*)realloc(b->vals, (size_t)cap * sizeof(double));
  if (!nv) return -1;
  b->vals = nv;
  double* na = (double*)realloc(b->absv, (size_t)cap * sizeof(double));
  if (!na) return -1;
  b->absv = na;
  b->cap = cap;
  return 0;
}

/* drain(sort=true) into the block, then reset — workspace.cpp:62-80 */
static int ws_drain_sorted(ws_t* w, blk_t* out) {
  sort_i64(w->list, w->n);
  if (blk_reserve(out, out->n + w->n)) return -1;
  for (int64_t t = 0; t < w->n; t++) {
    int64_t c = w->list[t];
    out->idx[out->n] = c;
    out->vals[out->n] = w->vals[c];
    out->absv[out->n] = w->absv[c];
    out->n++;
    w->vals[c] = 0.0;
    w->absv[c] = 0.0;
    w->flag[c] = 0;
  }
  w->n = 0;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* row-blocked driver: each block computes rows [r0,r1) into its blk_t and
 * records per-row counts; blocks are concatenated afterwards. */
typedef int (*row_fn)(const void* ctx, ws_t* w, int64_t row, blk_t* out, oracle_counters* cnt);

typedef struct rows_job {
  int64_t nrows, ws_size;
  int nthreads;
  const void* ctx;
  row_fn fn;
  int64_t* counts;
  blk_t* blocks;
  oracle_counters* cnts;
  int* errs;
} rows_job;

static void rows_worker(int b, void* arg) {
  rows_job* j = (rows_job*)arg;
  int64_t r0 = j->nrows * b / j->nthreads, r1 = j->nrows * (b + 1) / j->nthreads;
  ws_t w;
  if (ws_init(&w, j->ws_size)) {
    j->errs[b] = 1;
    return;
  }
  for (int64_t r = r0; r < r1; r++) {
    int64_t before = j->blocks[b].n;
    if (j->fn(j->ctx, &w, r, &j->blocks[b], &j->cnts[b])) {
      j->errs[b] = 1;
      break;
    }
    j->counts[r + 1] = j->blocks[b].n - before;
  }
  ws_destroy(&w);
}

typedef struct concat_job {
  int64_t nrows;
  int nthreads;
  const int64_t* counts;
  const blk_t* blocks;
  oracle_csr* res;
} concat_job;

static void concat_worker(int b, void* arg) {
  concat_job* j = (concat_job*)arg;
  int64_t r0 = j->nrows * b / j->nthreads;
  int64_t off = j->counts[r0];
  const blk_t* k = &j->blocks[b];
  if (k->n) {
    memcpy(j->res->idx + off, k->idx, (size_t)k->n * sizeof(int64_t));
    memcpy(j->res->vals + off, k->vals, (size_t)k->n * sizeof(double));
    memcpy(j->res->absv + off, k->absv, (size_t)k->n * sizeof(double));
  }
}

static int run_rows(int64_t nrows, int64_t ws_size, int nthreads, const void* ctx, row_fn fn,
                    int64_t ncols_out, oracle_csr* res) {
  memset(res, 0, sizeof(*res));
  if (nthreads < 1) nthreads = 1;
  if (nthreads > nrows) nthreads = (int)(nrows > 0 ? nrows : 1);
  int64_t* counts = (int64_t*)calloc((size_t)nrows + 1, sizeof(int64_t));
  blk_t* blocks = (blk_t*)calloc((size_t)nthreads, sizeof(blk_t));
  oracle_counters* cnts = (oracle_counters*)calloc((size_t)nthreads, sizeof(oracle_counters));
  int err = 0;
  if (!counts || !blocks || !cnts) {
    free(counts);
    free(blocks);
    free(cnts);
    return -1;
  }
  int* errs = (int*)calloc((size_t)nthreads, sizeof(int));
  rows_job job = {nrows, ws_size, nthreads, ctx, fn, counts, blocks, cnts, errs};
  par_run(nthreads, rows_worker, &job);
  for (int b = 0; b < nthreads; b++) err |= errs[b];
  free(errs);
  memset(&g_counters, 0, sizeof(g_counters));
  for (int b = 0; b < nthreads; b++) {
    g_counters.mults += cnts[b].mults;
    g_counters.adds += cnts[b].adds;
    g_counters.ws_inserts += cnts[b].ws_inserts;
    g_counters.ws_resets += cnts[b].ws_resets;
    g_counters.appends += cnts[b].appends;
  }
  if (!err) {
    for (int64_t r = 0; r < nrows; r++) counts[r + 1] += counts[r];
    int64_t nnz = counts[nrows];
    res->nrows = nrows;
    res->ncols = ncols_out;
    res->nnz = nnz;
    res->pos = counts;
    res->idx = (int64_t*)malloc((size_t)(nnz ? nnz : 1) * sizeof(int64_t));
    res->vals = (double*)malloc((size_t)(nnz ? nnz : 1) * sizeof(double));
    res->absv = (double*)malloc((size_t)(nnz ? nnz : 1) * sizeof(double));
    if (!res->idx || !res->vals || !res->absv) err = 1;
    if (!err) {
      concat_job cj = {nrows, nthreads, counts, blocks, res};
      par_run(nthreads, concat_worker, &cj);
    }
  }
  for (int b = 0; b < nthreads; b++) {
    free(blocks[b].idx);
    free(blocks[b].vals);
    free(blocks[b].absv);
  }
  free(blocks);
  free(cnts);
  if (err) {
    free(res->idx);
    free(res->vals);
    free(res->absv);
    free(counts);
    memset(res, 0, sizeof(*res));
    return -1;
  }
  return 0;
}

void oracle_free(oracle_csr* m) {
  if (!m) return;
  free(m->pos);
  free(m->idx);
  free(m->vals);
  free(m->absv);
  m->pos = m->idx = NULL;
  m->vals = m->absv = NULL;
}

/* ------------------------------------------------------------------------ */
/* SpGEMM */
typedef struct spgemm_ctx {
  const oracle_csr_in* A;
  const oracle_csr_in* B;
} spgemm_ctx;

static int spgemm_row(const void* vctx, ws_t* w, int64_t i, blk_t* out, oracle_counters* cnt) {
  const spgemm_ctx* c = (const spgemm_ctx*)vctx;
  const oracle_csr_in* A = c->A;
  const oracle_csr_in* B = c->B;
  /* forall(k in A(i,:)) forall(j in B(k,:)) w0(j) += A(i,k)*B(k,j) */
  for (int64_t p = A->pos[i]; p < A->pos[i + 1]; p++) {
    const int64_t k = A->idx[p];
    const double a = A->vals[p];
    for (int64_t q = B->pos[k]; q < B->pos[k + 1]; q++) {
      const double prod = a * B->vals[q];
      ws_insert(w, B->idx[q], prod, fabs(prod), 1);
      cnt->mults++;
      cnt->ws_inserts++;
    }
  }
  cnt->adds = cnt->mults;
  cnt->ws_resets++;
  /* forall(j) C(i,j) = w0(j): sorted drain appended to row i */
  int64_t before = out->n;
  if (ws_drain_sorted(w, out)) return -1;
  cnt->appends += out->n - before;
  return 0;
}

int oracle_spgemm(const oracle_csr_in* A, const oracle_csr_in* B, int nthreads, oracle_csr* C) {
  if (A->ncols != B->nrows) return -2;
  spgemm_ctx c = {A, B};
  return run_rows(A->nrows, B->ncols, nthreads, &c, spgemm_row, B->ncols, C);
}

/* ------------------------------------------------------------------------ */
/* SpAdd */
typedef struct spadd_ctx {
  int nops;
  const oracle_csr_in* ops;
} spadd_ctx;

static int spadd_row(const void* vctx, ws_t* w, int64_t i, blk_t* out, oracle_counters* cnt) {
  const spadd_ctx* c = (const spadd_ctx*)vctx;
  for (int o = 0; o < c->nops; o++) {
    const oracle_csr_in* X = &c->ops[o];
    /* forall(j) w0(j) = B(i,j)  then  forall(j) w0(j) += C(i,j) ; ... */
    for (int64_t q = X->pos[i]; q < X->pos[i + 1]; q++) {
      ws_insert(w, X->idx[q], X->vals[q], fabs(X->vals[q]), o > 0);
      cnt->ws_inserts++;
      if (o > 0) cnt->adds++;
    }
  }
  cnt->ws_resets++;
  int64_t before = out->n;
  if (ws_drain_sorted(w, out)) return -1;
  cnt->appends += out->n - before;
  return 0;
}

int oracle_spadd(int nops, const oracle_csr_in* ops, int nthreads, oracle_csr* D) {
  if (nops < 2) return -2;
  for (int o = 1; o < nops; o++)
    if (ops[o].nrows != ops[0].nrows || ops[o].ncols != ops[0].ncols) return -2;
  spadd_ctx c = {nops, ops};
  return run_rows(ops[0].nrows, ops[0].ncols, nthreads, &c, spadd_row, ops[0].ncols, D);
}

/* ------------------------------------------------------------------------ */
/* MTTKRP, dense factors:
 *   forall(i,j) ((forall(r) A(i,r) += w0(r)*C(j,r)) where
 *                (forall(k,r) w0(r) += B(i,j,k)*D(k,r)))                     */
typedef struct mttkrp_dense_job {
  const oracle_csf3* B;
  const double* C;
  const double* D;
  int64_t R;
  int nthreads;
  double* A;
  double* Aabs;
  int64_t* mults;
} mttkrp_dense_job;

static void mttkrp_dense_worker(int b, void* arg) {
  mttkrp_dense_job* j = (mttkrp_dense_job*)arg;
  const oracle_csf3* B = j->B;
  const int64_t R = j->R, I = B->dims[0];
  double* w0 = (double*)malloc((size_t)R * sizeof(double));
  double* w0a = (double*)malloc((size_t)R * sizeof(double));
  int64_t mults = 0;
  /* slices interleaved over threads (slice sizes are skewed) */
  for (int64_t i = b; i < I; i += j->nthreads) {
    double* Ai = j->A + i * R;
    double* Aai = j->Aabs + i * R;
    for (int64_t f = B->pos1[i]; f < B->pos1[i + 1]; f++) {
      const int64_t jj = B->idx1[f];
      for (int64_t r = 0; r < R; r++) {
        w0[r] = 0.0;
        w0a[r] = 0.0;
      }
      for (int64_t p = B->pos2[f]; p < B->pos2[f + 1]; p++) {
        const int64_t k = B->idx2[p];
        const double bv = B->vals[p];
        const double* Dk = j->D + k * R;
        for (int64_t r = 0; r < R; r++) {
          const double t = bv * Dk[r];
          w0[r] += t;
          w0a[r] += fabs(t);
        }
        mults += R;
      }
      const double* Cj = j->C + jj * R;
      for (int64_t r = 0; r < R; r++) {
        Ai[r] += w0[r] * Cj[r];
        Aai[r] += w0a[r] * fabs(Cj[r]);
      }
      mults += R;
    }
  }
  j->mults[b] = mults;
  free(w0);
  free(w0a);
}

int oracle_mttkrp_dense(const oracle_csf3* B, const double* C, const double* D, int64_t R,
                        int nthreads, double* A, double* Aabs) {
  const int64_t I = B->dims[0];
  if (nthreads < 1) nthreads = 1;
  memset(A, 0, (size_t)(I * R) * sizeof(double));
  memset(Aabs, 0, (size_t)(I * R) * sizeof(double));
  int64_t* mults = (int64_t*)calloc((size_t)nthreads, sizeof(int64_t));
  mttkrp_dense_job job = {B, C, D, R, nthreads, A, Aabs, mults};
  par_run(nthreads, mttkrp_dense_worker, &job);
  memset(&g_counters, 0, sizeof(g_counters));
  for (int b = 0; b < nthreads; b++) g_counters.mults += mults[b];
  g_counters.adds = g_counters.mults;
  free(mults);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* MTTKRP, sparse factors and sparse result:
 *   forall(i) ((forall(r) A(i,r) = w1(r)) where (forall(j) ((forall(r)
 *     w1(r) += w0(r)*C(j,r)) where (forall(k,r) w0(r) += B(i,j,k)*D(k,r)))))
 * w0 is consumed at C's stored coordinates with a presence check
 * (Workspace::present, workspace.h:35). */
typedef struct mttkrp_sp_ctx {
  const oracle_csf3* B;
  const oracle_csr_in* C;
  const oracle_csr_in* D;
  int64_t R;
} mttkrp_sp_ctx;

static int mttkrp_sparse_row(const void* vctx, ws_t* w1, int64_t i, blk_t* out,
                             oracle_counters* cnt) {
  const mttkrp_sp_ctx* c = (const mttkrp_sp_ctx*)vctx;
  const oracle_csf3* B = c->B;
  const oracle_csr_in* C = c->C;
  const oracle_csr_in* D = c->D;
  /* per-thread inner workspace w0 (R-wide), allocated lazily in w1's slack */
  static __thread ws_t w0;
  static __thread int64_t w0_size = -1;
  if (w0_size != c->R) {
    if (w0_size >= 0) ws_destroy(&w0);
    if (ws_init(&w0, c->R)) return -1;
    w0_size = c->R;
  }
  for (int64_t f = B->pos1[i]; f < B->pos1[i + 1]; f++) {
    const int64_t j = B->idx1[f];
    for (int64_t p = B->pos2[f]; p < B->pos2[f + 1]; p++) {
      const int64_t k = B->idx2[p];
      const double b = B->vals[p];
      for (int64_t q = D->pos[k]; q < D->pos[k + 1]; q++) {
        const double t = b * D->vals[q];
        ws_insert(&w0, D->idx[q], t, fabs(t), 1);
        cnt->mults++;
        cnt->ws_inserts++;
      }
    }
    for (int64_t q = C->pos[j]; q < C->pos[j + 1]; q++) {
      const int64_t r = C->idx[q];
      if (!w0.flag[r]) continue; /* present(r) */
      const double t = w0.vals[r] * C->vals[q];
      ws_insert(w1, r, t, w0.absv[r] * fabs(C->vals[q]), 1);
      cnt->mults++;
      cnt->ws_inserts++;
    }
    /* reset w0 (where-producer scope ends) */
    for (int64_t t = 0; t < w0.n; t++) {
      const int64_t r = w0.list[t];
      w0.vals[r] = 0.0;
      w0.absv[r] = 0.0;
      w0.flag[r] = 0;
    }
    w0.n = 0;
    cnt->ws_resets++;
  }
  cnt->adds = cnt->mults;
  cnt->ws_resets++;
  int64_t before = out->n;
  if (ws_drain_sorted(w1, out)) return -1;
  cnt->appends += out->n - before;
  return 0;
}

int oracle_mttkrp_sparse(const oracle_csf3* B, const oracle_csr_in* C, const oracle_csr_in* D,
                         int nthreads, oracle_csr* A) {
  if (C->nrows != B->dims[1] || D->nrows != B->dims[2] || C->ncols != D->ncols) return -2;
  mttkrp_sp_ctx c = {B, C, D, C->ncols};
  return run_rows(B->dims[0], C->ncols, nthreads, &c, mttkrp_sparse_row, C->ncols, A);
}

/* ------------------------------------------------------------------------ */
/* SPEC kernels outside the workspace plans                   */

int oracle_ttv(const oracle_csf3* B, const double* c, oracle_csr* A) {
  memset(A, 0, sizeof(*A));
  memset(&g_counters, 0, sizeof(g_counters));
  const int64_t I = B->dims[0], F = B->nfibers;
  A->nrows = I;
  A->ncols = B->dims[1];
  A->nnz = F;
  A->pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)(I + 1));
  A->idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(F > 0 ? F : 1));
  A->vals = (double*)malloc(sizeof(double) * (size_t)(F > 0 ? F : 1));
  A->absv = (double*)malloc(sizeof(double) * (size_t)(F > 0 ? F : 1));
  if (!A->pos || !A->idx || !A->vals || !A->absv) {
    oracle_free(A);
    return -1;
  }
  memcpy(A->pos, B->pos1, sizeof(int64_t) * (size_t)(I + 1));
  for (int64_t f = 0; f < F; f++) {
    double w = 0.0, wa = 0.0;
    for (int64_t p = B->pos2[f]; p < B->pos2[f + 1]; p++) {
      const double t = B->vals[p] * c[B->idx2[p]];
      w += t;
      wa += fabs(t);
      g_counters.mults++;
      g_counters.adds++;
    }
    A->idx[f] = B->idx1[f];
    A->vals[f] = w;
    A->absv[f] = wa;
  }
  g_counters.appends = F;
  return 0;
}

int oracle_rowdot(const oracle_csr_in* B, const oracle_csr_in* C, double* a, double* aabs) {
  if (B->nrows != C->nrows || B->ncols != C->ncols) return -2;
  memset(&g_counters, 0, sizeof(g_counters));
  for (int64_t i = 0; i < B->nrows; i++) {
    int64_t p = B->pos[i], q = C->pos[i];
    const int64_t pe = B->pos[i + 1], qe = C->pos[i + 1];
    double w = 0.0, wa = 0.0;
    while (p < pe && q < qe) {
      g_counters.merge_compares++;
      const int64_t x = B->idx[p], y = C->idx[q];
      if (x == y) {
        const double t = B->vals[p] * C->vals[q];
        w += t;
        wa += fabs(t);
        g_counters.mults++;
        g_counters.adds++;
        p++;
        q++;
      } else if (x < y) {
        p++;
      } else {
        q++;
      }
    }
    a[i] = w;
    if (aabs) aabs[i] = wa;
  }
  return 0;
}

/* one union co-iteration D = X + Y (row by row): the loop runs while either
 * row has entries left and compares the two current coordinates (an
 * exhausted row compares as +inf), one merge_compare per iteration = per
 * union coordinate (so merge_compares >= nnz(X u Y) - 1). */
static int union2(const oracle_csr_in* X, const oracle_csr_in* Y, const double* xabs,
                  const double* yabs, oracle_csr* D) {
  const int64_t n = X->nrows;
  memset(D, 0, sizeof(*D));
  D->nrows = n;
  D->ncols = X->ncols;
  const int64_t cap = X->nnz + Y->nnz;
  D->pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  D->idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(cap > 0 ? cap : 1));
  D->vals = (double*)malloc(sizeof(double) * (size_t)(cap > 0 ? cap : 1));
  D->absv = (double*)malloc(sizeof(double) * (size_t)(cap > 0 ? cap : 1));
  if (!D->pos || !D->idx || !D->vals || !D->absv) {
    oracle_free(D);
    return -1;
  }
  int64_t o = 0;
  D->pos[0] = 0;
  for (int64_t i = 0; i < n; i++) {
    int64_t p = X->pos[i], q = Y->pos[i];
    const int64_t pe = X->pos[i + 1], qe = Y->pos[i + 1];
    while (p < pe || q < qe) {
      g_counters.merge_compares++;
      const int64_t x = p < pe ? X->idx[p] : INT64_MAX;
      const int64_t y = q < qe ? Y->idx[q] : INT64_MAX;
      if (x == y) {
        D->idx[o] = x;
        D->vals[o] = X->vals[p] + Y->vals[q];
        D->absv[o] = (xabs ? xabs[p] : fabs(X->vals[p])) + (yabs ? yabs[q] : fabs(Y->vals[q]));
        g_counters.adds++;
        p++;
        q++;
      } else if (x < y) {
        D->idx[o] = x;
        D->vals[o] = X->vals[p];
        D->absv[o] = xabs ? xabs[p] : fabs(X->vals[p]);
        p++;
      } else {
        D->idx[o] = y;
        D->vals[o] = Y->vals[q];
        D->absv[o] = yabs ? yabs[q] : fabs(Y->vals[q]);
        q++;
      }
      o++;
    }
    D->pos[i + 1] = o;
  }
  D->nnz = o;
  g_counters.appends += o;
  return 0;
}

int oracle_spadd_merge(int nops, const oracle_csr_in* ops, oracle_csr* D) {
  if (nops < 2) return -2;
  for (int o = 1; o < nops; o++)
    if (ops[o].nrows != ops[0].nrows || ops[o].ncols != ops[0].ncols) return -2;
  memset(&g_counters, 0, sizeof(g_counters));
  oracle_csr acc;
  int err = union2(&ops[0], &ops[1], NULL, NULL, &acc);
  for (int o = 2; o < nops && !err; o++) {
    oracle_csr_in x = {acc.nrows, acc.ncols, acc.nnz, acc.pos, acc.idx, acc.vals};
    oracle_csr next;
    err = union2(&x, &ops[o], acc.absv, NULL, &next);
    oracle_free(&acc);
    acc = next;
  }
  if (err) return err;
  *D = acc;
  return 0;
}
