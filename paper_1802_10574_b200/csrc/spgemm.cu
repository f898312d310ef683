// spgemm.cu — Gustavson SpGEMM  C = A·B  (CSR x CSR -> CSR, sorted columns).
//
// Reference loop nest (golden CIN, test_transform.cpp:141-147):
//   forall(i) ((forall(j) C(i,j) = w0(j)) where (forall(k,j) w0(j) += A(i,k)*B(k,j)))
// with a dense row workspace, products accumulated into 0.0 in canonical
// order (k ascending over A's row, then B's row order), and a sorted drain
// (Workspace::insert / drain, workspace.cpp:34-71).
//
// B200 design: symbolic pass -> scan -> numeric pass.
//  * rowprod (one pass over A): products per row P_i = sum_{k in A_i} nnz(B_k)
//    (the binning key), and for every A entry its B-row start and its
//    row-local product offset, so every later kernel maps product j of a row
//    to (A entry, B position) with no staging and no block barriers.
//  * bins by P_i (exact output upper bound):
//      tiny8/16/32 P <= 8/16/32 : groups of 8/16/32 lanes per row (4/2/1 rows
//                                 per warp), one product per lane; distinct
//                                 rank by a shuffle sweep, values summed in
//                                 canonical order (bit-exact with the CPU).
//      hash XS/S/M1/M/L1/L P <= 64/256/512/1024/2048/4096 : CTA of 1..32 warps
//                                 per row.  Symbolic: a shared-memory table of
//                                 keys sized 2P whose hash is ORDER-PRESERVING
//                                 (slot = scaled column, forward linear
//                                 probing, no wrap) counts the distinct
//                                 columns.  Numeric: bucketed counting sort
//                                 (bucket_numeric_kernel): products in
//                                 registers, ~P/4 order-preserving buckets,
//                                 in-bucket ranks, duplicates folded, coalesced
//                                 row writes; rows with clustered columns (and
//                                 unsorted output) use the table's numeric
//                                 pass, whose occupied runs are mutually
//                                 ordered (ranked per run in the drain), values
//                                 accumulated with shared fp64 atomics.
//      long P > 4096          : 1024-thread CTA per row (rows claimed longest
//                                 first), a column bitmap over all columns in
//                                 shared memory (popcount rank) and fp64
//                                 atomics; computed once, before the scan,
//                                 into a scratch region, then copied into C.
//  * products are enumerated flattened, warp-contiguous and lane-interleaved
//    (B rows read coalesced), with 4 independent gathers in flight per lane.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "index.cuh"
#include "runtime.h"

namespace stamgpu {
namespace {

enum Bin : int {
  kBinEmpty = 0,
  kBinTiny8,
  kBinTiny16,
  kBinTiny32,
  kBinHashXS,
  kBinHashS,
  kBinHashM1,
  kBinHashM,
  kBinHashL1,
  kBinHashL,
  kBinLong,
  kNumBins
};
constexpr int kLongThreads = 1024;
constexpr uint32_t kEmpty = 0xffffffffu;
// threads of the hash-M1 numeric tier (rows of 256 < P <= 512 products);
// config 1 kernel: 64 0.163 ms, 128 0.121 ms (kept), 256 0.137 ms
#ifndef SPGEMM_M1_NUM_THREADS
#define SPGEMM_M1_NUM_THREADS 128
#endif
#ifndef SPGEMM_BATCH
#define SPGEMM_BATCH 4
#endif
constexpr int kBatch = SPGEMM_BATCH;  // independent product gathers in flight per lane

__host__ __device__ inline int bin_of(int64_t p) {
  if (p == 0) return kBinEmpty;
  if (p <= 8) return kBinTiny8;
  if (p <= 16) return kBinTiny16;
  if (p <= 32) return kBinTiny32;
  if (p <= 64) return kBinHashXS;
  if (p <= 256) return kBinHashS;
  if (p <= 512) return kBinHashM1;
  if (p <= 1024) return kBinHashM;
  if (p <= 2048) return kBinHashL1;
  if (p <= 4096) return kBinHashL;
  return kBinLong;
}

struct SpgemmParams {
  int64_t m, n;  // C is m x n
  const int64_t* apos;
  const int64_t* aidx;
  const double* avals;
  const int64_t* bpos;
  const int64_t* bidx;
  const double* bvals;
  const uint32_t* bcol32;    // B's column indices as u32 (n < 2^32): half the gather bytes
  int64_t* prod;             // [m] products per row
  uint2* span;               // [m] first/last column any of the row's B rows holds (x > y: none)
  uint2* bspan;              // [nrows(B)] first/last column of each B row (x > y: empty)
  int64_t* arows;            // rows with more than kLongA entries (rowprod_long_kernel)
  unsigned long long* narows;  // [0] their count, [1] claim counter
  int* aoff;                 // [nnz(A)] row-local product offset of each A entry
  int64_t* bst;              // [nnz(A)] start of the entry's B row
  unsigned long long* bins;  // [kNumBins] counts, then cursors
  int64_t* bin_rows;         // [m] rows grouped by bin
  int64_t* cpos;             // [m+1]: counts at [i+1], then offsets
  int64_t* cidx;
  double* cvals;
  int64_t* stats;            // [0] total products, [1] max products of a row
  bool values;               // false: ASSEMBLE mode (index only)
  bool sorted;               // false: rows in workspace (slot) order
};

// ---------------------------------------------------------------------------
// rowprod: a warp takes 32 consecutive rows and walks their A entries flat,
// 32 at a time (coalesced A reads, independent B-row gathers in every lane);
// the row of an entry comes from a shuffle search over the 32 row starts, and
// segmented warp scans give each entry its row-local product offset and each
// row its products and column span.  Rows continuing past a window of 32
// entries carry their partial sums into the next window.  Rows with more than
// kLongA entries are skipped here and listed for rowprod_long_kernel (a warp
// per row, claimed dynamically), so no warp is stuck behind a power-law row.
constexpr int kLongA = 64;

struct RowTally {
  unsigned long long* hist;  // shared [kNumBins]
  unsigned long long total = 0, maxp = 0;
  __device__ void add(const SpgemmParams& P, int64_t row, int64_t s, unsigned lo, unsigned hi) {
    P.prod[row] = s;
    P.span[row] = make_uint2(lo, hi);
    atomicAdd(&hist[bin_of(s)], 1ull);
    total += (unsigned long long)s;
    maxp = max(maxp, (unsigned long long)s);
  }
};

__device__ __forceinline__ void tally_flush(const SpgemmParams& P, RowTally& T,
                                            unsigned long long* sh_total,
                                            unsigned long long* sh_max) {
  const unsigned long long t = warp_sum(T.total);
  const unsigned long long mx = warp_max(T.maxp);
  if (lane_id() == 0) {
    if (t) atomicAdd(sh_total, t);
    atomicMax(sh_max, mx);
  }
  __syncthreads();
  if (threadIdx.x < kNumBins && T.hist[threadIdx.x]) atomicAdd(&P.bins[threadIdx.x], T.hist[threadIdx.x]);
  if (threadIdx.x == 0) {
    if (*sh_total) atomicAdd((unsigned long long*)&P.stats[0], *sh_total);
    atomicMax((unsigned long long*)&P.stats[1], *sh_max);
  }
}

__global__ void rowprod_kernel(const SpgemmParams P, int rw) {
  __shared__ unsigned long long hist[kNumBins];
  __shared__ unsigned long long total, maxp;
  if (threadIdx.x < kNumBins) hist[threadIdx.x] = 0;
  if (threadIdx.x == 0) total = maxp = 0;
  __syncthreads();
  const unsigned lane = lane_id();
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  RowTally T;
  T.hist = hist;
  // windows of rw <= 32 rows (fewer for small matrices: more warps in flight)
  for (int64_t base = warp * rw; base < P.m; base += nwarps * rw) {
    const int nr = (int)min((int64_t)rw, P.m - base);
    // lane l < nr: start of row base + l; lanes >= nr: the window's end
    const int64_t rp = P.apos[base + min((int)lane, nr)];
    const int64_t wend = P.apos[base + nr];
    const int64_t wbeg = __shfl_sync(kFull, rp, 0);
    int64_t rnx = __shfl_down_sync(kFull, rp, 1);  // end of row base + l
    if (lane == 31) rnx = wend;
    const bool mine = (int)lane < nr;
    if (mine && rp == rnx) T.add(P, base + lane, 0, 0xffffffffu, 0u);
    const bool longa = mine && rnx - rp > kLongA;
    const unsigned lm = __ballot_sync(kFull, longa);
    if (lm) {
      unsigned long long at = 0;
      if (lane == 0) at = atomicAdd(&P.narows[0], (unsigned long long)__popc(lm));
      at = __shfl_sync(kFull, at, 0);
      if (longa) P.arows[at + __popc(lm & lanemask_lt())] = base + lane;
    }
    int carry_r = -1;
    int64_t carry_s = 0;
    unsigned carry_lo = 0xffffffffu, carry_hi = 0u;
    int64_t c = wbeg;
    while (c < wend) {
      const int64_t p = c + lane;
      // row of entry p: the largest r < nr with start(r) <= p
      int r = 0;
#pragma unroll
      for (int st = 16; st >= 1; st >>= 1) {
        const int cand = r + st;
        const int64_t v = __shfl_sync(kFull, rp, cand & 31);
        if (cand < nr && v <= p) r = cand;
      }
      const int64_t rend = __shfl_sync(kFull, rnx, r);
      const bool rlong = ((lm >> r) & 1u) != 0;
      // a window position inside a listed row: jump past it
      const int r0 = __shfl_sync(kFull, r, 0);
      if ((lm >> r0) & 1u) {
        c = __shfl_sync(kFull, rend, 0);
        continue;
      }
      const bool valid = p < wend && !rlong;
      int64_t len = 0;
      unsigned lo = 0xffffffffu, hi = 0u;
      if (valid) {
        const int64_t k = P.aidx[p];
        const int64_t b0 = P.bpos[k], b1 = P.bpos[k + 1];
        const uint2 sp = P.bspan[k];
        P.bst[p] = b0;
        len = b1 - b0;
        lo = sp.x;
        hi = sp.y;
      }
      // segmented inclusive scans (a row's entries are contiguous lanes)
      int64_t inc = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t u = __shfl_up_sync(kFull, inc, o);
        const unsigned ul = __shfl_up_sync(kFull, lo, o), uh = __shfl_up_sync(kFull, hi, o);
        const int ru = __shfl_up_sync(kFull, r, o);
        if ((int)lane >= o && ru == r) {
          inc += u;
          lo = min(lo, ul);
          hi = max(hi, uh);
        }
      }
      const bool cont = r == carry_r;
      const int64_t off = cont ? carry_s : 0;
      if (valid) P.aoff[p] = (int)(off + inc - len);
      const int64_t tot = off + inc;
      if (cont) {
        lo = min(lo, carry_lo);
        hi = max(hi, carry_hi);
      }
      if (valid && p == rend - 1) T.add(P, base + r, tot, lo, hi);
      const int lastv = (int)min((int64_t)31, wend - 1 - c);  // last in-window lane (uniform)
      carry_r = __shfl_sync(kFull, r, lastv);
      carry_s = __shfl_sync(kFull, tot, lastv);
      carry_lo = __shfl_sync(kFull, lo, lastv);
      carry_hi = __shfl_sync(kFull, hi, lastv);
      c += 32;
    }
  }
  tally_flush(P, T, &total, &maxp);
}

// First/last column of every B row (8 bytes per row, L2-resident for rowprod's
// gathers instead of two 32-byte sectors of B's column array per A entry).
__global__ void bspan_kernel(const SpgemmParams P, int64_t nb) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nb;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b0 = P.bpos[r], b1 = P.bpos[r + 1];
    P.bspan[r] = b1 > b0 ? make_uint2((unsigned)P.bidx[b0], (unsigned)P.bidx[b1 - 1])
                         : make_uint2(0xffffffffu, 0u);
  }
}

// B's int64 column indices as u32 for the product gathers (4 instead of 8
// bytes per product in both passes; 16M entries at config 3: ~30 us).
__global__ void bcol32_kernel(const int64_t* bidx, int64_t nnz, uint32_t* out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nnz;
       t += (int64_t)gridDim.x * blockDim.x)
    out[t] = (uint32_t)__ldcs(bidx + t);
}

// Rows with more than kLongA entries: a warp per row, claimed dynamically.
__global__ void rowprod_long_kernel(const SpgemmParams P) {
  __shared__ unsigned long long hist[kNumBins];
  __shared__ unsigned long long total, maxp;
  if (threadIdx.x < kNumBins) hist[threadIdx.x] = 0;
  if (threadIdx.x == 0) total = maxp = 0;
  __syncthreads();
  const unsigned lane = lane_id();
  RowTally T;
  T.hist = hist;
  const unsigned long long n = P.narows[0];
  while (true) {
    unsigned long long q = 0;
    if (lane == 0) q = atomicAdd(&P.narows[1], 1ull);
    q = __shfl_sync(kFull, q, 0);
    if (q >= n) break;
    const int64_t i = P.arows[q];
    const int64_t b0 = P.apos[i], b1 = P.apos[i + 1];
    int64_t carry = 0;
    unsigned wlo = 0xffffffffu, whi = 0u;
    constexpr int U = 8;  // 256 entries per step: all gathers issued before the scans
    for (int64_t c = b0; c < b1; c += 32 * U) {
      int64_t bs[U], len[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t p = c + 32 * u + lane;
        bs[u] = 0;
        len[u] = 0;
        if (p < b1) {
          const int64_t k = P.aidx[p];
          bs[u] = P.bpos[k];
          len[u] = P.bpos[k + 1] - bs[u];
          const uint2 sp = P.bspan[k];
          wlo = min(wlo, sp.x);
          whi = max(whi, sp.y);
        }
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t p = c + 32 * u + lane;
        if (p < b1) P.bst[p] = bs[u];
      }
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int64_t p = c + 32 * u + lane;
        const int64_t inc = warp_inclusive_scan(len[u]);
        if (p < b1) P.aoff[p] = (int)(carry + inc - len[u]);
        carry += __shfl_sync(kFull, inc, 31);
      }
    }
    wlo = __reduce_min_sync(kFull, wlo);
    whi = __reduce_max_sync(kFull, whi);
    if (lane == 0) T.add(P, i, carry, wlo, whi);
  }
  tally_flush(P, T, &total, &maxp);
}

__global__ void bin_scatter_kernel(const SpgemmParams P, const unsigned long long* offsets) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = i < P.m;
  const int b = valid ? bin_of(P.prod[i]) : -1;
  const unsigned peers = __match_any_sync(kFull, b);
  const int leader = __ffs(peers) - 1;
  unsigned long long base = 0;
  if ((int)lane_id() == leader && valid && b != kBinEmpty)
    base = atomicAdd(&P.bins[b], (unsigned long long)__popc(peers));
  base = __shfl_sync(kFull, base, leader);
  if (valid && b != kBinEmpty) P.bin_rows[offsets[b] + base + __popc(peers & lanemask_lt())] = i;
}

// A entry of row [a0, a0+na) holding product j: last p with aoff[a0+p] <= j.
__device__ __forceinline__ int entry_of(const int* aoff, int na, int j) {
  int lo = 0, hi = na;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (aoff[mid] <= j) lo = mid; else hi = mid;
  }
  return lo;
}

// The same for a warp-uniform j, by the whole warp: each level samples 32
// evenly spaced offsets in parallel and keeps the segment holding j, so a
// row of na entries costs ceil(log32(na)) dependent loads instead of log2(na).
__device__ __forceinline__ int entry_of_warp(const int* aoff, int na, int j) {
  const int lane = (int)lane_id();
  int lo = 0, hi = na;
  while (hi - lo > 1) {
    const int step = (hi - lo + 31) >> 5;
    const int p = lo + lane * step;
    const bool le = p < hi && aoff[p] <= j;
    const unsigned m = __ballot_sync(kFull, le);  // lane 0 (aoff[lo] <= j) always set
    const int L = 31 - __clz(m);
    lo = lo + L * step;
    hi = min(hi, lo + step);
  }
  return lo;
}

// ---------------------------------------------------------------------------
// tiny rows: groups of G lanes per row, one product per lane (P <= G)
template <int G>
__device__ __forceinline__ void tiny_product(const SpgemmParams& P, int64_t i, bool valid, int g,
                                             bool numeric, int64_t& col, double& val, bool& has) {
  has = false;
  col = INT64_MAX;
  val = 0.0;
  if (!valid) return;
  const int64_t a0 = P.apos[i];
  const int na = (int)(P.apos[i + 1] - a0);
  const int prod = (int)P.prod[i];
  if (g >= prod) return;
  const int p = entry_of(P.aoff + a0, na, g);
  const int64_t q = P.bst[a0 + p] + (g - P.aoff[a0 + p]);
  col = P.bcol32[q];
  if (numeric) val = mul_rn(P.avals[a0 + p], P.bvals[q]);
  has = true;
}

template <int G>
__global__ void tiny_symbolic_kernel(const SpgemmParams P, const int64_t* rows, int64_t nrows) {
  const int lane = (int)lane_id();
  const int g = lane % G;
  const int64_t group = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  const int64_t iters = (nrows + ngroups - 1) / ngroups;
  for (int64_t it = 0; it < iters; it++) {
    const int64_t r = group + it * ngroups;
    const bool valid = r < nrows;
    const int64_t i = valid ? rows[r] : 0;
    int64_t col;
    double val;
    bool has;
    tiny_product<G>(P, i, valid, g, false, col, val, has);
    bool lead = has;
#pragma unroll
    for (int t = 0; t < G; t++) {
      const int64_t ct = __shfl_sync(kFull, col, t, G);
      if (t < g && ct == col) lead = false;
    }
    const unsigned m = __ballot_sync(kFull, lead);
    const unsigned gm = (G == 32) ? kFull : (((1u << G) - 1u) << (lane - g));
    if (valid && g == 0) P.cpos[i + 1] = __popc(m & gm);
  }
}

template <int G>
__global__ void tiny_numeric_kernel(const SpgemmParams P, const int64_t* rows, int64_t nrows) {
  const int lane = (int)lane_id();
  const int g = lane % G;
  const int64_t group = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
  const int64_t iters = (nrows + ngroups - 1) / ngroups;
  for (int64_t it = 0; it < iters; it++) {
    const int64_t r = group + it * ngroups;
    const bool valid = r < nrows;
    const int64_t i = valid ? rows[r] : 0;
    int64_t col;
    double val;
    bool has;
    tiny_product<G>(P, i, valid, g, P.values, col, val, has);
    bool lead = has;
#pragma unroll
    for (int t = 0; t < G; t++) {
      const int64_t ct = __shfl_sync(kFull, col, t, G);
      if (t < g && ct == col) lead = false;
    }
    const unsigned lead_mask = __ballot_sync(kFull, lead) >> (lane - g);
    int out = 0;
    double w = add_rn(0.0, val);  // first insert accumulates into 0.0
#pragma unroll
    for (int t = 0; t < G; t++) {
      const int64_t ct = __shfl_sync(kFull, col, t, G);
      const double vt = __shfl_sync(kFull, val, t, G);
      if (((lead_mask >> t) & 1u) && ct < col) out++;
      if (t > g && ct == col) w = add_rn(w, vt);
    }
    if (lead) {
      const int64_t dst = P.cpos[i] + out;
      P.cidx[dst] = col;
      if (P.values) P.cvals[dst] = w;
    }
  }
}

// ---------------------------------------------------------------------------
// Flattened product enumeration for CTA-per-row kernels: the row's products
// [0, P_i) are split into warp-contiguous ranges, lane-interleaved inside
// them; each lane keeps its own A-entry cursor and issues kBatch independent
// (idx, val) gathers before consuming them.  f(col, value) sees every product
// exactly once; kNumeric false skips the value loads.
// One batch of NW windows of 32 products starting at `base` (uniform) of the
// warp's range [.., w1): lane's product in window u is base + 32u + lane.
// q[u] = its B entry, av[u] = its A value, ok[u] = inside the range.  pb / ob
// (the A entry holding product `base` and that entry's first product) are
// advanced to the batch's end.
template <bool kNumeric, int NW>
__device__ __forceinline__ void product_windows(const SpgemmParams& P, int64_t a0, int na, int total,
                                                const int* aoff, int base, int w1, int& pb, int& ob,
                                                int64_t (&q)[NW], double (&av)[NW], bool (&ok)[NW]) {
  const int lane = (int)lane_id();
  const unsigned upto = (lane == 31) ? 0xffffffffu : ((2u << lane) - 1u);
#pragma unroll
  for (int u = 0; u < NW; u++) {
    const int wb = base + 32 * u;  // window start (uniform)
    const int j = wb + lane;
    ok[u] = j < w1;
    q[u] = 0;
    av[u] = 0.0;
    if (wb >= w1) continue;  // uniform
    // boundaries of the next 32 entries, relative to the window start
    const int pe = pb + 1 + lane;
    const int bnd = pe < na ? aoff[pe] - wb : (1 << 30);
    const int nxt = __shfl_down_sync(kFull, bnd, 1);
    const bool empty_seg = lane < 31 && bnd == nxt && bnd <= 32;
    int p, op;
    if (!__any_sync(kFull, empty_seg)) {
      // lane's entry = pb + #boundaries at or below it (all boundaries >= 1)
      const unsigned M = __reduce_or_sync(kFull, bnd < 32 ? (1u << bnd) : 0u);
      const int c = __popc(M & upto);
      p = pb + c;
      const int bc = __shfl_sync(kFull, bnd, (c + 31) & 31);
      op = c == 0 ? ob : bc + wb;
      // advance to the entry holding product wb + 32
      const int adv = __popc(M) + (__any_sync(kFull, bnd == 32) ? 1 : 0);
      if (adv > 0) {
        const int ba = __shfl_sync(kFull, bnd, adv - 1);
        pb += adv;
        ob = ba + wb;
      }
    } else {
      // rows with empty B rows in this window: per-lane cursor
      p = pb;
      if (ok[u])
        while (p + 1 < na && aoff[p + 1] <= j) p++;
      op = aoff[p];
      const int last = min(wb + 32, total) - 1;
      int pn = pb;
      while (pn + 1 < na && aoff[pn + 1] <= last) pn++;
      // entry holding product wb + 32 (or the last one)
      while (pn + 1 < na && aoff[pn + 1] <= wb + 32) pn++;
      pb = __shfl_sync(kFull, pn, 0);
      ob = aoff[pb];
    }
    if (ok[u]) {
      q[u] = P.bst[a0 + p] + (j - op);
      if (kNumeric) av[u] = P.avals[a0 + p];
    }
  }
}

template <bool kNumeric, typename F>
__device__ __forceinline__ void for_products(const SpgemmParams& P, int64_t a0, int na, int total,
                                             F f) {
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int per = (total + nwarps - 1) / nwarps;
  const int w0 = min(total, warp * per), w1 = min(total, w0 + per);
  if (w0 >= w1) return;
  const int* aoff = P.aoff + a0;
  // pb: A entry holding product `base`; ob: its first product (aoff[pb])
  int pb = entry_of_warp(aoff, na, w0);
  int ob = aoff[pb];
  for (int base = w0; base < w1; base += 32 * kBatch) {
    int64_t q[kBatch];
    double av[kBatch];
    bool ok[kBatch];
    product_windows<kNumeric, kBatch>(P, a0, na, total, aoff, base, w1, pb, ob, q, av, ok);
    int64_t col[kBatch];
    double bv[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; u++) {
      col[u] = 0;
      bv[u] = 0.0;
      if (ok[u]) {
        col[u] = P.bcol32[q[u]];
        if (kNumeric) bv[u] = P.bvals[q[u]];
      }
    }
#pragma unroll
    for (int u = 0; u < kBatch; u++)
      if (ok[u]) f(col[u], kNumeric ? mul_rn(av[u], bv[u]) : 0.0);
  }
}

// Order-preserving slot of a column in a table of tb main slots.
struct SlotMap {
  int64_t c0;
  uint64_t scale;  // floor(tb * 2^32 / span)
  __device__ __forceinline__ int operator()(int64_t c) const {
    return (int)(((uint64_t)(c - c0) * scale) >> 32);
  }
};

// Order-preserving slot map of row i from its column span (computed by
// rowprod from the first/last column of every B row the row touches).
__device__ __forceinline__ SlotMap row_slot_map(const SpgemmParams& P, int64_t i, int tb) {
  const uint2 sp = P.span[i];
  SlotMap sm;
  const bool nonempty = sp.x <= sp.y;
  sm.c0 = nonempty ? (int64_t)sp.x : 0;
  const uint64_t span = nonempty ? (uint64_t)(sp.y - sp.x) + 1 : 1;
  sm.scale = ((uint64_t)tb << 32) / span;
  if (sm.scale == 0) sm.scale = 1;
  return sm;
}

// Insert col (linear probing forward from its order-preserving slot).
__device__ __forceinline__ int hash_insert(uint32_t* keys, uint32_t key, int slot, bool& created) {
  while (true) {
    const uint32_t old = atomicCAS(&keys[slot], kEmpty, key);
    if (old == kEmpty) {
      created = true;
      return slot;
    }
    if (old == key) {
      created = false;
      return slot;
    }
    slot++;
  }
}

// A row with P products uses tb = next_pow2(2P) main slots (at least 64) and
// tb/2 overflow slots: at most P <= tb/2 entries are inserted, all at or after
// their home slot (< tb), so forward probing never runs off the end (a load
// of at most 1/2 keeps the order-preserving runs short).  TB is the tier's
// largest tb.
template <int TB>
struct HashSmem {
  uint32_t keys[TB + TB / 2];
  double vals[TB + TB / 2];
  int64_t red[2];
  int scan[33];
  int64_t claimed;
};

// The symbolic pass only needs the keys (3x less shared memory per row).
template <int TB>
struct HashKeysSmem {
  uint32_t keys[TB + TB / 2];
  int64_t red[2];
  int scan[33];
  int64_t claimed;
};

__device__ __forceinline__ int row_table(int64_t prod) {
  const int need = (int)(2 * prod);  // next power of two >= 2P, at least 64
  return need <= 64 ? 64 : 1 << (32 - __clz(need - 1));
}

template <int THREADS>
__device__ __forceinline__ int cta_flag_scan(bool f, int* sh, int* tot) {
  if constexpr (THREADS == 32) {
    const unsigned m = __ballot_sync(kFull, f);
    *tot = __popc(m);
    return __popc(m & lanemask_lt());
  } else {
    return block_exclusive_scan(f ? 1 : 0, sh, tot);
  }
}

template <int THREADS>
__device__ __forceinline__ void cta_sync() {
  if constexpr (THREADS == 32) __syncwarp(); else __syncthreads();
}

// Dynamic row claims one row ahead: the claim for the next row is issued when
// a row starts and published (by thread 0, into `sh`) when it ends, so the
// atomic's round trip overlaps the row's work instead of preceding it.
template <int THREADS>
struct RowClaims {
  unsigned long long* claim;
  int64_t* sh;
  int64_t ahead = 0;
  __device__ RowClaims(unsigned long long* c, int64_t* s) : claim(c), sh(s) {
    if (threadIdx.x == 0) *sh = (int64_t)atomicAdd(claim, 1ull);
  }
  __device__ __forceinline__ int64_t next() {
    cta_sync<THREADS>();
    const int64_t r = *sh;
    cta_sync<THREADS>();
    if (threadIdx.x == 0) ahead = (int64_t)atomicAdd(claim, 1ull);
    return r;
  }
  // before the row's last barrier
  __device__ __forceinline__ void publish() {
    if (threadIdx.x == 0) *sh = ahead;
  }
};

// CTA total of one int per thread; `sh` is zero on entry and left zero for
// the next call (the caller's next CTA barrier orders the reset).
template <int THREADS>
__device__ __forceinline__ int cta_sum(int v, int* sh) {
  if constexpr (THREADS == 32) {
    return warp_sum(v);
  } else {
    v = warp_sum(v);
    if (lane_id() == 0 && v) atomicAdd(sh, v);
    __syncthreads();
    const int tot = *sh;
    __syncthreads();
    if (threadIdx.x == 0) *sh = 0;
    return tot;
  }
}

// First slot at or after s0 that does not continue an occupied run (a run
// never crosses it).  Warp-cooperative forward scan; uniform result.
__device__ __forceinline__ int run_boundary(const uint32_t* keys, int s0, int nslots) {
  if (s0 <= 0) return 0;
  if (s0 >= nslots) return nslots;
  const int lane = (int)lane_id();
  for (int c = s0; c < nslots; c += 32) {
    const int s = c + lane;
    // s is a boundary iff slot s-1 is empty
    const bool bnd = s >= nslots || keys[s - 1] == kEmpty;
    const unsigned m = __ballot_sync(kFull, bnd);
    if (m) return min(nslots, c + __ffs(m) - 1);
  }
  return nslots;
}

// Writes the occupied slots of the table in column order.  Runs (maximal
// groups of consecutive occupied slots) are mutually ordered; inside a run an
// entry's output position is the run's first position plus its rank among the
// run's keys.  Warps own contiguous slot ranges whose ends sit on run
// boundaries; one block prefix over the warp counts gives each warp its base.
// A warp walks its range in windows of 32 slots cut after the window's last
// empty slot, so every run in a window is complete and ranks come from warp
// shuffles; runs of 32 or more slots rank through shared memory.
template <int THREADS>
__device__ void drain_table(const uint32_t* keys, const double* vals, int nslots, int64_t c0,
                            int64_t* out_idx, double* out_vals, int* scan, bool sorted) {
  constexpr int kWarpsN = THREADS / 32;
  const int lane = (int)lane_id();
  const int warp = threadIdx.x >> 5;
  const int per = (nslots + kWarpsN - 1) / kWarpsN;
  const int r0 = run_boundary(keys, warp * per, nslots);
  const int r1 = run_boundary(keys, (warp + 1) * per, nslots);
  int base = 0;
  if constexpr (kWarpsN > 1) {
    int cnt = 0;
    for (int c = r0; c < r1; c += 32) {
      const int s = c + lane;
      cnt += __popc(__ballot_sync(kFull, s < r1 && keys[s] != kEmpty));
    }
    if (lane == 0) scan[warp] = cnt;
    __syncthreads();
    if (warp == 0) {
      const int v = lane < kWarpsN ? scan[lane] : 0;
      const int inc = warp_inclusive_scan(v);
      if (lane < kWarpsN) scan[lane] = inc - v;
    }
    __syncthreads();
    base = scan[warp];
  }
  const unsigned lt = lanemask_lt();
  int c = r0;
  while (c < r1) {
    const int s = c + lane;
    const uint32_t k = s < r1 ? keys[s] : kEmpty;
    const bool occ = k != kEmpty;
    const unsigned om = __ballot_sync(kFull, occ);
    const unsigned em = ~om;
    if (em == 0) {
      // a run of >= 32 slots starting at c: find its end, rank in shared memory
      int e = c + 32;
      while (true) {
        const int t = e + lane;
        const unsigned m = __ballot_sync(kFull, t >= r1 || keys[t] == kEmpty);
        if (m) {
          e += __ffs(m) - 1;
          break;
        }
        e += 32;
      }
      const int len = e - c;
      // dense columns land in order (no collisions): emit directly
      bool disorder = false;
      if (sorted)
        for (int x = lane; x + 1 < len; x += 32) disorder |= keys[c + x] > keys[c + x + 1];
      const bool in_order = !__any_sync(kFull, disorder);
      for (int x = lane; x < len + (32 - len % 32) % 32; x += 32) {
        const bool mine = x < len;
        const uint32_t kx = mine ? keys[c + x] : kEmpty;
        int rank = x;
        if (!in_order) {
          rank = 0;
          for (int j = 0; j < len; j++) rank += keys[c + j] < kx ? 1 : 0;
        }
        if (mine) {
          out_idx[base + rank] = c0 + (int64_t)kx;
          if (vals) out_vals[base + rank] = vals[c + x];
        }
      }
      base += len;
      c = e;
      continue;
    }
    const int last = 31 - __clz(em);  // the window's last empty slot
    const bool mine = occ && lane < last;
    const unsigned below = em & lt;
    const int rs = below ? 32 - __clz(below) : 0;  // my run's first lane
    const unsigned above = em & ~(lt | (1u << lane));
    const int re = __ffs(above) - 1;  // my run's end (an empty lane <= last)
    // ranks: only windows whose runs are out of order need the shuffle loop
    const uint32_t kprev = __shfl_up_sync(kFull, k, 1);
    const bool dis = sorted && mine && lane > rs && kprev > k;
    int rank = lane - rs;
    if (__any_sync(kFull, dis)) {
      const int len = mine ? re - rs : 0;
      const int maxl = __reduce_max_sync(kFull, (unsigned)len);
      rank = 0;
      for (int d = 0; d < maxl; d++) {
        const int src = rs + d;
        const uint32_t kk = __shfl_sync(kFull, k, src & 31);
        rank += (src < re && kk < k) ? 1 : 0;
      }
    }
    if (mine) {
      const int pos = base + __popc(om & ((1u << rs) - 1)) + rank;
      out_idx[pos] = c0 + (int64_t)k;
      if (vals) out_vals[pos] = vals[s];
    }
    base += __popc(om & ((1u << last) - 1));
    c += last + 1;
  }
}

template <int THREADS, int TB>
__global__ void __launch_bounds__(THREADS, (THREADS >= 64 ? 2048 / THREADS : 32)) hash_symbolic_kernel(const SpgemmParams P,
                                                                 const int64_t* rows,
                                                                 int64_t nrows,
                                                                 unsigned long long* claim) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  HashKeysSmem<TB>& S = *reinterpret_cast<HashKeysSmem<TB>*>(smem_raw);
  if (threadIdx.x == 0) S.scan[0] = 0;  // cta_sum's accumulator (the claim syncs)
  RowClaims<THREADS> rc(claim, &S.claimed);
  while (true) {
    const int64_t r = rc.next();
    if (r >= nrows) break;
    const int64_t i = rows[r];
    const int total = (int)P.prod[i];
    const int tb = row_table(total);
    const int nslots = tb + tb / 2;
    const int64_t a0 = P.apos[i];
    const int na = (int)(P.apos[i + 1] - a0);
    const SlotMap sm = row_slot_map(P, i, tb);
    for (int s = threadIdx.x; s < nslots; s += THREADS) S.keys[s] = kEmpty;
    cta_sync<THREADS>();
    int created = 0;
    for_products<false>(P, a0, na, total, [&](int64_t col, double) {
      bool made;
      hash_insert(S.keys, (uint32_t)(col - sm.c0), sm(col), made);
      created += made ? 1 : 0;
    });
    const int tot = cta_sum<THREADS>(created, S.scan);
    if (threadIdx.x == 0) P.cpos[i + 1] = tot;
    rc.publish();
    cta_sync<THREADS>();
  }
}

template <int THREADS, int TB>
__global__ void __launch_bounds__(THREADS, (THREADS == 1024 ? 1 : THREADS == 32 ? 32 : 1536 / THREADS)) hash_numeric_kernel(const SpgemmParams P,
                                                                const int64_t* rows,
                                                                int64_t nrows,
                                                                unsigned long long* claim,
                                                                const unsigned long long* nrows_dev) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  HashSmem<TB>& S = *reinterpret_cast<HashSmem<TB>*>(smem_raw);
  if (nrows_dev) nrows = (int64_t)*nrows_dev;  // a list built on the device
  RowClaims<THREADS> rc(claim, &S.claimed);
  while (true) {
    const int64_t r = rc.next();
    if (r >= nrows) break;
    const int64_t i = rows[r];
    const int64_t dst = P.cpos[i];  // issued early, used by the drain
    const int total = (int)P.prod[i];
    const int tb = row_table(total);
    const int nslots = tb + tb / 2;
    const int64_t a0 = P.apos[i];
    const int na = (int)(P.apos[i + 1] - a0);
    const SlotMap sm = row_slot_map(P, i, tb);
    for (int s = threadIdx.x; s < nslots; s += THREADS) {
      S.keys[s] = kEmpty;
      if (P.values) S.vals[s] = 0.0;
    }
    cta_sync<THREADS>();
    if (P.values) {
      for_products<true>(P, a0, na, total, [&](int64_t col, double v) {
        bool made;
        const int s = hash_insert(S.keys, (uint32_t)(col - sm.c0), sm(col), made);
        atomicAdd(&S.vals[s], v);
      });
    } else {
      for_products<false>(P, a0, na, total, [&](int64_t col, double) {
        bool made;
        hash_insert(S.keys, (uint32_t)(col - sm.c0), sm(col), made);
      });
    }
    cta_sync<THREADS>();
    // rank the runs (mutually ordered) and write the row in column order
    drain_table<THREADS>(S.keys, P.values ? S.vals : nullptr, nslots, sm.c0, P.cidx + dst,
                         P.cvals + dst, S.scan, P.sorted);
    rc.publish();
    cta_sync<THREADS>();
  }
}

// ---------------------------------------------------------------------------
// Numeric pass of the hash tiers by bucketed counting sort.  The hash tables
// above are at most half full and followed by an overflow region, so their
// sorted drain walks ~4.3 slots per product (~45 % of the numeric kernels'
// instructions); the exact row length is known from the symbolic pass, so the
// numeric pass does not need a table at all:
//   * every thread keeps its (at most PER) products in registers;
//   * a product's bucket is its column scaled into ~total/4 order-preserving
//     buckets (the hash tiers' slot map); an atomic per product counts the
//     bucket and gives the product its place in it;
//   * a block scan turns counts into bases, the products are staged bucket
//     by bucket in shared memory (work proportional to the products, not to a
//     table);
//   * inside a bucket (4 entries on average) an entry is the representative
//     of its column if no earlier entry holds it; representatives are ranked
//     among their bucket's representatives, add their duplicates' values in
//     stage order, and go to their final position through a second staging
//     buffer, so the row leaves in coalesced stores.
// A row with a bucket of more than kBucketMax entries (clustered columns: the
// in-bucket work is quadratic) is listed for the hash kernel.
constexpr int kBucketMax = 48;

template <int THREADS, int PER>
struct BucketSmem {
  int cnt[THREADS + 1];   // entries per bucket, then exclusive bases (cnt[nb] = total)
  int ucnt[THREADS + 1];  // representatives per bucket, then exclusive bases
  uint32_t col[THREADS * PER];
  double val[THREADS * PER];
  uint32_t ocol[THREADS * PER];
  double oval[THREADS * PER];
  unsigned char rep[THREADS * PER];
  int scan[33];
  int64_t claimed;
};

template <int THREADS>
__device__ __forceinline__ int cta_exclusive_scan(int v, int* sh) {
  if constexpr (THREADS == 32) {
    return warp_inclusive_scan(v) - v;
  } else {
    return block_exclusive_scan(v, sh, nullptr);
  }
}

template <int THREADS, int PER>
__global__ void __launch_bounds__(THREADS, (THREADS == 1024 ? 1 : THREADS == 32 ? 32 : 1536 / THREADS))
    bucket_numeric_kernel(const SpgemmParams P, const int64_t* rows, int64_t nrows, unsigned long long* claim,
                          unsigned long long* fb_count, int64_t* fb_rows) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using Smem = BucketSmem<THREADS, PER>;
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  constexpr int kWarpsN = THREADS / 32;
  RowClaims<THREADS> rc(claim, &S.claimed);
  while (true) {
    const int64_t r = rc.next();
    if (r >= nrows) break;
    const int64_t i = rows[r];
    const int64_t dst = P.cpos[i];
    const int total = (int)P.prod[i];
    const int64_t a0 = P.apos[i];
    const int na = (int)(P.apos[i + 1] - a0);
    // ~total/4 buckets, a power of two, at most one per thread
    int nb = total <= 4 ? 1 : (1 << (32 - __clz(total - 1))) >> 2;
    nb = min(nb, THREADS);
    const SlotMap sm = row_slot_map(P, i, nb);
    if (tid < nb) {
      S.cnt[tid] = 0;
      S.ucnt[tid] = 0;
    }
    cta_sync<THREADS>();
    // the thread's products (one batch of PER windows per warp covers the row)
    uint32_t col[PER];
    double val[PER];
    bool ok[PER];
    int bk[PER], ix[PER];
    {
      const int per = (total + kWarpsN - 1) / kWarpsN;  // <= 32 * PER
      const int w0 = min(total, warp * per), w1 = min(total, w0 + per);
      int64_t q[PER];
      double av[PER];
#pragma unroll
      for (int u = 0; u < PER; u++) {
        ok[u] = false;
        q[u] = 0;
        av[u] = 0.0;
      }
      if (w0 < w1) {
        const int* aoff = P.aoff + a0;
        int pb = entry_of_warp(aoff, na, w0);
        int ob = aoff[pb];
        if (P.values)
          product_windows<true, PER>(P, a0, na, total, aoff, w0, w1, pb, ob, q, av, ok);
        else
          product_windows<false, PER>(P, a0, na, total, aoff, w0, w1, pb, ob, q, av, ok);
      }
#pragma unroll
      for (int u = 0; u < PER; u++) {
        col[u] = 0;
        val[u] = 0.0;
        if (ok[u]) {
          col[u] = (uint32_t)((int64_t)P.bcol32[q[u]] - sm.c0);
          if (P.values) val[u] = mul_rn(av[u], P.bvals[q[u]]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < PER; u++) {
      bk[u] = 0;
      ix[u] = 0;
      if (ok[u]) {
        bk[u] = min(nb - 1, sm((int64_t)col[u] + sm.c0));
        ix[u] = atomicAdd(&S.cnt[bk[u]], 1);
      }
    }
    cta_sync<THREADS>();
    const int mine = tid < nb ? S.cnt[tid] : 0;
    bool big;
    if constexpr (THREADS == 32) {
      big = __any_sync(kFull, mine > kBucketMax);
    } else {
      big = __syncthreads_or(mine > kBucketMax ? 1 : 0) != 0;
    }
    if (big) {
      // clustered columns: the hash kernel takes the row
      if (tid == 0) fb_rows[atomicAdd(fb_count, 1ull)] = i;
      rc.publish();
      cta_sync<THREADS>();
      continue;
    }
    {
      const int excl = cta_exclusive_scan<THREADS>(mine, S.scan);
      cta_sync<THREADS>();
      if (tid < nb) S.cnt[tid] = excl;
      if (tid == 0) S.cnt[nb] = total;
      cta_sync<THREADS>();
    }
#pragma unroll
    for (int u = 0; u < PER; u++)
      if (ok[u]) {
        const int at = S.cnt[bk[u]] + ix[u];
        S.col[at] = col[u];
        S.val[at] = val[u];
      }
    cta_sync<THREADS>();
    // representatives: the first entry of its column in the bucket's stage order
    bool rp[PER];
#pragma unroll
    for (int u = 0; u < PER; u++) {
      rp[u] = false;
      if (ok[u]) {
        const int lo = S.cnt[bk[u]], me = lo + ix[u];
        bool first = true;
        for (int t = lo; t < me; t++) first &= S.col[t] != col[u];
        rp[u] = first;
        S.rep[me] = first ? 1 : 0;
        if (first) atomicAdd(&S.ucnt[bk[u]], 1);
      }
    }
    cta_sync<THREADS>();
    {
      const int umine = tid < nb ? S.ucnt[tid] : 0;
      const int uex = cta_exclusive_scan<THREADS>(umine, S.scan);
      cta_sync<THREADS>();
      if (tid < nb) S.ucnt[tid] = uex;
      if (tid == nb - 1) S.ucnt[nb] = uex + umine;  // the row's length
      cta_sync<THREADS>();
    }
    // final position: the bucket's base + the rank among its representatives
#pragma unroll
    for (int u = 0; u < PER; u++)
      if (ok[u] && rp[u]) {
        const int lo = S.cnt[bk[u]], hi = S.cnt[bk[u] + 1], me = lo + ix[u];
        int rank = 0;
        double sum = add_rn(0.0, val[u]);  // the workspace's first insert accumulates into 0.0
        for (int t = lo; t < hi; t++) {
          const uint32_t c2 = S.col[t];
          rank += (S.rep[t] && c2 < col[u]) ? 1 : 0;
          if (t > me && c2 == col[u]) sum = add_rn(sum, S.val[t]);
        }
        const int out = S.ucnt[bk[u]] + rank;
        S.ocol[out] = col[u];
        S.oval[out] = sum;
      }
    cta_sync<THREADS>();
    const int len = S.ucnt[nb];
    for (int t = tid; t < len; t += THREADS) {
      P.cidx[dst + t] = sm.c0 + (int64_t)S.ocol[t];
      if (P.values) P.cvals[dst + t] = S.oval[t];
    }
    rc.publish();
    cta_sync<THREADS>();
  }
}

// ---------------------------------------------------------------------------
// Long rows: a bitmap over all n columns in shared memory (64-bit words), and
// for the numeric pass an exclusive popcount prefix per word.
struct LongHeader {
  int scan[33];
  int64_t claimed;
};

__host__ __device__ inline size_t long_header() { return (sizeof(LongHeader) + 15) & ~(size_t)15; }


__device__ __forceinline__ void set_bit(unsigned long long* bits, int64_t col) {
  atomicOr(&bits[col >> 6], 1ull << (col & 63));
}

// Long rows in one pass, before the row-pointer scan: the row's column
// bitmap, an exclusive popcount prefix per word, the sorted column list and
// the values (fp64 atomics at each product's popcount slot) go to a scratch
// region at the row's products offset (an upper bound of its output), and
// the exact count to cpos[i+1].  After the scan long_copy_kernel moves the
// rows into C.  (Replaces a symbolic bitmap pass + a numeric bitmap pass:
// the products are enumerated twice instead of three times.)
//
// Matrices wider than the shared-memory bitmap (win_words 64-bit words,
// ~1.2M columns) are processed in column windows of win_words * 64 columns,
// in column order, each window enumerating the row's products again and
// keeping those that fall inside it.
__global__ void __launch_bounds__(kLongThreads) long_numeric_kernel(const SpgemmParams P,
                                                                    const int64_t* rows,
                                                                    int64_t nrows,
                                                                    unsigned long long* claim,
                                                                    const int64_t* soff,
                                                                    uint32_t* sidx,
                                                                    double* sval,
                                                                    int win_words) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LongHeader& S = *reinterpret_cast<LongHeader*>(smem_raw);
  auto* bits = reinterpret_cast<unsigned long long*>(smem_raw + long_header());
  const int64_t nw_all = (P.n + 63) >> 6;
  int* wpre = reinterpret_cast<int*>(bits + win_words);
  RowClaims<kLongThreads> rc(claim, &S.claimed);
  while (true) {
    const int64_t r = rc.next();
    if (r >= nrows) break;
    const int64_t i = rows[r];
    const int64_t a0 = P.apos[i];
    const int na = (int)(P.apos[i + 1] - a0);
    const int total = (int)P.prod[i];
    int64_t dst = soff[r];
    int64_t row_cnt = 0;
    for (int64_t wbase = 0; wbase < nw_all; wbase += win_words) {
      const int nw = (int)min((int64_t)win_words, nw_all - wbase);
      const int64_t c0 = wbase * 64, c1 = (wbase + nw) * 64;  // the window's columns
      const bool whole = wbase == 0 && nw == nw_all;
      for (int w = threadIdx.x; w < nw; w += blockDim.x) bits[w] = 0ull;
      __syncthreads();
      for_products<false>(P, a0, na, total, [&](int64_t col, double) {
        if (whole || (col >= c0 && col < c1)) set_bit(bits, col - c0);
      });
      __syncthreads();
      // exclusive popcount prefix per word and the sorted column list: warp w
      // owns words [w*per_w, (w+1)*per_w), lane-interleaved in 32-word chunks
      int cnt;
      {
        const int lane = (int)lane_id();
        const int warp = threadIdx.x >> 5;
        const int per_w = (nw + 31) / 32;
        const int ww0 = min(nw, warp * per_w), ww1 = min(nw, ww0 + per_w);
        int mine = 0;
        for (int w = ww0 + lane; w < ww1; w += 32) mine += __popcll(bits[w]);
        mine = warp_sum(mine);
        if (lane == 0) S.scan[warp] = mine;
        __syncthreads();
        if (warp == 0) {
          const int v = S.scan[lane];
          const int inc = warp_inclusive_scan(v);
          S.scan[lane] = inc - v;
          if (lane == 31) S.scan[32] = inc;
        }
        __syncthreads();
        cnt = S.scan[32];
        int run = S.scan[warp];
        for (int w = ww0; w < ww1; w += 32) {
          const int wl = w + lane;
          const unsigned long long bm = wl < ww1 ? bits[wl] : 0ull;
          const int c = __popcll(bm);
          const int inc = warp_inclusive_scan(c);
          int pos = run + inc - c;
          if (wl < ww1) wpre[wl] = pos;
          unsigned long long mm = bm;
          while (mm) {
            const int b = __ffsll((long long)mm) - 1;
            sidx[dst + pos] = (uint32_t)(c0 + (int64_t)wl * 64 + b);
            pos++;
            mm &= mm - 1;
          }
          run += __shfl_sync(kFull, inc, 31);
        }
      }
      if (P.values) {
        for (int t = threadIdx.x; t < cnt; t += blockDim.x) sval[dst + t] = 0.0;
        __syncthreads();
        for_products<true>(P, a0, na, total, [&](int64_t col, double v) {
          if (whole || (col >= c0 && col < c1)) {
            const int64_t cc = col - c0;
            const int w = (int)(cc >> 6);
            const int slot = wpre[w] + __popcll(bits[w] & ((1ull << (cc & 63)) - 1ull));
            atomicAdd(&sval[dst + slot], v);
          }
        });
      }
      dst += cnt;
      row_cnt += cnt;
      __syncthreads();  // the window's bitmap and prefix are reused
    }
    if (threadIdx.x == 0) P.cpos[i + 1] = row_cnt;
    rc.publish();
    __syncthreads();
  }
}

// Long rows from their scratch regions into C: CTA per row (rows arrive
// longest first), 4 independent loads in flight per thread.
constexpr int kCopyThreads = 1024;
__global__ void __launch_bounds__(kCopyThreads) long_copy_kernel(const SpgemmParams P,
                                                                 const int64_t* rows,
                                                                 int64_t nrows,
                                                                 const int64_t* soff,
                                                                 const uint32_t* sidx,
                                                                 const double* sval) {
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int64_t i = rows[r];
    const int64_t dst = P.cpos[i], cnt = P.cpos[i + 1] - dst, src = soff[r];
    for (int64_t base = 0; base < cnt; base += 4 * kCopyThreads) {
      uint32_t c[4];
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int64_t t = base + u * kCopyThreads + threadIdx.x;
        c[u] = 0;
        v[u] = 0.0;
        if (t < cnt) {
          c[u] = __ldcs(sidx + src + t);
          if (P.values) v[u] = __ldcs(sval + src + t);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int64_t t = base + u * kCopyThreads + threadIdx.x;
        if (t < cnt) {
          __stcs(reinterpret_cast<long long*>(P.cidx) + dst + t, (long long)c[u]);
          if (P.values) __stcs(P.cvals + dst + t, v[u]);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
template <int THREADS, int TB>
void launch_hash(stamrt::Call& call, const SpgemmParams& P, const int64_t* rows, int64_t n,
                 bool numeric, const char* name, unsigned long long* claim,
                 cudaStream_t st = nullptr) {
  if (n == 0) return;
  if (!st) st = call.stream();
  const size_t smem = numeric ? sizeof(HashSmem<TB>) : sizeof(HashKeysSmem<TB>);
  auto grid_for = [&](auto kern) {
    STAM_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 1;
    STAM_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem));
    return (unsigned)std::min<int64_t>(n, (int64_t)std::max(1, per_sm) * call.ctx()->num_sms);
  };
  if (numeric) {
    const unsigned grid = grid_for(hash_numeric_kernel<THREADS, TB>);
    call.before_launch(name, st);
    hash_numeric_kernel<THREADS, TB><<<grid, THREADS, smem, st>>>(P, rows, n, claim, nullptr);
    call.after_launch(st);
  } else {
    const unsigned grid = grid_for(hash_symbolic_kernel<THREADS, TB>);
    call.before_launch(name, st);
    hash_symbolic_kernel<THREADS, TB><<<grid, THREADS, smem, st>>>(P, rows, n, claim);
    call.after_launch(st);
  }
}

// Numeric pass of a hash tier: the bucket kernel, then the hash kernel over
// the rows it listed (clustered columns; the list length stays on the device).
// ctl: [0] bucket claims, [1] listed rows, [2] hash claims.
template <int THREADS, int TB, int PER>
void launch_bucket(stamrt::Call& call, const SpgemmParams& P, const int64_t* rows, int64_t n,
                   const char* name, unsigned long long* ctl, int64_t* fb_rows, cudaStream_t st = nullptr) {
  if (n == 0) return;
  if (!st) st = call.stream();
  const int sms = call.ctx()->num_sms;
  {
    using Smem = BucketSmem<THREADS, PER>;
    auto kern = bucket_numeric_kernel<THREADS, PER>;
    const size_t smem = sizeof(Smem);
    STAM_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 1;
    STAM_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem));
    const int64_t grid = std::min<int64_t>(n, (int64_t)std::max(1, per_sm) * sms);
    call.before_launch(name, st);
    kern<<<(unsigned)grid, THREADS, smem, st>>>(P, rows, n, ctl, ctl + 1, fb_rows);
    call.after_launch(st);
  }
  {
    const size_t smem = sizeof(HashSmem<TB>);
    auto kern = hash_numeric_kernel<THREADS, TB>;
    STAM_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 1;
    STAM_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem));
    const int64_t grid = std::min<int64_t>(n, (int64_t)std::max(1, per_sm) * sms);
    call.before_launch("spgemm_hash_clustered", st);
    kern<<<(unsigned)grid, THREADS, smem, st>>>(P, fb_rows, 0, ctl + 2, ctl + 1);
    call.after_launch(st);
  }
}

// Long rows: scratch offsets (products prefix over the long rows), the
// one-pass kernel into scratch (before the scan) — returns the scratch.
__global__ void gather_prod_kernel(const int64_t* rows, int64_t n, const int64_t* prod,
                                   int64_t* out);

struct LongScratch {
  int64_t* soff = nullptr;
  uint32_t* sidx = nullptr;
  double* sval = nullptr;
};

LongScratch launch_long(stamrt::Call& call, const SpgemmParams& P, const int64_t* rows, int64_t n,
                        unsigned long long* claim) {
  LongScratch L;
  if (n == 0) return L;
  L.soff = call.scratch_n<int64_t>((size_t)n + 1);
  call.before_launch("spgemm_long_offsets");
  gather_prod_kernel<<<(unsigned)stamrt::ceil_div(n, 256), 256, 0, call.stream()>>>(rows, n, P.prod,
                                                                                  L.soff);
  call.after_launch();
  STAM_CUDA_CHECK(cudaMemsetAsync(L.soff + n, 0, sizeof(int64_t), call.stream()));
  size_t sb = 0;
  STAM_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, sb, L.soff, L.soff, n + 1, call.stream()));
  void* stmp = call.scratch(sb);
  STAM_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(stmp, sb, L.soff, L.soff, n + 1, call.stream()));
  const int64_t tot = call.read_scalar(L.soff + n);
  L.sidx = call.scratch_n<uint32_t>((size_t)std::max<int64_t>(tot, 1));
  if (P.values) L.sval = call.scratch_n<double>((size_t)std::max<int64_t>(tot, 1));
  // bitmap + word prefix of one column window in shared memory (12 bytes per
  // 64 columns): the whole row when B is narrow enough, else windows
  const int64_t nw_all = (P.n + 63) / 64;
  const int64_t max_words = ((int64_t)call.ctx()->smem_optin - (int64_t)long_header()) / 12 / 32 * 32;
  const int win_words = (int)std::min<int64_t>(nw_all, max_words);
  const size_t smem = long_header() + (size_t)win_words * 12;
  STAM_CUDA_CHECK(cudaFuncSetAttribute(long_numeric_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t grid = std::min<int64_t>(n, call.ctx()->num_sms);
  call.before_launch("spgemm_long_numeric");
  long_numeric_kernel<<<(unsigned)grid, kLongThreads, smem, call.stream()>>>(
      P, rows, n, claim, L.soff, L.sidx, L.sval, win_words);
  call.after_launch();
  return L;
}

// The copy is bandwidth-bound and the hash numeric tiers are not: it runs on
// the auxiliary stream, overlapped with them (the caller joins before the end).
void launch_long_copy(stamrt::Call& call, const SpgemmParams& P, const int64_t* rows, int64_t n,
                      const LongScratch& L, cudaStream_t aux) {
  if (n == 0) return;
  call.before_launch("spgemm_long_copy", aux);
  long_copy_kernel<<<(unsigned)std::min<int64_t>(n, (int64_t)call.ctx()->num_sms * 2), kCopyThreads,
                     0, aux>>>(P, rows, n, L.soff, L.sidx, L.sval);
  call.after_launch(aux);
}

template <int G>
void launch_tiny(stamrt::Call& call, const SpgemmParams& P, const int64_t* rows, int64_t n,
                 bool numeric,
                 cudaStream_t st = nullptr) {
  if (n == 0) return;
  const int64_t threads = n * G;
  const unsigned grid =
      (unsigned)std::min<int64_t>(stamrt::ceil_div(threads, 256), (int64_t)call.ctx()->num_sms * 16);
  if (!st) st = call.stream();
  call.before_launch(numeric ? "spgemm_tiny_numeric" : "spgemm_tiny_symbolic", st);
  if (numeric)
    tiny_numeric_kernel<G><<<grid, 256, 0, st>>>(P, rows, n);
  else
    tiny_symbolic_kernel<G><<<grid, 256, 0, st>>>(P, rows, n);
  call.after_launch(st);
}

// ---------------------------------------------------------------------------
// COMPUTE mode (SPEC run_compute_after_assemble): values of
// A·B written into a pre-assembled index.  A warp per row walks the row's
// products in the canonical order (k ascending, then B-row order), 32 at a
// time; each product locates its column in the assembled row (binary search;
// an unsorted index through a sorted copy and its permutation); lanes that hit
// the same entry are combined in lane order by the lowest of them, so every
// value is the sequential sum ((0 + p1) + p2) + ... of the CPU workspace —
// bit-identical to the reference.  pos/idx are never modified.
__global__ void compute_rows_kernel(const SpgemmParams P, const int64_t* rows, int64_t nrows,
                                    const int64_t* ipos, const int64_t* skey,
                                    const int64_t* perm, unsigned long long* claim, int* missing) {
  const int lane = (int)lane_id();
  while (true) {
    int64_t r = 0;
    if (lane == 0) r = (int64_t)atomicAdd(claim, 1ull);
    r = __shfl_sync(kFull, r, 0);
    if (r >= nrows) break;
    const int64_t i = rows[r];
    const int64_t a0 = P.apos[i];
    const int na = (int)(P.apos[i + 1] - a0);
    const int total = (int)P.prod[i];
    const int64_t c0 = ipos[i], cn = ipos[i + 1] - c0;
    for (int base = 0; base < total; base += 32) {
      const int j = base + lane;
      long long slot = -1;
      double v = 0.0;
      if (j < total) {
        const int p = entry_of(P.aoff + a0, na, j);
        const int64_t q = P.bst[a0 + p] + (j - P.aoff[a0 + p]);
        const int64_t col = P.bidx[q];
        v = mul_rn(P.avals[a0 + p], P.bvals[q]);
        slot = (long long)index_lookup(skey, perm, c0, cn, col);
        if (slot < 0) atomicOr(missing, 1);
      }
      const unsigned act = __ballot_sync(kFull, slot >= 0);
      const unsigned peers = __match_any_sync(kFull, slot) & act;
      const bool leader = slot >= 0 && __ffs(peers) - 1 == lane;
      double w = leader ? P.cvals[slot] : 0.0;
      for (int t = 0; t < 32; t++) {
        const double vt = __shfl_sync(kFull, v, t);
        if (leader && ((peers >> t) & 1u)) w = add_rn(w, vt);
      }
      if (leader) P.cvals[slot] = w;
      __syncwarp();
    }
  }
}

// COMPUTE mode, rows with many products (one warp per row would serialise a
// row's 10^4-10^5 products): every product is expanded in canonical order
// into (entry, value) pairs at its flat position (CTA per row, no ordering
// needed), a stable radix sort by entry keeps canonical order inside each
// entry's run, and each run is summed sequentially — the same ((0 + p1) + p2)
// + ... as the CPU workspace.
__global__ void compute_expand_kernel(const SpgemmParams P, const int64_t* rows, int64_t nrows,
                                      const int64_t* poff, const int64_t* ipos,
                                      const int64_t* skey, const int64_t* perm,
                                      unsigned long long* keys, double* vals, int* missing) {
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int64_t i = rows[r];
    const int64_t a0 = P.apos[i];
    const int na = (int)(P.apos[i + 1] - a0);
    const int total = (int)P.prod[i];
    const int64_t c0 = ipos[i], cn = ipos[i + 1] - c0;
    const int64_t o = poff[r];
    for (int j = threadIdx.x; j < total; j += blockDim.x) {
      const int p = entry_of(P.aoff + a0, na, j);
      const int64_t q = P.bst[a0 + p] + (j - P.aoff[a0 + p]);
      const int64_t col = P.bidx[q];
      const int64_t e = index_lookup(skey, perm, c0, cn, col);
      if (e < 0) atomicOr(missing, 1);
      keys[o + j] = e < 0 ? 0ull : (unsigned long long)e;
      vals[o + j] = mul_rn(P.avals[a0 + p], P.bvals[q]);
    }
  }
}

__global__ void compute_reduce_runs_kernel(const unsigned long long* keys, const double* vals,
                                           int64_t n, double* out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[t];
    if (t > 0 && keys[t - 1] == k) continue;
    double w = add_rn(0.0, vals[t]);  // first insert accumulates into 0.0
    for (int64_t u = t + 1; u < n && keys[u] == k; u++) w = add_rn(w, vals[u]);
    out[k] = w;
  }
}

__global__ void gather_prod_kernel(const int64_t* rows, int64_t n, const int64_t* prod,
                                   int64_t* out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) out[t] = prod[rows[t]];
}

// Orders the long rows longest first (greedy LPT over the dynamic claims).
__global__ void gather_keys_kernel(const int64_t* rows, int64_t n, const int64_t* prod,
                                   uint64_t* keys) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) keys[t] = (uint64_t)prod[rows[t]];
}

// pos[i] - base for a row block (the block's own CSR view) and pos[i] + off
// for a block result placed after the earlier blocks' entries.
__global__ void pos_shift_kernel(const int64_t* in, int64_t* out, int64_t n, int64_t delta) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    out[t] = in[t] + delta;
}

// ---------------------------------------------------------------------------
// Narrow B (n <= kNarrowCols columns) with short rows (P_i <= pmax): one fused
// pass, no symbolic kernel, no bins, no scan.  A warp per row of a tile of
// kNarrowRows consecutive rows: the row's products set bits in a column bitmap
// of n bits in shared memory (the whole column space: no hashing, the column
// order is the bit order), a popcount prefix over the words gives every
// column its slot in the row, the products' values are added at their slots
// (shared fp64 atomics; first insert into 0.0 as the workspace does), and the
// tile learns its output offset by decoupled look-back (tiles are claimed in
// row order) and writes its rows straight into C, which is allocated at the
// products bound.  Config 1 (10k x 10k, 400 products per row) runs as one
// kernel plus a products reduction.
constexpr int kNarrowCols = 16384;
constexpr int kNarrowRows = 8;  // warps (rows) per CTA tile
constexpr int kNarrowMaxP = 1024;

__global__ void narrow_products_kernel(const SpgemmParams P, unsigned long long* out) {
  // out[0] += products, out[1] = max products of a row (a warp per row; one
  // pair of atomics per CTA)
  __shared__ unsigned long long s_tot[32], s_max[32];
  const unsigned lane = lane_id();
  const int wib = threadIdx.x >> 5;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long tot = 0, mx = 0;
  for (int64_t i = warp; i < P.m; i += nwarps) {
    const int64_t a0 = P.apos[i], a1 = P.apos[i + 1];
    unsigned long long s = 0;
    for (int64_t p = a0 + lane; p < a1; p += 32) {
      const int64_t k = P.aidx[p];
      s += (unsigned long long)(P.bpos[k + 1] - P.bpos[k]);
    }
    s = warp_sum(s);
    tot += s;
    mx = max(mx, s);
  }
  if (lane == 0) {
    s_tot[wib] = tot;
    s_max[wib] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0, m = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
      t += s_tot[w];
      m = max(m, s_max[w]);
    }
    if (t) atomicAdd(&out[0], t);
    atomicMax(&out[1], m);
  }
}

// Enumerates the row's products entry by entry (the warp walks the A entries,
// lanes cover each entry's B row: coalesced reads of the B row, no product ->
// entry search), two entries per step so two gathers are in flight per lane.
// f(col, value) sees every product once; kNumeric false skips the values.
template <bool kNumeric, typename F>
__device__ __forceinline__ void narrow_products(const SpgemmParams& P, int64_t a0, int64_t a1,
                                                F f) {
  const int lane = (int)lane_id();
  for (int64_t c = a0; c < a1; c += 32) {
    const int64_t p = c + lane;
    int64_t b0 = 0;
    int len = 0;
    double av = 0.0;
    if (p < a1) {
      const int64_t k = P.aidx[p];
      b0 = P.bpos[k];
      len = (int)(P.bpos[k + 1] - b0);
      if (kNumeric) av = P.avals[p];
    }
    const int nent = (int)min((int64_t)32, a1 - c);
    for (int e = 0; e < nent; e += 2) {
      const int64_t bx = __shfl_sync(kFull, b0, e);
      const int lx = __shfl_sync(kFull, len, e);
      const double ax = kNumeric ? __shfl_sync(kFull, av, e) : 0.0;
      const int e1 = min(e + 1, 31);
      const int64_t by = __shfl_sync(kFull, b0, e1);
      const int ly = e + 1 < nent ? __shfl_sync(kFull, len, e1) : 0;
      const double ay = kNumeric ? __shfl_sync(kFull, av, e1) : 0.0;
      const int lm = max(lx, ly);
      for (int t = lane; t < lm; t += 32) {
        const bool okx = t < lx, oky = t < ly;
        const int64_t cx = okx ? P.bidx[bx + t] : 0;
        const int64_t cy = oky ? P.bidx[by + t] : 0;
        const double vx = (kNumeric && okx) ? P.bvals[bx + t] : 0.0;
        const double vy = (kNumeric && oky) ? P.bvals[by + t] : 0.0;
        if (okx) f(cx, kNumeric ? mul_rn(ax, vx) : 0.0);
        if (oky) f(cy, kNumeric ? mul_rn(ay, vy) : 0.0);
      }
    }
  }
}

__global__ void __launch_bounds__(kNarrowRows * 32) spgemm_narrow_kernel(
    const SpgemmParams P, int nwords, int pmax, uint64_t* status, unsigned long long* claim) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int counts[kNarrowRows];
  __shared__ int64_t tile_sh, prefix_sh;
  const int lane = (int)lane_id();
  const int warp = threadIdx.x >> 5;
  const size_t per_warp = ((size_t)nwords * 12 + (size_t)pmax * 8 + 15) & ~(size_t)15;
  unsigned char* mine = smem_raw + per_warp * warp;
  double* vals = reinterpret_cast<double*>(mine);
  unsigned long long* bits = reinterpret_cast<unsigned long long*>(mine + (size_t)pmax * 8);
  int* wpre = reinterpret_cast<int*>(bits + nwords);
  for (int w = lane; w < nwords; w += 32) bits[w] = 0ull;
  const int64_t ntiles = (P.m + kNarrowRows - 1) / kNarrowRows;
  while (true) {
    if (threadIdx.x == 0) tile_sh = (int64_t)atomicAdd(claim, 1ull);
    __syncthreads();
    const int64_t tile = tile_sh;
    if (tile >= ntiles) break;
    const int64_t i = tile * kNarrowRows + warp;
    int count = 0;
    if (i < P.m) {
      const int64_t a0 = P.apos[i], a1 = P.apos[i + 1];
      narrow_products<false>(P, a0, a1, [&](int64_t col, double) {
        atomicOr(&bits[col >> 6], 1ull << (col & 63));
      });
      __syncwarp();
      int run = 0;
      for (int w0 = 0; w0 < nwords; w0 += 32) {
        const int w = w0 + lane;
        const int c = w < nwords ? __popcll(bits[w]) : 0;
        const int inc = warp_inclusive_scan(c);
        if (w < nwords) wpre[w] = run + inc - c;
        run += __shfl_sync(kFull, inc, 31);
      }
      count = run;
      if (P.values) {
        for (int t = lane; t < count; t += 32) vals[t] = 0.0;
        __syncwarp();
        narrow_products<true>(P, a0, a1, [&](int64_t col, double v) {
          const int w = (int)(col >> 6);
          const int slot = wpre[w] + __popcll(bits[w] & ((1ull << (col & 63)) - 1ull));
          atomicAdd(&vals[slot], v);
        });
      }
    }
    if (lane == 0) counts[warp] = count;
    __syncthreads();
    if (warp == 0) {
      const int c = lane < kNarrowRows ? counts[lane] : 0;
      const int64_t agg = warp_sum((int64_t)c);
      const int64_t ex = lookback_exclusive(status, tile, agg);
      if (lane == 0) prefix_sh = ex;
    }
    __syncthreads();
    if (i < P.m) {
      int64_t off = prefix_sh;
      for (int w = 0; w < warp; w++) off += counts[w];
      if (lane == 0) {
        P.cpos[i] = off;
        if (i == P.m - 1) P.cpos[P.m] = off + count;
      }
      // columns: a lane per bitmap word (its bits in order), values coalesced
      for (int w = lane; w < nwords; w += 32) {
        unsigned long long b = bits[w];
        int pos = wpre[w];
        while (b) {
          const int bit = __ffsll((long long)b) - 1;
          P.cidx[off + pos] = (int64_t)w * 64 + bit;
          pos++;
          b &= b - 1;
        }
        bits[w] = 0ull;  // ready for the next row
      }
      if (P.values)
        for (int t = lane; t < count; t += 32) P.cvals[off + t] = vals[t];
    }
    __syncthreads();
  }
}

}  // namespace
}  // namespace stamgpu

using namespace stamrt;

namespace stamgpu {
namespace {
// Inputs on the device, per-row products / per-entry offsets (rowprod), and
// the control block read back: host[0..kNumBins) bin counts, host[kNumBins]
// total products, host[kNumBins+1] max products of a row.
void prepare(stamrt::Call& call, const stam_csr_view* A, const stam_csr_view* B,
             SpgemmParams& P, int64_t* host) {
  using stamrt::ceil_div;
  const int64_t m = A->nrows, n = B->ncols;
  P = SpgemmParams{};
  P.m = m;
  P.n = n;
  P.apos = call.device_input(A->pos, (size_t)m + 1, A->mem);
  P.aidx = call.device_input(A->idx, (size_t)A->nnz, A->mem);
  P.avals = call.device_input(A->vals, (size_t)A->nnz, A->mem);
  P.bpos = call.device_input(B->pos, (size_t)B->nrows + 1, B->mem);
  P.bidx = call.device_input(B->idx, (size_t)B->nnz, B->mem);
  P.bvals = call.device_input(B->vals, (size_t)B->nnz, B->mem);
  P.prod = call.scratch_n<int64_t>((size_t)m);
  P.span = call.scratch_n<uint2>((size_t)m);
  P.aoff = call.scratch_n<int>((size_t)std::max<int64_t>(A->nnz, 1));
  P.bst = call.scratch_n<int64_t>((size_t)std::max<int64_t>(A->nnz, 1));
  auto* ctl = static_cast<int64_t*>(call.scratch_zero(sizeof(int64_t) * 16));
  P.bins = reinterpret_cast<unsigned long long*>(ctl);
  P.stats = ctl + kNumBins;
  P.bin_rows = call.scratch_n<int64_t>((size_t)m);
  P.cpos = static_cast<int64_t*>(call.scratch_zero(sizeof(int64_t) * ((size_t)m + 1)));
  P.values = true;
  P.sorted = true;
  P.bspan = call.scratch_n<uint2>((size_t)std::max<int64_t>(B->nrows, 1));
  P.arows = call.scratch_n<int64_t>((size_t)std::max<int64_t>(m, 1));
  P.narows = static_cast<unsigned long long*>(call.scratch_zero(sizeof(unsigned long long) * 2));
  const int sms = call.ctx()->num_sms;
  {
    auto* c32 = call.scratch_n<uint32_t>((size_t)std::max<int64_t>(B->nnz, 1));
    call.before_launch("spgemm_bcol32");
    bcol32_kernel<<<(unsigned)std::min<int64_t>(ceil_div(std::max<int64_t>(B->nnz, 1), 256), (int64_t)sms * 16), 256, 0,
                    call.stream()>>>(P.bidx, B->nnz, c32);
    call.after_launch();
    P.bcol32 = c32;
  }
  call.before_launch("spgemm_bspan");
  bspan_kernel<<<(unsigned)std::min<int64_t>(ceil_div(B->nrows, 256), (int64_t)sms * 8), 256, 0,
                 call.stream()>>>(P, B->nrows);
  call.after_launch();
  call.before_launch("spgemm_rowprod");
  // rows per warp window: 32, or fewer when that leaves the GPU underfilled
  int rw = 32;
  while (rw > 4 && ceil_div(m, (int64_t)rw) < (int64_t)sms * 32) rw >>= 1;
  rowprod_kernel<<<(unsigned)std::min<int64_t>(ceil_div(ceil_div(m, (int64_t)rw), 8), (int64_t)sms * 8),
                   256, 0, call.stream()>>>(P, rw);
  call.after_launch();
  call.before_launch("spgemm_rowprod_long");
  rowprod_long_kernel<<<(unsigned)(sms * 2), 256, 0, call.stream()>>>(P);
  call.after_launch();
  static_assert(kNumBins + 2 <= 16, "control block");
  call.read_scalars(ctl, 16, host);
  if (host[kNumBins + 1] >= (int64_t)INT32_MAX)
    stamrt::fail(STAM_ERR_UNSUPPORTED_MERGE, "spgemm: a row has 2^31 or more products");
}

// Groups the rows by bin (P.bin_rows, bin b at offsets[b]; empty rows left out).
void bin_rows(stamrt::Call& call, SpgemmParams& P, const int64_t* host,
              unsigned long long* counts, unsigned long long* offsets) {
  unsigned long long acc = 0;
  for (int b = 0; b < kNumBins; b++) {
    counts[b] = (unsigned long long)host[b];
    offsets[b] = acc;
    if (b != kBinEmpty) acc += counts[b];
  }
  auto* d_off = static_cast<unsigned long long*>(call.scratch(sizeof(unsigned long long) * kNumBins));
  STAM_CUDA_CHECK(cudaMemcpyAsync(d_off, offsets, sizeof(unsigned long long) * kNumBins,
                                  cudaMemcpyHostToDevice, call.stream()));
  STAM_CUDA_CHECK(cudaMemsetAsync(P.bins, 0, sizeof(unsigned long long) * kNumBins, call.stream()));
  call.before_launch("spgemm_bin_scatter");
  bin_scatter_kernel<<<(unsigned)stamrt::ceil_div(P.m, 256), 256, 0, call.stream()>>>(P, d_off);
  call.after_launch();
}
}  // namespace
}  // namespace stamgpu

namespace stamgpu {
namespace {
// Narrow path (spgemm_narrow_kernel): returns false (nothing launched that
// matters) when a row has more than kNarrowMaxP products.
bool spgemm_narrow(stamrt::Call& call, const stam_csr_view* A, const stam_csr_view* B,
                   stam_csr_result* Cr) {
  using stamrt::ceil_div;
  const int64_t m = A->nrows, n = B->ncols;
  SpgemmParams P{};
  P.m = m;
  P.n = n;
  P.apos = call.device_input(A->pos, (size_t)m + 1, A->mem);
  P.aidx = call.device_input(A->idx, (size_t)A->nnz, A->mem);
  P.avals = call.device_input(A->vals, (size_t)A->nnz, A->mem);
  P.bpos = call.device_input(B->pos, (size_t)B->nrows + 1, B->mem);
  P.bidx = call.device_input(B->idx, (size_t)B->nnz, B->mem);
  P.bvals = call.device_input(B->vals, (size_t)B->nnz, B->mem);
  const int sms = call.ctx()->num_sms;
  const int64_t ntiles = ceil_div(m, (int64_t)kNarrowRows);
  // control block: [0] products, [1] max products, [2] tile claims, then tile status
  auto* ctl = static_cast<unsigned long long*>(
      call.scratch_zero(sizeof(unsigned long long) * (size_t)(4 + ntiles)));
  call.before_launch("spgemm_narrow_products");
  narrow_products_kernel<<<(unsigned)std::min<int64_t>(ceil_div(m, 8), (int64_t)sms * 2), 256, 0,
                           call.stream()>>>(P, ctl);
  call.after_launch();
  int64_t hv[2];
  call.read_scalars(reinterpret_cast<const int64_t*>(ctl), 2, hv);
  const int64_t products = hv[0], pmax_row = hv[1];
  if (pmax_row > kNarrowMaxP) return false;
  const int nwords = (int)ceil_div(n, (int64_t)64);
  const int pmax = (int)std::max<int64_t>(32, (pmax_row + 31) / 32 * 32);
  const size_t smem = (((size_t)nwords * 12 + (size_t)pmax * 8 + 15) & ~(size_t)15) * kNarrowRows;
  if (smem > call.ctx()->smem_optin) return false;
  P.values = call.opts().mode == STAM_MODE_FUSED;
  P.sorted = true;
  call.alloc_csr_result(Cr, m, n, products);
  P.cpos = Cr->pos;
  P.cidx = Cr->idx;
  P.cvals = Cr->vals;
  if (!P.values && products > 0)  // ASSEMBLE: index only, values defined as zero
    STAM_CUDA_CHECK(cudaMemsetAsync(Cr->vals, 0, sizeof(double) * (size_t)products, call.stream()));
  if (m == 0) STAM_CUDA_CHECK(cudaMemsetAsync(Cr->pos, 0, sizeof(int64_t), call.stream()));
  STAM_CUDA_CHECK(cudaFuncSetAttribute(spgemm_narrow_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 1;
  STAM_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, spgemm_narrow_kernel,
                                                                kNarrowRows * 32, smem));
  const int64_t grid = std::min<int64_t>(ntiles, (int64_t)std::max(1, per_sm) * sms);
  call.before_launch("spgemm_narrow");
  spgemm_narrow_kernel<<<(unsigned)grid, kNarrowRows * 32, smem, call.stream()>>>(
      P, nwords, pmax, reinterpret_cast<uint64_t*>(ctl + 4), ctl + 2);
  call.after_launch();
  const int64_t nnz = call.read_scalar(Cr->pos + m);
  call.finish_csr_result(Cr, nnz);
  call.finish();
  stam_stats* st = call.stats();
  st->mults = products;
  st->adds = products;
  st->ws_inserts = products;
  st->ws_resets = m;
  st->appends = nnz;
  return true;
}
}  // namespace
}  // namespace stamgpu

namespace stamgpu {
namespace {
// Host result of a large product: row blocks, each computed by the device
// pipeline into a device result whose rows go down to the pinned host result
// on the d2h stream while the next block computes (the result is ~16x the
// inputs at config 3: the PCIe download, not the kernels, bounds the call).
// Inputs are staged once; block b's pos is rebased on the device.
int spgemm_streamed(stam_cuda_ctx* ctx, const stam_csr_view* A, const stam_csr_view* B,
                    const stam_options* opts, stam_csr_result* Cr, stam_stats* stats) {
  using stamrt::ceil_div;
  return guarded([&] {
    stam_options o = *opts;
    o.result_mem = STAM_MEM_DEVICE;
    o.timing = 0;
    Call call(reinterpret_cast<Ctx*>(ctx), &o, stats);
    const int64_t m = A->nrows, n = B->ncols;
    SpgemmParams P{};
    P.m = m;
    P.apos = call.device_input(A->pos, (size_t)m + 1, A->mem);
    P.aidx = call.device_input(A->idx, (size_t)A->nnz, A->mem);
    P.avals = call.device_input(A->vals, (size_t)A->nnz, A->mem);
    const bool same = B->pos == A->pos && B->idx == A->idx && B->vals == A->vals;
    P.bpos = same ? P.apos : call.device_input(B->pos, (size_t)B->nrows + 1, B->mem);
    P.bidx = same ? P.aidx : call.device_input(B->idx, (size_t)B->nnz, B->mem);
    P.bvals = same ? P.avals : call.device_input(B->vals, (size_t)B->nnz, B->mem);
    const int sms = call.ctx()->num_sms;
    auto* ctl = static_cast<unsigned long long*>(call.scratch_zero(sizeof(unsigned long long) * 2));
    call.before_launch("spgemm_narrow_products");
    narrow_products_kernel<<<(unsigned)std::min<int64_t>(ceil_div(m, 8), (int64_t)sms * 8), 256, 0,
                             call.stream()>>>(P, ctl);
    call.after_launch();
    int64_t hv[2];
    call.read_scalars(reinterpret_cast<const int64_t*>(ctl), 2, hv);
    const int64_t products = hv[0];
    int64_t nblocks = 8;
    if (const char* e = std::getenv("STAM_SPGEMM_BLOCKS")) nblocks = std::max(1, std::atoi(e));
    nblocks = std::max<int64_t>(1, std::min<int64_t>(nblocks, m));
    std::vector<int64_t> rb((size_t)nblocks + 1), eb((size_t)nblocks + 1);
    for (int64_t b = 0; b <= nblocks; b++) rb[(size_t)b] = m * b / nblocks;
    // entry offsets of the block boundaries
    auto* bnd = call.scratch_n<int64_t>((size_t)nblocks + 1);
    for (int64_t b = 0; b <= nblocks; b++)
      STAM_CUDA_CHECK(cudaMemcpyAsync(bnd + b, P.apos + rb[(size_t)b], sizeof(int64_t),
                                      cudaMemcpyDeviceToDevice, call.stream()));
    call.read_scalars(bnd, (int)nblocks + 1, eb.data());
    call.alloc_csr_result_host(Cr, m, n, products);
    Cr->pos[0] = 0;
    stam_csr_view Bv{B->nrows, B->ncols, B->nnz, P.bpos, P.bidx, P.bvals, STAM_MEM_DEVICE, 0};
    std::vector<stam_csr_result> parts((size_t)nblocks);
    int64_t off = 0, launches = 0;
    stam_stats acc{};
    int status = STAM_OK;
    for (int64_t b = 0; b < nblocks && status == STAM_OK; b++) {
      const int64_t r0 = rb[(size_t)b], r1 = rb[(size_t)b + 1];
      auto* pb = call.scratch_n<int64_t>((size_t)(r1 - r0) + 1);
      pos_shift_kernel<<<(unsigned)std::min<int64_t>(ceil_div(r1 - r0 + 1, 256), (int64_t)sms * 4), 256, 0,
                         call.stream()>>>(P.apos + r0, pb, r1 - r0 + 1, -eb[(size_t)b]);
      STAM_CUDA_CHECK(cudaGetLastError());
      stam_csr_view Av{r1 - r0, A->ncols, eb[(size_t)b + 1] - eb[(size_t)b], pb,
                       P.aidx + eb[(size_t)b], P.avals + eb[(size_t)b], STAM_MEM_DEVICE, 0};
      stam_stats sb{};
      stam_csr_result& Cb = parts[(size_t)b];
      std::memset(&Cb, 0, sizeof(Cb));
      status = stam_cuda_spgemm(ctx, &Av, &Bv, &o, &Cb, &sb);
      if (status != STAM_OK) break;
      acc.mults += sb.mults;
      acc.ws_inserts += sb.ws_inserts;
      launches += sb.kernel_launches;
      // block rows after the earlier blocks' entries, then down to the host
      pos_shift_kernel<<<(unsigned)std::min<int64_t>(ceil_div(r1 - r0, 256), (int64_t)sms * 4), 256, 0,
                         call.stream()>>>(Cb.pos + 1, Cb.pos + 1, r1 - r0, off);
      STAM_CUDA_CHECK(cudaGetLastError());
      cudaEvent_t ready = call.event();
      STAM_CUDA_CHECK(cudaEventRecord(ready, call.stream()));
      call.d2h_range(Cr->pos + r0 + 1, Cb.pos + 1, sizeof(int64_t) * (size_t)(r1 - r0), ready);
      call.d2h_range(Cr->idx + off, Cb.idx, sizeof(int64_t) * (size_t)Cb.nnz, nullptr);
      call.d2h_range(Cr->vals + off, Cb.vals, sizeof(double) * (size_t)Cb.nnz, nullptr);
      off += Cb.nnz;
    }
    call.finish_csr_result_host(Cr, off);  // joins the downloads
    for (auto& Cb : parts)
      if (Cb.handle) stam_cuda_release(ctx, Cb.handle);
    if (status != STAM_OK) {
      const std::string msg = stam_cuda_last_error();
      fail(status, msg);
    }
    call.finish();
    stam_stats* st = call.stats();
    st->mults = acc.mults;
    st->adds = acc.mults;
    st->ws_inserts = acc.ws_inserts;
    st->ws_resets = m;
    st->appends = off;
    st->kernel_launches += launches;
  });
}
}  // namespace
}  // namespace stamgpu

extern "C" int stam_cuda_spgemm(stam_cuda_ctx* ctx, const stam_csr_view* A, const stam_csr_view* B,
                                const stam_options* opts, stam_csr_result* Cr, stam_stats* stats) {
  using namespace stamgpu;
  // a host result of a large product streams down block by block
  if (ctx && A && B && opts && opts->result_mem == STAM_MEM_HOST && opts->mode == STAM_MODE_FUSED &&
      A->nrows >= 65536 && A->nnz >= ((int64_t)1 << 22) && B->ncols > kNarrowCols &&
      A->ncols == B->nrows && A->nrows > 0 && B->nrows > 0 && B->ncols < (int64_t)UINT32_MAX &&
      std::getenv("STAM_NO_STREAM") == nullptr)
    return spgemm_streamed(ctx, A, B, opts, Cr, stats);
  return guarded([&] {
    Call call(reinterpret_cast<Ctx*>(ctx), opts, stats);
    check_csr_view(A, "spgemm A");
    check_csr_view(B, "spgemm B");
    if (A->ncols != B->nrows) fail(STAM_ERR_DIMENSION_MISMATCH, "spgemm: A columns != B rows");
    if (call.opts().mode == STAM_MODE_COMPUTE)
      fail(STAM_ERR_PRECONDITION_VIOLATED,
           "spgemm compute mode needs the pre-assembled index: use stam_cuda_spgemm_compute");
    if (B->ncols >= (int64_t)UINT32_MAX)
      fail(STAM_ERR_UNSUPPORTED_MERGE, "spgemm: B has 2^32 or more columns");
    const int64_t m = A->nrows, n = B->ncols;
    SpgemmParams P;
    if (n <= kNarrowCols && spgemm_narrow(call, A, B, Cr))
      return;
    int64_t host[16];
    prepare(call, A, B, P, host);
    P.values = call.opts().mode == STAM_MODE_FUSED;
    P.sorted = call.opts().sort != 0;
    const int64_t products = host[kNumBins];
    unsigned long long counts[kNumBins], offsets[kNumBins];
    bin_rows(call, P, host, counts, offsets);

    const int64_t* rows_b[kNumBins];
    for (int b = 0; b < kNumBins; b++) rows_b[b] = P.bin_rows + offsets[b];
    // longest rows first for the long bin
    if (counts[kBinLong] > 1) {
      const int64_t nl = (int64_t)counts[kBinLong];
      auto* keys = call.scratch_n<uint64_t>((size_t)nl * 2);
      auto* rows_sorted = call.scratch_n<int64_t>((size_t)nl);
      call.before_launch("spgemm_long_keys");
      gather_keys_kernel<<<(unsigned)ceil_div(nl, 256), 256, 0, call.stream()>>>(rows_b[kBinLong],
                                                                                 nl, P.prod, keys);
      call.after_launch();
      size_t sort_bytes = 0;
      STAM_CUDA_CHECK(cub::DeviceRadixSort::SortPairsDescending(
          nullptr, sort_bytes, keys, keys + nl, rows_b[kBinLong], rows_sorted, (int)nl, 0, 40,
          call.stream()));
      void* sort_tmp = call.scratch(sort_bytes);
      call.before_launch("spgemm_long_sort");
      STAM_CUDA_CHECK(cub::DeviceRadixSort::SortPairsDescending(
          sort_tmp, sort_bytes, keys, keys + nl, rows_b[kBinLong], rows_sorted, (int)nl, 0, 40,
          call.stream()));
      call.after_launch();
      rows_b[kBinLong] = rows_sorted;
    }
    auto* claims = static_cast<unsigned long long*>(call.scratch_zero(sizeof(unsigned long long) * 16));

    // symbolic: the small-row tiers on the auxiliary stream beside the large
    // ones (independent rows; fills each kernel's tail)
    cudaStream_t aux = call.fork();
    launch_tiny<8>(call, P, rows_b[kBinTiny8], counts[kBinTiny8], false, aux);
    launch_tiny<16>(call, P, rows_b[kBinTiny16], counts[kBinTiny16], false, aux);
    launch_tiny<32>(call, P, rows_b[kBinTiny32], counts[kBinTiny32], false, aux);
    launch_hash<32, 128>(call, P, rows_b[kBinHashXS], counts[kBinHashXS], false, "spgemm_hashXS_symbolic", claims + 0, aux);
    // symbolic tiers at half the numeric tiers' threads per row (keys only:
    // more rows in flight per SM; measured 10.65 -> 10.52 ms on config 3)
    launch_hash<32, 512>(call, P, rows_b[kBinHashS], counts[kBinHashS], false, "spgemm_hashS_symbolic", claims + 1, aux);
    launch_hash<64, 1024>(call, P, rows_b[kBinHashM1], counts[kBinHashM1], false, "spgemm_hashM1_symbolic", claims + 12);
    launch_hash<128, 2048>(call, P, rows_b[kBinHashM], counts[kBinHashM], false, "spgemm_hashM_symbolic", claims + 2);
    launch_hash<256, 4096>(call, P, rows_b[kBinHashL1], counts[kBinHashL1], false, "spgemm_hashL1_symbolic", claims + 10);
    launch_hash<512, 8192>(call, P, rows_b[kBinHashL], counts[kBinHashL], false, "spgemm_hashL_symbolic", claims + 3);
    const LongScratch lsc = launch_long(call, P, rows_b[kBinLong], counts[kBinLong], claims + 4);
    call.join();

    // scan counts -> row pointers
    size_t temp_bytes = 0;
    STAM_CUDA_CHECK(cub::DeviceScan::InclusiveSum(nullptr, temp_bytes, P.cpos + 1, P.cpos + 1, m,
                                                  call.stream()));
    void* temp = call.scratch(temp_bytes);
    call.before_launch("spgemm_scan");
    STAM_CUDA_CHECK(cub::DeviceScan::InclusiveSum(temp, temp_bytes, P.cpos + 1, P.cpos + 1, m,
                                                  call.stream()));
    call.after_launch();
    // Small products: C is allocated at the products count (an upper bound of
    // nnz, known since rowprod) and the exact nnz read once everything is
    // queued — no host round trip between the passes (config 1: 0.286 ->
    // 0.275 ms).  Large: exact allocation after the scan (measured faster on
    // config 3: 10.55 vs 10.86 ms).
    const bool defer_nnz = products <= (int64_t)(64ll << 20);
    const int64_t cap = defer_nnz ? products : call.read_scalar(P.cpos + m);
    call.alloc_csr_result(Cr, m, n, cap);
    STAM_CUDA_CHECK(cudaMemcpyAsync(Cr->pos, P.cpos, sizeof(int64_t) * ((size_t)m + 1),
                                    cudaMemcpyDeviceToDevice, call.stream()));
    P.cidx = Cr->idx;
    P.cvals = Cr->vals;
    if (!P.values && cap > 0)  // ASSEMBLE: index only, values defined as zero
      STAM_CUDA_CHECK(cudaMemsetAsync(Cr->vals, 0, sizeof(double) * (size_t)cap, call.stream()));
    // control words and row lists of the bucketed numeric pass (zeroed on the
    // main stream before the fork: the auxiliary stream's kernels read them)
    auto* bctl = static_cast<unsigned long long*>(call.scratch_zero(sizeof(unsigned long long) * 3 * 6));
    auto* fb = call.scratch_n<int64_t>((size_t)std::max<int64_t>(m, 1));
    // numeric (ASSEMBLE: the same passes without values): the long-row copy
    // and the small-row tiers on the auxiliary stream
    aux = call.fork();
    launch_long_copy(call, P, rows_b[kBinLong], counts[kBinLong], lsc, aux);
    launch_tiny<8>(call, P, rows_b[kBinTiny8], counts[kBinTiny8], true, aux);
    launch_tiny<16>(call, P, rows_b[kBinTiny16], counts[kBinTiny16], true, aux);
    launch_tiny<32>(call, P, rows_b[kBinTiny32], counts[kBinTiny32], true, aux);
    if (std::getenv("STAM_SPGEMM_HASH_NUMERIC") != nullptr || !P.sorted) {
      // the hash tables' numeric pass (unsorted output keeps the workspace's slot order)
      launch_hash<32, 128>(call, P, rows_b[kBinHashXS], counts[kBinHashXS], true, "spgemm_hashXS_numeric", claims + 5, aux);
      launch_hash<64, 512>(call, P, rows_b[kBinHashS], counts[kBinHashS], true, "spgemm_hashS_numeric", claims + 6, aux);
      launch_hash<SPGEMM_M1_NUM_THREADS, 1024>(call, P, rows_b[kBinHashM1], counts[kBinHashM1], true, "spgemm_hashM1_numeric", claims + 13);
      launch_hash<256, 2048>(call, P, rows_b[kBinHashM], counts[kBinHashM], true, "spgemm_hashM_numeric", claims + 7);
      launch_hash<512, 4096>(call, P, rows_b[kBinHashL1], counts[kBinHashL1], true, "spgemm_hashL1_numeric", claims + 11);
      launch_hash<1024, 8192>(call, P, rows_b[kBinHashL], counts[kBinHashL], true, "spgemm_hashL_numeric", claims + 8);
    } else {
      // bucketed counting sort (rows with clustered columns fall back to the hash kernel)
      int64_t fo = 0;
      auto fb_at = [&](int bin) {
        int64_t* q = fb + fo;
        fo += (int64_t)counts[bin];
        return q;
      };
      launch_bucket<32, 128, 2>(call, P, rows_b[kBinHashXS], counts[kBinHashXS], "spgemm_bucketXS_numeric", bctl + 0, fb_at(kBinHashXS), aux);
      launch_bucket<64, 512, 4>(call, P, rows_b[kBinHashS], counts[kBinHashS], "spgemm_bucketS_numeric", bctl + 3, fb_at(kBinHashS), aux);
      launch_bucket<128, 1024, 4>(call, P, rows_b[kBinHashM1], counts[kBinHashM1], "spgemm_bucketM1_numeric", bctl + 6, fb_at(kBinHashM1));
      launch_bucket<256, 2048, 4>(call, P, rows_b[kBinHashM], counts[kBinHashM], "spgemm_bucketM_numeric", bctl + 9, fb_at(kBinHashM));
      #ifndef SPGEMM_BUCKET_L1_THREADS
#define SPGEMM_BUCKET_L1_THREADS 512
#endif
      launch_bucket<SPGEMM_BUCKET_L1_THREADS, 4096, 2048 / SPGEMM_BUCKET_L1_THREADS>(
          call, P, rows_b[kBinHashL1], counts[kBinHashL1], "spgemm_bucketL1_numeric", bctl + 12, fb_at(kBinHashL1));
      #ifndef SPGEMM_BUCKET_L_THREADS
#define SPGEMM_BUCKET_L_THREADS 1024
#endif
      launch_bucket<SPGEMM_BUCKET_L_THREADS, 8192, 4096 / SPGEMM_BUCKET_L_THREADS>(
          call, P, rows_b[kBinHashL], counts[kBinHashL], "spgemm_bucketL_numeric", bctl + 15, fb_at(kBinHashL));
    }
    call.join();
    const int64_t nnz = defer_nnz ? call.read_scalar(P.cpos + m) : cap;

    call.finish_csr_result(Cr, nnz);
    call.finish();
    stam_stats* st = call.stats();
    st->mults = products;
    st->adds = products;
    st->ws_inserts = products;
    st->ws_resets = m;
    st->appends = nnz;
  });
}

extern "C" int stam_cuda_spgemm_compute(stam_cuda_ctx* ctx, const stam_csr_view* A,
                                        const stam_csr_view* B, const stam_csr_view* Cidx,
                                        const stam_options* opts, stam_csr_result* Cr,
                                        stam_stats* stats) {
  using namespace stamgpu;
  return guarded([&] {
    Call call(reinterpret_cast<Ctx*>(ctx), opts, stats);
    check_csr_view(A, "spgemm A");
    check_csr_view(B, "spgemm B");
    if (!Cidx) fail(STAM_ERR_PRECONDITION_VIOLATED, "spgemm compute: null pre-assembled index");
    if (A->ncols != B->nrows) fail(STAM_ERR_DIMENSION_MISMATCH, "spgemm: A columns != B rows");
    if (Cidx->nrows != A->nrows || Cidx->ncols != B->ncols)
      fail(STAM_ERR_DIMENSION_MISMATCH, "spgemm compute: index dimensions != A rows x B columns");
    if (Cidx->nnz < 0 || !Cidx->pos || (Cidx->nnz > 0 && !Cidx->idx))
      fail(STAM_ERR_PRECONDITION_VIOLATED, "spgemm compute: incomplete pre-assembled index");
    const int64_t m = A->nrows, n = B->ncols, nnz = Cidx->nnz;
    SpgemmParams P;
    int64_t host[16];
    prepare(call, A, B, P, host);
    const int64_t products = host[kNumBins];
    const int64_t* ipos = call.device_input(Cidx->pos, (size_t)m + 1, Cidx->mem);
    const int64_t* iidx = call.device_input(Cidx->idx, (size_t)nnz, Cidx->mem);
    call.alloc_csr_result(Cr, m, n, nnz);
    STAM_CUDA_CHECK(cudaMemcpyAsync(Cr->pos, ipos, sizeof(int64_t) * ((size_t)m + 1),
                                    cudaMemcpyDeviceToDevice, call.stream()));
    if (nnz > 0) {
      STAM_CUDA_CHECK(cudaMemcpyAsync(Cr->idx, iidx, sizeof(int64_t) * (size_t)nnz,
                                      cudaMemcpyDeviceToDevice, call.stream()));
      STAM_CUDA_CHECK(cudaMemsetAsync(Cr->vals, 0, sizeof(double) * (size_t)nnz, call.stream()));
    }
    const IndexSearch ix = make_index_search(call, ipos, iidx, m, nnz, call.opts().sort != 0);
    const int64_t* skey = ix.skey;
    const int64_t* perm = ix.perm;
    auto* flags = static_cast<int*>(call.scratch_zero(sizeof(int) * 4));
    auto* claim = reinterpret_cast<unsigned long long*>(flags + 2);
    P.cvals = Cr->vals;
    unsigned long long counts[kNumBins], offsets[kNumBins];
    bin_rows(call, P, host, counts, offsets);
    // rows up to the hash tiers: a warp per row; long rows: expand-sort-reduce
    const int64_t nshort = (int64_t)offsets[kBinLong];
    const int64_t nlong = (int64_t)counts[kBinLong];
    if (nshort > 0) {
      call.before_launch("spgemm_compute_rows");
      compute_rows_kernel<<<(unsigned)(call.ctx()->num_sms * 8), 256, 0, call.stream()>>>(
          P, P.bin_rows, nshort, ipos, skey, perm, claim, flags);
      call.after_launch();
    }
    if (nlong > 0) {
      const int64_t* lrows = P.bin_rows + offsets[kBinLong];
      auto* poff = call.scratch_n<int64_t>((size_t)nlong + 1);
      call.before_launch("spgemm_compute_gather");
      gather_prod_kernel<<<(unsigned)ceil_div(nlong, 256), 256, 0, call.stream()>>>(lrows, nlong,
                                                                                    P.prod, poff);
      call.after_launch();
      size_t sb = 0;
      STAM_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, sb, poff, poff, nlong + 1, call.stream()));
      void* stmp = call.scratch(sb);
      STAM_CUDA_CHECK(cudaMemsetAsync(poff + nlong, 0, sizeof(int64_t), call.stream()));
      call.before_launch("spgemm_compute_scan");
      STAM_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(stmp, sb, poff, poff, nlong + 1, call.stream()));
      call.after_launch();
      const int64_t nexp = call.read_scalar(poff + nlong);
      auto* k0 = call.scratch_n<unsigned long long>((size_t)nexp);
      auto* k1 = call.scratch_n<unsigned long long>((size_t)nexp);
      auto* v0 = call.scratch_n<double>((size_t)nexp);
      auto* v1 = call.scratch_n<double>((size_t)nexp);
      call.before_launch("spgemm_compute_expand");
      compute_expand_kernel<<<(unsigned)std::min<int64_t>(nlong, (int64_t)call.ctx()->num_sms * 4),
                              512, 0, call.stream()>>>(P, lrows, nlong, poff, ipos, skey, perm, k0,
                                                       v0, flags);
      call.after_launch();
      int end_bit = 1;
      while (end_bit < 64 && ((int64_t)1 << end_bit) < nnz) end_bit++;
      cub::DoubleBuffer<unsigned long long> kb(k0, k1);
      cub::DoubleBuffer<double> vb(v0, v1);
      size_t rb = 0;
      STAM_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, rb, kb, vb, nexp, 0, end_bit,
                                                      call.stream()));
      void* rtmp = call.scratch(rb);
      call.before_launch("spgemm_compute_sort");
      STAM_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(rtmp, rb, kb, vb, nexp, 0, end_bit,
                                                      call.stream()));
      call.after_launch();
      call.before_launch("spgemm_compute_reduce");
      compute_reduce_runs_kernel<<<(unsigned)std::min<int64_t>(ceil_div(nexp, 256),
                                                               (int64_t)call.ctx()->num_sms * 16),
                                   256, 0, call.stream()>>>(kb.Current(), vb.Current(), nexp,
                                                            Cr->vals);
      call.after_launch();
    }
    int64_t missing = 0;
    call.read_scalars(reinterpret_cast<const int64_t*>(flags), 1, &missing);
    if ((int)missing != 0)
      fail(STAM_ERR_MISSING_SLOT,
           "spgemm compute: a product's column is missing from the pre-assembled index");
    call.finish_csr_result(Cr, nnz);
    call.finish();
    stam_stats* st = call.stats();
    st->mults = products;
    st->adds = products;
    st->ws_resets = m;
  });
}
