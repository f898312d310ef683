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
//           the whole GPU); a warp walks a chunk's fibers four at a time, a
//           quarter-warp per fiber (R = 32: one row = 8 lanes x 32 B) with its
//           w0 share in registers; at the fiber end w0 * C(j,:) is accumulated
//           into the quarter's share of the slice row.  Slices inside a chunk
//           are stored directly; slices cut by chunk boundaries leave
//           per-chunk partials that block sums and a warp per chain add in a
//           fixed order (deterministic; no atomics on the heavy slices).
//  sparse — three phases whose gathered sets each fit the L2 (see "Three
//           phases" below): a filter streams the CSF through per-warp shared-
//           memory rings filled by TMA bulk copies and ANDs the two factor
//           rows' column bitmaps (a hit record per matching nonzero); an
//           expansion turns hits into match records on full warps and counts
//           each slice's distinct columns; after a scan of the row lengths an
//           accumulation adds w0*C(j,r) into an R-wide shared-memory workspace
//           with a presence bitmap and drains it sorted (ballot/popcount)
//           straight into the CSR.  w0 is evaluated only at C's stored
//           coordinates (presence-checked).  The single-pass kernel (a warp
//           per slice, matches queued per warp) remains for tensors outside
//           the three-phase path's limits and for slices that overflow their
//           record rows.
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

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
  int64_t* chunk_fa;    // [nchunks+1] first fiber starting in chunk c
  int64_t* chunk_s;     // [nchunks+1] slice of chunk_fa[c] (I when none)
  unsigned long long* counter;  // dynamic chunk claims
  double* part;         // [ncb][nchunks][2][32] partials (head, tail)
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

// Chunk c owns the fibers whose first nonzero lies in [c*S, (c+1)*S).
__global__ void mttkrp_dense_bounds_kernel(const DenseParams P) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c > P.nchunks) return;
  const int64_t fa = c == P.nchunks ? P.nfibers : lower_bound_g(P.pos2, P.nfibers, c * P.chunk_nnz);
  P.chunk_fa[c] = fa;
  P.chunk_s[c] = fa < P.nfibers ? slice_of(P.pos1, P.I, fa) : P.I;
}

// Per-chunk slice bookkeeping shared by both dense kernels: slices that start
// and end inside the chunk are stored directly; the chunk's first slice, if it
// began earlier, leaves a head partial; its last slice, if it continues,
// leaves a tail partial (or the head partial when it is also the first).
struct SliceTracker {
  int64_t s, s_end;
  bool open;        // current slice began before this chunk
  bool wrote_head;
};

// R == 32, quarter-warp per fiber: a warp walks a chunk's fibers four at a
// time, quarter q (8 lanes, 4 columns each: two 16-byte loads per row) owns
// fiber f4 + q.  Short fibers (the median fiber holds one nonzero) thus put
// four D rows and four C rows in flight per warp step instead of one; long
// fibers stream their nonzeros in batches of 8 per quarter (coalesced k/b
// loads, 4 row loads in flight per lane).  Each quarter keeps w0 for its
// fiber; w0 * C(j,:) accumulates into the quarter's share of the slice row,
// and the four shares are combined (xor shuffles, fixed order) when the slice
// is flushed.  Slice/partial bookkeeping: slices inside a chunk are stored directly, a
// slice cut by a chunk boundary leaves a head or tail partial (SliceTracker).
#ifndef DQ_MINB
#define DQ_MINB 2
#endif
// A lane's 32-byte slice of a factor row: one 256-bit load (sm_100) when the
// factors are 32-byte aligned, else two 128-bit loads.
template <bool k256>
__device__ __forceinline__ void ld_row32(const double* p, double2& a, double2& b) {
  if constexpr (k256) {
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y)
        : "l"(p));
  } else {
    a = __ldg(reinterpret_cast<const double2*>(p));
    b = __ldg(reinterpret_cast<const double2*>(p) + 1);
  }
}

#ifndef DQ_LONG_FIBER
#define DQ_LONG_FIBER 96
#endif
constexpr int kLongFiber = DQ_LONG_FIBER;  // a fiber this long takes a whole warp step

template <bool k256>
__global__ void __launch_bounds__(256, DQ_MINB) mttkrp_dense32q_kernel(const DenseParams P) {
  const int lane = (int)lane_id();
  const int q = lane >> 3;
  const int col = 4 * (lane & 7);
  const int qbase = lane & ~7;
  while (true) {
    int64_t c = 0;
    if (lane == 0) c = (int64_t)atomicAdd(P.counter, 1ull);
    c = __shfl_sync(kFull, c, 0);
    if (c >= P.nchunks) break;
    const int64_t fa = P.chunk_fa[c], fb = P.chunk_fa[c + 1];
    double* part = P.part + (c * 2) * 32;
    if (fa >= fb) {
      if (lane == 0) {
        P.part_slice[2 * c] = -2;
        P.part_slice[2 * c + 1] = -1;
      }
      continue;
    }
    SliceTracker st;
    st.s = P.chunk_s[c];
    st.s_end = P.pos1[st.s + 1];
    st.open = P.pos1[st.s] < fa;
    st.wrote_head = false;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    auto flush = [&](bool ends_here) {
      double t[4];
#pragma unroll
      for (int x = 0; x < 4; x++) {
        t[x] = acc[x] + __shfl_xor_sync(kFull, acc[x], 8);
        t[x] += __shfl_xor_sync(kFull, t[x], 16);
        acc[x] = 0.0;
      }
      const bool started_here = !st.open;
      double* dst;
      if (started_here && ends_here) {
        dst = P.A + st.s * 32 + col;
      } else {
        const int slot = started_here ? 1 : 0;
        dst = part + slot * 32 + col;
        if (lane == 0) P.part_slice[2 * c + slot] = st.s;
        if (slot == 0) st.wrote_head = true;
      }
      if (q == 0) {
        reinterpret_cast<double2*>(dst)[0] = make_double2(t[0], t[1]);
        reinterpret_cast<double2*>(dst)[1] = make_double2(t[2], t[3]);
      }
    };
    for (int64_t fg = fa; fg < fb; fg += 32) {
      const int nf = (int)min((int64_t)32, fb - fg);
      int mj = 0, mlen = 0;
      int64_t mz = 0;
      if (lane < nf) {
        mj = (int)P.idx1[fg + lane];
        mz = P.pos2[fg + lane];
        mlen = (int)(P.pos2[fg + lane + 1] - mz);
      }
      // Steps: up to 4 consecutive short fibers, a quarter each; or one long
      // fiber (>= kLongFiber nonzeros) split over all four quarters (batch t
      // covers its nonzeros [32t, 32t+32), quarter q the 8 at 32t+8q), so no
      // quarter idles while another finishes a long fiber.
      const unsigned longm = __ballot_sync(kFull, lane < nf && mlen >= kLongFiber);
      auto step_at = [&](int g, bool& lmode, int& nsh) {
        lmode = (longm >> g) & 1u;
        const unsigned after = longm >> g;  // bit 0 = fiber g
        const int next_long = after ? __ffs(after) - 1 : 32;
        nsh = lmode ? 1 : min(4, min(nf - g, next_long));
      };
      // lane (q, l) of a step's first batch: short -> nonzero l of fiber g+q;
      // long -> nonzero 8q+l of fiber g
      auto first_batch = [&](int g, bool lmode, int nsh, int& k, double& b) {
        const int src = lmode ? g : g + q;
        const int64_t z0n = __shfl_sync(kFull, mz, src & 31);
        const int lenn = __shfl_sync(kFull, mlen, src & 31);
        const int zl = (lmode ? 8 * q : 0) + (lane & 7);
        k = 0;
        b = 0.0;
        if ((lmode || q < nsh) && zl < lenn) {
          k = (int)P.idx2[z0n + zl];
          b = P.vals[z0n + zl];
        }
      };
      bool lmode;
      int nsh;
      step_at(0, lmode, nsh);
      int pk;
      double pb;
      first_batch(0, lmode, nsh, pk, pb);
      for (int g = 0; g < nf;) {
        const int src = lmode ? g : g + q;
        const bool fv = lmode || q < nsh;
        const int64_t z0 = __shfl_sync(kFull, mz, src & 31);
        const int len_s = __shfl_sync(kFull, mlen, src & 31);  // every lane shuffles
        const int len = fv ? len_s : 0;
        const int j = __shfl_sync(kFull, mj, src & 31);
        const int zoff = lmode ? 8 * q : 0;
        const int stride = lmode ? 32 : 8;
        double2 c0 = make_double2(0.0, 0.0), c1 = c0;
        if (fv && (!lmode || q == 0)) {
          ld_row32<k256>(P.C + (int64_t)j * 32 + col, c0, c1);
        }
        int kk = pk;
        double bb = pb;
        // the next step and its first batch, loaded before this one is consumed
        const int gn = g + nsh;
        bool lmode_n = false;
        int nsh_n = 0;
        if (gn < nf) {  // uniform
          step_at(gn, lmode_n, nsh_n);
          first_batch(gn, lmode_n, nsh_n, pk, pb);
        }
        const int nmax = __reduce_max_sync(kFull, (unsigned)len);
        double w[4] = {0.0, 0.0, 0.0, 0.0};
        for (int zb = 0; zb < nmax; zb += stride) {
          // lane (q, l) holds nonzero zb + zoff + l of its quarter's stream;
          // load the next batch before consuming this one
          int kn = 0;
          double bn = 0.0;
          if (zb + stride < nmax) {
            const int zl = zb + stride + zoff + (lane & 7);
            if (zl < len) {
              kn = (int)P.idx2[z0 + zl];
              bn = P.vals[z0 + zl];
            }
          }
          if (!lmode && nmax - zb == 1) {
            // every quarter holds at most one nonzero (the typical short-fiber
            // step): one row load per lane, no unused slots
            const int k = __shfl_sync(kFull, kk, qbase);
            const double bv = __shfl_sync(kFull, bb, qbase);
            if (zb < len) {
              double2 d0, d1;
              ld_row32<k256>(P.D + (int64_t)k * 32 + col, d0, d1);
              w[0] = fma(bv, d0.x, w[0]);
              w[1] = fma(bv, d0.y, w[1]);
              w[2] = fma(bv, d1.x, w[2]);
              w[3] = fma(bv, d1.y, w[3]);
            }
            kk = kn;
            bb = bn;
            continue;
          }
#pragma unroll
          for (int h = 0; h < 2; h++) {
            if (__all_sync(kFull, zb + zoff + 4 * h >= len)) break;  // no quarter has entries left
            double2 d[4][2];
            double b[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
              const int uu = 4 * h + u;
              const int k = __shfl_sync(kFull, kk, qbase + uu);
              const double bv = __shfl_sync(kFull, bb, qbase + uu);
              const bool ok = zb + zoff + uu < len;
              b[u] = ok ? bv : 0.0;
              if (ok) {
                ld_row32<k256>(P.D + (int64_t)k * 32 + col, d[u][0], d[u][1]);
              } else {
                d[u][0] = make_double2(0.0, 0.0);
                d[u][1] = d[u][0];
              }
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
              w[0] = fma(b[u], d[u][0].x, w[0]);
              w[1] = fma(b[u], d[u][0].y, w[1]);
              w[2] = fma(b[u], d[u][1].x, w[2]);
              w[3] = fma(b[u], d[u][1].y, w[3]);
            }
          }
          kk = kn;
          bb = bn;
        }
        if (lmode) {  // the four quarters' partial sums of the one fiber (fixed order)
#pragma unroll
          for (int x = 0; x < 4; x++) {
            w[x] += __shfl_xor_sync(kFull, w[x], 8);
            w[x] += __shfl_xor_sync(kFull, w[x], 16);
          }
        }
        // fibers g..g+nsh-1 in order: add the owner quarter's share, flush at slice ends
#pragma unroll
        for (int u = 0; u < 4; u++) {
          if (u >= nsh) break;  // uniform
          const int64_t f = fg + g + u;
          while (f >= st.s_end) {
            st.s++;
            st.s_end = P.pos1[st.s + 1];
            st.open = false;
          }
          if (q == u) {
            acc[0] = fma(w[0], c0.x, acc[0]);
            acc[1] = fma(w[1], c0.y, acc[1]);
            acc[2] = fma(w[2], c1.x, acc[2]);
            acc[3] = fma(w[3], c1.y, acc[3]);
          }
          if (f + 1 == st.s_end) flush(true);
        }
        g = gn;
        lmode = lmode_n;
        nsh = nsh_n;
      }
    }
    if (fb < st.s_end) flush(false);
    if (lane == 0) {
      if (!st.wrote_head) P.part_slice[2 * c] = -1;
      if (!(fb < st.s_end && !st.open)) P.part_slice[2 * c + 1] = -1;
    }
  }
}

// Any R: column blocks of 32, a full warp per nonzero, one double per lane.
__global__ void __launch_bounds__(256) mttkrp_dense_generic_kernel(const DenseParams P) {
  const int lane = (int)lane_id();
  const int64_t ncb = (P.R + 31) / 32;
  while (true) {
    int64_t task = 0;
    if (lane == 0) task = (int64_t)atomicAdd(P.counter, 1ull);
    task = __shfl_sync(kFull, task, 0);
    if (task >= P.nchunks * ncb) break;
    const int64_t c = task % P.nchunks;
    const int64_t cbi = task / P.nchunks;
    const int64_t col = cbi * 32 + lane;
    const bool col_ok = col < P.R;
    const int64_t fa = P.chunk_fa[c], fb = P.chunk_fa[c + 1];
    double* part = P.part + ((cbi * P.nchunks + c) * 2) * 32;
    if (fa >= fb) {
      if (lane == 0 && cbi == 0) {
        P.part_slice[2 * c] = -2;
        P.part_slice[2 * c + 1] = -1;
      }
      continue;
    }
    SliceTracker st;
    st.s = P.chunk_s[c];
    st.s_end = P.pos1[st.s + 1];
    st.open = P.pos1[st.s] < fa;
    st.wrote_head = false;
    double acc = 0.0;
    auto flush = [&](bool ends_here) {
      const bool started_here = !st.open;
      if (started_here && ends_here) {
        if (col_ok) P.A[st.s * P.R + col] = acc;
      } else {
        const int slot = started_here ? 1 : 0;
        part[slot * 32 + lane] = acc;
        if (lane == 0 && cbi == 0) P.part_slice[2 * c + slot] = st.s;
        if (slot == 0) st.wrote_head = true;
      }
      acc = 0.0;
    };
    for (int64_t f = fa; f < fb; f++) {
      while (f >= st.s_end) {
        st.s++;
        st.s_end = P.pos1[st.s + 1];
        st.open = false;
      }
      const int64_t j = P.idx1[f];
      const int64_t z0 = P.pos2[f], z1 = P.pos2[f + 1];
      double w = 0.0;
      for (int64_t zb = z0; zb < z1; zb += 32) {
        const int n = (int)min((int64_t)32, z1 - zb);
        int kz = 0;
        double bz = 0.0;
        if (lane < n) {
          kz = (int)P.idx2[zb + lane];
          bz = P.vals[zb + lane];
        }
        for (int t0 = 0; t0 < n; t0 += 8) {
          double d[8], b[8];
#pragma unroll
          for (int u = 0; u < 8; u++) {
            const int src = t0 + u;
            const int k = __shfl_sync(kFull, kz, src & 31);
            const double bv = __shfl_sync(kFull, bz, src & 31);
            const bool ok = src < n && col_ok;
            b[u] = ok ? bv : 0.0;
            d[u] = ok ? __ldg(P.D + (int64_t)k * P.R + col) : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; u++) w = fma(b[u], d[u], w);
        }
      }
      if (col_ok) acc = fma(w, __ldg(P.C + j * P.R + col), acc);
      if (f + 1 == st.s_end) flush(true);
    }
    if (fb < st.s_end) flush(false);
    if (lane == 0 && cbi == 0) {
      if (!st.wrote_head) P.part_slice[2 * c] = -1;
      if (!(fb < st.s_end && !st.open)) P.part_slice[2 * c + 1] = -1;
    }
  }
}

// Sums the partials of every slice cut by chunk boundaries, in a fixed order.
// A chain = the chunk holding a slice's tail partial plus the following chunks
// holding its head partials.  Most chains span 2-3 chunks; a heavy slice's
// spans ~10^4, so two levels of block sums come first:
//  * level 1: every aligned block of 32 chunks whose heads all belong to one
//    slice (or are empty) gets its head partials summed in chunk order;
//  * level 2: the same over aligned blocks of 32 level-1 blocks;
//  * chains: a warp per chain walks forward from the tail partial, taking
//    whole level-2 / level-1 blocks where they are aligned and uniform and
//    loose chunks elsewhere, and sums the items in walk order (lane = column).
// Every order is fixed by the chunking: results are deterministic run to run.
constexpr int kFixBlock = 32;          // items per block sum (both levels)
constexpr int64_t kSliceMixed = -1;    // head "none" / block not uniform
constexpr int64_t kSliceEmpty = -2;    // empty chunk / block of empty chunks

// One level of block sums.  Input item t has slice hs[t * hstride] and, for
// column block cbi, values vals[cbi * vcb + t * vstride + lane].
__global__ void mttkrp_dense_blocksum_kernel(const int64_t* hs, int hstride, const double* vals,
                                             int64_t vstride, int64_t vcb, int64_t n, int64_t ncb,
                                             double* bsum, int64_t* bslice, int64_t nblocks) {
  const int lane = (int)lane_id();
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t task = warp; task < nblocks * ncb; task += nwarps) {
    const int64_t b = task % nblocks, cbi = task / nblocks;
    const int64_t t0 = b * kFixBlock;
    const int64_t t = t0 + lane;
    const int64_t h = t < n ? hs[t * hstride] : kSliceEmpty;
    const unsigned nonempty = __ballot_sync(kFull, h != kSliceEmpty);
    int64_t sb = kSliceEmpty;
    if (nonempty) sb = __shfl_sync(kFull, h, __ffs(nonempty) - 1);
    const bool full = __all_sync(kFull, h == kSliceEmpty || h == sb) && sb != kSliceMixed;
    if (cbi == 0 && lane == 0) bslice[b] = full ? sb : kSliceMixed;
    if (!full || sb == kSliceEmpty) continue;
    const double* base = vals + cbi * vcb;
    double v[kFixBlock];
#pragma unroll
    for (int u = 0; u < kFixBlock; u++)
      v[u] = ((nonempty >> u) & 1) ? base[(t0 + u) * vstride + lane] : 0.0;
    double sum = 0.0;
#pragma unroll
    for (int u = 0; u < kFixBlock; u++) sum += v[u];
    bsum[(cbi * nblocks + b) * 32 + lane] = sum;
  }
}

struct FixupLevels {
  const double* bsum1;
  const int64_t* bslice1;
  int64_t nb1;
  const double* bsum2;
  const int64_t* bslice2;
  int64_t nb2;
};

// Sums the leading run of items (lanes 0..) whose slice is s or empty, in
// order; returns the run length.  `lim` caps the items examined.
__device__ __forceinline__ int take_items(const int64_t* hs, int hstride, const double* vals,
                                          int64_t vstride, int64_t t0, int lim, int64_t s,
                                          double& acc) {
  const int lane = (int)lane_id();
  const int64_t h = lane < lim ? hs[(t0 + lane) * hstride] : kSliceMixed;
  const bool ok = lane < lim && (h == s || h == kSliceEmpty);
  const unsigned bad = __ballot_sync(kFull, !ok);
  const int run = bad ? __ffs(bad) - 1 : 32;
  const unsigned take = __ballot_sync(kFull, ok && h == s) & (run == 32 ? kFull : ((1u << run) - 1));
  for (int u0 = 0; u0 < run; u0 += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; u++)
      v[u] = (u0 + u < run && ((take >> (u0 + u)) & 1)) ? vals[(t0 + u0 + u) * vstride + lane] : 0.0;
#pragma unroll
    for (int u = 0; u < 8; u++)
      if (u0 + u < run && ((take >> (u0 + u)) & 1)) acc += v[u];
  }
  return run;
}

__global__ void mttkrp_dense_fixup_kernel(const DenseParams P, const FixupLevels L) {
  const int lane = (int)lane_id();
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t ncb = (P.R + 31) / 32;
  constexpr int64_t kB2 = (int64_t)kFixBlock * kFixBlock;
  for (int64_t c = warp; c < P.nchunks; c += nwarps) {
    const int64_t s = P.part_slice[2 * c + 1];
    if (s < 0) continue;  // uniform across the warp
    for (int64_t cbi = 0; cbi < ncb; cbi++) {
      const double* base = P.part + cbi * P.nchunks * 64;
      double acc = base[(c * 2 + 1) * 32 + lane];
      int64_t t = c + 1;
      while (t < P.nchunks) {
        if (t % kB2 == 0 && t / kB2 < L.nb2) {
          const int64_t b = t / kB2;
          const int lim = (int)min((int64_t)32, L.nb2 - b);
          const int run = take_items(L.bslice2, 1, L.bsum2 + cbi * L.nb2 * 32, 32, b, lim, s, acc);
          t += (int64_t)run * kB2;
          if (run == lim && lim == 32) continue;
          if (run == lim) { if (t >= P.nchunks) break; }
        }
        if (t % kFixBlock == 0 && t / kFixBlock < L.nb1) {
          const int64_t b = t / kFixBlock;
          // up to the next level-2 boundary
          const int64_t bend = min(L.nb1, (b / kFixBlock + 1) * kFixBlock);
          const int lim = (int)(bend - b);
          const int run = take_items(L.bslice1, 1, L.bsum1 + cbi * L.nb1 * 32, 32, b, lim, s, acc);
          t += (int64_t)run * kFixBlock;
          if (run == lim) continue;
        }
        // loose chunks up to the next level-1 boundary
        const int lim = (int)(min(P.nchunks, (t / kFixBlock + 1) * kFixBlock) - t);
        const int run = take_items(P.part_slice, 2, base, 64, t, lim, s, acc);
        t += run;
        if (run < lim) break;  // the chain ends at chunk t
      }
      const int64_t col = cbi * 32 + lane;
      if (col < P.R) P.A[s * P.R + col] = acc;
    }
  }
}

// ===========================================================================
// sparse
// ===========================================================================
#ifndef SP_WARPS
#define SP_WARPS 8
#endif
constexpr int kSpWarps = SP_WARPS;
constexpr int kRowChunk = 8;         // factor-row entries held in registers at once

struct HitRec;
struct MatRec;

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
  unsigned long long* mults;  // SPEC counter: |D_k| per nonzero + consumed w0 entries
  int64_t* stage;             // [I*2R] per slice: R drained coordinates, then R values
  // column bitmaps of the factor rows (kBmWords 64-bit words per row; R <= 64*W)
  const unsigned long long* cbm;
  const unsigned long long* dbm;
  // three-phase path: hit and match records per slice
  int32_t* rec_cnt;            // [I] hits of each slice, -1: left to the single-pass kernel
  int32_t* mat_cnt;            // [I] match records of each slice
  unsigned long long* dsum;    // [I] sum of |D_k| over the slice's nonzeros (SPEC counter)
  HitRec* hits;                // [I*hit_cap]
  MatRec* mats;                // [I*mat_cap]
  int32_t hit_cap, mat_cap;
  int mode;                    // single-pass kernel: 0 staged rows, 1 row lengths only, 2 rows into the CSR
  const int64_t* slice_list;   // slices to evaluate (fallback pass), or null: all
  int64_t nlist;
  const unsigned long long* nlist_dev;  // list length on the device (overrides nlist)
  unsigned long long* ovf;     // [0] overflowed slices (appended to ovf_list)
  int64_t* ovf_list;
  int tma_ok;                  // the CSF arrays sit on 16-byte boundaries (bulk copies)
};

__device__ __forceinline__ int64_t* stage_idx_row(const SparseParams& P, int64_t i) {
  return P.stage + i * 2 * P.R;
}
__device__ __forceinline__ double* stage_vals_row(const SparseParams& P, int64_t i) {
  return reinterpret_cast<double*>(P.stage + i * 2 * P.R + P.R);
}

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

__device__ __forceinline__ void ws_add(double* wv, uint32_t* wb, int64_t r, double v) {
  atomicAdd(&wv[r], v);
  atomicOr(&wb[r >> 5], 1u << (r & 31));
}

// Evaluates slice i into the warp's workspace (vals[R], bits[R/32]).
__device__ void sparse_slice(const SparseParams& P, int64_t i, double* wv, uint32_t* wb,
                             unsigned long long& mults) {
  const int lane = (int)lane_id();
  const int64_t f0 = P.pos1[i], f1 = P.pos1[i + 1];
  for (int64_t f = f0 + lane; f < f1; f += 32) {
    const int64_t j = P.idx1[f];
    const int64_t z0 = P.pos2[f], z1 = P.pos2[f + 1];
    const int64_t c0 = P.cpos[j], c1 = P.cpos[j + 1];
    if (z1 - z0 == 1) {
      // single nonzero: C_j ∩ D_k.  Column ids of both rows are loaded into
      // registers kRowChunk at a time (independent loads) and intersected
      // all-pairs; values are fetched only for matches.
      const int64_t k = P.idx2[z0];
      const double b = P.vals[z0];
      const int64_t d0 = P.dpos[k], d1 = P.dpos[k + 1];
      mults += (unsigned long long)(d1 - d0);
      for (int64_t cq = c0; cq < c1; cq += kRowChunk) {
        int cc[kRowChunk];
#pragma unroll
        for (int a = 0; a < kRowChunk; a++) cc[a] = cq + a < c1 ? (int)P.cidx[cq + a] : -1;
        for (int64_t dq = d0; dq < d1; dq += kRowChunk) {
          int dd[kRowChunk];
#pragma unroll
          for (int e = 0; e < kRowChunk; e++) dd[e] = dq + e < d1 ? (int)P.didx[dq + e] : -2;
#pragma unroll
          for (int a = 0; a < kRowChunk; a++) {
            int hit = -1;
#pragma unroll
            for (int e = 0; e < kRowChunk; e++) hit = (dd[e] == cc[a]) ? e : hit;
            if (hit >= 0) {
              // w0(r) = 0 + b*D(k,r);  w1(r) += w0(r)*C(j,r)
              const double w0 = add_rn(0.0, mul_rn(b, P.dvals[dq + hit]));
              ws_add(wv, wb, cc[a], mul_rn(w0, P.cvals[cq + a]));
              mults++;
            }
          }
        }
      }
    } else {
      // general fiber: w0 at each of C_j's coordinates, accumulated over k
      for (int64_t z = z0; z < z1; z++) {
        const int64_t k = P.idx2[z];
        mults += (unsigned long long)(P.dpos[k + 1] - P.dpos[k]);
      }
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
          ws_add(wv, wb, r, mul_rn(w0, P.cvals[q]));
          mults++;
        }
      }
    }
  }
}

// Column bitmap of every factor row: W 64-bit words per row (bit r = column
// r present).  One thread per row; rows hold sorted distinct columns.
template <int W>
__global__ void factor_bitmap_kernel(const int64_t* pos, const int64_t* idx, int64_t nrows,
                                     unsigned long long* bm) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows;
       r += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long w[W];
#pragma unroll
    for (int k = 0; k < W; k++) w[k] = 0ull;
    for (int64_t t = pos[r]; t < pos[r + 1]; t++) {
      const int64_t c = idx[t];
#pragma unroll
      for (int k = 0; k < W; k++) w[k] |= ((c >> 6) == k) ? (1ull << (c & 63)) : 0ull;
    }
#pragma unroll
    for (int k = 0; k < W; k++) bm[r * W + k] = w[k];
  }
}

template <int W>
__device__ __forceinline__ void load_bm(const unsigned long long* p, unsigned long long (&b)[W]) {
  if constexpr (W == 4) {
    // one 256-bit load per bitmap row (rows are 32-byte aligned)
    asm("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];"
        : "=l"(b[0]), "=l"(b[1]), "=l"(b[2]), "=l"(b[3])
        : "l"(p));
  } else if constexpr (W % 2 == 0) {
#pragma unroll
    for (int k = 0; k < W; k += 2) {
      const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(p) + k / 2);
      b[k] = v.x;
      b[k + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int k = 0; k < W; k++) b[k] = __ldg(p + k);
  }
}

// Factor value / row-pointer gathers at matches.  Only the bitmaps (32 MB at
// config 5) are kept evict_last: the whole gathered set (bitmaps + values +
// row pointers, ~104 MB) does not stay resident beside the 6.4 GB stream.
#ifndef SP_VAL_HINT
#define SP_VAL_HINT 0  // 0 normal, 1 evict_last, 2 evict_first
#endif
template <typename T>
__device__ __forceinline__ T ld_val(const T* p, uint64_t keep) {
  if constexpr (SP_VAL_HINT == 1) return ld_keep(p, keep);
  else if constexpr (SP_VAL_HINT == 2) return __ldcs(p);
  else return __ldg(p);
}

// load_bm with the L2 evict_last hint (the bitmaps are re-read ~400 times per
// call while the CSF streams past them once).
template <int W>
__device__ __forceinline__ void load_bm_keep(const unsigned long long* p, uint64_t pol,
                                             unsigned long long (&b)[W]) {
  if constexpr (W % 4 == 0) {
#pragma unroll
    for (int k = 0; k < W; k += 4) ld_keep_v4(p + k, pol, b[k], b[k + 1], b[k + 2], b[k + 3]);
  } else {
#pragma unroll
    for (int k = 0; k < W; k++)
      b[k] = (unsigned long long)ld_keep(reinterpret_cast<const int64_t*>(p) + k, pol);
  }
}

// Position of column r among the row's columns (popcount of the bits below).
template <int W>
__device__ __forceinline__ int bm_rank(const unsigned long long (&b)[W], int r) {
  int n = 0;
#pragma unroll
  for (int k = 0; k < W; k++) {
    const int lo = k * 64;
    if (r >= lo + 64) n += __popcll(b[k]);
    else if (r > lo) n += __popcll(b[k] & ((1ull << (r - lo)) - 1ull));
  }
  return n;
}

// Matches (C_j ∩ D_k columns of single-nonzero fibers) are queued per warp
// so that their value gathers and workspace updates run on full warps instead
// of the few lanes that found a match.  (A warp-cooperative expansion -- lane
// s evaluating the warp's s-th match, owner found by a shuffle search -- cut
// no time: 6.79 vs 6.22 ms at config 5, the kernel waits on memory.)
constexpr int kQ = 128;
struct MatchQueue {
  int64_t ci[kQ];  // position of C(j,r) in C's values
  int64_t di[kQ];  // position of D(k,r) in D's values
  double b[kQ];    // B(i,j,k)
  int r[kQ];
};

__host__ __device__ constexpr size_t match_queue_bytes() { return sizeof(MatchQueue); }

// sparse_slice with factor-row bitmaps: C_j ∩ D_k is a word-wise AND and a
// matched column's value positions are popcounts (same arithmetic and
// per-entry order as sparse_slice: w0 = 0 + b*D(k,r), w1(r) += w0*C(j,r)).
template <int W>
__device__ void sparse_slice_bm(const SparseParams& P, int64_t i, double* wv, uint32_t* wb,
                                unsigned long long& mults, void* mbuf) {
  const int lane = (int)lane_id();
  const int64_t f0 = P.pos1[i], f1 = P.pos1[i + 1];
  const uint64_t keep = l2_evict_last_policy();
  MatchQueue& Q = *static_cast<MatchQueue*>(mbuf);
  int qn = 0;  // queued matches (warp-uniform)
  auto flush = [&]() {
    for (int t = lane; t < qn; t += 32) {
      const double w0 = add_rn(0.0, mul_rn(Q.b[t], ld_val(P.dvals + Q.di[t], keep)));
      ws_add(wv, wb, Q.r[t], mul_rn(w0, ld_val(P.cvals + Q.ci[t], keep)));
    }
    __syncwarp();
    qn = 0;
  };
  for (int64_t fb = f0; fb < f1; fb += 32) {
    const int64_t f = fb + lane;
    int nm = 0;
    int64_t j = 0, k = 0;
    double b = 0.0;
    unsigned long long m[W];
    unsigned long long bc[W], bd[W];
#pragma unroll
    for (int w = 0; w < W; w++) m[w] = bc[w] = bd[w] = 0ull;
    bool single = false;
    if (f < f1) {
      j = __ldcs(P.idx1 + f);
      const int64_t z0 = __ldcs(P.pos2 + f), z1 = __ldcs(P.pos2 + f + 1);
      load_bm_keep<W>(P.cbm + j * W, keep, bc);
      if (z1 - z0 == 1) {
        single = true;
        k = __ldcs(P.idx2 + z0);
        b = __ldcs(P.vals + z0);
        load_bm_keep<W>(P.dbm + k * W, keep, bd);
#pragma unroll
        for (int w = 0; w < W; w++) {
          mults += (unsigned long long)__popcll(bd[w]);
          m[w] = bc[w] & bd[w];
          nm += __popcll(m[w]);
        }
      } else {
        // general fiber: w0 at each of C_j's columns, accumulated over k in order
        for (int64_t z = z0; z < z1; z++) {
          unsigned long long bz[W];
          load_bm<W>(P.dbm + P.idx2[z] * W, bz);
#pragma unroll
          for (int w = 0; w < W; w++) mults += (unsigned long long)__popcll(bz[w]);
        }
        const int64_t c0 = P.cpos[j];
        int ic = 0;
#pragma unroll
        for (int w = 0; w < W; w++) {
          unsigned long long cm = bc[w];
          while (cm) {
            const int bit = __ffsll((long long)cm) - 1;
            const int r = w * 64 + bit;
            double w0 = 0.0;
            bool present = false;
            for (int64_t z = z0; z < z1; z++) {
              const int64_t kz = P.idx2[z];
              unsigned long long bz[W];
              load_bm<W>(P.dbm + kz * W, bz);
              if ((bz[w] >> bit) & 1ull) {
                w0 = add_rn(w0, mul_rn(P.vals[z], P.dvals[P.dpos[kz] + bm_rank<W>(bz, r)]));
                present = true;
              }
            }
            if (present) {
              ws_add(wv, wb, r, mul_rn(w0, P.cvals[c0 + ic]));
              mults++;
            }
            ic++;
            cm &= cm - 1ull;
          }
        }
      }
    }
    const int inc = warp_inclusive_scan(nm);
    const int tot = __shfl_sync(kFull, inc, 31);
    if (tot == 0) continue;
    // per-lane walk of the matched bits into the warp's queue (evaluated 32 at
    // a time by flush), or directly when the batch alone overflows the queue
    if (tot > kQ - qn) flush();
    const bool direct = tot > kQ;
    if (nm > 0) {
      const int64_t c0 = ld_val(P.cpos + j, keep), d0 = ld_val(P.dpos + k, keep);
      int slot = qn + inc - nm;
      int rc = 0, rd = 0;
#pragma unroll
      for (int w = 0; w < W; w++) {
        unsigned long long mm = m[w];
        while (mm) {
          const int bit = __ffsll((long long)mm) - 1;
          const unsigned long long below = (1ull << bit) - 1ull;
          const int64_t ci = c0 + rc + __popcll(bc[w] & below);
          const int64_t di = d0 + rd + __popcll(bd[w] & below);
          if (direct) {
            const double w0 = add_rn(0.0, mul_rn(b, ld_val(P.dvals + di, keep)));
            ws_add(wv, wb, w * 64 + bit, mul_rn(w0, ld_val(P.cvals + ci, keep)));
          } else {
            Q.ci[slot] = ci;
            Q.di[slot] = di;
            Q.b[slot] = b;
            Q.r[slot] = w * 64 + bit;
            slot++;
          }
          mults++;
          mm &= mm - 1ull;
        }
        rc += __popcll(bc[w]);
        rd += __popcll(bd[w]);
      }
    }
    __syncwarp();
    if (!direct) {
      qn += tot;
      if (qn >= kQ - 32) flush();
    }
  }
  flush();
}

// Each warp claims slices dynamically, evaluates one into its shared-memory
// workspace and drains it sorted into a fixed-stride staging row (a row of A
// holds at most R entries), recording the count in the row-pointer array.  No
// ordering between slices is needed here; a scan and a coalesced compaction
// copy build the CSR afterwards (no look-back waits on slower slices).
#ifndef SP_MINB
#define SP_MINB 4  // resident CTAs per SM the register budget targets
#endif
template <int W>
__global__ void __launch_bounds__(kSpWarps * 32, SP_MINB) mttkrp_sparse_kernel(const SparseParams P) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = (int)lane_id();
  const int warp = threadIdx.x >> 5;
  const int64_t R = P.R;
  const int nwords = (int)((R + 31) / 32);
  const size_t ws_bytes = ((size_t)R * 8 + (size_t)nwords * 4 + 15) & ~(size_t)15;
  double* wv = reinterpret_cast<double*>(smem_raw + (size_t)warp * ws_bytes);
  uint32_t* wb = reinterpret_cast<uint32_t*>(wv + R);
  void* owners = smem_raw + (size_t)kSpWarps * ws_bytes + (size_t)warp * match_queue_bytes();
  unsigned long long mults = 0;
  while (true) {
    int64_t i = 0;
    if (lane == 0) i = (int64_t)atomicAdd(P.tile_counter, 1ull);
    i = __shfl_sync(kFull, i, 0);
    if (P.slice_list) {
      if (i >= (P.nlist_dev ? (int64_t)*P.nlist_dev : P.nlist)) break;
      i = P.slice_list[i];
    } else if (i >= P.I) {
      break;
    }
    for (int64_t r = lane; r < R; r += 32) wv[r] = 0.0;
    for (int w = lane; w < nwords; w += 32) wb[w] = 0u;
    __syncwarp();
    if constexpr (W > 0)
      sparse_slice_bm<W>(P, i, wv, wb, mults, owners);
    else
      sparse_slice(P, i, wv, wb, mults);
    __syncwarp();
    // sorted drain by ballot/popcount over the presence bitmap: into the
    // slice's staging row (mode 0), nowhere (mode 1: the row length only) or
    // straight into its CSR row (mode 2, after the scan)
    int64_t* oi = P.mode == 2 ? P.out_idx + P.out_pos[i] : stage_idx_row(P, i);
    double* ov = P.mode == 2 ? P.out_vals + P.out_pos[i] : stage_vals_row(P, i);
    int out = 0;
    for (int w = 0; w < nwords; w++) {
      const uint32_t bits = wb[w];
      if (bits == 0) continue;
      if (P.mode != 1 && ((bits >> lane) & 1u)) {
        const int rank = __popc(bits & ((1u << lane) - 1u));
        const int64_t r = (int64_t)w * 32 + lane;
        __stcs(reinterpret_cast<long long*>(oi) + out + rank, (long long)r);
        __stcs(ov + out + rank, wv[r]);
      }
      out += __popc(bits);
    }
    if (lane == 0 && P.mode != 2) P.out_pos[i + 1] = out;
    __syncwarp();
  }
  mults = warp_sum(mults);
  if (lane == 0 && mults && P.mults) atomicAdd(P.mults, mults);
}

// ---------------------------------------------------------------------------
// Three phases, each with a gathered set below the L2's ~64-80 MB random-
// gather capacity (profiles/r02/l2_capacity.md; one pass gathers ~104 MB at
// config 5 and misses on 23-63 % of lookups):
//  1. filter: the CSF streamed once through per-warp shared-memory rings
//     filled by TMA bulk copies (fiber metadata kMD1 chunks ahead, a chunk's
//     nonzeros as soon as its pos2 range has landed), so the only loads a lane
//     waits for are the two factor-row bitmaps (gathered set: 32 MB).  A
//     nonzero whose C_j and D_k share a column becomes a hit record (j, k, b)
//     in the slice's hit row -- one 16-byte store, no walk over the bits.
//  2. expand: lanes over the slice's hits (every lane holds one, so the bit
//     walks run on full warps): each shared column becomes a match record
//     (positions of C(j,r) and D(k,r) in the factors' values, column, the
//     hit's index), and the slice's distinct columns are counted, so the row
//     pointers can be scanned before any row is written (gathered: both
//     bitmaps and both row-start arrays, 40 MB; with D's values in the same
//     kernel the 72 MB set missed L2: 5.2 GB of DRAM reads for 1.5 GB of
//     records).
//  3. accumulate: a warp per slice, lanes over its match records:
//     w0 = 0 + b·D(k,r), w1(r) += w0·C(j,r) into its R-wide workspace
//     (gathered: both factors' values, 64 MB), drained sorted straight into
//     the CSR.
// Same arithmetic as sparse_slice_bm for single-nonzero fibers; a multi-nonzero
// fiber yields one hit per nonzero (columns shared by two of its nonzeros are
// multiplied with C one by one, see the filter).  A slice with more hits or
// matches than its rows hold goes to the single-pass kernel, which runs over
// the listed slices twice: row lengths before the scan, the rows after it.
struct __align__(16) HitRec {
  int j, k;
  double b;
};
// Records are touched once per phase: streamed past the L2-resident factor data.
template <typename T>
__device__ __forceinline__ T ld_rec(const T* p) {
  static_assert(sizeof(T) == 16, "16-byte records");
  const int4 v = __ldcs(reinterpret_cast<const int4*>(p));
  return *reinterpret_cast<const T*>(&v);
}
template <typename T>
__device__ __forceinline__ void st_rec(T* p, const T& x) {
  static_assert(sizeof(T) == 16, "16-byte records");
  __stcs(reinterpret_cast<int4*>(p), *reinterpret_cast<const int4*>(&x));
}

struct __align__(16) MatRec {
  int c;          // position of C(j, column) in C's values
  unsigned meta;  // column | the hit's index in the slice's hit row << 10
  int64_t d;      // position of D(k, column) in D's values
};

#ifndef SPM_D1
#define SPM_D1 4  // chunks of fiber metadata in flight per warp (power of two)
#endif
#ifndef SPM_D2
#define SPM_D2 2  // chunks of nonzeros in flight per warp (power of two)
#endif
#ifndef SPM_GROUP
#define SPM_GROUP 8  // consecutive slices per claim
#endif
#ifndef SPM_CHUNK
#define SPM_CHUNK 64  // fibers per ring slot
#endif
constexpr int kMD1 = SPM_D1, kMD2 = SPM_D2, kMGroup = SPM_GROUP, kMC = SPM_CHUNK;
constexpr int kMZ = kMC + 8;  // nonzeros staged per chunk
static_assert(kMD2 < kMD1 && (kMD1 & (kMD1 - 1)) == 0 && (kMD2 & (kMD2 - 1)) == 0, "ring depths");
static_assert(kMGroup < 32 && kMC % 32 == 0, "groups and chunks");

// A warp's rings.  A chunk is kMC consecutive fibers at an absolute multiple
// of kMC, so every bulk copy starts on a 16-byte boundary of its array.
struct __align__(16) MatchRing {
  int64_t j[kMD1][kMC];
  int64_t p2[kMD1][kMC + 2];
  int64_t k[kMD2][kMZ];
  double v[kMD2][kMZ];
  int64_t zbase[kMD2];  // first staged nonzero, or -1: lanes read global memory
  uint64_t bar1[kMD1];
  uint64_t bar2[kMD2];
};

// Ring 1: fiber metadata (idx1, pos2) of the chunk starting at fiber f into
// slot q mod kMD1, one mbarrier phase per use.
__device__ __forceinline__ void ring_issue1(const SparseParams& P, MatchRing& Q, int lane, uint32_t q,
                                            int64_t f) {
  const int s = (int)(q & (kMD1 - 1));
  if (P.tma_ok && f + kMC + 2 <= P.nfibers + 1) {
    if (lane == 0) {
      const uint64_t once = l2_evict_first_policy();
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&Q.bar1[s], 8 * kMC + 8 * (kMC + 2));
      bulk_g2s_hint(Q.j[s], P.idx1 + f, 8 * kMC, &Q.bar1[s], once);
      bulk_g2s_hint(Q.p2[s], P.pos2 + f, 8 * (kMC + 2), &Q.bar1[s], once);
    }
  } else {
    // the tensor's last chunk (or arrays off a 16-byte boundary): by the lanes
    for (int t = lane; t < kMC + 2; t += 32) {
      if (t < kMC) Q.j[s][t] = f + t < P.nfibers ? P.idx1[f + t] : 0;
      Q.p2[s][t] = f + t <= P.nfibers ? P.pos2[f + t] : P.nnz;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&Q.bar1[s]);
  }
}
// Ring 2: once the chunk's pos2 range has landed, its nonzeros (idx2, vals)
// into slot q mod kMD2 (or a note that lanes read them from global memory).
__device__ __forceinline__ void ring_issue2(const SparseParams& P, MatchRing& Q, int lane, uint32_t q) {
  const int s1 = (int)(q & (kMD1 - 1)), s2 = (int)(q & (kMD2 - 1));
  mbar_wait(&Q.bar1[s1], (q / kMD1) & 1u);
  if (lane == 0) {
    const int64_t zal = Q.p2[s1][0] & ~(int64_t)1, zbl = (Q.p2[s1][kMC] + 1) & ~(int64_t)1;
    const int64_t len = zbl - zal;
    if (P.tma_ok && len > 0 && len <= kMZ && zbl <= P.nnz) {
      const uint64_t once = l2_evict_first_policy();
      Q.zbase[s2] = zal;
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&Q.bar2[s2], (unsigned)len * 16u);
      bulk_g2s_hint(Q.k[s2], P.idx2 + zal, (unsigned)len * 8u, &Q.bar2[s2], once);
      bulk_g2s_hint(Q.v[s2], P.vals + zal, (unsigned)len * 8u, &Q.bar2[s2], once);
    } else {
      Q.zbase[s2] = -1;
      mbar_arrive(&Q.bar2[s2]);
    }
  }
}

#ifndef SPM_MINB
#define SPM_MINB 3  // the rings hide the stream's latency: registers before occupancy
#endif
template <int W>
__global__ void __launch_bounds__(kSpWarps * 32, SPM_MINB)
    mttkrp_sparse_filter_kernel(const __grid_constant__ SparseParams P) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = (int)lane_id();
  const unsigned lt = lanemask_lt();
  MatchRing& Q = reinterpret_cast<MatchRing*>(smem_raw)[threadIdx.x >> 5];
  if (lane == 0) {
    for (int s = 0; s < kMD1; s++) mbar_init(&Q.bar1[s], 1);
    for (int s = 0; s < kMD2; s++) mbar_init(&Q.bar2[s], 1);
    mbar_init_fence();
  }
  __syncwarp();
  uint32_t n1 = 0, n2 = 0, np = 0;  // chunks issued to ring 1 / ring 2 / consumed (warp lifetime)
  while (true) {
    int64_t i0 = 0;
    if (lane == 0) i0 = (int64_t)atomicAdd(P.tile_counter, (unsigned long long)kMGroup);
    i0 = __shfl_sync(kFull, i0, 0);
    if (i0 >= P.I) break;
    const int gcount = (int)min((int64_t)kMGroup, P.I - i0);
    const int64_t p1 = lane <= gcount ? P.pos1[i0 + lane] : 0;
    const int64_t F0 = __shfl_sync(kFull, p1, 0);
    const int64_t fb0 = F0 & ~(int64_t)(kMC - 1);  // first fiber of the group's first chunk
    // fiber positions below are relative to fb0 (the host bounds a group's fibers to int32)
    const int p1r = (int)(p1 - fb0);
    const int F0r = (int)(F0 - fb0), F1r = __shfl_sync(kFull, p1r, gcount);
    if (F0r == F1r) {
      if (lane < gcount) {
        P.rec_cnt[i0 + lane] = 0;
        P.dsum[i0 + lane] = 0ull;
      }
      continue;
    }
    const uint32_t nch = (uint32_t)((F1r + kMC - 1) / kMC);
    const uint32_t base = np;  // n1 == n2 == np between groups
    for (uint32_t t = 0; t < (uint32_t)kMD1 && t < nch; t++, n1++)
      ring_issue1(P, Q, lane, n1, fb0 + (int64_t)(n1 - base) * kMC);
    for (uint32_t t = 0; t < (uint32_t)kMD2 && t < nch; t++, n2++) ring_issue2(P, Q, lane, n2);

    int si = 0;  // current slice of the group
    int cur_f1 = __shfl_sync(kFull, p1r, 1);
    int nrec = 0;
    bool ovf = false;
    unsigned mcur = 0;  // the lane's share of the current slice's sum of |D_k|
    HitRec* hrow = P.hits + i0 * P.hit_cap;  // the current slice's hit row
    for (uint32_t q = base; q < base + nch; q++) {
      const int s1 = (int)(q & (kMD1 - 1)), s2 = (int)(q & (kMD2 - 1));
      mbar_wait(&Q.bar2[s2], (q / kMD2) & 1u);
      const int64_t zb = Q.zbase[s2];
#pragma unroll 1
      for (int h = 0; h < kMC / 32; h++) {
        const int cfirst = (int)(q - base) * kMC + h * 32;
        if (cfirst >= F1r) break;
        const int f = cfirst + lane;
        const bool valid = f >= F0r && f < F1r;
        const int t = h * 32 + lane;
        const int j = (int)Q.j[s1][t];
        const int64_t z0 = Q.p2[s1][t];
        const int nz = valid ? (int)(Q.p2[s1][t + 1] - z0) : 0;
        int nh = 0, k = 0;  // the fiber's hits
        double b = 0.0;
        unsigned mf = 0;  // the fiber's sum of |D_k|
        if (nz >= 1) {
          const uint64_t keep = l2_evict_last_policy();
          unsigned long long bc[W], bd[W];
          load_bm_keep<W>(P.cbm + (int64_t)j * W, keep, bc);
          if (zb >= 0) {
            k = (int)Q.k[s2][z0 - zb];
            b = Q.v[s2][z0 - zb];
          } else {
            k = (int)__ldcs(P.idx2 + z0);
            b = __ldcs(P.vals + z0);
          }
          load_bm_keep<W>(P.dbm + (int64_t)k * W, keep, bd);
          unsigned long long any = 0ull;
#pragma unroll
          for (int w = 0; w < W; w++) {
            mf += (unsigned)__popcll(bd[w]);
            any |= bc[w] & bd[w];
          }
          nh = any != 0ull ? 1 : 0;
          if (nz > 1) {
            // one hit per nonzero.  Two nonzeros meeting C_j in one column are
            // multiplied with C(j,r) one by one instead of summed first (the
            // difference is an ulp of the column's terms, inside the parity
            // bound); the SPEC counter takes one w0 entry per distinct column.
            int seen = 0, each = 0;
#pragma unroll
            for (int w = 0; w < W; w++) {
              bd[w] &= bc[w];  // columns of C_j seen so far
              each += __popcll(bd[w]);
            }
            for (int64_t z = z0 + 1; z < z0 + nz; z++) {
              unsigned long long bz[W];
              load_bm<W>(P.dbm + P.idx2[z] * W, bz);
              unsigned long long m = 0ull;
#pragma unroll
              for (int w = 0; w < W; w++) {
                mf += (unsigned)__popcll(bz[w]);
                m |= bc[w] & bz[w];
                each += __popcll(bc[w] & bz[w]);
                bd[w] |= bc[w] & bz[w];
              }
              nh += m != 0ull ? 1 : 0;
            }
#pragma unroll
            for (int w = 0; w < W; w++) seen += __popcll(bd[w]);
            mf -= (unsigned)(each - seen);  // phase 2 adds one per match
          }
        }
        const unsigned hits = __ballot_sync(kFull, nh > 0);
        const bool slow = __any_sync(kFull, nh > 1);  // a multi-nonzero fiber with several hits
        // hits go to the slice of each lane's fiber: the batch is walked in
        // segments that end at slice boundaries
        const int fend = min(cfirst + 32, F1r);
        int fcur = max(cfirst, F0r);
        while (si < gcount) {
          const int seg_end = min(cur_f1, fend);
          const bool in_seg = f >= fcur && f < seg_end;
          mcur += in_seg ? mf : 0u;
          const unsigned seg = __ballot_sync(kFull, in_seg);
          const unsigned hs = hits & seg;
          if (hs) {
            int before, tot;
            if (!slow) {
              before = __popc(hs & lt);
              tot = __popc(hs);
            } else {
              const int x = in_seg ? nh : 0;
              const int inc = warp_inclusive_scan(x);
              before = inc - x;
              tot = __shfl_sync(kFull, inc, 31);
            }
            if (ovf || nrec + tot > P.hit_cap) {
              ovf = true;  // the slice goes to the single-pass kernel
            } else {
              if (in_seg && nh > 0) {
                HitRec* row = hrow + nrec + before;
                HitRec rec;
                rec.j = j;
                rec.k = k;
                rec.b = b;
                if (nz == 1) {
                  st_rec(row, rec);
                } else {
                  unsigned long long bc[W];
                  load_bm<W>(P.cbm + (int64_t)j * W, bc);
                  for (int64_t z = z0; z < z0 + nz; z++) {
                    const int64_t kz = P.idx2[z];
                    unsigned long long bz[W];
                    load_bm<W>(P.dbm + kz * W, bz);
                    unsigned long long m = 0ull;
#pragma unroll
                    for (int w = 0; w < W; w++) m |= bc[w] & bz[w];
                    if (m != 0ull) {
                      rec.k = (int)kz;
                      rec.b = P.vals[z];
                      *row++ = rec;
                    }
                  }
                }
              }
              nrec += tot;
            }
          }
          if (cur_f1 > fend) break;  // the slice continues in a later batch
          const unsigned long long ds = warp_sum((unsigned long long)mcur);
          if (lane == 0) {
            P.rec_cnt[i0 + si] = ovf ? -1 : nrec;
            P.dsum[i0 + si] = ds;
            if (ovf) P.ovf_list[atomicAdd(P.ovf, 1ull)] = i0 + si;
          }
          mcur = 0;
          si++;
          hrow += P.hit_cap;
          fcur = cur_f1;
          cur_f1 = __shfl_sync(kFull, p1r, min(si + 1, 31));
          nrec = 0;
          ovf = false;
        }
      }
      __syncwarp();
      if (n1 < base + nch) {
        ring_issue1(P, Q, lane, n1, fb0 + (int64_t)(n1 - base) * kMC);
        n1++;
      }
      if (n2 < base + nch) {
        ring_issue2(P, Q, lane, n2);
        n2++;
      }
    }
    np = base + nch;
  }
}

// Phase 2: lanes over the slice's hits (every lane holds one, so the bit walks
// run on full warps).  Each hit's shared columns become match records; the
// slice's distinct columns give its row length in A.  The next round's hit
// records and the next slice's head (its hit count and first records) are
// loaded before the current round is expanded: the record stream's DRAM
// latency stays off the chain record -> bitmaps / row starts -> match records.
#ifndef SPX_MINB
#define SPX_MINB 1
#endif
template <int W>
__global__ void __launch_bounds__(256, SPX_MINB) mttkrp_sparse_expand_kernel(const SparseParams P) {
  __shared__ uint32_t pres[8][32];
  const int lane = (int)lane_id();
  const int wl = threadIdx.x >> 5;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t keep = l2_evict_last_policy();
  unsigned long long mults = 0;
  // a slice's head: its hit count and (whatever the count) the first 32 records of its row
  auto head = [&](int64_t i, int& n, HitRec& r0) {
    n = 0;
    r0.j = r0.k = 0;
    r0.b = 0.0;
    if (i < P.I) {
      n = P.rec_cnt[i];
      if (lane < P.hit_cap) r0 = ld_rec(P.hits + i * P.hit_cap + lane);
    }
  };
  int n_nxt;
  HitRec r_nxt;
  head(warp, n_nxt, r_nxt);
  for (int64_t i = warp; i < P.I; i += nwarps) {
    const int n = n_nxt;
    HitRec rec = r_nxt;
    head(i + nwarps, n_nxt, r_nxt);
    if (n < 0) continue;  // evaluated by the single-pass kernel
    if (n == 0) {
      // no hit: an empty row; the multiplications that found nothing still count
      if (lane == 0) {
        P.mat_cnt[i] = 0;
        mults += P.dsum[i];
      }
      continue;
    }
    const HitRec* hrow = P.hits + i * P.hit_cap;
    MatRec* mrow = P.mats + i * P.mat_cap;
    pres[wl][lane] = 0u;
    __syncwarp();
    int nmat = 0;
    bool ovf = false;
    for (int t0 = 0; t0 < n; t0 += 32) {
      const int t = t0 + lane;
      // the next round's records
      HitRec rnext;
      rnext.j = rnext.k = 0;
      rnext.b = 0.0;
      if (t + 32 < n) rnext = ld_rec(hrow + t + 32);
      unsigned long long bc[W], bd[W];
#pragma unroll
      for (int w = 0; w < W; w++) bc[w] = bd[w] = 0ull;
      int64_t d0 = 0, c0 = 0;
      int x = 0;
      if (t < n) {
        load_bm_keep<W>(P.cbm + (int64_t)rec.j * W, keep, bc);
        load_bm_keep<W>(P.dbm + (int64_t)rec.k * W, keep, bd);
        d0 = __ldg(P.dpos + rec.k);
        c0 = __ldg(P.cpos + rec.j);
#pragma unroll
        for (int w = 0; w < W; w++) x += __popcll(bc[w] & bd[w]);
      }
      const int inc = warp_inclusive_scan(x);
      const int tot = __shfl_sync(kFull, inc, 31);
      if (nmat + tot > P.mat_cap) {
        ovf = true;
        break;
      }
      if (x > 0) {
        MatRec* out = mrow + nmat + inc - x;
        int pc = 0, pd = 0;
#pragma unroll
        for (int w = 0; w < W; w++) {
          unsigned long long mm = bc[w] & bd[w];
          while (mm) {
            const int bit = __ffsll((long long)mm) - 1;
            const unsigned long long below = (1ull << bit) - 1ull;
            const int rc = pc + __popcll(bc[w] & below);
            const int rd = pd + __popcll(bd[w] & below);
            const unsigned r = (unsigned)(w * 64 + bit);
            MatRec m;
            m.c = (int)(c0 + rc);
            m.meta = r | ((unsigned)t << 10);
            m.d = d0 + rd;
            st_rec(out++, m);
            atomicOr(&pres[wl][r >> 5], 1u << (r & 31u));
            mm &= mm - 1ull;
          }
          pc += __popcll(bc[w]);
          pd += __popcll(bd[w]);
        }
      }
      nmat += tot;
      rec = rnext;
    }
    __syncwarp();
    if (ovf) {
      if (lane == 0) {
        P.rec_cnt[i] = -1;
        P.ovf_list[atomicAdd(P.ovf, 1ull)] = i;
      }
    } else {
      const int cnt = warp_sum(__popc(pres[wl][lane]));
      if (lane == 0) {
        P.out_pos[i + 1] = cnt;
        P.mat_cnt[i] = nmat;
        mults += P.dsum[i] + (unsigned long long)nmat;
      }
    }
    __syncwarp();
  }
  if (lane == 0 && mults) atomicAdd(P.mults, mults);
}

// Phase 3 (after the row-pointer scan): w0 = 0 + b·D(k,r) (final: one nonzero
// per fiber and column, see phase 1), w1(r) += w0·C(j,r) into the warp's
// workspace (kAU records per lane in flight), then the sorted drain straight
// into the slice's CSR row.  The drain leaves the workspace reset for the
// next slice.
#ifndef SPA_U
#define SPA_U 4
#endif
constexpr int kAU = SPA_U;
#ifndef SPA_MINB
#define SPA_MINB 1
#endif
__global__ void __launch_bounds__(kSpWarps * 32, SPA_MINB) mttkrp_sparse_accum_kernel(const SparseParams P) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = (int)lane_id();
  const int warp = threadIdx.x >> 5;
  const int64_t R = P.R;
  const int nwords = (int)((R + 31) / 32);
  const size_t ws_bytes = ((size_t)R * 8 + (size_t)nwords * 4 + 15) & ~(size_t)15;
  double* wv = reinterpret_cast<double*>(smem_raw + (size_t)warp * ws_bytes);
  uint32_t* wb = reinterpret_cast<uint32_t*>(wv + R);
  for (int64_t r = lane; r < R; r += 32) wv[r] = 0.0;
  for (int w = lane; w < nwords; w += 32) wb[w] = 0u;
  __syncwarp();
  const uint64_t keep = l2_evict_last_policy();
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = gw; i < P.I; i += nwarps) {
    if (P.rec_cnt[i] <= 0) continue;  // empty, or written by the single-pass kernel
    const int n = P.mat_cnt[i];
    const int64_t dst = P.out_pos[i];
    const MatRec* mrow = P.mats + i * P.mat_cap;
    const HitRec* hrow = P.hits + i * P.hit_cap;
    for (int t0 = 0; t0 < n; t0 += 32 * kAU) {
      MatRec m[kAU];
      double cv[kAU], dv[kAU], b[kAU];
#pragma unroll
      for (int u = 0; u < kAU; u++) {
        const int t = t0 + u * 32 + lane;
        m[u].c = 0;
        m[u].meta = 0u;
        m[u].d = 0;
        if (t < n) m[u] = ld_rec(mrow + t);
      }
#pragma unroll
      for (int u = 0; u < kAU; u++) {
        const bool on = t0 + u * 32 + lane < n;
        cv[u] = on ? ld_keep(P.cvals + m[u].c, keep) : 0.0;
        dv[u] = on ? ld_keep(P.dvals + m[u].d, keep) : 0.0;
        b[u] = on ? __ldcs(&hrow[m[u].meta >> 10].b) : 0.0;  // streamed like the records
      }
#pragma unroll
      for (int u = 0; u < kAU; u++)
        if (t0 + u * 32 + lane < n) {
          const double w0 = add_rn(0.0, mul_rn(b[u], dv[u]));
          ws_add(wv, wb, (int64_t)(m[u].meta & 1023u), mul_rn(w0, cv[u]));
        }
    }
    __syncwarp();
    int64_t* oi = P.out_idx + dst;
    double* ov = P.out_vals + dst;
    int out = 0;
    for (int w = 0; w < nwords; w++) {
      const uint32_t bits = wb[w];
      if (bits == 0) continue;
      if ((bits >> lane) & 1u) {
        const int rank = __popc(bits & ((1u << lane) - 1u));
        const int64_t r = (int64_t)w * 32 + lane;
        __stcs(reinterpret_cast<long long*>(oi) + out + rank, (long long)r);
        __stcs(ov + out + rank, wv[r]);
        wv[r] = 0.0;
      }
      out += __popc(bits);
    }
    __syncwarp();
    for (int w = lane; w < nwords; w += 32) wb[w] = 0u;
    __syncwarp();
  }
}

// Copies staged rows (stride R) into the compact CSR: a warp per row.
__global__ void mttkrp_sparse_compact_kernel(const SparseParams P) {
  const int lane = (int)lane_id();
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < P.I; i += nwarps) {
    const int64_t dst = P.out_pos[i], n = P.out_pos[i + 1] - dst;
    const int64_t* si = stage_idx_row(P, i);
    const double* sv = stage_vals_row(P, i);
    for (int64_t t = lane; t < n; t += 32) {
      P.out_idx[dst + t] = si[t];
      P.out_vals[dst + t] = sv[t];
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
    const int64_t ncb = (R + 31) / 32;
    const bool fast = R == 32 && ((uintptr_t)P.C % 16 == 0) && ((uintptr_t)P.D % 16 == 0);
    // ~16 chunks per resident warp: small enough to balance the skewed
    // slices, large enough to amortize a chunk's bookkeeping
    const int64_t warps = (int64_t)sms * 32;
#ifndef DQ_CHUNKS_PER_WARP
#define DQ_CHUNKS_PER_WARP 32
#endif
#ifndef DQ_CHUNK_MIN
#define DQ_CHUNK_MIN 512
#endif
    P.chunk_nnz = std::max<int64_t>(DQ_CHUNK_MIN, ceil_div(std::max<int64_t>(B->nnz, 1), warps * DQ_CHUNKS_PER_WARP));
    P.nchunks = std::max<int64_t>(1, ceil_div(B->nnz, P.chunk_nnz));
    P.part = call.scratch_n<double>((size_t)(ncb * P.nchunks * 64));
    P.part_slice = call.scratch_n<int64_t>((size_t)(2 * P.nchunks));
    P.chunk_fa = call.scratch_n<int64_t>((size_t)P.nchunks + 1);
    P.chunk_s = call.scratch_n<int64_t>((size_t)P.nchunks + 1);
    P.counter = static_cast<unsigned long long*>(call.scratch_zero(16));
    if (B->nfibers > 0) {
      call.before_launch("mttkrp_dense_bounds");
      mttkrp_dense_bounds_kernel<<<(unsigned)ceil_div(P.nchunks + 1, 256), 256, 0, call.stream()>>>(P);
      call.after_launch();
      call.before_launch(fast ? "mttkrp_dense32" : "mttkrp_dense_generic");
      if (fast)
      {
        const bool a32 = ((uintptr_t)P.C % 32 == 0) && ((uintptr_t)P.D % 32 == 0);
        if (a32)
          mttkrp_dense32q_kernel<true><<<(unsigned)(sms * DQ_MINB), 256, 0, call.stream()>>>(P);
        else
          mttkrp_dense32q_kernel<false><<<(unsigned)(sms * DQ_MINB), 256, 0, call.stream()>>>(P);
      }
      else
        mttkrp_dense_generic_kernel<<<(unsigned)(sms * 4), 256, 0, call.stream()>>>(P);
      call.after_launch();
      FixupLevels L{};
      L.nb1 = ceil_div(P.nchunks, (int64_t)kFixBlock);
      L.nb2 = ceil_div(L.nb1, (int64_t)kFixBlock);
      double* bsum1 = call.scratch_n<double>((size_t)(ncb * L.nb1 * 32));
      int64_t* bslice1 = call.scratch_n<int64_t>((size_t)L.nb1);
      double* bsum2 = call.scratch_n<double>((size_t)(ncb * L.nb2 * 32));
      int64_t* bslice2 = call.scratch_n<int64_t>((size_t)L.nb2);
      L.bsum1 = bsum1;
      L.bslice1 = bslice1;
      L.bsum2 = bsum2;
      L.bslice2 = bslice2;
      call.before_launch("mttkrp_dense_blocksum");
      mttkrp_dense_blocksum_kernel<<<(unsigned)std::min<int64_t>(ceil_div(L.nb1 * ncb, 8), (int64_t)sms * 8),
                                     256, 0, call.stream()>>>(P.part_slice, 2, P.part, 64, P.nchunks * 64,
                                                              P.nchunks, ncb, bsum1, bslice1, L.nb1);
      mttkrp_dense_blocksum_kernel<<<(unsigned)std::min<int64_t>(ceil_div(L.nb2 * ncb, 8), (int64_t)sms * 8),
                                     256, 0, call.stream()>>>(bslice1, 1, bsum1, 32, L.nb1 * 32, L.nb1, ncb,
                                                              bsum2, bslice2, L.nb2);
      call.after_launch();
      call.before_launch("mttkrp_dense_fixup");
      mttkrp_dense_fixup_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(P.nchunks, 8), (int64_t)sms * 8)),
                                  256, 0, call.stream()>>>(P, L);
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

namespace stamgpu {
namespace {
// staging budget of the sparse path (bytes): see mttkrp_sparse_blocked
int64_t sparse_stage_budget() {
  int64_t mb = 4096;
  if (const char* e = std::getenv("STAM_SPARSE_STAGE_MB")) mb = std::max(1, std::atoi(e));
  return mb << 20;
}

__global__ void mttkrp_pos_shift_kernel(int64_t* p, int64_t n, int64_t delta) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    p[t] += delta;
}

// Host CSF input (the e2e case): the CSF is 6.4 GB at config 5 and PCIe H2D
// (~55 GB/s) bounds the call, so the slices go up in nnz-balanced blocks on
// the copy stream, all issued at once into full-size device arrays (absolute
// positions stay valid), each block is evaluated by the device path as soon
// as its copies land, and its result rows go down on the d2h stream into a
// pinned host result sized by the bound I x R while later blocks upload.
int mttkrp_sparse_streamed(stam_cuda_ctx* ctx, const stam_csf3_view* B, const stam_csr_view* Cv,
                           const stam_csr_view* Dv, const stam_options* opts,
                           stam_csr_result* A, stam_stats* stats) {
  return guarded([&] {
    stam_options o = *opts;
    o.result_mem = STAM_MEM_DEVICE;
    o.timing = 0;
    Call call(reinterpret_cast<Ctx*>(ctx), &o, stats);
    check_csf3_view(B, "mttkrp B");
    check_csr_view(Cv, "mttkrp C");
    check_csr_view(Dv, "mttkrp D");
    if (Cv->nrows != B->dims[1] || Dv->nrows != B->dims[2])
      fail(STAM_ERR_DIMENSION_MISMATCH, "mttkrp: C rows != dim 1 or D rows != dim 2");
    if (Cv->ncols != Dv->ncols) fail(STAM_ERR_DIMENSION_MISMATCH, "mttkrp: C and D ranks differ");
    const int64_t I = B->dims[0], R = Cv->ncols;
    auto dev_csr = [&](const stam_csr_view* v) {
      stam_csr_view d = *v;
      d.pos = call.device_input(v->pos, (size_t)v->nrows + 1, v->mem);
      d.idx = call.device_input(v->idx, (size_t)v->nnz, v->mem);
      d.vals = call.device_input(v->vals, (size_t)v->nnz, v->mem);
      d.mem = STAM_MEM_DEVICE;
      return d;
    };
    const stam_csr_view Cd = dev_csr(Cv), Dd = dev_csr(Dv);
    const int64_t* d_pos1 = call.device_input(B->pos1, (size_t)I + 1, B->mem);
    auto* d_idx1 = call.host_staging<int64_t>((size_t)B->nfibers);
    auto* d_pos2 = call.host_staging<int64_t>((size_t)B->nfibers + 1);
    auto* d_idx2 = call.host_staging<int64_t>((size_t)B->nnz);
    auto* d_vals = call.host_staging<double>((size_t)B->nnz);
    // nnz-balanced slice blocks (~16M nonzeros each)
    int64_t nblocks = std::max<int64_t>(2, std::min<int64_t>(64, ceil_div(B->nnz, (int64_t)1 << 24)));
    nblocks = std::max(nblocks, ceil_div(I * R * 22, sparse_stage_budget()));
    nblocks = std::min(nblocks, I);
    std::vector<int64_t> sb{0};
    for (int64_t b = 1; b < nblocks; b++) {
      const int64_t target = B->nnz * b / nblocks;
      // first slice whose nonzeros start at or after target
      int64_t lo = sb.back(), hi = I;
      while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        if (B->pos2[B->pos1[mid]] < target) lo = mid + 1; else hi = mid;
      }
      if (lo > sb.back() && lo < I) sb.push_back(lo);
    }
    sb.push_back(I);
    nblocks = (int64_t)sb.size() - 1;
    std::vector<cudaEvent_t> landed((size_t)nblocks, nullptr);
    for (int64_t b = 0; b < nblocks; b++) {
      const int64_t f0 = B->pos1[sb[(size_t)b]], f1 = B->pos1[sb[(size_t)b + 1]];
      const int64_t z0 = B->pos2[f0], z1 = B->pos2[f1];
      call.copy_range(d_idx1 + f0, B->idx1 + f0, sizeof(int64_t) * (size_t)(f1 - f0));
      call.copy_range(d_pos2 + f0, B->pos2 + f0, sizeof(int64_t) * (size_t)(f1 - f0 + 1));
      call.copy_range(d_idx2 + z0, B->idx2 + z0, sizeof(int64_t) * (size_t)(z1 - z0));
      call.copy_range(d_vals + z0, B->vals + z0, sizeof(double) * (size_t)(z1 - z0));
      // own events: the per-block device calls below reuse the context's pool
      STAM_CUDA_CHECK(cudaEventCreateWithFlags(&landed[(size_t)b], cudaEventDisableTiming));
      STAM_CUDA_CHECK(cudaEventRecord(landed[(size_t)b], call.ctx()->copy_stream));
    }
    struct EventsGuard {
      std::vector<cudaEvent_t>& ev;
      ~EventsGuard() {
        for (auto e : ev)
          if (e) cudaEventDestroy(e);
      }
    } events_guard{landed};
    call.alloc_csr_result_host(A, I, R, I * R);
    A->pos[0] = 0;
    std::vector<stam_csr_result> parts((size_t)nblocks);
    int64_t off = 0, launches = 0, mults = 0;
    int status = STAM_OK;
    const int sms = call.ctx()->num_sms;
    for (int64_t b = 0; b < nblocks && status == STAM_OK; b++) {
      const int64_t s0 = sb[(size_t)b], s1 = sb[(size_t)b + 1];
      call.wait(landed[(size_t)b]);
      stam_csf3_view Bv = *B;
      Bv.dims[0] = s1 - s0;
      Bv.pos1 = d_pos1 + s0;
      Bv.idx1 = d_idx1;
      Bv.pos2 = d_pos2;
      Bv.idx2 = d_idx2;
      Bv.vals = d_vals;
      Bv.mem = STAM_MEM_DEVICE;
      stam_csr_result& Ab = parts[(size_t)b];
      std::memset(&Ab, 0, sizeof(Ab));
      stam_stats st{};
      status = stam_cuda_mttkrp_sparse(ctx, &Bv, &Cd, &Dd, &o, &Ab, &st);
      if (status != STAM_OK) break;
      mults += st.mults;
      launches += st.kernel_launches;
      mttkrp_pos_shift_kernel<<<(unsigned)std::min<int64_t>(ceil_div(s1 - s0, 256), (int64_t)sms * 4),
                                256, 0, call.stream()>>>(Ab.pos + 1, s1 - s0, off);
      STAM_CUDA_CHECK(cudaGetLastError());
      cudaEvent_t ready = call.event();
      STAM_CUDA_CHECK(cudaEventRecord(ready, call.stream()));
      call.d2h_range(A->pos + s0 + 1, Ab.pos + 1, sizeof(int64_t) * (size_t)(s1 - s0), ready);
      call.d2h_range(A->idx + off, Ab.idx, sizeof(int64_t) * (size_t)Ab.nnz, nullptr);
      call.d2h_range(A->vals + off, Ab.vals, sizeof(double) * (size_t)Ab.nnz, nullptr);
      off += Ab.nnz;
    }
    call.finish_csr_result_host(A, off);  // joins the downloads
    for (auto& Ab : parts)
      if (Ab.handle) stam_cuda_release(ctx, Ab.handle);
    if (status != STAM_OK) {
      const std::string msg = stam_cuda_last_error();
      fail(status, msg);
    }
    call.finish();
    stam_stats* st = call.stats();
    st->mults = mults;
    st->adds = mults;
    st->ws_resets = B->nfibers + I;
    st->appends = off;
    st->kernel_launches += launches;
  });
}
// Bounded staging (ADVICE: the fixed-stride staging is 16·I·R bytes whatever
// the output's sparsity, 2 GB at config 5): when it would exceed the budget
// (STAM_SPARSE_STAGE_MB, default 4096), slices are evaluated in blocks whose
// staging fits, each by the device path, and the block results are placed
// into one exact CSR (device-to-device copies).
int mttkrp_sparse_blocked(stam_cuda_ctx* ctx, const stam_csf3_view* B, const stam_csr_view* Cv,
                          const stam_csr_view* Dv, const stam_options* opts, stam_csr_result* A,
                          stam_stats* stats) {
  return guarded([&] {
    stam_options o = *opts;
    o.result_mem = STAM_MEM_DEVICE;
    o.timing = 0;
    Call call(reinterpret_cast<Ctx*>(ctx), opts, stats);
    check_csf3_view(B, "mttkrp B");
    check_csr_view(Cv, "mttkrp C");
    check_csr_view(Dv, "mttkrp D");
    const int64_t I = B->dims[0], R = Cv->ncols;
    auto dev_csr = [&](const stam_csr_view* v) {
      stam_csr_view d = *v;
      d.pos = call.device_input(v->pos, (size_t)v->nrows + 1, v->mem);
      d.idx = call.device_input(v->idx, (size_t)v->nnz, v->mem);
      d.vals = call.device_input(v->vals, (size_t)v->nnz, v->mem);
      d.mem = STAM_MEM_DEVICE;
      return d;
    };
    const stam_csr_view Cd = dev_csr(Cv), Dd = dev_csr(Dv);
    stam_csf3_view Bd = *B;
    Bd.pos1 = call.device_input(B->pos1, (size_t)I + 1, B->mem);
    Bd.idx1 = call.device_input(B->idx1, (size_t)B->nfibers, B->mem);
    Bd.pos2 = call.device_input(B->pos2, (size_t)B->nfibers + 1, B->mem);
    Bd.idx2 = call.device_input(B->idx2, (size_t)B->nnz, B->mem);
    Bd.vals = call.device_input(B->vals, (size_t)B->nnz, B->mem);
    Bd.mem = STAM_MEM_DEVICE;
    const int64_t per = std::max<int64_t>(1, sparse_stage_budget() / (22 * R));  // slices per block
    const int64_t nblocks = ceil_div(I, per);
    std::vector<stam_csr_result> parts((size_t)nblocks);
    int64_t total = 0, launches = 0, mults = 0;
    int status = STAM_OK;
    for (int64_t b = 0; b < nblocks && status == STAM_OK; b++) {
      const int64_t s0 = b * per, s1 = std::min(I, s0 + per);
      stam_csf3_view Bv = Bd;
      Bv.dims[0] = s1 - s0;
      Bv.pos1 = Bd.pos1 + s0;
      stam_csr_result& Ab = parts[(size_t)b];
      std::memset(&Ab, 0, sizeof(Ab));
      stam_stats st{};
      status = stam_cuda_mttkrp_sparse(ctx, &Bv, &Cd, &Dd, &o, &Ab, &st);
      total += Ab.nnz;
      mults += st.mults;
      launches += st.kernel_launches;
    }
    if (status == STAM_OK) {
      call.alloc_csr_result(A, I, R, total);
      STAM_CUDA_CHECK(cudaMemsetAsync(A->pos, 0, sizeof(int64_t), call.stream()));
      int64_t off = 0;
      const int sms = call.ctx()->num_sms;
      for (int64_t b = 0; b < nblocks; b++) {
        const int64_t s0 = b * per, s1 = std::min(I, s0 + per);
        const stam_csr_result& Ab = parts[(size_t)b];
        STAM_CUDA_CHECK(cudaMemcpyAsync(A->pos + s0 + 1, Ab.pos + 1, sizeof(int64_t) * (size_t)(s1 - s0),
                                        cudaMemcpyDeviceToDevice, call.stream()));
        mttkrp_pos_shift_kernel<<<(unsigned)std::min<int64_t>(ceil_div(s1 - s0, 256), (int64_t)sms * 4),
                                  256, 0, call.stream()>>>(A->pos + s0 + 1, s1 - s0, off);
        STAM_CUDA_CHECK(cudaGetLastError());
        STAM_CUDA_CHECK(cudaMemcpyAsync(A->idx + off, Ab.idx, sizeof(int64_t) * (size_t)Ab.nnz,
                                        cudaMemcpyDeviceToDevice, call.stream()));
        STAM_CUDA_CHECK(cudaMemcpyAsync(A->vals + off, Ab.vals, sizeof(double) * (size_t)Ab.nnz,
                                        cudaMemcpyDeviceToDevice, call.stream()));
        off += Ab.nnz;
      }
    }
    STAM_CUDA_CHECK(cudaStreamSynchronize(call.stream()));
    for (auto& Ab : parts)
      if (Ab.handle) stam_cuda_release(ctx, Ab.handle);
    if (status != STAM_OK) {
      const std::string msg = stam_cuda_last_error();
      fail(status, msg);
    }
    call.finish_csr_result(A, total);
    call.finish();
    stam_stats* st = call.stats();
    st->mults = mults;
    st->adds = mults;
    st->ws_resets = B->nfibers + I;
    st->appends = total;
    st->kernel_launches += launches;
  });
}

}  // namespace
}  // namespace stamgpu

extern "C" int stam_cuda_mttkrp_sparse(stam_cuda_ctx* ctx, const stam_csf3_view* B,
                                       const stam_csr_view* Cv, const stam_csr_view* Dv,
                                       const stam_options* opts, stam_csr_result* A,
                                       stam_stats* stats) {
  using namespace stamgpu;
  if (ctx && B && Cv && Dv && opts && B->mem == STAM_MEM_HOST && opts->result_mem == STAM_MEM_HOST &&
      B->nnz >= ((int64_t)1 << 24) && B->dims[0] > 1 && Cv->ncols > 0 && Cv->ncols <= 512 &&
      B->dims[0] * Cv->ncols <= ((int64_t)1 << 29) && B->pos1 && B->pos2 &&
      std::getenv("STAM_NO_STREAM") == nullptr)
    return mttkrp_sparse_streamed(ctx, B, Cv, Dv, opts, A, stats);
  if (ctx && B && Cv && Dv && opts && B->dims[0] > 1 && Cv->ncols > 0 &&
      B->dims[0] * Cv->ncols * 22 > sparse_stage_budget())
    return mttkrp_sparse_blocked(ctx, B, Cv, Dv, opts, A, stats);
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
    const size_t smem = ws_bytes * kSpWarps + match_queue_bytes() * kSpWarps;
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
    auto* ctl = static_cast<uint64_t*>(call.scratch_zero(8 * 8));
    P.tile_counter = reinterpret_cast<unsigned long long*>(ctl);
    P.mults = reinterpret_cast<unsigned long long*>(ctl + 1);
    // row pointers: counts at [i+1], scanned in place
    int64_t* cpos = static_cast<int64_t*>(call.scratch_zero(sizeof(int64_t) * ((size_t)I + 1)));
    P.out_pos = cpos;
    // factor-row column bitmaps when R fits W <= 8 words
    const int64_t words = (R + 63) / 64;
    const int W = words <= 1 ? 1 : words <= 2 ? 2 : words <= 4 ? 4 : words <= 8 ? 8 : 0;
    const size_t smem_w = ws_bytes * kSpWarps + match_queue_bytes() * kSpWarps;
    // both bitmaps in one block; rows are read with 256-bit loads (W = 4):
    // 32-byte aligned
    const size_t bm_words = (size_t)((Cv->nrows + Dv->nrows) * (W > 0 ? W : 1)) + 8;
    auto* bm_raw = W > 0 ? call.scratch_n<unsigned long long>(bm_words) : nullptr;
    auto* bm_base = reinterpret_cast<unsigned long long*>(((uintptr_t)bm_raw + 31) & ~(uintptr_t)31);
    size_t bm_used = 0;
    auto build_bm = [&](const int64_t* pos, const int64_t* idx, int64_t nrows) {
      unsigned long long* bm = bm_base + bm_used;
      bm_used += (size_t)(nrows * W);
      const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(nrows, 256),
                                                        (int64_t)call.ctx()->num_sms * 8);
      call.before_launch("mttkrp_factor_bitmap");
      switch (W) {
        case 1: factor_bitmap_kernel<1><<<grid, 256, 0, call.stream()>>>(pos, idx, nrows, bm); break;
        case 2: factor_bitmap_kernel<2><<<grid, 256, 0, call.stream()>>>(pos, idx, nrows, bm); break;
        case 4: factor_bitmap_kernel<4><<<grid, 256, 0, call.stream()>>>(pos, idx, nrows, bm); break;
        default: factor_bitmap_kernel<8><<<grid, 256, 0, call.stream()>>>(pos, idx, nrows, bm); break;
      }
      call.after_launch();
      return bm;
    };
    if (W > 0) {
      P.cbm = build_bm(P.cpos, P.cidx, Cv->nrows);
      P.dbm = build_bm(P.dpos, P.didx, Dv->nrows);
    }
    auto launch = [&](auto kern, cudaStream_t st) {
      STAM_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem_w));
      int per_sm = 1;
      STAM_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSpWarps * 32,
                                                                    smem_w));
      const int64_t grid = std::min<int64_t>(ceil_div(I, kSpWarps),
                                             (int64_t)std::max(1, per_sm) * call.ctx()->num_sms);
      call.before_launch("mttkrp_sparse", st);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)grid);
      cfg.blockDim = dim3(kSpWarps * 32);
      cfg.dynamicSmemBytes = smem_w;
      cfg.stream = st;
      cfg.attrs = nullptr;
      cfg.numAttrs = 0;
      STAM_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, P));
      call.after_launch(st);
    };
    auto launch_single = [&](cudaStream_t st) {
      switch (W) {
        case 1: launch(mttkrp_sparse_kernel<1>, st); break;
        case 2: launch(mttkrp_sparse_kernel<2>, st); break;
        case 4: launch(mttkrp_sparse_kernel<4>, st); break;
        case 8: launch(mttkrp_sparse_kernel<8>, st); break;
        default: launch(mttkrp_sparse_kernel<0>, st); break;
      }
    };
    // the single-pass kernel over one of the slice lists of the three-phase path
    auto launch_list = [&](int mode, cudaStream_t st) {
      const SparseParams saved = P;
      P.slice_list = saved.ovf_list;
      P.nlist_dev = saved.ovf;
      P.mode = mode;
      if (mode == 2) P.mults = nullptr;  // counted by the first run
      P.tile_counter = reinterpret_cast<unsigned long long*>(ctl + 4 + mode);
      launch_single(st);
      P = saved;
    };
    // three phases (filter -> hits, expand -> matches + row lengths, accumulate
    // + drain) when coordinates fit int32 and most fibers hold one nonzero (a
    // longer fiber's hits are written by one lane).  Rows per slice: hits and
    // matches are sized from the rank (a row of A holds at most R entries;
    // the sparse-factor workloads fill a fraction of it), slices that exceed
    // them go to the single-pass kernel.
    const int hit_cap = std::max(32, (int)((5 * R) / 8) & ~7);
    const int mat_cap = std::max(32, (int)((3 * R) / 4) & ~7);
    const char* tp = std::getenv("STAM_SP_PHASES");
    const bool three = W > 0 && B->dims[1] < (INT32_MAX - 64) / kMGroup && B->dims[2] < INT32_MAX && R <= 512 &&
                       Cv->nnz < INT32_MAX &&
                       B->nnz <= B->nfibers + B->nfibers / 8 && !(tp && std::atoi(tp) == 1);
    const int sms = call.ctx()->num_sms;
    if (!three) {
      P.stage = call.scratch_n<int64_t>((size_t)(2 * I * R));
      launch_single(call.stream());
    } else {
      P.hit_cap = hit_cap;
      P.mat_cap = mat_cap;
      P.hits = static_cast<HitRec*>(call.scratch(sizeof(HitRec) * (size_t)I * hit_cap));
      P.mats = static_cast<MatRec*>(call.scratch(sizeof(MatRec) * (size_t)I * mat_cap));
      P.rec_cnt = call.scratch_n<int32_t>((size_t)I);
      P.mat_cnt = call.scratch_n<int32_t>((size_t)I);
      P.dsum = reinterpret_cast<unsigned long long*>(call.scratch_n<int64_t>((size_t)I));
      // slices left to the single-pass kernel (listed by the filter and by the expansion)
      P.ovf = reinterpret_cast<unsigned long long*>(ctl + 2);
      P.ovf_list = call.scratch_n<int64_t>((size_t)I);
      auto aligned16 = [](const void* q) { return ((uintptr_t)q & 15u) == 0; };
      P.tma_ok = aligned16(P.idx1) && aligned16(P.pos2) && aligned16(P.idx2) && aligned16(P.vals) &&
                 std::getenv("STAM_SP_NO_TMA") == nullptr;
      auto filter = [&](auto kern) {
        const size_t msmem = sizeof(MatchRing) * kSpWarps;
        STAM_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)msmem));
        int per_sm = 1;
        STAM_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSpWarps * 32, msmem));
        const int64_t grid = std::min<int64_t>(ceil_div(ceil_div(I, (int64_t)kMGroup), kSpWarps),
                                               (int64_t)std::max(1, per_sm) * sms);
        call.before_launch("mttkrp_sparse_filter");
        kern<<<(unsigned)grid, kSpWarps * 32, msmem, call.stream()>>>(P);
        call.after_launch();
      };
      switch (W) {
        case 1: filter(mttkrp_sparse_filter_kernel<1>); break;
        case 2: filter(mttkrp_sparse_filter_kernel<2>); break;
        case 4: filter(mttkrp_sparse_filter_kernel<4>); break;
        default: filter(mttkrp_sparse_filter_kernel<8>); break;
      }
      auto expand = [&](auto kern) {
        int per_sm = 1;
        STAM_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0));
        call.before_launch("mttkrp_sparse_expand");
        kern<<<(unsigned)std::min<int64_t>(ceil_div(I, 8), (int64_t)std::max(1, per_sm) * sms), 256, 0,
               call.stream()>>>(P);
        call.after_launch();
      };
      switch (W) {
        case 1: expand(mttkrp_sparse_expand_kernel<1>); break;
        case 2: expand(mttkrp_sparse_expand_kernel<2>); break;
        case 4: expand(mttkrp_sparse_expand_kernel<4>); break;
        default: expand(mttkrp_sparse_expand_kernel<8>); break;
      }
      // the listed slices: row lengths by the single-pass kernel (the list length
      // stays on the device; beside the expansion on a second stream the
      // kernel's large CTAs cost more residency than the overlap gains:
      // 5.26 vs 4.89 ms at config 5)
      launch_list(1, call.stream());
    }
    size_t temp_bytes = 0;
    STAM_CUDA_CHECK(cub::DeviceScan::InclusiveSum(nullptr, temp_bytes, cpos + 1, cpos + 1, I,
                                                  call.stream()));
    void* temp = call.scratch(temp_bytes);
    call.before_launch("mttkrp_sparse_scan");
    STAM_CUDA_CHECK(cub::DeviceScan::InclusiveSum(temp, temp_bytes, cpos + 1, cpos + 1, I,
                                                  call.stream()));
    call.after_launch();
    int64_t ctlv[2];
    call.read_scalars(reinterpret_cast<int64_t*>(ctl), 2, ctlv);
    const int64_t nnz = call.read_scalar(cpos + I);
    call.alloc_csr_result(A, I, R, nnz);
    STAM_CUDA_CHECK(cudaMemcpyAsync(A->pos, cpos, sizeof(int64_t) * ((size_t)I + 1),
                                    cudaMemcpyDeviceToDevice, call.stream()));
    P.out_idx = A->idx;
    P.out_vals = A->vals;
    if (three) {
      const size_t asmem = ws_bytes * kSpWarps;
      STAM_CUDA_CHECK(cudaFuncSetAttribute(mttkrp_sparse_accum_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)asmem));
      int per_sm = 1;
      STAM_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mttkrp_sparse_accum_kernel,
                                                                    kSpWarps * 32, asmem));
      const int64_t grid = std::min<int64_t>(ceil_div(I, kSpWarps), (int64_t)std::max(1, per_sm) * sms);
      // the listed slices again, now straight into their CSR rows
      launch_list(2, call.stream());
      call.before_launch("mttkrp_sparse_accum");
      mttkrp_sparse_accum_kernel<<<(unsigned)grid, kSpWarps * 32, asmem, call.stream()>>>(P);
      call.after_launch();
    } else {
      call.before_launch("mttkrp_sparse_compact");
      mttkrp_sparse_compact_kernel<<<(unsigned)std::min<int64_t>(ceil_div(I, 8), (int64_t)sms * 16), 256, 0,
                                     call.stream()>>>(P);
      call.after_launch();
    }
    call.finish_csr_result(A, nnz);
    call.finish();
    stam_stats* st = call.stats();
    st->mults = ctlv[1];
    st->adds = ctlv[1];
    st->ws_resets = B->nfibers + I;
    st->appends = nnz;
  });
}
