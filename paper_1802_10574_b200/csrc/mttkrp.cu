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
//  sparse — a warp per slice (claimed dynamically), lanes over fibers; per
//           fiber, w0 is evaluated only at C_j's stored coordinates
//           (presence-checked; the C_j and D_k column ids are held in
//           registers and intersected all-pairs); w1 is a dense R-wide
//           shared-memory workspace with a presence bitmap, drained sorted by
//           ballot/popcount into a fixed-stride staging row (a row holds <= R
//           entries); scan + coalesced compaction build the CSR.  (An ordered
//           look-back made every slice wait for the slowest earlier one: 41% of
//           warp samples asleep, profiles/r01_ncu_summary.md.)
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <string>
#include <vector>

#include "common.cuh"
#include "runtime.h"

namespace stamgpu {
namespace {

// Runtime switch for A/B measurements of alternative paths (default on).
inline bool env_flag(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) != 0 : dflt != 0;
}

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
  // heavy slices (computed by mttkrp_dense_heavy_kernel; skipped by the chunked kernels)
  int nheavy;
  const int64_t* heavy_f;     // [nheavy][2] fiber range of each heavy slice
  const unsigned char* heavy_flag;  // [I] 1 for a heavy slice
};

__device__ __forceinline__ bool fiber_is_heavy(const DenseParams& P, int64_t f) {
  bool h = false;
  for (int t = 0; t < P.nheavy; t++) h |= (f >= P.heavy_f[2 * t]) && (f < P.heavy_f[2 * t + 1]);
  return h;
}

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
      if (P.nheavy && P.heavy_flag[st.s]) return;  // mttkrp_dense_heavy_kernel's row
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
        if (P.nheavy && fiber_is_heavy(P, fg + lane)) mlen = 0;  // tiled kernel's fiber
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
      if (!(fb < st.s_end && !st.open) || (P.nheavy && P.heavy_flag[st.s]))
        P.part_slice[2 * c + 1] = -1;
    }
  }
}

// ---------------------------------------------------------------------------
// Heavy slices (R == 32): slices whose fibers are long enough that D rows
// repeat many times inside a block of fibers (config 4's top slices: fibers of
// ~3,200 / 1,100 / 600 nonzeros over K = 28,818).  Work items are blocks of
// kHvFibers consecutive fibers of one heavy slice times a range of k.  A CTA
// walks its item's k range in tiles of kHvTile D rows; each tile is copied
// global -> shared by one cp.async.bulk (TMA, 48 KB contiguous: D is
// row-major) on an mbarrier, double-buffered so the next tile lands while this
// one is consumed.  Every quarter-warp owns 4 fibers and consumes, per tile,
// the nonzeros whose k falls inside it, reading D from shared memory: each D
// row is fetched from L2 once per item instead of once per nonzero (the
// chunked kernel's 256 B per nonzero).  A fiber's w0 partial over the item's k
// range is multiplied into C(j,:) and summed (fixed order) into the item's
// partial row; mttkrp_dense_heavy_reduce adds an item's partials per slice in
// item order (deterministic).
#ifndef HV_FPQ
#define HV_FPQ 2
#endif
constexpr int kHvWarps = 16;
constexpr int kHvFpq = HV_FPQ;                      // fibers per quarter-warp
constexpr int kHvFibers = kHvWarps * 4 * kHvFpq;   // fibers per work item
constexpr int kHvDepth = 3;                          // batches of 8 nonzeros held per fiber
#ifndef HV_TILE
#define HV_TILE 192
#endif
constexpr int kHvTile = HV_TILE;  // D rows per stage (48 KB at R = 32)

struct HeavyItem {
  int64_t f0, f1;  // fibers [f0, f1), f1 - f0 <= kHvFibers, one slice
  int32_t k0, k1;  // k range [k0, k1)
  int32_t slot;    // heavy slice index
  int32_t pad;
};

struct HeavySmem {
  double tile[2][kHvTile * 32];
  double red[kHvWarps][32];
  uint64_t bar[2];
  int item;
};

// Quarter-cooperative lower bound: first z in [z0, z1) with idx2[z] >= k.
// Every quarter of the warp searches its own range; the loop runs while any
// quarter is still narrowing (ballots are warp-wide).
__device__ __forceinline__ int64_t quarter_lower_bound(const int64_t* idx2, int64_t z0, int64_t z1,
                                                       int64_t k, int ql, unsigned qmask) {
  int64_t lo = z0, hi = z1;  // answer in [lo, hi]
  while (__any_sync(kFull, hi - lo > 8)) {
    const bool act = hi - lo > 8;  // uniform within the quarter
    const int64_t step = act ? (hi - lo + 7) >> 3 : 0;
    const int64_t p = lo + (int64_t)ql * step;
    const bool lt = act && p < hi && idx2[p] < k;
    const int nlt = __popc(__ballot_sync(kFull, lt) & qmask);  // samples below k: a prefix
    if (act) {
      if (nlt == 0) {
        hi = lo;
      } else {
        lo = lo + (int64_t)(nlt - 1) * step + 1;
        hi = min(hi, lo - 1 + step);
      }
    }
  }
  // final pass over <= 8 candidates
  const int64_t p = lo + ql;
  const bool lt = p < hi && idx2[p] < k;
  return lo + __popc(__ballot_sync(kFull, lt) & qmask);
}

__global__ void __launch_bounds__(kHvWarps * 32, 1) mttkrp_dense_heavy_kernel(
    const DenseParams P, const HeavyItem* items, int nitems, unsigned long long* claim,
    double* hpart) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  HeavySmem& S = *reinterpret_cast<HeavySmem*>(smem_raw);
  const int lane = (int)lane_id();
  const int warp = threadIdx.x >> 5;
  const int q = lane >> 3, ql = lane & 7;
  const int qbase = lane & ~7;
  const unsigned qmask = 0xffu << qbase;
  // lane columns: 2ql, 2ql+1 and 16+2ql, 16+2ql+1 (a quarter's 16-byte loads
  // of one row are contiguous: conflict-free shared reads)
  const int ca = 2 * ql, cb = 16 + 2 * ql;
  if (threadIdx.x == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t gt = 0;  // tiles consumed by this CTA (stage = gt & 1, parity = (gt >> 1) & 1)
  auto issue = [&](const HeavyItem& it, int t, uint32_t g) {
    const int kt0 = it.k0 + t * kHvTile;
    const int rows = min(kHvTile, it.k1 - kt0);
    const uint32_t bytes = (uint32_t)rows * 256u;
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&S.bar[g & 1], bytes);
    bulk_g2s(S.tile[g & 1], P.D + (int64_t)kt0 * 32, bytes, &S.bar[g & 1]);
  };
  while (true) {
    if (threadIdx.x == 0) S.item = (int)atomicAdd(claim, 1ull);
    __syncthreads();
    const int itn = S.item;
    if (itn >= nitems) break;
    const HeavyItem it = items[itn];
    const int nt = (it.k1 - it.k0 + kHvTile - 1) / kHvTile;
    if (threadIdx.x == 0) {
      issue(it, 0, gt);
      if (nt > 1) issue(it, 1, gt + 1);
    }
    // this quarter's fibers: kHvDepth batches of 8 nonzeros in flight (lane ql
    // holds entry cur + 8d + ql of batch d); batch 0 is being consumed
    int64_t cur[kHvFpq];
    int32_t zrem[kHvFpq];  // entries from cur to the fiber's end
    int used[kHvFpq];
    int kb[kHvFpq][kHvDepth];
    double bb[kHvFpq][kHvDepth];
    double w[kHvFpq][4];
#pragma unroll
    for (int u = 0; u < kHvFpq; u++) {
      const int64_t f = it.f0 + (warp * 4 + q) * kHvFpq + u;
      int64_t z0 = 0, z1 = 0;
      if (f < it.f1) {
        z0 = P.pos2[f];
        z1 = P.pos2[f + 1];
      }
      if (it.k0 > 0) z0 = quarter_lower_bound(P.idx2, z0, z1, it.k0, ql, qmask);
      cur[u] = z0;
      zrem[u] = (int32_t)(z1 - z0);
      used[u] = 0;
#pragma unroll
      for (int d = 0; d < kHvDepth; d++) {
        const int e = 8 * d + ql;
        kb[u][d] = e < zrem[u] ? (int)P.idx2[z0 + e] : INT_MAX;
        bb[u][d] = e < zrem[u] ? P.vals[z0 + e] : 0.0;
      }
#pragma unroll
      for (int x = 0; x < 4; x++) w[u][x] = 0.0;
    }
    for (int t = 0; t < nt; t++, gt++) {
      const int kt0 = it.k0 + t * kHvTile;
      const int kt1 = min(it.k1, kt0 + kHvTile);
      mbar_wait_parity(&S.bar[gt & 1], (gt >> 1) & 1);
      const double* tile = S.tile[gt & 1];
#pragma unroll
      for (int u = 0; u < kHvFpq; u++) {
        while (true) {
          // entries [used, 8) of batch 0 with k < kt1 (a prefix: k sorted)
          const bool in = ql >= used[u] && kb[u][0] < kt1;
          const unsigned m = (__ballot_sync(kFull, in) & qmask) >> qbase;
          const int n = __popc(m);
          const int nmax = __reduce_max_sync(kFull, (unsigned)n);
          if (nmax == 0) break;  // uniform
          for (int e0 = 0; e0 < nmax; e0 += 4) {
            double2 da[4], db[4];
            double b[4];
#pragma unroll
            for (int v = 0; v < 4; v++) {
              const int e = e0 + v;
              const int src = qbase + min(7, used[u] + e);
              const int k = __shfl_sync(kFull, kb[u][0], src);
              const double bv = __shfl_sync(kFull, bb[u][0], src);
              const bool ok = e < n;
              b[v] = ok ? bv : 0.0;
              const double* row = tile + (ok ? (k - kt0) : 0) * 32;
              da[v] = *reinterpret_cast<const double2*>(row + ca);
              db[v] = *reinterpret_cast<const double2*>(row + cb);
            }
#pragma unroll
            for (int v = 0; v < 4; v++) {
              w[u][0] = fma(b[v], da[v].x, w[u][0]);
              w[u][1] = fma(b[v], da[v].y, w[u][1]);
              w[u][2] = fma(b[v], db[v].x, w[u][2]);
              w[u][3] = fma(b[v], db[v].y, w[u][3]);
            }
          }
          used[u] += n;
          // a fully consumed batch: shift the ring, prefetch kHvDepth batches ahead
          const bool adv = used[u] == 8;
          if (adv) {
            cur[u] += 8;
            zrem[u] -= 8;
            used[u] = 0;
#pragma unroll
            for (int d = 0; d + 1 < kHvDepth; d++) {
              kb[u][d] = kb[u][d + 1];
              bb[u][d] = bb[u][d + 1];
            }
            const int e = 8 * (kHvDepth - 1) + ql;
            kb[u][kHvDepth - 1] = e < zrem[u] ? (int)P.idx2[cur[u] + e] : INT_MAX;
            bb[u][kHvDepth - 1] = e < zrem[u] ? P.vals[cur[u] + e] : 0.0;
          }
          if (!__any_sync(kFull, adv)) break;
        }
      }
      __syncthreads();  // every warp is done with this stage
      if (threadIdx.x == 0 && t + 2 < nt) issue(it, t + 2, gt + 2);
    }
    // w0 (partial over [k0, k1)) x C(j,:), summed over the quarter's fibers,
    // the warp's quarters and the CTA's warps in a fixed order
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int u = 0; u < kHvFpq; u++) {
      const int64_t f = it.f0 + (warp * 4 + q) * kHvFpq + u;
      if (f < it.f1) {
        const int64_t j = P.idx1[f];
        const double2 c0 = __ldg(reinterpret_cast<const double2*>(P.C + j * 32 + ca));
        const double2 c1 = __ldg(reinterpret_cast<const double2*>(P.C + j * 32 + cb));
        acc[0] = fma(w[u][0], c0.x, acc[0]);
        acc[1] = fma(w[u][1], c0.y, acc[1]);
        acc[2] = fma(w[u][2], c1.x, acc[2]);
        acc[3] = fma(w[u][3], c1.y, acc[3]);
      }
    }
#pragma unroll
    for (int x = 0; x < 4; x++) {
      acc[x] += __shfl_xor_sync(kFull, acc[x], 8);
      acc[x] += __shfl_xor_sync(kFull, acc[x], 16);
    }
    if (q == 0) {
      S.red[warp][ca] = acc[0];
      S.red[warp][ca + 1] = acc[1];
      S.red[warp][cb] = acc[2];
      S.red[warp][cb + 1] = acc[3];
    }
    __syncthreads();
    if (warp == 0) {
      double sum = 0.0;
#pragma unroll
      for (int x = 0; x < kHvWarps; x++) sum += S.red[x][lane];
      hpart[(int64_t)itn * 32 + lane] = sum;
    }
  }
}

// Heavy slice rows: a CTA per slice; warp w adds the slice's items w, w+32,
// ... in order, then warp 0 adds the 32 warp sums in order (deterministic).
__global__ void mttkrp_dense_heavy_reduce_kernel(const DenseParams P, const int* slot_items,
                                                 const double* hpart, const int64_t* heavy_s) {
  __shared__ double ws[32][33];
  const int lane = (int)lane_id();
  const int warp = threadIdx.x >> 5;
  const int hs = blockIdx.x;
  const int t0 = slot_items[hs], t1 = slot_items[hs + 1];
  double sum = 0.0;
  for (int t = t0 + warp; t < t1; t += 32) sum += hpart[(int64_t)t * 32 + lane];
  ws[warp][lane] = sum;
  __syncthreads();
  if (warp == 0) {
    double tot = 0.0;
    for (int x = 0; x < 32; x++) tot += ws[x][lane];
    P.A[heavy_s[hs] * 32 + lane] = tot;
  }
}

// Per-slice nnz and fibers; slices whose average fiber is long enough for a
// block of kHvFibers fibers to reuse each staged D row (avg length > 2K /
// kHvFibers) and that hold at least one full block are listed as heavy.
constexpr int kMaxHeavy = 64;
__global__ void mttkrp_dense_heavy_select_kernel(const DenseParams P, int64_t min_len,
                                                 unsigned char* flag, int64_t* list,
                                                 unsigned long long* count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P.I;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f0 = P.pos1[i], f1 = P.pos1[i + 1];
    const int64_t nz = f1 > f0 ? P.pos2[f1] - P.pos2[f0] : 0;
    bool heavy = f1 - f0 >= kHvFibers && nz >= min_len * (f1 - f0);
    if (heavy) {
      const unsigned long long at = atomicAdd(count, 1ull);
      if (at < kMaxHeavy) {
        list[4 * at] = i;
        list[4 * at + 1] = f0;
        list[4 * at + 2] = f1;
        list[4 * at + 3] = nz;
      } else {
        heavy = false;
      }
    }
    flag[i] = heavy ? 1 : 0;
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
  int64_t* stage_idx;         // [I*R] drained rows at a fixed stride
  double* stage_vals;
  // column bitmaps of the factor rows (kBmWords 64-bit words per row; R <= 64*W)
  const unsigned long long* cbm;
  const unsigned long long* dbm;
};

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

// Matches (C_j ∩ D_k columns of single-nonzero fibers) are expanded warp-
// cooperatively: every lane with matches parks its fiber's (C row start, D
// row start, b, match / C / D bitmaps) in a per-warp shared buffer, then the
// warp's matches are numbered (a warp scan) and taken 32 at a time, lane s
// evaluating match s: owner lane by a shuffle search over the scan, the
// owner's t-th matched column by popcounts over its bitmap, the value
// positions by popcounts of the C and D bitmaps below it.  No per-lane bit
// walk (a lane with two matches no longer holds 31 others back).
template <int W>
struct MatchOwners {
  int64_t c0[32];
  int64_t d0[32];
  double b[32];
  unsigned long long m[W][32];
  unsigned long long bc[W][32];
  unsigned long long bd[W][32];
};
__host__ __device__ constexpr size_t match_owners_bytes(int W) { return (size_t)(3 + 3 * W) * 32 * 8; }

// sparse_slice with factor-row bitmaps: C_j ∩ D_k is a word-wise AND and a
// matched column's value positions are popcounts (same arithmetic and
// per-entry order as sparse_slice: w0 = 0 + b*D(k,r), w1(r) += w0*C(j,r)).
template <int W>
__device__ void sparse_slice_bm(const SparseParams& P, int64_t i, double* wv, uint32_t* wb,
                                unsigned long long& mults, MatchOwners<W>& O) {
  const int lane = (int)lane_id();
  const int64_t f0 = P.pos1[i], f1 = P.pos1[i + 1];
  const uint64_t keep = l2_evict_last_policy();
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
    if (nm > 0) {
      O.c0[lane] = ld_keep(P.cpos + j, keep);
      O.d0[lane] = ld_keep(P.dpos + k, keep);
      O.b[lane] = b;
#pragma unroll
      for (int w = 0; w < W; w++) {
        O.m[w][lane] = m[w];
        O.bc[w][lane] = bc[w];
        O.bd[w][lane] = bd[w];
      }
    }
    __syncwarp();
    mults += (unsigned long long)nm;
    for (int g0 = 0; g0 < tot; g0 += 32) {  // warp-uniform
      const int g = g0 + lane;
      // owner: the lowest lane whose inclusive count exceeds g
      int o = 0;
#pragma unroll
      for (int st = 16; st >= 1; st >>= 1) {
        const int iv = __shfl_sync(kFull, inc, (o + st - 1) & 31);
        if (iv <= g) o += st;
      }
      const int ex = __shfl_sync(kFull, inc, o) - __shfl_sync(kFull, nm, o);
      if (g < tot) {
        int t = g - ex;  // the owner's t-th match
        int r = 0, below_c = 0, below_d = 0;
        bool found = false;
#pragma unroll
        for (int w = 0; w < W; w++) {
          const unsigned long long mw = O.m[w][o];
          const unsigned long long cw = O.bc[w][o], dw = O.bd[w][o];
          const int pc = __popcll(mw);
          if (!found && t < pc) {
            // t-th set bit of mw (32-bit halves: __fns)
            const unsigned lo = (unsigned)mw;
            const int plo = __popc(lo);
            const int bit = t < plo ? (int)__fns(lo, 0, t + 1)
                                    : 32 + (int)__fns((unsigned)(mw >> 32), 0, t - plo + 1);
            const unsigned long long bl = (1ull << bit) - 1ull;
            r = w * 64 + bit;
            below_c += __popcll(cw & bl);
            below_d += __popcll(dw & bl);
            found = true;
          } else if (!found) {
            t -= pc;
            below_c += __popcll(cw);
            below_d += __popcll(dw);
          }
        }
        const double w0 = add_rn(0.0, mul_rn(O.b[o], ld_keep(P.dvals + O.d0[o] + below_d, keep)));
        ws_add(wv, wb, r, mul_rn(w0, ld_keep(P.cvals + O.c0[o] + below_c, keep)));
      }
    }
    __syncwarp();  // the owner buffer is rewritten by the next batch
  }
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
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = (int)lane_id();
  const int warp = threadIdx.x >> 5;
  const int64_t R = P.R;
  const int nwords = (int)((R + 31) / 32);
  const size_t ws_bytes = ((size_t)R * 8 + (size_t)nwords * 4 + 15) & ~(size_t)15;
  double* wv = reinterpret_cast<double*>(smem_raw + (size_t)warp * ws_bytes);
  uint32_t* wb = reinterpret_cast<uint32_t*>(wv + R);
  auto* owners = reinterpret_cast<MatchOwners<(W > 0 ? W : 1)>*>(
      smem_raw + (size_t)kSpWarps * ws_bytes + (size_t)warp * match_owners_bytes(W > 0 ? W : 1));
  unsigned long long mults = 0;
  while (true) {
    int64_t i = 0;
    if (lane == 0) i = (int64_t)atomicAdd(P.tile_counter, 1ull);
    i = __shfl_sync(kFull, i, 0);
    if (i >= P.I) break;
    for (int64_t r = lane; r < R; r += 32) wv[r] = 0.0;
    for (int w = lane; w < nwords; w += 32) wb[w] = 0u;
    __syncwarp();
    if constexpr (W > 0)
      sparse_slice_bm<W>(P, i, wv, wb, mults, *owners);
    else
      sparse_slice(P, i, wv, wb, mults);
    __syncwarp();
    // sorted drain by ballot/popcount over the presence bitmap
    int64_t* oi = P.stage_idx + i * R;
    double* ov = P.stage_vals + i * R;
    int out = 0;
    for (int w = 0; w < nwords; w++) {
      const uint32_t bits = wb[w];
      if (bits == 0) continue;
      if ((bits >> lane) & 1u) {
        const int rank = __popc(bits & ((1u << lane) - 1u));
        const int64_t r = (int64_t)w * 32 + lane;
        __stcs(reinterpret_cast<long long*>(oi) + out + rank, (long long)r);
        __stcs(ov + out + rank, wv[r]);
      }
      out += __popc(bits);
    }
    if (lane == 0) P.out_pos[i + 1] = out;
    __syncwarp();
  }
  mults = warp_sum(mults);
  if (lane == 0 && mults) atomicAdd(P.mults, mults);
}

// Copies staged rows (stride R) into the compact CSR: a warp per row.
__global__ void mttkrp_sparse_compact_kernel(const SparseParams P) {
  const int lane = (int)lane_id();
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < P.I; i += nwarps) {
    const int64_t dst = P.out_pos[i], n = P.out_pos[i + 1] - dst;
    const int64_t* si = P.stage_idx + i * P.R;
    const double* sv = P.stage_vals + i * P.R;
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
      // heavy slices -> the TMA-tiled kernel (beside the chunked one)
      const bool a16 = ((uintptr_t)P.D % 16 == 0);
      std::vector<HeavyItem> items;
      int64_t* heavy_s = nullptr;
      double* hpart = nullptr;
      HeavyItem* d_items = nullptr;
      int* slot_items = nullptr;
#ifndef HV_DISABLE
      if (fast && a16 && P.K >= 4 * kHvTile && env_flag("STAM_HV", 1)) {
        auto* hflag = static_cast<unsigned char*>(call.scratch((size_t)I));
        auto* hlist = static_cast<int64_t*>(call.scratch_zero(sizeof(int64_t) * (4 * kMaxHeavy + 1)));
        auto* hcount = reinterpret_cast<unsigned long long*>(hlist + 4 * kMaxHeavy);
        const int64_t min_len = std::max<int64_t>(64, ceil_div(2 * P.K, (int64_t)kHvFibers));
        call.before_launch("mttkrp_dense_heavy_select");
        mttkrp_dense_heavy_select_kernel<<<(unsigned)std::min<int64_t>(ceil_div(I, 256), (int64_t)sms * 8),
                                           256, 0, call.stream()>>>(P, min_len, hflag, hlist, hcount);
        call.after_launch();
        int64_t hl[4 * kMaxHeavy + 1];
        call.read_scalars(hlist, 4 * kMaxHeavy + 1, hl);
        const int nh = (int)std::min<int64_t>(hl[4 * kMaxHeavy], kMaxHeavy);
        if (nh > 0) {
          // heaviest first; fiber blocks of kHvFibers, each split over k so an
          // item holds ~1/4 of a fair share of the heavy nonzeros per CTA slot
          std::vector<int> order(nh);
          for (int h = 0; h < nh; h++) order[h] = h;
          std::sort(order.begin(), order.end(), [&](int a, int b) { return hl[4 * a + 3] > hl[4 * b + 3]; });
          int64_t hnz = 0;
          for (int h = 0; h < nh; h++) hnz += hl[4 * h + 3];
          const int64_t target = std::max<int64_t>(16384, hnz / ((int64_t)sms * 4));
          std::vector<int64_t> hs(nh), hf(2 * nh);
          const int64_t ktiles = ceil_div(P.K, (int64_t)kHvTile);
          for (int o = 0; o < nh; o++) {
            const int h = order[o];
            hs[o] = hl[4 * h];
            hf[2 * o] = hl[4 * h + 1];
            hf[2 * o + 1] = hl[4 * h + 2];
            const int64_t nf = hf[2 * o + 1] - hf[2 * o];
            const double per_fiber = (double)hl[4 * h + 3] / (double)nf;
            for (int64_t b0 = hf[2 * o]; b0 < hf[2 * o + 1]; b0 += kHvFibers) {
              const int64_t b1 = std::min<int64_t>(hf[2 * o + 1], b0 + kHvFibers);
              const int64_t est = (int64_t)(per_fiber * (double)(b1 - b0));
              const int64_t ks = std::max<int64_t>(1, std::min<int64_t>(ktiles, (est + target / 2) / target));
              for (int64_t p = 0; p < ks; p++) {
                HeavyItem itm{};
                itm.f0 = b0;
                itm.f1 = b1;
                itm.k0 = (int32_t)std::min<int64_t>(P.K, ktiles * p / ks * kHvTile);
                itm.k1 = (int32_t)std::min<int64_t>(P.K, ktiles * (p + 1) / ks * kHvTile);
                itm.slot = o;
                if (itm.k1 > itm.k0) items.push_back(itm);
              }
            }
          }
          std::vector<int> slot_first(nh + 1, 0);
          for (size_t t = 0; t < items.size(); t++) slot_first[items[t].slot + 1] = (int)t + 1;
          for (int o = 0; o < nh; o++) slot_first[o + 1] = std::max(slot_first[o + 1], slot_first[o]);
          slot_items = call.scratch_n<int>((size_t)nh + 1);
          STAM_CUDA_CHECK(cudaMemcpyAsync(slot_items, slot_first.data(), sizeof(int) * (nh + 1),
                                          cudaMemcpyHostToDevice, call.stream()));
          P.nheavy = nh;
          P.heavy_flag = hflag;
          auto* d_hf = call.scratch_n<int64_t>((size_t)(2 * nh));
          heavy_s = call.scratch_n<int64_t>((size_t)nh);
          d_items = call.scratch_n<HeavyItem>(items.size());
          hpart = call.scratch_n<double>(items.size() * 32);
          STAM_CUDA_CHECK(cudaMemcpyAsync(d_hf, hf.data(), sizeof(int64_t) * hf.size(),
                                          cudaMemcpyHostToDevice, call.stream()));
          STAM_CUDA_CHECK(cudaMemcpyAsync(heavy_s, hs.data(), sizeof(int64_t) * hs.size(),
                                          cudaMemcpyHostToDevice, call.stream()));
          STAM_CUDA_CHECK(cudaMemcpyAsync(d_items, items.data(), sizeof(HeavyItem) * items.size(),
                                          cudaMemcpyHostToDevice, call.stream()));
          P.heavy_f = d_hf;
          // the host vectors must outlive the async copies
          STAM_CUDA_CHECK(cudaStreamSynchronize(call.stream()));
          auto* hclaim = static_cast<unsigned long long*>(call.scratch_zero(16));
          cudaStream_t aux = call.fork();
          const size_t hsm = sizeof(HeavySmem);
          STAM_CUDA_CHECK(cudaFuncSetAttribute(mttkrp_dense_heavy_kernel,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm));
          call.before_launch("mttkrp_dense_heavy", aux);
          mttkrp_dense_heavy_kernel<<<(unsigned)std::min<int64_t>((int64_t)items.size(), (int64_t)sms),
                                      kHvWarps * 32, hsm, aux>>>(P, d_items, (int)items.size(), hclaim,
                                                                hpart);
          call.after_launch(aux);
        }
      }
#endif
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
      if (P.nheavy > 0) {
        call.join();
        call.before_launch("mttkrp_dense_heavy_reduce");
        mttkrp_dense_heavy_reduce_kernel<<<(unsigned)P.nheavy, 1024, 0, call.stream()>>>(
            P, slot_items, hpart, heavy_s);
        call.after_launch();
      }
    }
    call.finish_dense_result(A);
    call.finish();
    stam_stats* st = call.stats();
    st->mults = (B->nnz + B->nfibers) * R;  // SPEC.md:416 hoisted count
    st->adds = st->mults;
    st->ws_resets = B->nfibers;
  });
}

extern "C" int stam_cuda_mttkrp_sparse(stam_cuda_ctx* ctx, const stam_csf3_view* B,
                                       const stam_csr_view* Cv, const stam_csr_view* Dv,
                                       const stam_options* opts, stam_csr_result* A,
                                       stam_stats* stats) {
  using namespace stamgpu;
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
    const size_t smem = ws_bytes * kSpWarps + match_owners_bytes(8) * kSpWarps;
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
    P.stage_idx = call.scratch_n<int64_t>((size_t)(I * R));
    P.stage_vals = call.scratch_n<double>((size_t)(I * R));
    auto* ctl = static_cast<uint64_t*>(call.scratch_zero(4 * 8));
    P.tile_counter = reinterpret_cast<unsigned long long*>(ctl);
    P.mults = reinterpret_cast<unsigned long long*>(ctl + 1);
    // row pointers: counts at [i+1], scanned in place
    int64_t* cpos = static_cast<int64_t*>(call.scratch_zero(sizeof(int64_t) * ((size_t)I + 1)));
    P.out_pos = cpos;
    // factor-row column bitmaps when R fits W <= 8 words
    const int64_t words = (R + 63) / 64;
    const int W = words <= 1 ? 1 : words <= 2 ? 2 : words <= 4 ? 4 : words <= 8 ? 8 : 0;
    const size_t smem_w = ws_bytes * kSpWarps + match_owners_bytes(W > 0 ? W : 1) * kSpWarps;
    auto build_bm = [&](const int64_t* pos, const int64_t* idx, int64_t nrows) {
      // rows are read with 256-bit loads (W = 4): align the array to 32 bytes
      auto* raw = call.scratch_n<unsigned long long>((size_t)(nrows * W) + 4);
      auto* bm = reinterpret_cast<unsigned long long*>(((uintptr_t)raw + 31) & ~(uintptr_t)31);
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
    auto launch = [&](auto kern) {
      STAM_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem_w));
      int per_sm = 1;
      STAM_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSpWarps * 32,
                                                                    smem_w));
      const int64_t grid = std::min<int64_t>(ceil_div(I, kSpWarps),
                                             (int64_t)std::max(1, per_sm) * call.ctx()->num_sms);
      call.before_launch("mttkrp_sparse");
      kern<<<(unsigned)grid, kSpWarps * 32, smem_w, call.stream()>>>(P);
      call.after_launch();
    };
    switch (W) {
      case 1: launch(mttkrp_sparse_kernel<1>); break;
      case 2: launch(mttkrp_sparse_kernel<2>); break;
      case 4: launch(mttkrp_sparse_kernel<4>); break;
      case 8: launch(mttkrp_sparse_kernel<8>); break;
      default: launch(mttkrp_sparse_kernel<0>); break;
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
    call.before_launch("mttkrp_sparse_compact");
    mttkrp_sparse_compact_kernel<<<(unsigned)std::min<int64_t>(ceil_div(I, 8),
                                                               (int64_t)call.ctx()->num_sms * 16),
                                   256, 0, call.stream()>>>(P);
    call.after_launch();
    call.finish_csr_result(A, nnz);
    call.finish();
    stam_stats* st = call.stats();
    st->mults = ctlv[1];
    st->adds = ctlv[1];
    st->ws_resets = B->nfibers + I;
    st->appends = nnz;
  });
}
