// spadd.cu — multi-operand SpAdd  D = ops[0] + ops[1] + ... (CSR, sorted).
//
// Reference semantics: one row workspace per output row, the
// first operand assigned and the others accumulated in operand order, then a
// sorted drain (golden CIN test_transform.cpp:275-284; Workspace::insert
// workspace.cpp:34-46; drain workspace.cpp:62-71).  No pairwise merge.
//
// B200 design:
//  * one kernel, one pass over the inputs: ordered tiles of 16 rows claimed
//    through an atomic counter; every tile merges its rows in shared memory,
//    publishes its output count and learns its output offset by decoupled
//    look-back, then streams its staged rows out.  Inputs are read once and the
//    output written once, the HBM minimum.
//  * the row workspace is a rank-merge in shared memory: each stored element
//    finds its position in the operand-ordered merge by binary search into the
//    other operands' rows (already staged in smem), so the row is "scattered"
//    into its sorted slot; equal columns land adjacent in operand order and are
//    combined exactly as the workspace would (w = a; w += b; w += c ...), so
//    values are bit-identical to the CPU reference.
//  * rows too long for a warp's staging go to a CTA-per-row kernel with a
//    windowed column bitmap (also operand-ordered, also bit-exact).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "index.cuh"
#include "runtime.h"

namespace stamgpu {
namespace {

constexpr int kMaxOps = 16;

// Tile shapes: warps per CTA, rows per warp, staged entries per warp.  Short
// rows (the common case) use many rows per tile; rows averaging a few hundred
// entries use one row per warp and a deeper staging buffer.
template <int W, int RPW, int STAGE>
struct TileCfg {
  static constexpr int kWarps = W;
  static constexpr int kRowsPerWarp = RPW;
  static constexpr int kTileRows = W * RPW;
  static constexpr int kStage = STAGE;
};
// 1: a look-back tile per warp (no CTA barriers after the tile claim);
// 0: one look-back tile per CTA.  Measured on config 2: 0.485 ms (per CTA)
// vs 0.614 ms (per warp: 24x more look-back tiles lengthen the prefix chain)
#ifndef SPADD_WARP_LOOKBACK
#define SPADD_WARP_LOOKBACK 0
#endif
// -DSPADD_MINB=n: minimum resident CTAs per SM the tiles kernel's register
// budget targets.  Unset by default: an explicit minimum of 1 makes ptxas use
// 64 registers instead of 40 (config 2: 0.714 vs 0.480 ms).
#ifdef SPADD_MINB
#define SPADD_TILES_BOUNDS(t) __launch_bounds__(t, SPADD_MINB)
#else
#define SPADD_TILES_BOUNDS(t) __launch_bounds__(t)
#endif
#ifndef SPADD_MIDTHRESH
#define SPADD_MIDTHRESH 360
#endif
#ifndef SPADD_MID_WARPS
#define SPADD_MID_WARPS 4
#endif
#ifndef SPADD_MID_STAGE
#define SPADD_MID_STAGE 768
#endif
#ifndef SPADD_SHORT_W
#define SPADD_SHORT_W 24
#define SPADD_SHORT_RPW 1
#define SPADD_SHORT_STAGE 256
#endif
using ShortRows = TileCfg<SPADD_SHORT_W, SPADD_SHORT_RPW, SPADD_SHORT_STAGE>;
using MediumRows = TileCfg<16, 1, 384>;
using MidRowsCfg = TileCfg<SPADD_MID_WARPS, 1, SPADD_MID_STAGE>;
constexpr int kStageMin = SPADD_SHORT_STAGE < SPADD_MID_STAGE ? SPADD_SHORT_STAGE : SPADD_MID_STAGE;

enum RowState : int { kStaged = 0, kPostponed = 1, kDeferred = 2 };

struct SpaddParams {
  const int64_t* pos[kMaxOps];
  const int64_t* idx[kMaxOps];
  const double* vals[kMaxOps];
  int nops;
  int64_t nrows;
  int64_t ntiles;
  int64_t tile_base;  // first tile of this launch (row blocks of a streamed call)
  int64_t last_tile;  // last tile of this launch: publishes its end offset
  int64_t* block_end; // (host-mapped) end offset of this launch's rows
  int64_t* out_pos;
  int64_t* out_idx;
  double* out_vals;
  uint64_t* tile_status;
  unsigned long long* tile_counter;
  int64_t* deferred_rows;
  bool values;  // false: ASSEMBLE mode (index only, values written as zero)
  unsigned long long* deferred_count;
  int64_t* total_nnz;
};

template <typename ColT, int STAGE>
struct WarpStage {
  ColT in_col[STAGE];
  ColT st_col[STAGE];
  double st_val[STAGE];
  uint8_t st_op[STAGE];
  // current row's operand segments
  int64_t seg_beg[kMaxOps];
  int seg_len[kMaxOps];
  int seg_co[kMaxOps];
};

template <typename ColT, typename Cfg>
struct TileSmem {
  WarpStage<ColT, Cfg::kStage> w[Cfg::kWarps];
  int64_t tpos[kMaxOps][Cfg::kTileRows + 1];
  int64_t row_cnt[Cfg::kTileRows];
  int64_t row_dst[Cfg::kTileRows];
  int row_state[Cfg::kTileRows];
  int row_off[Cfg::kTileRows];
  int64_t tile_id;
};

// Number of elements < x (lower) or <= x (upper) in sorted s[0..n).
// Branchless; trip count = bit length of n, uniform across a warp searching
// one operand row.
// The search depth (bit length of n) is warp-uniform: every lane searches the
// same operand row.  A fall-through switch enters the fully unrolled steps at
// that depth (no per-step loop control).
#define STAM_RANK_STEP(B, CMP)                                    \
  case (B) + 1: {                                                 \
    const int probe = pos + (1 << (B));                           \
    pos = (probe <= n && CMP(s[probe - 1], x)) ? probe : pos;     \
  }                                                               \
    [[fallthrough]];
#define STAM_LT(a, b) ((a) < (b))
#define STAM_LE(a, b) ((a) <= (b))
template <bool kUpper, bool kSwitch, typename ColT>
__device__ __forceinline__ int rank_of(const ColT* s, int n, ColT x) {
  int pos = 0;
  const int depth = n ? 32 - __clz(n) : 0;  // steps 2^(depth-1) .. 1
  if (!kSwitch || depth > 12) {  // longer than any staging here: plain loop
    for (int step = 1 << (depth - 1); step > 0; step >>= 1) {
      const int probe = pos + step;
      pos = (probe <= n && (kUpper ? s[probe - 1] <= x : s[probe - 1] < x)) ? probe : pos;
    }
    return pos;
  }
  if constexpr (kUpper) {
    switch (depth) {
      STAM_RANK_STEP(11, STAM_LE)
      STAM_RANK_STEP(10, STAM_LE)
      STAM_RANK_STEP(9, STAM_LE)
      STAM_RANK_STEP(8, STAM_LE)
      STAM_RANK_STEP(7, STAM_LE)
      STAM_RANK_STEP(6, STAM_LE)
      STAM_RANK_STEP(5, STAM_LE)
      STAM_RANK_STEP(4, STAM_LE)
      STAM_RANK_STEP(3, STAM_LE)
      STAM_RANK_STEP(2, STAM_LE)
      STAM_RANK_STEP(1, STAM_LE)
      STAM_RANK_STEP(0, STAM_LE)
      default:
        break;
    }
  } else {
    switch (depth) {
      STAM_RANK_STEP(11, STAM_LT)
      STAM_RANK_STEP(10, STAM_LT)
      STAM_RANK_STEP(9, STAM_LT)
      STAM_RANK_STEP(8, STAM_LT)
      STAM_RANK_STEP(7, STAM_LT)
      STAM_RANK_STEP(6, STAM_LT)
      STAM_RANK_STEP(5, STAM_LT)
      STAM_RANK_STEP(4, STAM_LT)
      STAM_RANK_STEP(3, STAM_LT)
      STAM_RANK_STEP(2, STAM_LT)
      STAM_RANK_STEP(1, STAM_LT)
      STAM_RANK_STEP(0, STAM_LT)
      default:
        break;
    }
  }
  return pos;
}
// kSwitch = false keeps the plain loop (generic operand counts: the unrolled
// switch inside 16 x 16 operand loops would blow up code size).
template <bool kSwitch = true, typename ColT>
__device__ __forceinline__ int rank_lower(const ColT* s, int n, ColT x) {
  return rank_of<false, kSwitch>(s, n, x);
}
template <bool kSwitch = true, typename ColT>
__device__ __forceinline__ int rank_upper(const ColT* s, int n, ColT x) {
  return rank_of<true, kSwitch>(s, n, x);
}

__device__ __forceinline__ int64_t lower_bound_global(const int64_t* s, int64_t n, int64_t x) {
  int64_t lo = 0;
  while (n > 0) {
    const int64_t h = n >> 1;
    if (__ldg(s + lo + h) < x) {
      lo += h + 1;
      n -= h + 1;
    } else {
      n = h;
    }
  }
  return lo;
}

// Fill the warp's segment table for tile row r; returns the exact total.
template <typename SM, typename WS>
__device__ __forceinline__ int64_t row_segments(const SM& S, WS& W, int nops, int r) {
  const unsigned lane = lane_id();
  int64_t b = 0, e = 0;
  if ((int)lane < nops) {
    b = S.tpos[lane][r];
    e = S.tpos[lane][r + 1];
  }
  const int64_t len = e - b;
  const int64_t inc = warp_inclusive_scan(len);
  const int64_t tot = __shfl_sync(kFull, inc, 31);
  if ((int)lane < nops) {
    W.seg_beg[lane] = b;
    // only trusted when tot fits the staging buffer
    W.seg_len[lane] = (int)min(len, (int64_t)0x3fffffff);
    W.seg_co[lane] = (int)min(inc - len, (int64_t)0x3fffffff);
  }
  __syncwarp();
  return tot;
}

// Stage the row's column segments, concatenated in operand order, into in_col.
template <int NOPS, typename ColT, int STAGE>
__device__ __forceinline__ void load_cols(const SpaddParams& P, WarpStage<ColT, STAGE>& W) {
  const unsigned lane = lane_id();
  const int nops = NOPS ? NOPS : P.nops;
#pragma unroll
  for (int p = 0; p < (NOPS ? NOPS : kMaxOps); p++) {
    if (!NOPS && p >= nops) break;
    const int64_t* src = P.idx[p] + W.seg_beg[p];
    const int len = W.seg_len[p];
    ColT* dst = W.in_col + W.seg_co[p];
    for (int t = lane; t < len; t += 32) dst[t] = (ColT)ldg_stream(src + t);
  }
  __syncwarp();
}

// Combines runs of equal columns of the merged row st_*[out, out+L) in
// operand order (assign, then accumulate: the workspace semantics) and
// compacts in place.  any_dup (warp-uniform) false: nothing to combine.
template <typename ColT, int STAGE>
__device__ __forceinline__ int combine_staged(WarpStage<ColT, STAGE>& W, int L, int out, bool any_dup) {
  const unsigned lane = lane_id();
  ColT* st_col = W.st_col + out;
  double* st_val = W.st_val + out;
  const uint8_t* st_op = W.st_op + out;
  __syncwarp();
  // no column in two operands: the merge is already the compact row
  if (!any_dup) return L;
  // combine runs of equal columns in operand order; compact in place
  int count = 0;
  ColT prev = 0;
  for (int base = 0; base < L; base += 32) {
    const int m = base + (int)lane;
    ColT x = 0;
    double w = 0.0;
    bool lead = false;
    if (m < L) {
      x = st_col[m];
      const ColT before = (lane == 0) ? prev : st_col[m - 1];
      lead = (m == 0) || (before != x);
      if (lead) {
        const double v0 = st_val[m];
        w = (st_op[m] == 0) ? v0 : add_rn(0.0, v0);  // assign vs accumulate into 0.0
        for (int n = m + 1; n < L && st_col[n] == x; n++) w = add_rn(w, st_val[n]);
      }
    }
    prev = __shfl_sync(kFull, x, 31);
    const unsigned lead_mask = __ballot_sync(kFull, lead);
    const int slot = count + __popc(lead_mask & lanemask_lt());
    __syncwarp();
    if (lead) {
      st_col[slot] = x;
      st_val[slot] = w;
    }
    __syncwarp();
    count += __popc(lead_mask);
  }
  return count;
}


// Rank-merge the staged row into st_* at [out, out+L) (operand order on ties),
// then combine equal columns in place.  Returns the number of distinct columns.
template <int NOPS, typename ColT, int STAGE>
__device__ int merge_row(const SpaddParams& P, WarpStage<ColT, STAGE>& W, int L, int out) {
  const unsigned lane = lane_id();
  const int nops = NOPS ? NOPS : P.nops;
  ColT* st_col = W.st_col + out;
  double* st_val = W.st_val + out;
  uint8_t* st_op = W.st_op + out;
  // scatter every element to its merged slot
  bool dup = false;
  auto scatter_operand = [&](int o) {
    const double* vsrc = P.vals[o] + W.seg_beg[o];
    const int len = W.seg_len[o];
    const int co = W.seg_co[o];
    for (int t = lane; t < len; t += 32) {
      const double v = P.values ? ldg_stream(vsrc + t) : 0.0;
      const ColT x = W.in_col[co + t];
      int m = t;
      auto rank_in = [&](int q) {
        const ColT* sq = W.in_col + W.seg_co[q];
        const int nq = W.seg_len[q];
        if (q < o) {
          const int r = rank_upper<NOPS != 0>(sq, nq, x);
          dup |= r > 0 && sq[r - 1] == x;
          m += r;
        } else if (q > o) {
          m += rank_lower<NOPS != 0>(sq, nq, x);
        }
      };
      if constexpr (NOPS != 0) {
#pragma unroll
        for (int q = 0; q < NOPS; q++) rank_in(q);
      } else {
#pragma unroll 1
        for (int q = 0; q < nops; q++) rank_in(q);
      }
      st_col[m] = x;
      st_val[m] = v;
      st_op[m] = (uint8_t)o;
    }
  };
  if constexpr (NOPS != 0) {
#pragma unroll
    for (int o = 0; o < NOPS; o++) scatter_operand(o);
  } else {
#pragma unroll 1
    for (int o = 0; o < nops; o++) scatter_operand(o);
  }
  return combine_staged(W, L, out, __any_sync(kFull, dup));
}

// ---------------------------------------------------------------------------
// Padded rank-merge (specialised operand counts).  Operand q's columns are
// staged at in_col[q*D, q*D + len_q) and padded with a sentinel above every
// column up to D = 2^DLOG > every len_q, so a rank is exactly DLOG
// branchless probes with no bounds test.  The row's elements are walked
// flattened across operands (lane e -> operand o, index t), every lane
// searching the NOPS-1 other operands: rank of x among operand q's columns
// counts s < x for q > o and s <= x (= s < x + 1) for q < o, which puts equal
// columns adjacent in operand order — the same merged position as merge_row.
template <typename ColT>
__device__ __forceinline__ ColT rank_sentinel() {
  return sizeof(ColT) == 8 ? (ColT)0x7fffffffffffffffll : (ColT)0xffffffffu;
}

template <int NOPS, typename ColT, int STAGE>
__device__ __forceinline__ void load_cols_padded(const SpaddParams& P, WarpStage<ColT, STAGE>& W,
                                                 int D) {
  const unsigned lane = lane_id();
#pragma unroll
  for (int q = 0; q < NOPS; q++) {
    const int64_t* src = P.idx[q] + W.seg_beg[q];
    const int len = W.seg_len[q];
    ColT* dst = W.in_col + q * D;
    for (int t = lane; t < D; t += 32) dst[t] = t < len ? (ColT)ldg_stream(src + t) : rank_sentinel<ColT>();
  }
  __syncwarp();
}

template <int NOPS, int DLOG, typename ColT, int STAGE>
__device__ __forceinline__ int merge_flat(const SpaddParams& P, WarpStage<ColT, STAGE>& W, int L,
                                          int out) {
  constexpr int D = 1 << DLOG;
  const unsigned lane = lane_id();
  int co[NOPS];
  const double* vb[NOPS];
#pragma unroll
  for (int q = 0; q < NOPS; q++) {
    co[q] = W.seg_co[q];
    vb[q] = P.vals[q] + W.seg_beg[q];
  }
  bool dup = false;
  for (int e = lane; e < L; e += 32) {
    int o = 0;
    int c0 = 0;
    const double* vp = vb[0];
#pragma unroll
    for (int q = 1; q < NOPS; q++) {
      const bool ge = e >= co[q];
      o += ge;
      c0 = ge ? co[q] : c0;
      vp = ge ? vb[q] : vp;
    }
    const int t = e - c0;
    const ColT x = W.in_col[o * D + t];
    const double v = P.values ? ldg_stream(vp + t) : 0.0;
    int m = t;
#pragma unroll
    for (int k = 1; k < NOPS; k++) {
      int q = o + k;
      q = q >= NOPS ? q - NOPS : q;
      const bool upper = q < o;
      const ColT xx = x + (ColT)upper;
      const ColT* sq = W.in_col + q * D;
      int r = 0;
#pragma unroll
      for (int b = DLOG - 1; b >= 0; b--) r = (sq[r + (1 << b) - 1] < xx) ? r + (1 << b) : r;
      dup |= upper && r > 0 && sq[r - 1] == x;
      m += r;
    }
    W.st_col[out + m] = x;
    W.st_val[out + m] = v;
    W.st_op[out + m] = (uint8_t)o;
  }
  return combine_staged(W, L, out, __any_sync(kFull, dup));
}

// Stages and merges the row through the padded path when NOPS * D fits the
// staging; returns -1 (nothing staged) otherwise.
template <int NOPS, typename ColT, int STAGE>
__device__ __forceinline__ int merge_row_padded(const SpaddParams& P, WarpStage<ColT, STAGE>& W, int L,
                                                int out) {
  if constexpr (NOPS == 2 || NOPS == 3) {
    int maxlen = 0;
#pragma unroll
    for (int q = 0; q < NOPS; q++) maxlen = max(maxlen, W.seg_len[q]);
    const int dlog = 32 - __clz(maxlen);  // D = 2^dlog > maxlen: a rank reaches len
    if (dlog > 8 || (NOPS << dlog) > STAGE) return -1;
    load_cols_padded<NOPS>(P, W, 1 << dlog);
    switch (dlog) {
      case 0: return merge_flat<NOPS, 0>(P, W, L, out);
      case 1: return merge_flat<NOPS, 1>(P, W, L, out);
      case 2: return merge_flat<NOPS, 2>(P, W, L, out);
      case 3: return merge_flat<NOPS, 3>(P, W, L, out);
      case 4: return merge_flat<NOPS, 4>(P, W, L, out);
      case 5: return merge_flat<NOPS, 5>(P, W, L, out);
      case 6: return merge_flat<NOPS, 6>(P, W, L, out);
      case 7: return merge_flat<NOPS, 7>(P, W, L, out);
      default: return merge_flat<NOPS, 8>(P, W, L, out);
    }
  }
  return -1;
}

// Distinct-column count of a staged row (in_col only, no merge written).
template <int NOPS, typename ColT, int STAGE>
__device__ int count_row(const SpaddParams& P, const WarpStage<ColT, STAGE>& W) {
  const unsigned lane = lane_id();
  int count = W.seg_len[0];  // every first-operand entry starts a column
  for (int o = 1; o < P.nops; o++) {
    const int len = W.seg_len[o];
    const int co = W.seg_co[o];
    for (int t0 = 0; t0 < len; t0 += 32) {
      const int t = t0 + (int)lane;
      bool lead = false;
      if (t < len) {
        const ColT x = W.in_col[co + t];
        lead = true;
        for (int q = 0; q < o && lead; q++) {
          const ColT* sq = W.in_col + W.seg_co[q];
          const int nq = W.seg_len[q];
          const int r = rank_lower(sq, nq, x);
          if (r < nq && sq[r] == x) lead = false;
        }
      }
      count += __popc(__ballot_sync(kFull, lead));
    }
  }
  return count;
}

// Distinct-column count of a row read straight from global memory (rows that
// exceed the staging buffer; their values are written by the long-row kernel).
template <typename SM>
__device__ int64_t count_row_global(const SpaddParams& P, const SM& S, int r) {
  const unsigned lane = lane_id();
  int64_t count = S.tpos[0][r + 1] - S.tpos[0][r];
  for (int o = 1; o < P.nops; o++) {
    const int64_t bo = S.tpos[o][r], lo = S.tpos[o][r + 1] - bo;
    for (int64_t t0 = 0; t0 < lo; t0 += 32) {
      const int64_t t = t0 + lane;
      bool lead = false;
      if (t < lo) {
        const int64_t x = __ldg(P.idx[o] + bo + t);
        lead = true;
        for (int q = 0; q < o && lead; q++) {
          const int64_t bq = S.tpos[q][r], lq = S.tpos[q][r + 1] - bq;
          const int64_t k = lower_bound_global(P.idx[q] + bq, lq, x);
          if (k < lq && __ldg(P.idx[q] + bq + k) == x) lead = false;
        }
      }
      count += __popc(__ballot_sync(kFull, lead));
    }
  }
  return count;
}

template <typename ColT, typename Cfg, int NOPS>
__global__ void SPADD_TILES_BOUNDS(Cfg::kWarps * 32) spadd_tiles_kernel(const SpaddParams P) {
  constexpr int kRowsPerWarp = Cfg::kRowsPerWarp;
  constexpr int kTileRowsC = Cfg::kTileRows;
  constexpr int kStage = Cfg::kStage;
  static_assert(kRowsPerWarp <= 32 && Cfg::kWarps <= 32, "warp look-back tiles");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  TileSmem<ColT, Cfg>& S = *reinterpret_cast<TileSmem<ColT, Cfg>*>(smem_raw);
  const unsigned lane = lane_id();
  const int warp = threadIdx.x >> 5;
  const int nops = P.nops;

  if (threadIdx.x == 0) S.tile_id = P.tile_base + (int64_t)atomicAdd(P.tile_counter, 1ull);
  __syncthreads();
  const int64_t tile = S.tile_id;
  const int64_t row0 = tile * kTileRowsC;
  const int nrows_tile = (int)min((int64_t)kTileRowsC, P.nrows - row0);

#if SPADD_WARP_LOOKBACK
  // each warp loads its own rows' operand row pointers (row bounds shared with
  // the neighbouring warp are written by both, with the same value)
  for (int i = lane; i < nops * (kRowsPerWarp + 1); i += 32) {
    const int p = i / (kRowsPerWarp + 1);
    const int r = warp * kRowsPerWarp + i % (kRowsPerWarp + 1);
    S.tpos[p][r] = (r <= nrows_tile) ? __ldg(P.pos[p] + row0 + r) : 0;
  }
  __syncwarp();
#else
  // tile-wide operand row pointers
  for (int i = threadIdx.x; i < nops * (kTileRowsC + 1); i += blockDim.x) {
    const int p = i / (kTileRowsC + 1);
    const int r = i % (kTileRowsC + 1);
    S.tpos[p][r] = (r <= nrows_tile) ? __ldg(P.pos[p] + row0 + r) : 0;
  }
  __syncthreads();
#endif

  WarpStage<ColT, kStage>& W = S.w[warp];
  int stage_off = 0;
  for (int k = 0; k < kRowsPerWarp; k++) {
    const int r = warp * kRowsPerWarp + k;
    if (r >= nrows_tile) break;
    const int64_t tot = row_segments(S, W, nops, r);
    int64_t cnt;
    int state;
    int padded = -1;
    if (tot <= kStage - stage_off) padded = merge_row_padded<NOPS>(P, W, (int)tot, stage_off);
    if (padded >= 0) {
      cnt = padded;
      state = kStaged;
    } else if (tot <= kStage - stage_off) {
      load_cols<NOPS>(P, W);
      cnt = merge_row<NOPS>(P, W, (int)tot, stage_off);
      state = kStaged;
    } else if (tot <= kStage) {
      load_cols<NOPS>(P, W);
      cnt = count_row<NOPS>(P, W);
      state = kPostponed;
    } else {
      cnt = count_row_global(P, S, r);
      state = kDeferred;
    }
    if (lane == 0) {
      S.row_cnt[r] = cnt;
      S.row_state[r] = state;
      S.row_off[r] = stage_off;
    }
    if (state == kStaged) stage_off += (int)cnt;
    __syncwarp();
  }
#if SPADD_WARP_LOOKBACK
  // Every warp is its own look-back tile (warp tile = tile * kWarps + warp):
  // no CTA barrier between a warp's merge and its writes, so a warp with a
  // long row does not hold up the other warps of its CTA.  Warps without rows
  // publish a zero aggregate.  Predecessors are resident or done (earlier
  // warps of this CTA, or CTAs that claimed earlier tiles).
  {
    const int rw0 = warp * kRowsPerWarp;
    const int rr = rw0 + (int)lane;
    const bool mine = (int)lane < kRowsPerWarp && rr < nrows_tile;
    const int64_t c = mine ? S.row_cnt[rr] : 0;
    const int64_t inc = warp_inclusive_scan(c);
    const int64_t agg = __shfl_sync(kFull, inc, 31);
    const int64_t wtile = tile * Cfg::kWarps + warp;
    const int64_t base = lookback_exclusive(P.tile_status, wtile, agg);
    if (mine) {
      S.row_dst[rr] = base + inc - c;
      P.out_pos[row0 + rr + 1] = base + inc;
    }
    if (lane == 0) {
      if (wtile == 0) P.out_pos[0] = 0;
      if (wtile == P.ntiles * Cfg::kWarps - 1) *P.total_nnz = base + agg;
      if (wtile == (P.last_tile + 1) * Cfg::kWarps - 1 && P.block_end) *P.block_end = base + agg;
    }
    __syncwarp();
  }
#else
  __syncthreads();

  // tile aggregate and look-back (warp 0)
  if (warp == 0) {
    const int64_t c = (int)lane < nrows_tile ? S.row_cnt[lane] : 0;
    const int64_t inc = warp_inclusive_scan(c);
    const int64_t agg = __shfl_sync(kFull, inc, 31);
    const int64_t base = lookback_exclusive(P.tile_status, tile, agg);
    if ((int)lane < nrows_tile) {
      S.row_dst[lane] = base + inc - c;
      P.out_pos[row0 + lane + 1] = base + inc;
    }
    if (lane == 0) {
      if (tile == 0) P.out_pos[0] = 0;
      if (tile == P.ntiles - 1) *P.total_nnz = base + agg;
      if (tile == P.last_tile && P.block_end) *P.block_end = base + agg;
    }
  }
  __syncthreads();
#endif

  // stream out staged rows; redo postponed rows with the (now free) staging
  for (int k = 0; k < kRowsPerWarp; k++) {
    const int r = warp * kRowsPerWarp + k;
    if (r >= nrows_tile) break;
    if (S.row_state[r] != kStaged) continue;
    const int64_t dst = S.row_dst[r];
    const int off = S.row_off[r];
    const int cnt = (int)S.row_cnt[r];
    for (int t = lane; t < cnt; t += 32) {
      stg_stream(P.out_idx + dst + t, (int64_t)W.st_col[off + t]);
      stg_stream(P.out_vals + dst + t, W.st_val[off + t]);
    }
  }
  __syncwarp();
  for (int k = 0; k < kRowsPerWarp; k++) {
    const int r = warp * kRowsPerWarp + k;
    if (r >= nrows_tile) break;
    const int state = S.row_state[r];
    if (state == kPostponed) {
      const int64_t dst = S.row_dst[r];
      const int64_t tot = row_segments(S, W, nops, r);
      load_cols<NOPS>(P, W);
      const int cnt = merge_row<NOPS>(P, W, (int)tot, 0);
      for (int t = lane; t < cnt; t += 32) {
        stg_stream(P.out_idx + dst + t, (int64_t)W.st_col[t]);
        stg_stream(P.out_vals + dst + t, W.st_val[t]);
      }
      __syncwarp();
    } else if (state == kDeferred && lane == 0) {
      const unsigned long long slot = atomicAdd(P.deferred_count, 1ull);
      P.deferred_rows[slot] = row0 + r;
    }
  }
}

// ---------------------------------------------------------------------------
// Long rows: one CTA per row, windowed column bitmap.  For each window of
// kWinBits columns the CTA marks present columns, ranks them by popcount
// prefix, zeroes the window's output slots and then applies the operands in
// order (assign, then accumulate) — the workspace semantics, bit-exact.
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// Mid rows (a warp's staging < row <= kMid elements): one CTA per row, the
// same rank-scatter as merge_row over the whole CTA (elements ranked by
// binary search in the other operands' staged segments), then equal columns
// combined in operand order and compacted by a block scan.
constexpr int kMid = 3072;
constexpr int kMidThreads = 256;

struct MidSmem {
  int64_t in_col[kMid];
  double in_val[kMid];
  int64_t st_col[kMid];
  double st_val[kMid];
  uint8_t st_op[kMid];
  int64_t seg_beg[kMaxOps];
  int seg_len[kMaxOps];
  int seg_co[kMaxOps + 1];
  int scan[33];
  int dup;
};

__device__ __forceinline__ int rank_g(const int64_t* s, int n, int64_t x, bool upper) {
  int lo = 0;
  while (n > 0) {
    const int h = n >> 1;
    const bool before = upper ? s[lo + h] <= x : s[lo + h] < x;
    if (before) {
      lo += h + 1;
      n -= h + 1;
    } else {
      n = h;
    }
  }
  return lo;
}

__global__ void __launch_bounds__(kMidThreads) spadd_mid_rows_kernel(const SpaddParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MidSmem& S = *reinterpret_cast<MidSmem*>(smem_raw);
  const int tid = threadIdx.x;
  const int nops = P.nops;
  const unsigned long long ndef = *P.deferred_count;
  for (unsigned long long d = blockIdx.x; d < ndef; d += gridDim.x) {
    const int64_t r = P.deferred_rows[d];
    if (tid < nops) {
      S.seg_beg[tid] = __ldg(P.pos[tid] + r);
      S.seg_len[tid] = (int)min((int64_t)kMid + 1, __ldg(P.pos[tid] + r + 1) - S.seg_beg[tid]);
    }
    if (tid == 0) S.dup = 0;
    __syncthreads();
    if (tid == 0) {
      int co = 0;
      for (int p = 0; p < nops; p++) {
        S.seg_co[p] = co;
        co = min(co + S.seg_len[p], kMid + 1);
      }
      S.seg_co[nops] = co;
    }
    __syncthreads();
    const int L = S.seg_co[nops];
    if (L > kMid) {  // spadd_long_rows_kernel's row
      __syncthreads();
      continue;
    }
    const int64_t dst = P.out_pos[r];
    for (int p = 0; p < nops; p++) {
      const int64_t b = S.seg_beg[p];
      const int co = S.seg_co[p];
      for (int t = tid; t < S.seg_len[p]; t += kMidThreads) {
        S.in_col[co + t] = __ldg(P.idx[p] + b + t);
        S.in_val[co + t] = P.values ? __ldg(P.vals[p] + b + t) : 0.0;
      }
    }
    __syncthreads();
    bool dup = false;
    for (int e = tid; e < L; e += kMidThreads) {
      int o = 0;
      while (o + 1 < nops && S.seg_co[o + 1] <= e) o++;
      const int64_t x = S.in_col[e];
      int m = e - S.seg_co[o];
      for (int q = 0; q < nops; q++) {
        if (q == o) continue;
        const int64_t* sq = S.in_col + S.seg_co[q];
        const int rq = rank_g(sq, S.seg_len[q], x, q < o);
        if (q < o && rq > 0 && sq[rq - 1] == x) dup = true;
        m += rq;
      }
      S.st_col[m] = x;
      S.st_val[m] = S.in_val[e];
      S.st_op[m] = (uint8_t)o;
    }
    if (dup) S.dup = 1;
    __syncthreads();
    if (!S.dup) {
      for (int m = tid; m < L; m += kMidThreads) {
        P.out_idx[dst + m] = S.st_col[m];
        P.out_vals[dst + m] = S.st_val[m];
      }
    } else {
      int run = 0;
      for (int base = 0; base < L; base += kMidThreads) {
        const int m = base + tid;
        bool lead = false;
        double w = 0.0;
        int64_t x = 0;
        if (m < L) {
          x = S.st_col[m];
          lead = m == 0 || S.st_col[m - 1] != x;
          if (lead) {
            w = S.st_op[m] == 0 ? S.st_val[m] : add_rn(0.0, S.st_val[m]);
            for (int n = m + 1; n < L && S.st_col[n] == x; n++) w = add_rn(w, S.st_val[n]);
          }
        }
        int tot;
        const int ex = block_exclusive_scan(lead ? 1 : 0, S.scan, &tot);
        if (lead) {
          P.out_idx[dst + run + ex] = x;
          P.out_vals[dst + run + ex] = w;
        }
        run += tot;
      }
    }
    __syncthreads();
  }
}

constexpr int kLongThreads = 512;
constexpr int kWinWords = 2048;
constexpr int64_t kWinBits = (int64_t)kWinWords * 32;

__global__ void __launch_bounds__(kLongThreads) spadd_long_rows_kernel(const SpaddParams P) {
  __shared__ uint32_t bits[kWinWords];
  __shared__ int wpre[kWinWords];
  __shared__ int64_t head[kMaxOps], stop[kMaxOps], wend[kMaxOps];
  __shared__ int64_t c0_sh;
  __shared__ int scan_sh[33];
  const int tid = threadIdx.x;
  const int nops = P.nops;
  const unsigned long long ndef = *P.deferred_count;
  for (unsigned long long d = blockIdx.x; d < ndef; d += gridDim.x) {
    const int64_t r = P.deferred_rows[d];
    if (tid < nops) {
      head[tid] = __ldg(P.pos[tid] + r);
      stop[tid] = __ldg(P.pos[tid] + r + 1);
    }
    for (int w = tid; w < kWinWords; w += blockDim.x) bits[w] = 0u;
    int64_t dst = P.out_pos[r];
    __syncthreads();
    int64_t row_len = 0;
    for (int p = 0; p < nops; p++) row_len += stop[p] - head[p];
    if (row_len <= kMid) {  // spadd_mid_rows_kernel's row
      __syncthreads();
      continue;
    }
    while (true) {
      if (tid == 0) {
        int64_t c0 = INT64_MAX;
        for (int p = 0; p < nops; p++)
          if (head[p] < stop[p]) c0 = min(c0, __ldg(P.idx[p] + head[p]));
        c0_sh = c0;
      }
      __syncthreads();
      const int64_t c0 = c0_sh;
      if (c0 == INT64_MAX) break;
      if (tid < nops) {
        wend[tid] = head[tid] +
                    lower_bound_global(P.idx[tid] + head[tid], stop[tid] - head[tid], c0 + kWinBits);
      }
      __syncthreads();
      for (int p = 0; p < nops; p++) {
        for (int64_t t = head[p] + tid; t < wend[p]; t += blockDim.x) {
          const int64_t c = __ldg(P.idx[p] + t) - c0;
          atomicOr(&bits[c >> 5], 1u << (c & 31));
        }
      }
      __syncthreads();
      // exclusive popcount prefix over the window's words
      constexpr int kPer = kWinWords / kLongThreads;
      int local[kPer];
      int sum = 0;
#pragma unroll
      for (int q = 0; q < kPer; q++) {
        local[q] = sum;
        sum += __popc(bits[tid * kPer + q]);
      }
      int total;
      const int base = block_exclusive_scan(sum, scan_sh, &total);
#pragma unroll
      for (int q = 0; q < kPer; q++) wpre[tid * kPer + q] = base + local[q];
      for (int t = tid; t < total; t += blockDim.x) P.out_vals[dst + t] = 0.0;
      __syncthreads();
      for (int p = 0; p < nops; p++) {
        for (int64_t t = head[p] + tid; t < wend[p]; t += blockDim.x) {
          const int64_t col = __ldg(P.idx[p] + t);
          const int64_t c = col - c0;
          const int w = (int)(c >> 5);
          const int rank = wpre[w] + __popc(bits[w] & ((1u << (c & 31)) - 1u));
          const double v = P.values ? __ldg(P.vals[p] + t) : 0.0;
          P.out_idx[dst + rank] = col;
          P.out_vals[dst + rank] = (p == 0) ? v : add_rn(P.out_vals[dst + rank], v);
        }
        __syncthreads();
      }
      for (int w = tid; w < kWinWords; w += blockDim.x) bits[w] = 0u;
      if (tid < nops) head[tid] = wend[tid];
      dst += total;
      __syncthreads();
    }
    __syncthreads();
  }
}

template <typename ColT, typename Cfg>
void launch_tiles(stamrt::Call& call, const SpaddParams& P, int64_t ntiles) {
  if (ntiles <= 0) return;
  const size_t smem = sizeof(TileSmem<ColT, Cfg>);
  // operand counts specialised at compile time (loops unrolled)
  auto kern = P.nops == 2 ? spadd_tiles_kernel<ColT, Cfg, 2>
              : P.nops == 3 ? spadd_tiles_kernel<ColT, Cfg, 3>
                            : spadd_tiles_kernel<ColT, Cfg, 0>;
  STAM_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  call.before_launch(sizeof(ColT) == 4 ? "spadd_tiles<u32>" : "spadd_tiles<i64>");
  kern<<<(unsigned)ntiles, Cfg::kWarps * 32, smem, call.stream()>>>(P);
  call.after_launch();
}

// COMPUTE mode (SPEC run_compute_after_assemble): operand values written into
// a pre-assembled index, a warp per row, operands in order (operand 0
// assigns, later operands accumulate; an entry first reached by a later
// operand accumulates into 0.0) — the workspace sequence, bit-identical.
__global__ void spadd_compute_rows_kernel(const SpaddParams P, const int64_t* ipos,
                                          const int64_t* skey, const int64_t* perm,
                                          int* missing) {
  const int lane = (int)lane_id();
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < P.nrows; i += nwarps) {
    const int64_t c0 = ipos[i], cn = ipos[i + 1] - c0;
    for (int o = 0; o < P.nops; o++) {
      const int64_t b = P.pos[o][i], e = P.pos[o][i + 1];
      for (int64_t t = b + lane; t < e; t += 32) {
        const int64_t slot = index_lookup(skey, perm, c0, cn, __ldg(P.idx[o] + t));
        const double v = __ldg(P.vals[o] + t);
        if (slot < 0) {
          atomicOr(missing, 1);
        } else {
          P.out_vals[slot] = o == 0 ? v : add_rn(P.out_vals[slot], v);
        }
      }
      __syncwarp();
    }
  }
}

}  // namespace
}  // namespace stamgpu

using namespace stamrt;

namespace {
int spadd_call(stam_cuda_ctx* ctx, int32_t nops, const stam_csr_view* ops,
               const stam_options* opts, stam_csr_result* D, stam_stats* stats) {
  using namespace stamgpu;
  return guarded([&] {
    Call call(reinterpret_cast<Ctx*>(ctx), opts, stats);
    if (!ops) fail(STAM_ERR_PRECONDITION_VIOLATED, "null operand array");
    if (nops < 2) fail(STAM_ERR_ARITY_MISMATCH, "spadd needs at least two operands");
    if (nops > kMaxOps)
      fail(STAM_ERR_UNSUPPORTED_MERGE, "spadd supports at most 16 operands per kernel call");
    for (int p = 0; p < nops; p++) {
      check_csr_view(&ops[p], "spadd operand");
      if (ops[p].nrows != ops[0].nrows || ops[p].ncols != ops[0].ncols)
        fail(STAM_ERR_DIMENSION_MISMATCH, "spadd operands must have equal dimensions");
    }
    if (call.opts().mode == STAM_MODE_COMPUTE)
      fail(STAM_ERR_PRECONDITION_VIOLATED,
           "spadd compute mode needs the pre-assembled index: use stam_cuda_spadd_compute");
    const int64_t nrows = ops[0].nrows, ncols = ops[0].ncols;
    SpaddParams P{};
    P.nops = nops;
    P.nrows = nrows;
    P.values = call.opts().mode == STAM_MODE_FUSED;
    int64_t cap = 0, accum = 0, in_bytes = 0;
    bool host_in = false;
    for (int p = 0; p < nops; p++) {
      cap += ops[p].nnz;
      if (p > 0) accum += ops[p].nnz;
      host_in |= ops[p].mem == STAM_MEM_HOST;
      in_bytes += ops[p].nnz * 16;
    }
    // rows averaging a few hundred entries: one row per warp, deeper staging
    // tile shape by the average row (sum over operands): rows fitting 256
    // staged entries, 384, or longer (measured: profiles/r01_suite_spadd_k.csv)
    const int64_t avg_row = nrows > 0 ? cap / nrows : 0;
    const int shape = ncols > (int64_t)UINT32_MAX ? 0 : avg_row <= 224 ? 0 : avg_row <= SPADD_MIDTHRESH ? 1 : 2;
    const int64_t kTileRows = shape == 0 ? ShortRows::kTileRows
                              : shape == 1 ? MediumRows::kTileRows : MidRowsCfg::kTileRows;
    P.ntiles = ceil_div(nrows, kTileRows);
    const bool host_out = call.opts().result_mem == STAM_MEM_HOST;
    // Host operands or a host result: stream row blocks.  Block k's operand
    // ranges go up on the copy stream while earlier blocks merge, and each
    // finished block's output range comes down on the d2h stream while later
    // blocks merge (PCIe carries both directions at once).
    std::vector<int64_t> blk{0, P.ntiles};  // block boundaries in tiles
    if (host_in || host_out) {
      int64_t block_mb = 64;
      if (const char* e = std::getenv("STAM_STREAM_BLOCK_MB")) block_mb = std::max(1, std::atoi(e));
      blk = stream_blocks(P.ntiles, in_bytes, block_mb << 20, Ctx::kMarks);
    }
    const int64_t nblocks = (int64_t)blk.size() - 1;
    const int64_t* hpos[kMaxOps] = {};
    for (int p = 0; p < nops; p++) {
      P.pos[p] = call.device_input(ops[p].pos, (size_t)nrows + 1, ops[p].mem);
      if (ops[p].mem == STAM_MEM_HOST) {
        hpos[p] = ops[p].pos;
        P.idx[p] = call.host_staging<int64_t>((size_t)ops[p].nnz);
        P.vals[p] = call.host_staging<double>((size_t)ops[p].nnz);
      } else {
        P.idx[p] = ops[p].idx;
        P.vals[p] = ops[p].vals;
      }
    }
    int64_t* h_pos = nullptr;
    int64_t* h_idx = nullptr;
    double* h_vals = nullptr;
    if (host_out)
      call.alloc_csr_result_streamed(D, nrows, ncols, cap, &h_pos, &h_idx, &h_vals);
    else
      call.alloc_csr_result(D, nrows, ncols, cap);
    P.out_pos = D->pos;
    P.out_idx = D->idx;
    P.out_vals = D->vals;
    // control block: [deferred count, total, pad, pad] + one tile counter per
    // block + tile status words
    const size_t ctl_words = 4 + (size_t)nblocks + (size_t)P.ntiles * (SPADD_WARP_LOOKBACK ? 32 : 1);
    auto* ctl = static_cast<uint64_t*>(call.scratch_zero(ctl_words * sizeof(uint64_t)));
    P.deferred_count = reinterpret_cast<unsigned long long*>(ctl);
    P.total_nnz = reinterpret_cast<int64_t*>(ctl + 1);
    P.tile_status = ctl + 4 + nblocks;
    const int64_t max_deferred = std::min<int64_t>(nrows, cap / kStageMin + 1);
    P.deferred_rows = call.scratch_n<int64_t>((size_t)max_deferred);
    int64_t* marks = host_out ? call.marks() : nullptr;

    std::vector<cudaEvent_t> done((size_t)nblocks);
    // STAM_DEBUG_STREAM=1: per-block timeline (copy done, kernel done, d2h done) on stderr
    const bool dbg = std::getenv("STAM_DEBUG_STREAM") != nullptr;
    struct TlPoint {
      std::chrono::steady_clock::time_point t;
      std::string name;
    };
    static std::vector<TlPoint*> tl;
    auto mark_n = [&](cudaStream_t st, std::string n) {
      if (!dbg) return;
      auto* p = new TlPoint{{}, std::move(n)};
      tl.push_back(p);
      STAM_CUDA_CHECK(cudaLaunchHostFunc(
          st, [](void* u) { static_cast<TlPoint*>(u)->t = std::chrono::steady_clock::now(); }, p));
    };
    mark_n(call.stream(), "start");
    auto issue_block = [&](int64_t k) {
      const int64_t t0 = blk[(size_t)k];
      const int64_t t1 = blk[(size_t)k + 1];
      if (host_in) {
        const int64_t r0 = t0 * kTileRows, r1 = std::min(nrows, t1 * kTileRows);
        for (int p = 0; p < nops; p++) {
          if (!hpos[p]) continue;
          const int64_t e0 = hpos[p][r0], e1 = hpos[p][r1];
          call.copy_range(const_cast<int64_t*>(P.idx[p]) + e0, ops[p].idx + e0,
                          (size_t)(e1 - e0) * sizeof(int64_t));
          if (P.values)
            call.copy_range(const_cast<double*>(P.vals[p]) + e0, ops[p].vals + e0,
                            (size_t)(e1 - e0) * sizeof(double));
        }
        call.wait(call.copy_fence());
        mark_n(call.ctx()->copy_stream, "h2d " + std::to_string(k));
      }
      P.tile_base = t0;
      P.last_tile = t1 - 1;
      P.block_end = marks ? marks + k : nullptr;
      P.tile_counter = reinterpret_cast<unsigned long long*>(ctl + 4 + k);
      if (ncols <= (int64_t)UINT32_MAX) {
        if (shape == 2)
          launch_tiles<uint32_t, MidRowsCfg>(call, P, t1 - t0);
        else if (shape == 1)
          launch_tiles<uint32_t, MediumRows>(call, P, t1 - t0);
        else
          launch_tiles<uint32_t, ShortRows>(call, P, t1 - t0);
      } else {
        launch_tiles<int64_t, ShortRows>(call, P, t1 - t0);
      }
      mark_n(call.stream(), "kern " + std::to_string(k));
      if (host_out) {
        done[(size_t)k] = call.event();
        STAM_CUDA_CHECK(cudaEventRecord(done[(size_t)k], call.stream()));
      }
    };
    if (!host_out) {
      for (int64_t k = 0; k < nblocks; k++) issue_block(k);
    } else {
      // keep a few blocks of uploads ahead; bring finished blocks down while
      // later ones compute (uploads and downloads interleave in issue order)
      constexpr int64_t kAhead = 3;
      int64_t issued = 0, prev = 0;
      for (; issued < std::min(nblocks, kAhead); issued++) issue_block(issued);
      for (int64_t k = 0; k < nblocks; k++) {
        STAM_CUDA_CHECK(cudaEventSynchronize(done[(size_t)k]));
        const int64_t end = *(volatile int64_t*)(marks + k);
        const int64_t r0 = blk[(size_t)k] * kTileRows;
        const int64_t r1 = std::min(nrows, blk[(size_t)k + 1] * kTileRows);
        call.d2h_range(h_pos + r0 + (k == 0 ? 0 : 1), D->pos + r0 + (k == 0 ? 0 : 1),
                       (size_t)(r1 - r0 + (k == 0 ? 1 : 0)) * sizeof(int64_t), done[(size_t)k]);
        call.d2h_range(h_idx + prev, D->idx + prev, (size_t)(end - prev) * sizeof(int64_t), nullptr);
        call.d2h_range(h_vals + prev, D->vals + prev, (size_t)(end - prev) * sizeof(double), nullptr);
        mark_n(call.ctx()->d2h_stream, "d2h " + std::to_string(k) + " " + std::to_string((end - prev) >> 10) + "K");
        prev = end;
        if (issued < nblocks) issue_block(issued++);
      }
    }
    // rows too long for a warp's staging (deferred by their tiles): mid rows
    // by a CTA each, the longest by the windowed bitmap kernel
    {
      const size_t msmem = sizeof(MidSmem);
      STAM_CUDA_CHECK(cudaFuncSetAttribute(spadd_mid_rows_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)msmem));
      call.before_launch("spadd_mid_rows");
      spadd_mid_rows_kernel<<<(unsigned)std::max(1, call.ctx()->num_sms * 2), kMidThreads, msmem,
                              call.stream()>>>(P);
      call.after_launch();
    }
    call.before_launch("spadd_long_rows");
    spadd_long_rows_kernel<<<(unsigned)std::max(1, call.ctx()->num_sms), kLongThreads, 0,
                             call.stream()>>>(P);
    call.after_launch();
    int64_t tail[2];
    call.read_scalars(reinterpret_cast<const int64_t*>(ctl), 2, tail);  // deferred, total
    const int64_t nnz = tail[1];
    if (dbg) {
      STAM_CUDA_CHECK(cudaDeviceSynchronize());
      for (auto* q : tl) {
        const double ms = std::chrono::duration<double, std::milli>(q->t - tl[0]->t).count();
        fprintf(stderr, "[spadd] %8.3f ms  %s\n", ms, q->name.c_str());
      }
      for (auto* q : tl) delete q;
      tl.clear();
    }
    if (host_out) {
      if (tail[0] > 0) {
        // long rows were filled after their blocks came down (the stream
        // was synchronised above): bring the entries down again
        call.d2h_range(h_idx, D->idx, (size_t)nnz * sizeof(int64_t), nullptr);
        call.d2h_range(h_vals, D->vals, (size_t)nnz * sizeof(double), nullptr);
      }
      call.finish_csr_result_streamed(D, nnz);
    } else {
      call.finish_csr_result(D, nnz);
    }
    call.finish();
    stam_stats* st = call.stats();
    st->adds = accum;
    st->ws_inserts = cap;
    st->ws_resets = nrows;
    st->appends = nnz;
  });
}

}  // namespace

// More than kMaxOps operands: the workspace sequence continued across calls.
// The partial sum of the first 16 operands is operand 0 of the next call
// (assigned — the value the workspace holds at that point), the next 15
// operands accumulate, and so on; a column first seen in a later operand
// accumulates into 0.0 either way, so the result is bit-identical to one
// workspace pass over all operands in order.  Partial sums stay on the device.
extern "C" int stam_cuda_spadd(stam_cuda_ctx* ctx, int32_t nops, const stam_csr_view* ops,
                               const stam_options* opts, stam_csr_result* D, stam_stats* stats) {
  using namespace stamgpu;
  if (nops <= kMaxOps || !ops) return spadd_call(ctx, nops, ops, opts, D, stats);
  stam_options o = opts ? *opts : stam_options{1, STAM_MODE_FUSED, STAM_MEM_DEVICE, 0};
  stam_options mid = o;
  mid.result_mem = STAM_MEM_DEVICE;
  stam_stats total{}, part{};
  stam_csr_result acc{};
  int st = spadd_call(ctx, kMaxOps, ops, &mid, &acc, &part);
  // counters of one workspace pass: the partial sum re-entering as operand 0
  // is not a new insert, and the rows are reset once
  auto add_stats = [&](int64_t reentered) {
    total.adds += part.adds;
    total.ws_inserts += part.ws_inserts - reentered;
    total.ws_resets = part.ws_resets;
    total.appends = part.appends;
    total.kernel_launches += part.kernel_launches;
    total.total_kernel_ms += part.total_kernel_ms;
    if (part.main_kernel_ms > total.main_kernel_ms) {
      total.main_kernel_ms = part.main_kernel_ms;
      std::memcpy(total.main_kernel, part.main_kernel, sizeof(total.main_kernel));
    }
  };
  if (st != 0) return st;
  add_stats(0);
  int32_t next = kMaxOps;
  while (st == 0) {
    const int32_t take = std::min<int32_t>(kMaxOps - 1, nops - next);
    const bool last = next + take == nops;
    std::vector<stam_csr_view> v((size_t)take + 1);
    v[0] = stam_csr_view{acc.nrows, acc.ncols, acc.nnz, acc.pos, acc.idx, acc.vals, acc.mem, 0};
    for (int32_t q = 0; q < take; q++) v[(size_t)q + 1] = ops[next + q];
    stam_csr_result out{};
    part = stam_stats{};
    const int64_t reentered = acc.nnz;
    st = spadd_call(ctx, take + 1, v.data(), last ? &o : &mid, last ? D : &out, &part);
    stam_cuda_release(ctx, acc.handle);
    if (st != 0) break;
    add_stats(reentered);
    next += take;
    if (last) break;
    acc = out;
  }
  if (st == 0 && stats) *stats = total;
  return st;
}

extern "C" int stam_cuda_spadd_compute(stam_cuda_ctx* ctx, int32_t nops, const stam_csr_view* ops,
                                       const stam_csr_view* Didx, const stam_options* opts,
                                       stam_csr_result* D, stam_stats* stats) {
  using namespace stamgpu;
  return guarded([&] {
    Call call(reinterpret_cast<Ctx*>(ctx), opts, stats);
    if (!ops) fail(STAM_ERR_PRECONDITION_VIOLATED, "null operand array");
    if (nops < 2) fail(STAM_ERR_ARITY_MISMATCH, "spadd needs at least two operands");
    if (nops > kMaxOps)
      fail(STAM_ERR_UNSUPPORTED_MERGE, "spadd supports at most 16 operands per call");
    for (int p = 0; p < nops; p++) {
      check_csr_view(&ops[p], "spadd operand");
      if (ops[p].nrows != ops[0].nrows || ops[p].ncols != ops[0].ncols)
        fail(STAM_ERR_DIMENSION_MISMATCH, "spadd operands must have equal dimensions");
    }
    if (!Didx) fail(STAM_ERR_PRECONDITION_VIOLATED, "spadd compute: null pre-assembled index");
    if (Didx->nrows != ops[0].nrows || Didx->ncols != ops[0].ncols)
      fail(STAM_ERR_DIMENSION_MISMATCH, "spadd compute: index dimensions != operand dimensions");
    if (Didx->nnz < 0 || !Didx->pos || (Didx->nnz > 0 && !Didx->idx))
      fail(STAM_ERR_PRECONDITION_VIOLATED, "spadd compute: incomplete pre-assembled index");
    const int64_t nrows = ops[0].nrows, ncols = ops[0].ncols, nnz = Didx->nnz;
    SpaddParams P{};
    P.nops = nops;
    P.nrows = nrows;
    int64_t accum = 0;
    for (int p = 0; p < nops; p++) {
      P.pos[p] = call.device_input(ops[p].pos, (size_t)nrows + 1, ops[p].mem);
      P.idx[p] = call.device_input(ops[p].idx, (size_t)ops[p].nnz, ops[p].mem);
      P.vals[p] = call.device_input(ops[p].vals, (size_t)ops[p].nnz, ops[p].mem);
      if (p > 0) accum += ops[p].nnz;
    }
    const int64_t* ipos = call.device_input(Didx->pos, (size_t)nrows + 1, Didx->mem);
    const int64_t* iidx = call.device_input(Didx->idx, (size_t)nnz, Didx->mem);
    call.alloc_csr_result(D, nrows, ncols, nnz);
    STAM_CUDA_CHECK(cudaMemcpyAsync(D->pos, ipos, sizeof(int64_t) * ((size_t)nrows + 1),
                                    cudaMemcpyDeviceToDevice, call.stream()));
    if (nnz > 0) {
      STAM_CUDA_CHECK(cudaMemcpyAsync(D->idx, iidx, sizeof(int64_t) * (size_t)nnz,
                                      cudaMemcpyDeviceToDevice, call.stream()));
      STAM_CUDA_CHECK(cudaMemsetAsync(D->vals, 0, sizeof(double) * (size_t)nnz, call.stream()));
    }
    const IndexSearch ix = make_index_search(call, ipos, iidx, nrows, nnz, call.opts().sort != 0);
    P.out_vals = D->vals;
    auto* missing = static_cast<int*>(call.scratch_zero(sizeof(int64_t)));
    call.before_launch("spadd_compute_rows");
    spadd_compute_rows_kernel<<<(unsigned)std::min<int64_t>(ceil_div(nrows, 8),
                                                            (int64_t)call.ctx()->num_sms * 16),
                                256, 0, call.stream()>>>(P, ipos, ix.skey, ix.perm, missing);
    call.after_launch();
    const int64_t miss = call.read_scalar(reinterpret_cast<const int64_t*>(missing));
    if (miss != 0)
      fail(STAM_ERR_MISSING_SLOT, "spadd compute: an operand column is missing from the index");
    call.finish_csr_result(D, nnz);
    call.finish();
    stam_stats* st = call.stats();
    st->adds = accum;
    st->ws_resets = nrows;
  });
}
