// spgemm.cu — Gustavson SpGEMM  C = A·B  (CSR x CSR -> CSR, sorted columns).
//
// Reference loop nest (golden CIN, test_transform.cpp:141-147):
//   forall(i) ((forall(j) C(i,j) = w0(j)) where (forall(k,j) w0(j) += A(i,k)*B(k,j)))
// with a dense row workspace, products accumulated into 0.0 in canonical
// order (k ascending over A's row, then B's row order), and a sorted drain
// (Workspace::insert / drain, workspace.cpp:34-71).
//
// B200 design: symbolic pass -> scan -> numeric pass.
//  * rowprod: products per row P_i = sum_{k in A_i} nnz(B_k) (also the
//    binning key), and per-bin row lists.
//  * bins by P_i (exact output upper bound):
//      tiny   P <= 32   : warp per row, one product per lane; distinct rank by
//                         a shuffle sweep, values summed in canonical order
//                         (bit-exact with the reference).
//      hash-S P <= 256  : one-warp CTA per row,
//      hash-M P <= 1024 : 128-thread CTA per row,
//      hash-L P <= 4096 : 256-thread CTA per row — a shared-memory hash table
//                         whose hash is ORDER-PRESERVING (slot = scaled column,
//                         linear probing forward, no wrap): occupied runs are
//                         mutually ordered, so sorting the few entries of each
//                         run gives the sorted row; values accumulate with
//                         shared-memory fp64 atomics.
//      long   P > 4096  : 512-thread CTA per row, a column bitmap over all
//                         columns in shared memory (popcount rank) and fp64
//                         atomics into the pre-assembled output row.
//  * products are enumerated flattened (prefix of B-row lengths over the A
//    row), warp-contiguous and lane-interleaved, so B rows are read coalesced.
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <string>

#include "common.cuh"
#include "runtime.h"

namespace stamgpu {
namespace {

enum Bin : int { kBinEmpty = 0, kBinTiny, kBinHashXS, kBinHashS, kBinHashM, kBinHashL, kBinLong, kNumBins };
constexpr int64_t kTinyMax = 32, kHashXSMax = 64, kHashSMax = 256, kHashMMax = 1024, kHashLMax = 4096;
constexpr int kAChunk = 1024;        // A entries staged per chunk (long rows)
constexpr int kLongThreads = 512;
constexpr uint32_t kEmpty = 0xffffffffu;

__host__ __device__ inline int bin_of(int64_t p) {
  if (p == 0) return kBinEmpty;
  if (p <= kTinyMax) return kBinTiny;
  if (p <= kHashXSMax) return kBinHashXS;
  if (p <= kHashSMax) return kBinHashS;
  if (p <= kHashMMax) return kBinHashM;
  if (p <= kHashLMax) return kBinHashL;
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
  int64_t* prod;             // [m] products per row
  unsigned long long* bins;  // [kNumBins] counts, then cursors
  int64_t* bin_rows;         // [m] rows grouped by bin
  int64_t* cpos;             // [m+1]: counts at [i+1], then offsets
  int64_t* cidx;
  double* cvals;
  int64_t* stats;            // [0] total products
};

// ---------------------------------------------------------------------------
__global__ void rowprod_kernel(const SpgemmParams P) {
  __shared__ unsigned long long hist[kNumBins];
  __shared__ unsigned long long total;
  if (threadIdx.x < kNumBins) hist[threadIdx.x] = 0;
  if (threadIdx.x == 0) total = 0;
  __syncthreads();
  // 8 lanes per row, 4 rows in flight per warp
  const unsigned lane = lane_id();
  const unsigned sub = lane & 7;
  const int64_t group = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) >> 3;
  const int64_t iters = (P.m + ngroups - 1) / ngroups;
  unsigned long long local_total = 0;
  for (int64_t it = 0; it < iters; it++) {
    const int64_t i = group + it * ngroups;
    int64_t s = 0;
    if (i < P.m) {
      const int64_t a0 = P.apos[i], a1 = P.apos[i + 1];
      for (int64_t p = a0 + sub; p < a1; p += 8) {
        const int64_t k = P.aidx[p];
        s += P.bpos[k + 1] - P.bpos[k];
      }
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    if (sub == 0 && i < P.m) {
      P.prod[i] = s;
      atomicAdd(&hist[bin_of(s)], 1ull);
      local_total += (unsigned long long)s;
    }
  }
  local_total = warp_sum(local_total);
  if (lane == 0 && local_total) atomicAdd(&total, local_total);
  __syncthreads();
  if (threadIdx.x < kNumBins && hist[threadIdx.x]) atomicAdd(&P.bins[threadIdx.x], hist[threadIdx.x]);
  if (threadIdx.x == 0 && total) atomicAdd((unsigned long long*)&P.stats[0], total);
}

__global__ void bin_scatter_kernel(const SpgemmParams P, const unsigned long long* offsets) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = i < P.m;
  const int b = valid ? bin_of(P.prod[i]) : -1;
  // warp-aggregated slot claims
  const unsigned peers = __match_any_sync(kFull, b);
  const int leader = __ffs(peers) - 1;
  unsigned long long base = 0;
  if ((int)lane_id() == leader && valid && b != kBinEmpty)
    base = atomicAdd(&P.bins[b], (unsigned long long)__popc(peers));
  base = __shfl_sync(kFull, base, leader);
  if (valid && b != kBinEmpty) {
    const unsigned rank = __popc(peers & lanemask_lt());
    P.bin_rows[offsets[b] + base + rank] = i;
  }
}

// ---------------------------------------------------------------------------
// tiny rows: one product per lane (P <= 32)
// Enumerates row i's products into lanes in canonical order.
__device__ __forceinline__ void tiny_products(const SpgemmParams& P, int64_t i, int64_t& col,
                                              double& val, bool& has) {
  const unsigned lane = lane_id();
  const int64_t a0 = P.apos[i], a1 = P.apos[i + 1];
  has = false;
  col = INT64_MAX;
  val = 0.0;
  int64_t done = 0;  // products emitted before this chunk of A entries
  for (int64_t c = a0; c < a1; c += 32) {
    const int64_t p = c + lane;
    int64_t b0 = 0, len = 0;
    double a = 0.0;
    if (p < a1) {
      const int64_t k = P.aidx[p];
      b0 = P.bpos[k];
      len = P.bpos[k + 1] - b0;
      a = P.avals[p];
    }
    const int64_t inc = warp_inclusive_scan(len);
    const int64_t exc = inc - len;
    const int64_t total = __shfl_sync(kFull, inc, 31);
    // product j (= lane - done) comes from the A entry whose range holds it
    const int64_t j = (int64_t)lane - done;
    int src = 0;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      const int cand = src + s;
      const int64_t e = __shfl_sync(kFull, exc, cand & 31);
      if (cand < 32 && e <= j) src = cand;
    }
    const int64_t sb0 = __shfl_sync(kFull, b0, src);
    const int64_t sexc = __shfl_sync(kFull, exc, src);
    const double sa = __shfl_sync(kFull, a, src);
    if (j >= 0 && j < total) {
      const int64_t q = sb0 + (j - sexc);
      col = P.bidx[q];
      val = mul_rn(sa, P.bvals[q]);
      has = true;
    }
    done += total;
  }
}

__global__ void tiny_symbolic_kernel(const SpgemmParams P, const int64_t* rows, int64_t nrows) {
  const unsigned lane = lane_id();
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < nrows; r += nwarps) {
    const int64_t i = rows[r];
    int64_t col;
    double val;
    bool has;
    tiny_products(P, i, col, val, has);
    // leader: no lower lane holds the same column
    bool lead = has;
    for (int j = 0; j < 32; j++) {
      const int64_t cj = __shfl_sync(kFull, col, j);
      if (j < (int)lane && cj == col) lead = false;
    }
    const int cnt = __popc(__ballot_sync(kFull, lead));
    if (lane == 0) P.cpos[i + 1] = cnt;
  }
}

__global__ void tiny_numeric_kernel(const SpgemmParams P, const int64_t* rows, int64_t nrows) {
  const unsigned lane = lane_id();
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < nrows; r += nwarps) {
    const int64_t i = rows[r];
    int64_t col;
    double val;
    bool has;
    tiny_products(P, i, col, val, has);
    bool lead = has;
    int out = 0;
    double w = add_rn(0.0, val);  // first insert accumulates into 0.0
    // pass 1: leader flags
    for (int j = 0; j < 32; j++) {
      const int64_t cj = __shfl_sync(kFull, col, j);
      if (j < (int)lane && cj == col) lead = false;
    }
    const unsigned lead_mask = __ballot_sync(kFull, lead);
    // pass 2: slot = leaders with a smaller column; sum later equal products
    for (int j = 0; j < 32; j++) {
      const int64_t cj = __shfl_sync(kFull, col, j);
      const double vj = __shfl_sync(kFull, val, j);
      if (((lead_mask >> j) & 1u) && cj < col) out++;
      if (j > (int)lane && cj == col) w = add_rn(w, vj);
    }
    if (lead) {
      const int64_t dst = P.cpos[i] + out;
      P.cidx[dst] = col;
      P.cvals[dst] = w;
    }
  }
}

// ---------------------------------------------------------------------------
// Flattened product enumeration for CTA-per-row kernels.
//
// A chunk of up to kAChunk A entries of row i is staged in smem (B row start,
// A value, exclusive prefix of B row lengths).  Products [0, total) of the
// chunk are split into warp-contiguous ranges, lane-interleaved inside them.
template <int AC>
struct ChunkSmem {
  int64_t bstart[AC];
  double aval[AC];
  int off[AC + 1];
  int scan[33];
};

// Stages A entries [c0, c1) (c1 - c0 <= AC); returns the product total.
template <int AC>
__device__ int stage_chunk(const SpgemmParams& P, ChunkSmem<AC>& S, int64_t c0, int64_t c1) {
  const int n = (int)(c1 - c0);
  int carry = 0;
  for (int base = 0; base < n; base += blockDim.x) {
    const int t = base + threadIdx.x;
    int len = 0;
    if (t < n) {
      const int64_t k = P.aidx[c0 + t];
      const int64_t b0 = P.bpos[k];
      len = (int)(P.bpos[k + 1] - b0);
      S.bstart[t] = b0;
      S.aval[t] = P.avals[c0 + t];
    }
    int tot;
    const int exc = block_exclusive_scan(len, S.scan, &tot);
    if (t < n) S.off[t] = carry + exc;
    carry += tot;
  }
  if (threadIdx.x == 0) S.off[n] = carry;
  __syncthreads();
  return carry;
}

// Calls f(col, value) for every product of the staged chunk, each exactly once.
template <int AC, typename F>
__device__ __forceinline__ void for_products(const SpgemmParams& P, const ChunkSmem<AC>& S, int nA,
                                             int total, F f) {
  const int lane = (int)lane_id();
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int per = (total + nwarps - 1) / nwarps;
  const int w0 = min(total, warp * per), w1 = min(total, w0 + per);
  // A entry holding product w0 (binary search), then advance monotonically
  int p = 0;
  {
    int lo = 0, hi = nA;  // last p with off[p] <= w0
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (S.off[mid] <= w0) lo = mid; else hi = mid;
    }
    p = lo;
  }
  for (int j = w0 + lane; j < w1; j += 32) {
    while (S.off[p + 1] <= j) p++;
    const int64_t q = S.bstart[p] + (j - S.off[p]);
    f(P.bidx[q], mul_rn(S.aval[p], P.bvals[q]));
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

// Column span of row i from the first/last column of every B row it touches.
__device__ SlotMap row_slot_map(const SpgemmParams& P, int64_t i, int tb, int64_t* red) {
  int64_t lo = INT64_MAX, hi = -1;
  const int64_t a0 = P.apos[i], a1 = P.apos[i + 1];
  for (int64_t p = a0 + threadIdx.x; p < a1; p += blockDim.x) {
    const int64_t k = P.aidx[p];
    const int64_t b0 = P.bpos[k], b1 = P.bpos[k + 1];
    if (b1 > b0) {
      lo = min(lo, P.bidx[b0]);
      hi = max(hi, P.bidx[b1 - 1]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(kFull, lo, o));
    hi = max(hi, __shfl_xor_sync(kFull, hi, o));
  }
  if (threadIdx.x == 0) {
    red[0] = INT64_MAX;
    red[1] = -1;
  }
  __syncthreads();
  if (lane_id() == 0) {
    atomicMin((long long*)&red[0], (long long)lo);
    atomicMax((long long*)&red[1], (long long)hi);
  }
  __syncthreads();
  SlotMap sm;
  sm.c0 = red[0];
  const uint64_t span = red[1] >= red[0] ? (uint64_t)(red[1] - red[0] + 1) : 1;
  sm.scale = ((uint64_t)tb << 32) / span;
  if (sm.scale == 0) sm.scale = 1;
  __syncthreads();
  return sm;
}

// Insert col (linear probing forward from its order-preserving slot).
// Returns the slot and whether this call created the entry.
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

// Table layout for the hash kernels: up to TB main slots + TB/2 overflow
// slots.  A row with P products uses tb = next_pow2(2P) main slots (at least
// 64) and tb/2 overflow slots: at most P <= tb/2 entries are inserted, so
// forward probing never runs off the end.
// A entries staged per chunk: a row of a hash bin has at most TB/2 products,
// hence at most TB/2 non-empty A entries; empty ones cost extra chunks only.
template <int TB>
constexpr int hash_achunk() { return TB / 2 < kAChunk ? TB / 2 : kAChunk; }

template <int TB>
struct HashSmem {
  ChunkSmem<hash_achunk<TB>()> chunk;
  uint32_t keys[TB + TB / 2];
  double vals[TB + TB / 2];
  int64_t red[2];
  int scan[33];
};

__device__ __forceinline__ int row_table(int64_t prod) {
  int tb = 64;
  while (tb < 2 * prod) tb <<= 1;
  return tb;
}

// Exclusive scan of one flag per thread across the CTA (warp-only CTAs use a
// ballot), returning the total through *tot.
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

template <int THREADS, int TB>
__global__ void __launch_bounds__(THREADS) hash_symbolic_kernel(const SpgemmParams P,
                                                                 const int64_t* rows,
                                                                 int64_t nrows) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  HashSmem<TB>& S = *reinterpret_cast<HashSmem<TB>*>(smem_raw);
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int64_t i = rows[r];
    const int tb = row_table(P.prod[i]);
    const int nslots = tb + tb / 2;
    const SlotMap sm = row_slot_map(P, i, tb, S.red);
    for (int s = threadIdx.x; s < nslots; s += THREADS) S.keys[s] = kEmpty;
    __syncthreads();
    const int64_t a0 = P.apos[i], a1 = P.apos[i + 1];
    int created = 0;
    constexpr int AC = hash_achunk<TB>();
    for (int64_t c0 = a0; c0 < a1; c0 += AC) {
      const int64_t c1 = min(a1, c0 + AC);
      const int total = stage_chunk(P, S.chunk, c0, c1);
      for_products(P, S.chunk, (int)(c1 - c0), total, [&](int64_t col, double) {
        bool made;
        hash_insert(S.keys, (uint32_t)(col - sm.c0), sm(col), made);
        created += made ? 1 : 0;
      });
      __syncthreads();
    }
    int tot;
    block_exclusive_scan(created, S.scan, &tot);
    if (threadIdx.x == 0) P.cpos[i + 1] = tot;
  }
}

template <int THREADS, int TB>
__global__ void __launch_bounds__(THREADS) hash_numeric_kernel(const SpgemmParams P,
                                                                const int64_t* rows,
                                                                int64_t nrows) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  HashSmem<TB>& S = *reinterpret_cast<HashSmem<TB>*>(smem_raw);
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int64_t i = rows[r];
    const int tb = row_table(P.prod[i]);
    const int nslots = tb + tb / 2;
    const SlotMap sm = row_slot_map(P, i, tb, S.red);
    for (int s = threadIdx.x; s < nslots; s += THREADS) {
      S.keys[s] = kEmpty;
      S.vals[s] = 0.0;
    }
    __syncthreads();
    const int64_t a0 = P.apos[i], a1 = P.apos[i + 1];
    constexpr int AC = hash_achunk<TB>();
    for (int64_t c0 = a0; c0 < a1; c0 += AC) {
      const int64_t c1 = min(a1, c0 + AC);
      const int total = stage_chunk(P, S.chunk, c0, c1);
      for_products(P, S.chunk, (int)(c1 - c0), total, [&](int64_t col, double v) {
        bool made;
        const int s = hash_insert(S.keys, (uint32_t)(col - sm.c0), sm(col), made);
        atomicAdd(&S.vals[s], v);
      });
      __syncthreads();
    }
    // sort every occupied run (runs are mutually ordered), started by the
    // thread that owns the run's first slot
    for (int s = threadIdx.x; s < nslots; s += THREADS) {
      if (S.keys[s] == kEmpty || (s > 0 && S.keys[s - 1] != kEmpty)) continue;
      int e = s + 1;
      while (e < nslots && S.keys[e] != kEmpty) e++;
      for (int a = s + 1; a < e; a++) {  // insertion sort of the run
        const uint32_t k = S.keys[a];
        const double v = S.vals[a];
        int b = a - 1;
        while (b >= s && S.keys[b] > k) {
          S.keys[b + 1] = S.keys[b];
          S.vals[b + 1] = S.vals[b];
          b--;
        }
        S.keys[b + 1] = k;
        S.vals[b + 1] = v;
      }
    }
    __syncthreads();
    // compact occupied slots in order, straight to the output row
    const int64_t dst = P.cpos[i];
    int64_t written = 0;
    for (int c = 0; c < nslots; c += THREADS) {
      const int s = c + threadIdx.x;
      const bool occ = s < nslots && S.keys[s] != kEmpty;
      int tot;
      const int pos = cta_flag_scan<THREADS>(occ, S.scan, &tot);
      if (occ) {
        P.cidx[dst + written + pos] = sm.c0 + (int64_t)S.keys[s];
        P.cvals[dst + written + pos] = S.vals[s];
      }
      written += tot;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Long rows: a bitmap over all n columns in shared memory (64-bit words), and
// for the numeric pass an exclusive popcount prefix per word.
struct LongSmem {
  ChunkSmem<kAChunk> chunk;
  int scan[33];
};

__host__ __device__ inline size_t long_header() { return (sizeof(LongSmem) + 15) & ~(size_t)15; }

__host__ __device__ inline size_t long_smem_bytes(int64_t n, bool numeric) {
  const size_t nw = (size_t)((n + 63) / 64);
  return long_header() + nw * 8 + (numeric ? nw * 4 : 0);
}

__device__ __forceinline__ void set_bit(unsigned long long* bits, int64_t col) {
  atomicOr(&bits[col >> 6], 1ull << (col & 63));
}

__global__ void __launch_bounds__(kLongThreads) long_symbolic_kernel(const SpgemmParams P,
                                                                     const int64_t* rows,
                                                                     int64_t nrows) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LongSmem& S = *reinterpret_cast<LongSmem*>(smem_raw);
  auto* bits = reinterpret_cast<unsigned long long*>(smem_raw + long_header());
  const int nw = (int)((P.n + 63) >> 6);
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int64_t i = rows[r];
    for (int w = threadIdx.x; w < nw; w += blockDim.x) bits[w] = 0ull;
    __syncthreads();
    const int64_t a0 = P.apos[i], a1 = P.apos[i + 1];
    for (int64_t c0 = a0; c0 < a1; c0 += kAChunk) {
      const int64_t c1 = min(a1, c0 + kAChunk);
      const int total = stage_chunk(P, S.chunk, c0, c1);
      for_products(P, S.chunk, (int)(c1 - c0), total,
                   [&](int64_t col, double) { set_bit(bits, col); });
      __syncthreads();
    }
    int cnt = 0;
    for (int w = threadIdx.x; w < nw; w += blockDim.x) cnt += __popcll(bits[w]);
    int tot;
    block_exclusive_scan(cnt, S.scan, &tot);
    if (threadIdx.x == 0) P.cpos[i + 1] = tot;
  }
}

__global__ void __launch_bounds__(kLongThreads) long_numeric_kernel(const SpgemmParams P,
                                                                    const int64_t* rows,
                                                                    int64_t nrows) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LongSmem& S = *reinterpret_cast<LongSmem*>(smem_raw);
  auto* bits = reinterpret_cast<unsigned long long*>(smem_raw + long_header());
  const int nw = (int)((P.n + 63) >> 6);
  int* wpre = reinterpret_cast<int*>(bits + nw);
  const int per = (nw + kLongThreads - 1) / kLongThreads;  // words per thread
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int64_t i = rows[r];
    const int64_t dst = P.cpos[i];
    const int64_t cnt = P.cpos[i + 1] - dst;
    for (int w = threadIdx.x; w < nw; w += blockDim.x) bits[w] = 0ull;
    for (int64_t t = threadIdx.x; t < cnt; t += blockDim.x) P.cvals[dst + t] = 0.0;
    __syncthreads();
    const int64_t a0 = P.apos[i], a1 = P.apos[i + 1];
    for (int64_t c0 = a0; c0 < a1; c0 += kAChunk) {
      const int64_t c1 = min(a1, c0 + kAChunk);
      const int total = stage_chunk(P, S.chunk, c0, c1);
      for_products(P, S.chunk, (int)(c1 - c0), total,
                   [&](int64_t col, double) { set_bit(bits, col); });
      __syncthreads();
    }
    // exclusive popcount prefix per word; write the sorted column list
    const int w0 = threadIdx.x * per, w1 = min(nw, w0 + per);
    int mine = 0;
    for (int w = w0; w < w1; w++) mine += __popcll(bits[w]);
    int tot;
    int run = block_exclusive_scan(mine, S.scan, &tot);
    for (int w = w0; w < w1; w++) {
      wpre[w] = run;
      unsigned long long m = bits[w];
      while (m) {
        const int b = __ffsll((long long)m) - 1;
        P.cidx[dst + run] = (int64_t)w * 64 + b;
        run++;
        m &= m - 1;
      }
    }
    __syncthreads();
    for (int64_t c0 = a0; c0 < a1; c0 += kAChunk) {
      const int64_t c1 = min(a1, c0 + kAChunk);
      const int total = stage_chunk(P, S.chunk, c0, c1);
      for_products(P, S.chunk, (int)(c1 - c0), total, [&](int64_t col, double v) {
        const int w = (int)(col >> 6);
        const int slot = wpre[w] + __popcll(bits[w] & ((1ull << (col & 63)) - 1ull));
        atomicAdd(&P.cvals[dst + slot], v);
      });
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
template <int THREADS, int TB>
void launch_hash(stamrt::Call& call, const SpgemmParams& P, const int64_t* rows, int64_t n,
                 bool numeric, const char* name) {
  if (n == 0) return;
  const size_t smem = sizeof(HashSmem<TB>);
  auto kern = numeric ? hash_numeric_kernel<THREADS, TB> : hash_symbolic_kernel<THREADS, TB>;
  STAM_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 1;
  STAM_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem));
  const int64_t grid = std::min<int64_t>(n, (int64_t)std::max(1, per_sm) * call.ctx()->num_sms * 4);
  call.before_launch(name);
  kern<<<(unsigned)grid, THREADS, smem, call.stream()>>>(P, rows, n);
  call.after_launch();
}

void launch_long(stamrt::Call& call, const SpgemmParams& P, const int64_t* rows, int64_t n,
                 bool numeric) {
  if (n == 0) return;
  const size_t smem = long_smem_bytes(P.n, numeric);
  auto kern = numeric ? long_numeric_kernel : long_symbolic_kernel;
  STAM_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t grid = std::min<int64_t>(n, call.ctx()->num_sms);
  call.before_launch(numeric ? "spgemm_long_numeric" : "spgemm_long_symbolic");
  kern<<<(unsigned)grid, kLongThreads, smem, call.stream()>>>(P, rows, n);
  call.after_launch();
}

}  // namespace
}  // namespace stamgpu

using namespace stamrt;

extern "C" int stam_cuda_spgemm(stam_cuda_ctx* ctx, const stam_csr_view* A, const stam_csr_view* B,
                                const stam_options* opts, stam_csr_result* Cr, stam_stats* stats) {
  using namespace stamgpu;
  return guarded([&] {
    Call call(reinterpret_cast<Ctx*>(ctx), opts, stats);
    check_csr_view(A, "spgemm A");
    check_csr_view(B, "spgemm B");
    if (A->ncols != B->nrows)
      fail(STAM_ERR_DIMENSION_MISMATCH, "spgemm: A columns != B rows");
    if (call.opts().mode != STAM_MODE_FUSED)
      fail(STAM_ERR_UNSUPPORTED_MERGE, "spgemm supports fused mode only in ABI v1");
    if (B->ncols >= (int64_t)UINT32_MAX)
      fail(STAM_ERR_UNSUPPORTED_MERGE, "spgemm: B has 2^32 or more columns");
    const int64_t m = A->nrows, n = B->ncols;
    const size_t long_smem = long_smem_bytes(n, true);
    SpgemmParams P{};
    P.m = m;
    P.n = n;
    P.apos = call.device_input(A->pos, (size_t)m + 1, A->mem);
    P.aidx = call.device_input(A->idx, (size_t)A->nnz, A->mem);
    P.avals = call.device_input(A->vals, (size_t)A->nnz, A->mem);
    P.bpos = call.device_input(B->pos, (size_t)B->nrows + 1, B->mem);
    P.bidx = call.device_input(B->idx, (size_t)B->nnz, B->mem);
    P.bvals = call.device_input(B->vals, (size_t)B->nnz, B->mem);
    P.prod = call.scratch_n<int64_t>((size_t)m);
    auto* ctl = static_cast<int64_t*>(call.scratch_zero(sizeof(int64_t) * 16));
    P.bins = reinterpret_cast<unsigned long long*>(ctl);
    P.stats = ctl + 8;
    P.bin_rows = call.scratch_n<int64_t>((size_t)m);
    P.cpos = static_cast<int64_t*>(call.scratch_zero(sizeof(int64_t) * ((size_t)m + 1)));
    const int sms = call.ctx()->num_sms;

    // products per row and bins
    call.before_launch("spgemm_rowprod");
    rowprod_kernel<<<(unsigned)std::min<int64_t>(ceil_div(m, 32), (int64_t)sms * 8), 256, 0,
                     call.stream()>>>(P);
    call.after_launch();
    int64_t host[16];
    call.read_scalars(ctl, 16, host);
    static_assert(kNumBins <= 8, "bin counters share the control block");
    unsigned long long counts[kNumBins], offsets[kNumBins];
    unsigned long long acc = 0;
    for (int b = 0; b < kNumBins; b++) {
      counts[b] = (unsigned long long)host[b];
      offsets[b] = acc;
      if (b != kBinEmpty) acc += counts[b];
    }
    const int64_t products = host[8];
    if (counts[kBinLong] > 0 && long_smem > call.ctx()->smem_optin)
      fail(STAM_ERR_UNSUPPORTED_MERGE,
           "spgemm: rows with more than 4096 products need a column bitmap of B's columns in "
           "shared memory (at most ~1.2M columns in ABI v1)");
    auto* d_off = static_cast<unsigned long long*>(call.scratch(sizeof(offsets)));
    STAM_CUDA_CHECK(cudaMemcpyAsync(d_off, offsets, sizeof(offsets), cudaMemcpyHostToDevice,
                                    call.stream()));
    STAM_CUDA_CHECK(cudaMemsetAsync(P.bins, 0, sizeof(unsigned long long) * kNumBins, call.stream()));
    call.before_launch("spgemm_bin_scatter");
    bin_scatter_kernel<<<(unsigned)ceil_div(m, 256), 256, 0, call.stream()>>>(P, d_off);
    call.after_launch();

    const int64_t* rows_b[kNumBins];
    for (int b = 0; b < kNumBins; b++) rows_b[b] = P.bin_rows + offsets[b];
    auto tiny_grid = [&](int64_t n) {
      return (unsigned)std::min<int64_t>(ceil_div(n, 8), (int64_t)sms * 16);
    };
    // symbolic
    if (counts[kBinTiny]) {
      call.before_launch("spgemm_tiny_symbolic");
      tiny_symbolic_kernel<<<tiny_grid(counts[kBinTiny]), 256, 0, call.stream()>>>(
          P, rows_b[kBinTiny], counts[kBinTiny]);
      call.after_launch();
    }
    launch_hash<32, 128>(call, P, rows_b[kBinHashXS], counts[kBinHashXS], false, "spgemm_hashXS_symbolic");
    launch_hash<32, 512>(call, P, rows_b[kBinHashS], counts[kBinHashS], false, "spgemm_hashS_symbolic");
    launch_hash<128, 2048>(call, P, rows_b[kBinHashM], counts[kBinHashM], false, "spgemm_hashM_symbolic");
    launch_hash<256, 8192>(call, P, rows_b[kBinHashL], counts[kBinHashL], false, "spgemm_hashL_symbolic");
    launch_long(call, P, rows_b[kBinLong], counts[kBinLong], false);

    // scan counts -> row pointers
    size_t temp_bytes = 0;
    STAM_CUDA_CHECK(cub::DeviceScan::InclusiveSum(nullptr, temp_bytes, P.cpos + 1, P.cpos + 1, m,
                                                  call.stream()));
    void* temp = call.scratch(temp_bytes);
    call.before_launch("spgemm_scan");
    STAM_CUDA_CHECK(cub::DeviceScan::InclusiveSum(temp, temp_bytes, P.cpos + 1, P.cpos + 1, m,
                                                  call.stream()));
    call.after_launch();
    const int64_t nnz = call.read_scalar(P.cpos + m);

    call.alloc_csr_result(Cr, m, n, nnz);
    STAM_CUDA_CHECK(cudaMemcpyAsync(Cr->pos, P.cpos, sizeof(int64_t) * ((size_t)m + 1),
                                    cudaMemcpyDeviceToDevice, call.stream()));
    P.cidx = Cr->idx;
    P.cvals = Cr->vals;
    if (counts[kBinTiny]) {
      call.before_launch("spgemm_tiny_numeric");
      tiny_numeric_kernel<<<tiny_grid(counts[kBinTiny]), 256, 0, call.stream()>>>(
          P, rows_b[kBinTiny], counts[kBinTiny]);
      call.after_launch();
    }
    launch_hash<32, 128>(call, P, rows_b[kBinHashXS], counts[kBinHashXS], true, "spgemm_hashXS_numeric");
    launch_hash<32, 512>(call, P, rows_b[kBinHashS], counts[kBinHashS], true, "spgemm_hashS_numeric");
    launch_hash<128, 2048>(call, P, rows_b[kBinHashM], counts[kBinHashM], true, "spgemm_hashM_numeric");
    launch_hash<256, 8192>(call, P, rows_b[kBinHashL], counts[kBinHashL], true, "spgemm_hashL_numeric");
    launch_long(call, P, rows_b[kBinLong], counts[kBinLong], true);

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
