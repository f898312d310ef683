// common.cuh — shared device helpers for the sm_100a workspace kernels.
//
// Everything here is plain CUDA C++ for sm_100a: warp primitives
// (shfl/ballot/match), an ordered-tile decoupled look-back used by the
// single-pass kernels (SpAdd, sparse MTTKRP) to turn per-tile output counts
// into output offsets without a separate symbolic pass, and a few math
// helpers that pin the rounding of the reference's accumulations.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace stamgpu {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;

// The reference accumulates `w += a*b` with the product rounded first
// (Workspace::insert receives the already-rounded product,
// workspace.cpp:34-46).  The oracle is compiled with -ffp-contract=off; these
// helpers stop nvcc from contracting into an FMA so results stay bit-exact.
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T u = __shfl_xor_sync(kFull, v, o);
    v = u > v ? u : v;
  }
  return v;
}

// Inclusive warp prefix sum.
template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
  const unsigned lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(kFull, v, o);
    if (lane >= (unsigned)o) v += u;
  }
  return v;
}

// Read-only streaming loads (bypass L1 allocation for data touched once).
#ifndef STAM_STREAM_PLAIN
__device__ __forceinline__ int64_t ldg_stream(const int64_t* p) {
  return (int64_t)__ldcs((const long long*)p);
}
__device__ __forceinline__ double ldg_stream(const double* p) { return __ldcs(p); }
__device__ __forceinline__ void stg_stream(int64_t* p, int64_t v) {
  __stcs((long long*)p, (long long)v);
}
__device__ __forceinline__ void stg_stream(double* p, double v) { __stcs(p, v); }
#else  // tuning experiment: default cache policy
__device__ __forceinline__ int64_t ldg_stream(const int64_t* p) { return __ldg(p); }
__device__ __forceinline__ double ldg_stream(const double* p) { return __ldg(p); }
__device__ __forceinline__ void stg_stream(int64_t* p, int64_t v) { *p = v; }
__device__ __forceinline__ void stg_stream(double* p, double v) { *p = v; }
#endif

// ---------------------------------------------------------------------------
// Ordered tiles with decoupled look-back.
//
// Tiles are claimed in increasing order through an atomic counter, so every
// predecessor of a claimed tile is already running; a tile publishes its
// aggregate, looks back over its predecessors' published values and publishes
// its inclusive prefix.  Status word: bits 63..62 flag (0 none, 1 aggregate,
// 2 inclusive prefix), bits 61..0 value.
// ---------------------------------------------------------------------------
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagInc = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Called by one full warp of the tile.  Returns the exclusive prefix (sum of
// all predecessors' aggregates) in every lane.
// look-back polling backoff (ns): first sleep and cap of the doubling.
// SpAdd config 2 kernel, two sweeps: cap 2048 0.486/0.485 ms, 8192 0.484,
// 256 0.480/0.480, 64 0.481/0.478, 16..128 0.478/0.480
#ifndef STAM_LB_NS0
#define STAM_LB_NS0 32
#endif
#ifndef STAM_LB_NSMAX
#define STAM_LB_NSMAX 256
#endif
__device__ __forceinline__ int64_t lookback_exclusive(uint64_t* status, int64_t tile,
                                                      int64_t aggregate) {
  const unsigned lane = lane_id();
  if (tile == 0) {
    if (lane == 0) st_release(&status[0], kFlagInc | (uint64_t)aggregate);
    return 0;
  }
  if (lane == 0) st_release(&status[tile], kFlagAgg | (uint64_t)aggregate);
  int64_t exclusive = 0;
  int64_t base = tile - 1;  // window covers [base-31, base]
  while (true) {
    const int64_t t = base - (int64_t)lane;
    uint64_t s = kFlagInc;  // lanes before tile 0 behave like a zero prefix
    if (t >= 0) {
      // predecessors still computing: back off so spinning warps do not steal
      // issue slots from the warps doing the work
      unsigned ns = STAM_LB_NS0;
      while (((s = ld_acquire(&status[t])) >> 62) == 0) {
        __nanosleep(ns);
        ns = ns < STAM_LB_NSMAX ? ns * 2 : ns;
      }
    }
    const unsigned inc_mask = __ballot_sync(kFull, (s >> 62) == 2);
    // closest predecessor holding an inclusive prefix = lowest set lane
    const int stop = inc_mask ? __ffs(inc_mask) - 1 : 32;
    int64_t v = (lane <= (unsigned)stop && t >= 0) ? (int64_t)(s & kValMask) : 0;
    exclusive += warp_sum(v);
    if (inc_mask) break;
    base -= 32;
  }
  if (lane == 0) st_release(&status[tile], kFlagInc | (uint64_t)(exclusive + aggregate));
  return exclusive;
}

// Block-wide exclusive scan of one int per thread (blockDim.x multiple of 32,
// <= 1024).  `sh` needs 33 ints.  Returns exclusive prefix, total in *total.
__device__ __forceinline__ int block_exclusive_scan(int v, int* sh, int* total) {
  const unsigned lane = lane_id();
  const unsigned warp = threadIdx.x >> 5;
  const unsigned nwarps = blockDim.x >> 5;
  int inc = warp_inclusive_scan(v);
  if (lane == 31) sh[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int w = lane < nwarps ? sh[lane] : 0;
    int winc = warp_inclusive_scan(w);
    if (lane < nwarps) sh[lane] = winc - w;
    if (lane == nwarps - 1) sh[32] = winc;
  }
  __syncthreads();
  int res = inc - v + sh[warp];
  if (total) *total = sh[32];
  __syncthreads();
  return res;
}


// ---------------------------------------------------------------------------
// L2 eviction-priority hints.  Kernels that stream a large array once while
// gathering from a small, heavily re-read one (the MTTKRP factor bitmaps and
// values: 32-70 MB re-read ~400 times per call beside 6.4 GB of CSF streamed
// once) keep the gathered array resident by loading it evict_last and the
// stream evict_first (__ldcs).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int64_t ld_keep(const int64_t* a, uint64_t pol) {
  int64_t v;
  asm("ld.global.nc.L2::cache_hint.s64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_keep(const double* a, uint64_t pol) {
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void ld_keep_v4(const unsigned long long* a, uint64_t pol,
                                           unsigned long long& x, unsigned long long& y,
                                           unsigned long long& z, unsigned long long& w) {
  asm("ld.global.nc.L2::cache_hint.v4.u64 {%0,%1,%2,%3}, [%4], %5;"
      : "=l"(x), "=l"(y), "=l"(z), "=l"(w)
      : "l"(a), "l"(pol));
}

__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ---------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk, SASS UBLKCP) into shared memory, completed
// on an mbarrier.  Callers: the sparse MTTKRP match kernel (per-warp rings of
// CSF fiber metadata and nonzeros), the dense MTTKRP heavy-slice kernel (its
// stationary tile of factor rows) and SpAdd (the tile's CSR row segments).
// Source, destination and size must be multiples of 16 bytes.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// makes initialised barriers visible to the async proxy
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// generic-proxy accesses to a buffer ordered before later async-proxy writes
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                              uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
      "[%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

}  // namespace stamgpu
