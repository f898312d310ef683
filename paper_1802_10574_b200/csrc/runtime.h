// runtime.h — host-side runtime shared by the kernel translation units:
// the context (device, stream, stream-ordered pool, pinned result cache,
// timing events), per-call scratch scopes, input staging, and the error
// convention of the C ABI (stam_cuda.h).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "stam_cuda.h"

namespace stamrt {

// Internal failure; converted to a status code at the C ABI boundary.
struct Failure {
  int code;
  std::string message;
};

[[noreturn]] void fail(int code, const std::string& message);
void set_last_error(const std::string& message);

#define STAM_CUDA_CHECK(expr)                                                   \
  do {                                                                          \
    cudaError_t _e = (expr);                                                    \
    if (_e != cudaSuccess) {                                                    \
      ::stamrt::fail(_e == cudaErrorMemoryAllocation ? STAM_ERR_OUT_OF_MEMORY   \
                                                     : STAM_ERR_CUDA,           \
                     std::string(#expr) + ": " + cudaGetErrorString(_e));       \
    }                                                                           \
  } while (0)

struct TimedLaunch {
  const char* name;
  cudaEvent_t start, stop;
};

struct Ctx {
  int device = 0;
  int num_sms = 148;
  size_t smem_optin = 227 * 1024;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // host->device staging overlapped with kernels
  cudaStream_t d2h_stream = nullptr;   // device->host result blocks overlapped with kernels
  cudaStream_t aux_stream = nullptr;   // bandwidth-bound kernels overlapped with compute-bound ones
  // pinned, device-mapped marks written by kernels (e.g. a row block's end
  // offset) and read by the host after the block's event
  int64_t* h_marks = nullptr;
  static constexpr int kMarks = 128;
  cudaMemPool_t pool = nullptr;
  // pinned host memory returned by released host results, reused by size
  std::vector<std::pair<void*, size_t>> pinned_free;
  // small pinned scalars for count read-back (grown on demand)
  int64_t* h_scalars = nullptr;
  int h_scalars_cap = 0;
  std::vector<cudaEvent_t> event_pool;  // timing-capable (kernel timings, H2D / D2H times)
  size_t event_next = 0;
  std::vector<cudaEvent_t> sync_pool;   // cudaEventDisableTiming (stream ordering only)
  size_t sync_next = 0;
};

// Result ownership record behind stam_*_result.handle.
struct Owned {
  void* dev = nullptr;
  void* host = nullptr;
  size_t host_bytes = 0;
  void* host_pending = nullptr;  // streamed host buffer, handed out by finish
};

// Per-call state: temporary device allocations (freed stream-ordered at the
// end of the call), timing events and launch counts.
class Call {
 public:
  Call(Ctx* ctx, const stam_options* opts, stam_stats* stats);
  ~Call();

  Ctx* ctx() const { return ctx_; }
  cudaStream_t stream() const { return ctx_->stream; }
  const stam_options& opts() const { return opts_; }

  // Temporary device allocation released when the call ends.
  void* scratch(size_t bytes);
  template <typename T>
  T* scratch_n(size_t n) {
    return static_cast<T*>(scratch(n * sizeof(T)));
  }
  // Zero-filled temporary allocation.
  void* scratch_zero(size_t bytes);

  // Device pointer for a possibly-host input array (copied H2D when needed).
  template <typename T>
  const T* device_input(const T* p, size_t n, int32_t mem) {
    return static_cast<const T*>(stage(p, n * sizeof(T), mem));
  }

  // Streamed staging: a device buffer for a host array whose ranges are
  // copied on the context's copy stream (copy_range), each batch of copies
  // closed by copy_fence() -> an event the kernel stream waits on.
  template <typename T>
  T* host_staging(size_t n) {
    return static_cast<T*>(scratch(n * sizeof(T)));
  }
  void copy_range(void* dst, const void* src, size_t bytes);
  cudaEvent_t copy_fence();
  void wait(cudaEvent_t ev);
  cudaEvent_t event();
  // Every event acquisition goes through here: grows the context's pool
  // (timing-capable events) when a call needs more than it holds.
  cudaEvent_t next_event();

  // Launch bookkeeping: call before/after each kernel launch.
  void before_launch(const char* name, cudaStream_t st = nullptr);
  void after_launch(cudaStream_t st = nullptr);
  // Second kernel stream: fork() orders it after the main stream's work so
  // far and returns it; join() orders the main stream after it (before the
  // call's temporaries are released).
  cudaStream_t fork();
  void join();

  // Read one int64 from device memory (synchronizes the stream).
  int64_t read_scalar(const int64_t* dptr);
  void read_scalars(const int64_t* dptr, int n, int64_t* out);

  // Result buffers: one device block holding pos/idx/vals (or vals only).
  void alloc_csr_result(stam_csr_result* r, int64_t nrows, int64_t ncols, int64_t nnz_capacity);
  void finish_csr_result(stam_csr_result* r, int64_t nnz);
  // Host result filled block by block while later blocks compute: device
  // result + a pinned host buffer of the same capacity; d2h_range copies a
  // finished range on the d2h stream (after `ready`), finish_csr_result_streamed
  // joins the copies and hands out the host buffer.
  void alloc_csr_result_streamed(stam_csr_result* r, int64_t nrows, int64_t ncols,
                                 int64_t nnz_capacity, int64_t** hpos, int64_t** hidx,
                                 double** hvals);
  void d2h_range(void* dst, const void* src, size_t bytes, cudaEvent_t ready);
  // Host-only CSR result (pinned, capacity nnz_capacity) filled by the caller
  // with d2h_range; finish_csr_result_host sets nnz after joining the copies.
  void alloc_csr_result_host(stam_csr_result* r, int64_t nrows, int64_t ncols,
                             int64_t nnz_capacity);
  void finish_csr_result_host(stam_csr_result* r, int64_t nnz);
  void finish_csr_result_streamed(stam_csr_result* r, int64_t nnz);
  int64_t* marks();
  void alloc_dense_result(stam_dense_result* r, int64_t nrows, int64_t ncols);
  void finish_dense_result(stam_dense_result* r);

  // Synchronize, harvest timings into stats.
  void finish();

  stam_stats* stats() { return stats_; }

 private:
  const void* stage(const void* p, size_t bytes, int32_t mem);
  void* pinned_alloc(size_t bytes);
  void pinned_recycle(void* p, size_t bytes);
  // The result allocated by this call: released by the destructor unless
  // finish() succeeded (a call that fails after allocating its result must
  // not hand the caller a handle it has no reason to release).
  void adopt_result(void** handle_slot);
  void** result_slot_ = nullptr;

  Ctx* ctx_;
  stam_options opts_;
  stam_stats* stats_;
  stam_stats local_stats_;
  std::vector<void*> temps_;
  std::vector<TimedLaunch> launches_;
  cudaEvent_t h2d_start_ = nullptr, h2d_stop_ = nullptr;
  cudaEvent_t d2h_start_ = nullptr, d2h_stop_ = nullptr;
  bool finished_ = false;
  bool copies_open_ = false;
  bool d2h_open_ = false;
  bool aux_open_ = false;
  int pending_ = -1;
};

// Runs `fn` translating Failure / std::exception into status codes.
template <typename F>
int guarded(F&& fn) {
  try {
    fn();
    return STAM_OK;
  } catch (const Failure& f) {
    set_last_error(f.message);
    return f.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return STAM_ERR_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return STAM_ERR_INTERNAL;
  }
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Block boundaries (in units, first 0, last nunits) for a streamed call
// moving `total_bytes` spread evenly over `nunits`: small blocks first and
// last (short pipeline fill and drain), `steady_bytes` blocks in between,
// at most max_blocks blocks.
std::vector<int64_t> stream_blocks(int64_t nunits, int64_t total_bytes, int64_t steady_bytes,
                                   int64_t max_blocks);

// Validates a CSR view's scalar fields (array contents are trusted; the C++
// wrapper validates storage before calling, as TensorStorage::validate does).
void check_csr_view(const stam_csr_view* v, const char* what);
void check_csf3_view(const stam_csf3_view* v, const char* what);
void check_dense_view(const stam_dense_view* v, const char* what);

}  // namespace stamrt
