// runtime.cpp — context, memory and error plumbing behind the C ABI.
#include "runtime.h"

#include <algorithm>
#include <new>

namespace stamrt {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& message) { g_last_error = message; }

void fail(int code, const std::string& message) { throw Failure{code, message}; }

// ---------------------------------------------------------------------------
Call::Call(Ctx* ctx, const stam_options* opts, stam_stats* stats) : ctx_(ctx) {
  if (!ctx) fail(STAM_ERR_PRECONDITION_VIOLATED, "null context");
  if (opts) {
    opts_ = *opts;
  } else {
    stam_cuda_default_options(&opts_);
  }
  stats_ = stats ? stats : &local_stats_;
  std::memset(stats_, 0, sizeof(stam_stats));
  STAM_CUDA_CHECK(cudaSetDevice(ctx_->device));
  ctx_->event_next = 0;
  ctx_->sync_next = 0;
}

Call::~Call() {
  // Temporaries go back to the pool in stream order; nothing here may throw.
  if (copies_open_ && ctx_->event_next < ctx_->event_pool.size()) {
    // staging copies still in flight must land before their buffers are freed
    cudaEvent_t ev = ctx_->event_pool[ctx_->event_next++];
    cudaEventRecord(ev, ctx_->copy_stream);
    cudaStreamWaitEvent(ctx_->stream, ev, 0);
  } else if (copies_open_) {
    cudaStreamSynchronize(ctx_->copy_stream);
  }
  if (d2h_open_) cudaStreamSynchronize(ctx_->d2h_stream);
  if (aux_open_) cudaStreamSynchronize(ctx_->aux_stream);
  for (void* p : temps_) cudaFreeAsync(p, ctx_->stream);
  if (!finished_) cudaStreamSynchronize(ctx_->stream);
  if (!finished_ && result_slot_ && *result_slot_) {
    // failed after allocating the result: release it here
    auto* own = static_cast<Owned*>(*result_slot_);
    if (own->dev) cudaFreeAsync(own->dev, ctx_->stream);
    if (own->host_pending && !own->host) own->host = own->host_pending;
    if (own->host) pinned_recycle(own->host, own->host_bytes);
    delete own;
    *result_slot_ = nullptr;
  }
}

void Call::adopt_result(void** handle_slot) { result_slot_ = handle_slot; }

void Call::pinned_recycle(void* p, size_t bytes) {
  ctx_->pinned_free.emplace_back(p, bytes);
  if (ctx_->pinned_free.size() > 8) {
    cudaFreeHost(ctx_->pinned_free.front().first);
    ctx_->pinned_free.erase(ctx_->pinned_free.begin());
  }
}

cudaEvent_t Call::next_event() {
  if (ctx_->event_next >= ctx_->event_pool.size()) {
    for (int e = 0; e < 64; e++) {
      cudaEvent_t ev;
      STAM_CUDA_CHECK(cudaEventCreate(&ev));
      ctx_->event_pool.push_back(ev);
    }
  }
  return ctx_->event_pool[ctx_->event_next++];
}

void* Call::scratch(size_t bytes) {
  void* p = nullptr;
  if (bytes == 0) bytes = 16;
  STAM_CUDA_CHECK(cudaMallocFromPoolAsync(&p, bytes, ctx_->pool, ctx_->stream));
  temps_.push_back(p);
  stats_->bytes_allocated += (int64_t)bytes;
  return p;
}

void* Call::scratch_zero(size_t bytes) {
  void* p = scratch(bytes);
  STAM_CUDA_CHECK(cudaMemsetAsync(p, 0, bytes ? bytes : 16, ctx_->stream));
  return p;
}

const void* Call::stage(const void* p, size_t bytes, int32_t mem) {
  if (mem == STAM_MEM_DEVICE || bytes == 0) return p;
  if (mem != STAM_MEM_HOST) fail(STAM_ERR_PRECONDITION_VIOLATED, "unknown memory kind");
  if (!p) fail(STAM_ERR_PRECONDITION_VIOLATED, "null host input array");
  if (opts_.timing && !h2d_start_) {
    h2d_start_ = next_event();
    h2d_stop_ = next_event();
    STAM_CUDA_CHECK(cudaEventRecord(h2d_start_, ctx_->stream));
  }
  void* d = scratch(bytes);
  STAM_CUDA_CHECK(cudaMemcpyAsync(d, p, bytes, cudaMemcpyHostToDevice, ctx_->stream));
  if (opts_.timing) STAM_CUDA_CHECK(cudaEventRecord(h2d_stop_, ctx_->stream));
  return d;
}

cudaEvent_t Call::event() {
  // ordering-only events: no timestamps (cheaper to record and wait on)
  if (ctx_->sync_next >= ctx_->sync_pool.size()) {
    for (int e = 0; e < 64; e++) {
      cudaEvent_t ev;
      STAM_CUDA_CHECK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      ctx_->sync_pool.push_back(ev);
    }
  }
  return ctx_->sync_pool[ctx_->sync_next++];
}

void Call::copy_range(void* dst, const void* src, size_t bytes) {
  if (!ctx_->copy_stream)
    STAM_CUDA_CHECK(cudaStreamCreateWithFlags(&ctx_->copy_stream, cudaStreamNonBlocking));
  if (!copies_open_) {
    // the staging buffers were allocated in kernel-stream order
    cudaEvent_t ready = event();
    STAM_CUDA_CHECK(cudaEventRecord(ready, ctx_->stream));
    STAM_CUDA_CHECK(cudaStreamWaitEvent(ctx_->copy_stream, ready, 0));
    copies_open_ = true;
  }
  if (bytes)
    STAM_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx_->copy_stream));
}

cudaEvent_t Call::copy_fence() {
  cudaEvent_t ev = event();
  STAM_CUDA_CHECK(cudaEventRecord(ev, ctx_->copy_stream ? ctx_->copy_stream : ctx_->stream));
  return ev;
}

cudaStream_t Call::fork() {
  if (!ctx_->aux_stream)
    STAM_CUDA_CHECK(cudaStreamCreateWithFlags(&ctx_->aux_stream, cudaStreamNonBlocking));
  cudaEvent_t ev = event();
  STAM_CUDA_CHECK(cudaEventRecord(ev, ctx_->stream));
  STAM_CUDA_CHECK(cudaStreamWaitEvent(ctx_->aux_stream, ev, 0));
  aux_open_ = true;
  return ctx_->aux_stream;
}

void Call::join() {
  if (!aux_open_) return;
  aux_open_ = false;
  cudaEvent_t ev = event();
  STAM_CUDA_CHECK(cudaEventRecord(ev, ctx_->aux_stream));
  STAM_CUDA_CHECK(cudaStreamWaitEvent(ctx_->stream, ev, 0));
}

void Call::wait(cudaEvent_t ev) { STAM_CUDA_CHECK(cudaStreamWaitEvent(ctx_->stream, ev, 0)); }

void Call::before_launch(const char* name, cudaStream_t st) {
  stats_->kernel_launches++;
  if (!opts_.timing) return;
  TimedLaunch t{name, nullptr, nullptr};
  t.start = next_event();
  t.stop = next_event();
  STAM_CUDA_CHECK(cudaEventRecord(t.start, st ? st : ctx_->stream));
  launches_.push_back(t);
  pending_ = (int)launches_.size() - 1;
}

void Call::after_launch(cudaStream_t st) {
  STAM_CUDA_CHECK(cudaGetLastError());
  if (!opts_.timing || pending_ < 0) return;
  STAM_CUDA_CHECK(cudaEventRecord(launches_[pending_].stop, st ? st : ctx_->stream));
  pending_ = -1;
}

int64_t Call::read_scalar(const int64_t* dptr) {
  int64_t v = 0;
  read_scalars(dptr, 1, &v);
  return v;
}

void Call::read_scalars(const int64_t* dptr, int n, int64_t* out) {
  if (n > ctx_->h_scalars_cap) {
    STAM_CUDA_CHECK(cudaStreamSynchronize(ctx_->stream));
    if (ctx_->h_scalars) STAM_CUDA_CHECK(cudaFreeHost(ctx_->h_scalars));
    ctx_->h_scalars = nullptr;
    ctx_->h_scalars_cap = 0;
    STAM_CUDA_CHECK(cudaMallocHost(&ctx_->h_scalars, (size_t)n * sizeof(int64_t)));
    ctx_->h_scalars_cap = n;
  }
  STAM_CUDA_CHECK(cudaMemcpyAsync(ctx_->h_scalars, dptr, n * sizeof(int64_t),
                                  cudaMemcpyDeviceToHost, ctx_->stream));
  STAM_CUDA_CHECK(cudaStreamSynchronize(ctx_->stream));
  std::memcpy(out, ctx_->h_scalars, n * sizeof(int64_t));
}

void* Call::pinned_alloc(size_t bytes) {
  auto& fl = ctx_->pinned_free;
  // best fit among cached buffers
  size_t best = fl.size();
  for (size_t i = 0; i < fl.size(); i++) {
    if (fl[i].second >= bytes && (best == fl.size() || fl[i].second < fl[best].second)) best = i;
  }
  if (best != fl.size()) {
    void* p = fl[best].first;
    fl.erase(fl.begin() + best);
    return p;
  }
  void* p = nullptr;
  STAM_CUDA_CHECK(cudaMallocHost(&p, bytes));
  return p;
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

void Call::alloc_csr_result(stam_csr_result* r, int64_t nrows, int64_t ncols,
                            int64_t nnz_capacity) {
  if (!r) fail(STAM_ERR_PRECONDITION_VIOLATED, "null result");
  std::memset(r, 0, sizeof(*r));
  size_t pos_b = align_up((size_t)(nrows + 1) * sizeof(int64_t), 256);
  size_t idx_b = align_up((size_t)std::max<int64_t>(nnz_capacity, 1) * sizeof(int64_t), 256);
  size_t val_b = align_up((size_t)std::max<int64_t>(nnz_capacity, 1) * sizeof(double), 256);
  auto* own = new Owned();
  void* d = nullptr;
  cudaError_t e = cudaMallocFromPoolAsync(&d, pos_b + idx_b + val_b, ctx_->pool, ctx_->stream);
  if (e != cudaSuccess) {
    delete own;
    fail(e == cudaErrorMemoryAllocation ? STAM_ERR_OUT_OF_MEMORY : STAM_ERR_CUDA,
         std::string("result allocation: ") + cudaGetErrorString(e));
  }
  own->dev = d;
  stats_->bytes_allocated += (int64_t)(pos_b + idx_b + val_b);
  r->handle = own;
  adopt_result(&r->handle);
  r->nrows = nrows;
  r->ncols = ncols;
  r->pos = (int64_t*)d;
  r->idx = (int64_t*)((char*)d + pos_b);
  r->vals = (double*)((char*)d + pos_b + idx_b);
  r->mem = STAM_MEM_DEVICE;
}

void Call::alloc_csr_result_streamed(stam_csr_result* r, int64_t nrows, int64_t ncols,
                                     int64_t nnz_capacity, int64_t** hpos, int64_t** hidx,
                                     double** hvals) {
  alloc_csr_result(r, nrows, ncols, nnz_capacity);
  auto* own = static_cast<Owned*>(r->handle);
  const size_t pos_b = align_up((size_t)(nrows + 1) * sizeof(int64_t), 256);
  const size_t idx_b = align_up((size_t)std::max<int64_t>(nnz_capacity, 1) * sizeof(int64_t), 256);
  const size_t val_b = align_up((size_t)std::max<int64_t>(nnz_capacity, 1) * sizeof(double), 256);
  char* h = static_cast<char*>(pinned_alloc(pos_b + idx_b + val_b));
  own->host_pending = h;
  own->host_bytes = pos_b + idx_b + val_b;
  *hpos = (int64_t*)h;
  *hidx = (int64_t*)(h + pos_b);
  *hvals = (double*)(h + pos_b + idx_b);
}

void Call::d2h_range(void* dst, const void* src, size_t bytes, cudaEvent_t ready) {
  if (!ctx_->d2h_stream)
    STAM_CUDA_CHECK(cudaStreamCreateWithFlags(&ctx_->d2h_stream, cudaStreamNonBlocking));
  if (ready) STAM_CUDA_CHECK(cudaStreamWaitEvent(ctx_->d2h_stream, ready, 0));
  d2h_open_ = true;
  if (bytes)
    STAM_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx_->d2h_stream));
}

void Call::finish_csr_result_streamed(stam_csr_result* r, int64_t nnz) {
  auto* own = static_cast<Owned*>(r->handle);
  r->nnz = nnz;
  if (d2h_open_) {
    cudaEvent_t done = event();
    STAM_CUDA_CHECK(cudaEventRecord(done, ctx_->d2h_stream));
    STAM_CUDA_CHECK(cudaStreamWaitEvent(ctx_->stream, done, 0));
  }
  char* h = static_cast<char*>(own->host_pending);
  const size_t pos_b = align_up((size_t)(r->nrows + 1) * sizeof(int64_t), 256);
  const size_t idx_b = (size_t)((char*)r->vals - (char*)r->idx);
  STAM_CUDA_CHECK(cudaFreeAsync(own->dev, ctx_->stream));
  own->dev = nullptr;
  own->host = h;
  own->host_pending = nullptr;
  r->pos = (int64_t*)h;
  r->idx = (int64_t*)(h + pos_b);
  r->vals = (double*)(h + pos_b + idx_b);
  r->mem = STAM_MEM_HOST;
}

void Call::alloc_csr_result_host(stam_csr_result* r, int64_t nrows, int64_t ncols,
                                 int64_t nnz_capacity) {
  if (!r) fail(STAM_ERR_PRECONDITION_VIOLATED, "null result");
  std::memset(r, 0, sizeof(*r));
  const size_t pos_b = align_up((size_t)(nrows + 1) * sizeof(int64_t), 256);
  const size_t idx_b = align_up((size_t)std::max<int64_t>(nnz_capacity, 1) * sizeof(int64_t), 256);
  const size_t val_b = align_up((size_t)std::max<int64_t>(nnz_capacity, 1) * sizeof(double), 256);
  auto* own = new Owned();
  char* h = nullptr;
  try {
    h = static_cast<char*>(pinned_alloc(pos_b + idx_b + val_b));
  } catch (...) {
    delete own;
    throw;
  }
  own->host = h;
  own->host_bytes = pos_b + idx_b + val_b;
  r->handle = own;
  adopt_result(&r->handle);
  r->nrows = nrows;
  r->ncols = ncols;
  r->pos = (int64_t*)h;
  r->idx = (int64_t*)(h + pos_b);
  r->vals = (double*)(h + pos_b + idx_b);
  r->mem = STAM_MEM_HOST;
}

void Call::finish_csr_result_host(stam_csr_result* r, int64_t nnz) {
  if (d2h_open_) STAM_CUDA_CHECK(cudaStreamSynchronize(ctx_->d2h_stream));
  d2h_open_ = false;
  r->nnz = nnz;
}

int64_t* Call::marks() {
  if (!ctx_->h_marks) {
    void* p = nullptr;
    STAM_CUDA_CHECK(cudaHostAlloc(&p, Ctx::kMarks * sizeof(int64_t), cudaHostAllocMapped));
    ctx_->h_marks = static_cast<int64_t*>(p);
  }
  return ctx_->h_marks;
}

void Call::finish_csr_result(stam_csr_result* r, int64_t nnz) {
  r->nnz = nnz;
  if (opts_.result_mem != STAM_MEM_HOST) return;
  auto* own = static_cast<Owned*>(r->handle);
  size_t pos_b = (size_t)(r->nrows + 1) * sizeof(int64_t);
  size_t idx_b = (size_t)nnz * sizeof(int64_t);
  size_t val_b = (size_t)nnz * sizeof(double);
  size_t total = pos_b + idx_b + val_b;
  void* h = pinned_alloc(total ? total : 16);
  own->host = h;
  own->host_bytes = total ? total : 16;
  if (opts_.timing) {
    d2h_start_ = next_event();
    d2h_stop_ = next_event();
    STAM_CUDA_CHECK(cudaEventRecord(d2h_start_, ctx_->stream));
  }
  char* hc = (char*)h;
  STAM_CUDA_CHECK(cudaMemcpyAsync(hc, r->pos, pos_b, cudaMemcpyDeviceToHost, ctx_->stream));
  if (nnz) {
    STAM_CUDA_CHECK(cudaMemcpyAsync(hc + pos_b, r->idx, idx_b, cudaMemcpyDeviceToHost, ctx_->stream));
    STAM_CUDA_CHECK(cudaMemcpyAsync(hc + pos_b + idx_b, r->vals, val_b, cudaMemcpyDeviceToHost,
                                    ctx_->stream));
  }
  if (opts_.timing) STAM_CUDA_CHECK(cudaEventRecord(d2h_stop_, ctx_->stream));
  STAM_CUDA_CHECK(cudaFreeAsync(own->dev, ctx_->stream));
  own->dev = nullptr;
  r->pos = (int64_t*)hc;
  r->idx = (int64_t*)(hc + pos_b);
  r->vals = (double*)(hc + pos_b + idx_b);
  r->mem = STAM_MEM_HOST;
}

void Call::alloc_dense_result(stam_dense_result* r, int64_t nrows, int64_t ncols) {
  if (!r) fail(STAM_ERR_PRECONDITION_VIOLATED, "null result");
  std::memset(r, 0, sizeof(*r));
  size_t b = align_up((size_t)std::max<int64_t>(nrows * ncols, 1) * sizeof(double), 256);
  auto* own = new Owned();
  void* d = nullptr;
  cudaError_t e = cudaMallocFromPoolAsync(&d, b, ctx_->pool, ctx_->stream);
  if (e != cudaSuccess) {
    delete own;
    fail(e == cudaErrorMemoryAllocation ? STAM_ERR_OUT_OF_MEMORY : STAM_ERR_CUDA,
         std::string("result allocation: ") + cudaGetErrorString(e));
  }
  own->dev = d;
  stats_->bytes_allocated += (int64_t)b;
  r->handle = own;
  adopt_result(&r->handle);
  r->nrows = nrows;
  r->ncols = ncols;
  r->vals = (double*)d;
  r->mem = STAM_MEM_DEVICE;
}

void Call::finish_dense_result(stam_dense_result* r) {
  if (opts_.result_mem != STAM_MEM_HOST) return;
  auto* own = static_cast<Owned*>(r->handle);
  size_t b = (size_t)(r->nrows * r->ncols) * sizeof(double);
  void* h = pinned_alloc(b ? b : 16);
  own->host = h;
  own->host_bytes = b ? b : 16;
  if (opts_.timing) {
    d2h_start_ = next_event();
    d2h_stop_ = next_event();
    STAM_CUDA_CHECK(cudaEventRecord(d2h_start_, ctx_->stream));
  }
  if (b) STAM_CUDA_CHECK(cudaMemcpyAsync(h, r->vals, b, cudaMemcpyDeviceToHost, ctx_->stream));
  if (opts_.timing) STAM_CUDA_CHECK(cudaEventRecord(d2h_stop_, ctx_->stream));
  STAM_CUDA_CHECK(cudaFreeAsync(own->dev, ctx_->stream));
  own->dev = nullptr;
  r->vals = (double*)h;
  r->mem = STAM_MEM_HOST;
}

void Call::finish() {
  STAM_CUDA_CHECK(cudaStreamSynchronize(ctx_->stream));
  STAM_CUDA_CHECK(cudaGetLastError());
  finished_ = true;
  if (!opts_.timing) return;
  float best = -1.f, total = 0.f;
  for (const auto& t : launches_) {
    float ms = 0.f;
    STAM_CUDA_CHECK(cudaEventElapsedTime(&ms, t.start, t.stop));
    total += ms;
    if (ms > best) {
      best = ms;
      std::strncpy(stats_->main_kernel, t.name, sizeof(stats_->main_kernel) - 1);
    }
  }
  stats_->main_kernel_ms = best < 0 ? 0.f : best;
  stats_->total_kernel_ms = total;
  if (h2d_start_) STAM_CUDA_CHECK(cudaEventElapsedTime(&stats_->h2d_ms, h2d_start_, h2d_stop_));
  if (d2h_start_) STAM_CUDA_CHECK(cudaEventElapsedTime(&stats_->d2h_ms, d2h_start_, d2h_stop_));
}

// ---------------------------------------------------------------------------
std::vector<int64_t> stream_blocks(int64_t nunits, int64_t total_bytes, int64_t steady_bytes,
                                   int64_t max_blocks) {
  std::vector<int64_t> b{0};
  if (nunits <= 0) {
    b.push_back(0);
    return b;
  }
  const double per_unit = std::max(1.0, (double)total_bytes / (double)nunits);
  // ramp 1/16, 1/8, 1/4, 1/2 of the steady size at both ends
  std::vector<int64_t> sizes;
  int64_t left = total_bytes;
  std::vector<int64_t> tail;
  for (int64_t s = steady_bytes / 16; s < steady_bytes && left > 4 * s; s *= 2) {
    sizes.push_back(s);
    tail.push_back(s);
    left -= 2 * s;
  }
  while (left > 0) {
    sizes.push_back(std::min(left, steady_bytes));
    left -= steady_bytes;
  }
  for (auto it = tail.rbegin(); it != tail.rend(); ++it) sizes.push_back(*it);
  if ((int64_t)sizes.size() > max_blocks) {
    sizes.assign((size_t)max_blocks, (total_bytes + max_blocks - 1) / max_blocks);
  }
  double acc = 0.0;
  for (int64_t s : sizes) {
    acc += (double)s;
    const int64_t u = std::min<int64_t>(nunits, std::max<int64_t>(b.back() + 1, (int64_t)(acc / per_unit)));
    if (u > b.back()) b.push_back(u);
    if (b.back() == nunits) break;
  }
  if (b.back() != nunits) b.push_back(nunits);
  return b;
}

void check_csr_view(const stam_csr_view* v, const char* what) {
  if (!v) fail(STAM_ERR_PRECONDITION_VIOLATED, std::string(what) + ": null view");
  if (v->nrows <= 0 || v->ncols <= 0)
    fail(STAM_ERR_DIMENSION_MISMATCH, std::string(what) + ": dimensions must be positive");
  if (v->nnz < 0) fail(STAM_ERR_PRECONDITION_VIOLATED, std::string(what) + ": negative nnz");
  if (!v->pos) fail(STAM_ERR_PRECONDITION_VIOLATED, std::string(what) + ": null pos");
  if (v->nnz > 0 && (!v->idx || !v->vals))
    fail(STAM_ERR_PRECONDITION_VIOLATED, std::string(what) + ": null idx/vals");
  if (v->nnz >= (int64_t)1 << 61)
    fail(STAM_ERR_OUT_OF_RANGE, std::string(what) + ": nnz exceeds 2^61");
}

void check_csf3_view(const stam_csf3_view* v, const char* what) {
  if (!v) fail(STAM_ERR_PRECONDITION_VIOLATED, std::string(what) + ": null view");
  for (int d = 0; d < 3; d++)
    if (v->dims[d] <= 0)
      fail(STAM_ERR_DIMENSION_MISMATCH, std::string(what) + ": dimensions must be positive");
  if (v->nfibers < 0 || v->nnz < 0)
    fail(STAM_ERR_PRECONDITION_VIOLATED, std::string(what) + ": negative sizes");
  if (!v->pos1) fail(STAM_ERR_PRECONDITION_VIOLATED, std::string(what) + ": null pos1");
  if (v->nfibers > 0 && (!v->idx1 || !v->pos2))
    fail(STAM_ERR_PRECONDITION_VIOLATED, std::string(what) + ": null fiber arrays");
  if (v->nnz > 0 && (!v->idx2 || !v->vals))
    fail(STAM_ERR_PRECONDITION_VIOLATED, std::string(what) + ": null idx2/vals");
}

void check_dense_view(const stam_dense_view* v, const char* what) {
  if (!v) fail(STAM_ERR_PRECONDITION_VIOLATED, std::string(what) + ": null view");
  if (v->nrows <= 0 || v->ncols <= 0)
    fail(STAM_ERR_DIMENSION_MISMATCH, std::string(what) + ": dimensions must be positive");
  if (!v->vals) fail(STAM_ERR_PRECONDITION_VIOLATED, std::string(what) + ": null vals");
}

}  // namespace stamrt

// ===========================================================================
// C ABI: context management
// ===========================================================================
using namespace stamrt;

struct stam_cuda_ctx : public stamrt::Ctx {};

extern "C" {

int stam_cuda_abi_version(void) { return STAM_CUDA_ABI_VERSION; }

const char* stam_cuda_last_error(void) { return g_last_error.c_str(); }

void stam_cuda_default_options(stam_options* opts) {
  if (!opts) return;
  opts->sort = 1;
  opts->mode = STAM_MODE_FUSED;
  opts->result_mem = STAM_MEM_DEVICE;
  opts->timing = 0;
}

int stam_cuda_ctx_create(int device, stam_cuda_ctx** out) {
  return guarded([&] {
    if (!out) fail(STAM_ERR_PRECONDITION_VIOLATED, "null output pointer");
    *out = nullptr;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
      fail(STAM_ERR_NO_DEVICE, std::string("no CUDA device: ") + cudaGetErrorString(e));
    if (device < 0 || device >= n) fail(STAM_ERR_OUT_OF_RANGE, "device index out of range");
    STAM_CUDA_CHECK(cudaSetDevice(device));
    cudaDeviceProp prop;
    STAM_CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      fail(STAM_ERR_NO_DEVICE, std::string("kernels are built for sm_100a; device is ") +
                                   prop.name);
    auto* c = new stam_cuda_ctx();
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    c->smem_optin = prop.sharedMemPerBlockOptin;
    STAM_CUDA_CHECK(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
    c->stream = c->own_stream;
    // a private stream-ordered pool: results and per-call temporaries are
    // recycled without touching the OS allocator, and the device's default
    // pool (shared with every other library in the process) stays as it was
    cudaMemPoolProps pp;
    std::memset(&pp, 0, sizeof(pp));
    pp.allocType = cudaMemAllocationTypePinned;
    pp.handleTypes = cudaMemHandleTypeNone;
    pp.location.type = cudaMemLocationTypeDevice;
    pp.location.id = device;
    STAM_CUDA_CHECK(cudaMemPoolCreate(&c->pool, &pp));
    uint64_t threshold = UINT64_MAX;
    STAM_CUDA_CHECK(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    STAM_CUDA_CHECK(cudaMallocHost(&c->h_scalars, 64 * sizeof(int64_t)));
    c->h_scalars_cap = 64;
    for (int i = 0; i < 64; i++) {
      cudaEvent_t ev;
      STAM_CUDA_CHECK(cudaEventCreate(&ev));
      c->event_pool.push_back(ev);
    }
    *out = c;
  });
}

int stam_cuda_ctx_destroy(stam_cuda_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto& p : ctx->pinned_free) cudaFreeHost(p.first);
    for (auto ev : ctx->event_pool) cudaEventDestroy(ev);
    for (auto ev : ctx->sync_pool) cudaEventDestroy(ev);
    if (ctx->h_scalars) cudaFreeHost(ctx->h_scalars);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->d2h_stream) cudaStreamDestroy(ctx->d2h_stream);
    if (ctx->aux_stream) cudaStreamDestroy(ctx->aux_stream);
    if (ctx->h_marks) cudaFreeHost(ctx->h_marks);
    // results still held by the caller keep the pool alive until released
    if (ctx->pool) cudaMemPoolDestroy(ctx->pool);
    delete ctx;
  });
}

int stam_cuda_ctx_set_stream(stam_cuda_ctx* ctx, void* stream) {
  return guarded([&] {
    if (!ctx) fail(STAM_ERR_PRECONDITION_VIOLATED, "null context");
    ctx->stream = stream ? (cudaStream_t)stream : ctx->own_stream;
  });
}

int stam_cuda_ctx_device(const stam_cuda_ctx* ctx) { return ctx ? ctx->device : -1; }

int stam_cuda_synchronize(stam_cuda_ctx* ctx) {
  return guarded([&] {
    if (!ctx) fail(STAM_ERR_PRECONDITION_VIOLATED, "null context");
    STAM_CUDA_CHECK(cudaSetDevice(ctx->device));
    STAM_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  });
}

int stam_cuda_release(stam_cuda_ctx* ctx, void* handle) {
  return guarded([&] {
    if (!ctx) fail(STAM_ERR_PRECONDITION_VIOLATED, "null context");
    if (!handle) return;
    auto* own = static_cast<Owned*>(handle);
    STAM_CUDA_CHECK(cudaSetDevice(ctx->device));
    if (own->dev) STAM_CUDA_CHECK(cudaFreeAsync(own->dev, ctx->stream));
    if (own->host_pending && !own->host) own->host = own->host_pending;
    if (own->host) {
      // keep a bounded cache of pinned buffers (pinning is slow)
      ctx->pinned_free.emplace_back(own->host, own->host_bytes);
      if (ctx->pinned_free.size() > 8) {
        cudaFreeHost(ctx->pinned_free.front().first);
        ctx->pinned_free.erase(ctx->pinned_free.begin());
      }
    }
    delete own;
  });
}

}  // extern "C"
