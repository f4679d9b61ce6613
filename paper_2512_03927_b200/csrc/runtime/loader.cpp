#include "loader.h"

#include <cuda.h>

#include <algorithm>
#include <chrono>

namespace odmoe {

// cuStreamWriteValue32 through the runtime's driver entry point (no link-time libcuda dependency)
typedef CUresult (*PFN_writeValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static PFN_writeValue32 write_value32() {
  static PFN_writeValue32 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_writeValue32>(p);
  }
  return fn;
}
bool stream_write_available() { return write_value32() != nullptr; }
static cudaError_t write_flag(cudaStream_t s, uint32_t* p, uint32_t v) {
  // default flags: the write is ordered after (and makes visible) the stream's earlier copies
  return write_value32()(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(p), v, 0) == CUDA_SUCCESS
             ? cudaSuccess : cudaErrorUnknown;
}

void Loader::start(int device, cudaStream_t copy, int64_t chunk_bytes, int max_inflight) {
  device_ = device;
  copy_ = copy;
  chunk_ = chunk_bytes > 0 ? chunk_bytes : (32 << 20);
  max_inflight_ = max_inflight > 0 ? max_inflight : 2;
  stop_ = false;
  started_ = true;
  th_ = std::thread([this] { run(); });
}

void Loader::stop() {
  if (!started_) return;
  {
    std::lock_guard<std::mutex> lk(mu_);
    stop_ = true;
    for (auto& r : pending_) r->cancelled = true;
    pending_.clear();
  }
  cv_work_.notify_all();
  if (th_.joinable()) th_.join();
  for (auto e : ev_pool_) cudaEventDestroy(e);
  ev_pool_.clear();
  started_ = false;
}

void Loader::submit(const std::shared_ptr<LoadReq>& r) {
  {
    std::lock_guard<std::mutex> lk(mu_);
    r->issued = 0;
    r->cancelled = r->fully_issued = r->done = false;
    pending_.push_back(r);
    loads_issued++;
  }
  cv_work_.notify_all();
}

bool Loader::cancel(const std::shared_ptr<LoadReq>& r) {
  std::lock_guard<std::mutex> lk(mu_);
  if (r->fully_issued || r->cancelled) return false;
  r->cancelled = true;
  pending_.erase(std::remove(pending_.begin(), pending_.end(), r), pending_.end());
  loads_cancelled++;
  cv_issued_.notify_all();
  return true;
}

bool Loader::wait_issued(const std::shared_ptr<LoadReq>& r) {
  std::unique_lock<std::mutex> lk(mu_);
  cv_issued_.wait(lk, [&] { return r->fully_issued || r->cancelled || stop_ || err_.load() != cudaSuccess; });
  return r->fully_issued && err_.load() == cudaSuccess;
}

bool Loader::is_done(const std::shared_ptr<LoadReq>& r) {
  std::lock_guard<std::mutex> lk(mu_);
  return r->done;
}

bool Loader::settled(const std::shared_ptr<LoadReq>& r, int64_t* bytes) {
  std::lock_guard<std::mutex> lk(mu_);
  if (bytes) *bytes = r->issued;
  return r->fully_issued || r->cancelled || err_.load() != cudaSuccess || !started_;
}

void Loader::run() {
  cudaSetDevice(device_);
  std::unique_lock<std::mutex> lk(mu_);
  for (;;) {
    // After a copy-stream error nothing more will land: hand the chunk events back, drop every
    // request (waiters see err_) and leave as soon as stop() asks, without waiting for inflight_.
    if (err_.load() != cudaSuccess) {
      for (auto& c : inflight_) ev_pool_.push_back(c.ev);
      inflight_.clear();
      for (auto& r : pending_) r->cancelled = true;
      pending_.clear();
      cv_issued_.notify_all();
      if (stop_) break;
      cv_work_.wait(lk, [&] { return stop_ || !pending_.empty(); });
      continue;
    }
    // Retire completed chunks (FIFO on one stream: completion is in order).
    while (!inflight_.empty()) {
      const cudaError_t q = cudaEventQuery(inflight_.front().ev);
      if (q == cudaErrorNotReady) break;
      if (q != cudaSuccess) { err_ = q; cv_issued_.notify_all(); break; }
      Chunk c = inflight_.front();
      inflight_.pop_front();
      ev_pool_.push_back(c.ev);
      if (c.last) { c.req->done = true; loads_completed++; }
    }
    // Issue chunks of the most urgent request while the copy queue is short.
    while ((int)inflight_.size() < max_inflight_ && err_.load() == cudaSuccess) {
      int bi = -1;
      for (int i = 0; i < (int)pending_.size(); ++i)
        if (bi < 0 || pending_[i]->key < pending_[bi]->key) bi = i;
      if (bi < 0) break;
      std::shared_ptr<LoadReq> r = pending_[bi];
      cudaError_t e = cudaSuccess;
      if (r->issued == 0 && r->wait_ev != nullptr) e = cudaStreamWaitEvent(copy_, r->wait_ev, 0);
      if (e == cudaSuccess && r->issued == 0 && r->tr_start) e = cudaEventRecord(r->tr_start, copy_);
      int64_t n = std::min(chunk_, r->bytes - r->issued);
      if (r->issued < r->w13_bytes && r->issued + n > r->w13_bytes) n = r->w13_bytes - r->issued;
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(r->dst + r->issued, r->src + r->issued, (size_t)n, cudaMemcpyHostToDevice, copy_);
      r->issued += n;
      bytes_h2d += n;
      if (e == cudaSuccess && r->tr_end) e = cudaEventRecord(r->tr_end, copy_);  // end of the last chunk issued
      if (e == cudaSuccess && r->issued == r->w13_bytes && r->ev_w13) e = cudaEventRecord(r->ev_w13, copy_);
      if (e == cudaSuccess && r->issued == r->w13_bytes && r->flag) e = write_flag(copy_, r->flag, r->epoch);
      const bool last = r->issued == r->bytes;
      if (e == cudaSuccess && last) e = cudaEventRecord(r->ev_done, copy_);
      if (e == cudaSuccess && last && r->flag) e = write_flag(copy_, r->flag + 1, r->epoch);
      cudaEvent_t ev = nullptr;
      if (e == cudaSuccess) {
        if (ev_pool_.empty()) {
          e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        } else {
          ev = ev_pool_.back();
          ev_pool_.pop_back();
        }
      }
      if (e == cudaSuccess) e = cudaEventRecord(ev, copy_);
      if (e != cudaSuccess) { err_ = e; cv_issued_.notify_all(); break; }
      inflight_.push_back(Chunk{ev, r, last});
      if (last) {
        r->fully_issued = true;
        pending_.erase(pending_.begin() + bi);
        cv_issued_.notify_all();
      }
    }
    if (stop_ && inflight_.empty()) break;
    if (inflight_.empty() && pending_.empty()) {
      cv_work_.wait(lk, [&] { return stop_ || !pending_.empty(); });
    } else {
      lk.unlock();
      std::this_thread::sleep_for(std::chrono::microseconds(20));
      lk.lock();
    }
  }
}

}  // namespace odmoe
