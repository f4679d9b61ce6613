// Copy-stream expert loader ("dynamically loads each target expert ...
// just-in-time ... and promptly evicts it afterward").
//
// One host thread per GPU feeds the GPU's H2D copy engine from the pinned host pool in fixed
// chunks, keeping at most `max_inflight` chunks queued on the copy stream. Because only a couple
// of chunks are ever queued, the loader can (a) always serve the most urgent request first
// (smallest key = earliest layer in decode order, so a misprediction reload for the layer being
// computed jumps ahead of prefetches) and (b) stop a mispredicted load after the chunk in
// flight instead of copying the whole 352 MB expert.
//
// Per request two events are recorded on the copy stream: after the W13 part (the first GEMV may
// start) and after the whole blob. A request may carry a `wait_ev` (the compute-done event of the
// slot's previous occupant) that the copy stream waits on before the first chunk, so a slot is
// never overwritten while a GEMV still reads it.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

namespace odmoe {

bool stream_write_available();  // cuStreamWriteValue32 reachable (the warm wait needs it)

struct LoadReq {
  int layer = -1, expert = -1, slot = -1;
  int64_t key = 0;                 // need order; smaller is served first
  const char* src = nullptr;       // pinned host
  char* dst = nullptr;             // device slot
  int64_t bytes = 0, w13_bytes = 0;
  cudaEvent_t ev_w13 = nullptr, ev_done = nullptr;  // owned by the slot
  cudaEvent_t wait_ev = nullptr;   // optional: copy stream waits on it before the first chunk
  uint32_t* flag = nullptr;        // optional device words [w13 landed, blob landed] the copy stream sets to
  uint32_t epoch = 0;              // `epoch` (stream memory writes) for a compute-stream spin wait
  cudaEvent_t tr_start = nullptr, tr_end = nullptr;  // optional timing events (event trace): before the
                                   // first chunk / after every chunk (the last record = end of the copy)
  // loader-owned state (guarded by Loader::mu_)
  int64_t issued = 0;
  bool cancelled = false, fully_issued = false, done = false;
};

class Loader {
 public:
  Loader() = default;
  ~Loader() { stop(); }
  void start(int device, cudaStream_t copy, int64_t chunk_bytes, int max_inflight);
  void stop();
  void submit(const std::shared_ptr<LoadReq>& r);
  // Stop issuing further chunks of r (chunks already queued still land). Returns true if the
  // request had not been fully issued.
  bool cancel(const std::shared_ptr<LoadReq>& r);
  // Block until every chunk of r is queued (its events are recorded). Returns false on error.
  bool wait_issued(const std::shared_ptr<LoadReq>& r);
  bool is_done(const std::shared_ptr<LoadReq>& r);
  // No further chunk of r will be issued (fully issued, cancelled or the loader failed); *bytes =
  // bytes issued for it.
  bool settled(const std::shared_ptr<LoadReq>& r, int64_t* bytes);
  cudaError_t error() const { return err_.load(); }

  std::atomic<int64_t> bytes_h2d{0}, loads_issued{0}, loads_completed{0}, loads_cancelled{0};

 private:
  void run();
  struct Chunk {
    cudaEvent_t ev;
    std::shared_ptr<LoadReq> req;
    bool last;
  };
  int device_ = 0;
  cudaStream_t copy_ = nullptr;
  int64_t chunk_ = 32 << 20;
  int max_inflight_ = 2;
  std::mutex mu_;
  std::condition_variable cv_work_, cv_issued_;
  std::vector<std::shared_ptr<LoadReq>> pending_;
  std::deque<Chunk> inflight_;
  std::vector<cudaEvent_t> ev_pool_;
  bool stop_ = false, started_ = false;
  std::atomic<cudaError_t> err_{cudaSuccess};
  std::thread th_;
};

}  // namespace odmoe
