// Executor pool with dynamic request batching (service.cu).
#pragma once

#include <chrono>
#include <condition_variable>
#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "device.cuh"

namespace hyreb {

struct Executor;

class Pool {
 public:
  Pool(DevIndex* ix, uint32_t workers, uint32_t max_batch, uint32_t max_wait_us);
  ~Pool();
  // Blocking and thread-safe: queues the query, waits for its batch.
  // hits needs min(k, rows) entries.  Validation errors throw.
  void search(const hyre_query& q, hyre_hit* hits, uint32_t* n_hits);
  void stats(uint64_t* batches, uint64_t* queries) const;

 private:
  struct Request {
    const hyre_query* q = nullptr;
    hyre_hit* hits = nullptr;
    uint32_t count = 0;
    int32_t status = HYRE_OK;
    std::string error;
    bool done = false;
    std::mutex mu;
    std::condition_variable cv;
  };
  void worker(uint32_t w);

  uint32_t max_batch_;
  std::chrono::microseconds max_wait_;
  std::vector<std::unique_ptr<Executor>> execs_;
  std::vector<std::thread> threads_;
  mutable std::mutex mu_;
  std::condition_variable cv_;
  std::deque<Request*> queue_;
  bool stop_ = false;
  uint64_t batches_ = 0, queries_ = 0;
};

}  // namespace hyreb
