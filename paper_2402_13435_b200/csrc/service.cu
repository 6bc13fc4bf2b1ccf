// Executor pool with dynamic request batching: the B200 replacement for the
// reference's SearchService::ExecutorPool (service.cpp:99-141), SURVEY.md §8
// row f3.
//
// The reference leases one CPU Executor per HTTP request; each query pays a
// full index scan.  On the GPU a scan costs about the same for 1 or 64
// queries (the batched scorer is bandwidth-bound), so the pool turns
// concurrent single-query requests into execute_batch calls: a request joins
// a shared queue; a worker (one per executor, each with its own CUDA stream)
// takes up to max_batch queued requests, waiting at most max_wait_us for the
// batch to fill once the first request is there, runs them as one batch and
// hands every caller its own result or validation error.  Requests are
// served in arrival order; per-query semantics are those of
// Executor::execute (execute_batch(b)[i] == execute(b[i]) up to the scorer's
// float rounding, pipeline.cpp:146-281).
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "executor.cuh"
#include "service.cuh"

namespace hyreb {

Pool::Pool(DevIndex* ix, uint32_t workers, uint32_t max_batch, uint32_t max_wait_us)
    : max_batch_(max_batch), max_wait_(std::chrono::microseconds(max_wait_us)) {
  if (workers < 1) validation("workers must be >= 1");
  if (max_batch < 1) validation("maxBatch must be >= 1");
  for (uint32_t i = 0; i < workers; ++i) execs_.emplace_back(new Executor(ix, max_batch));
  for (uint32_t i = 0; i < workers; ++i) threads_.emplace_back([this, i] { worker(i); });
}

Pool::~Pool() {
  {
    std::lock_guard<std::mutex> lk(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  for (auto& t : threads_) t.join();
}

void Pool::search(const hyre_query& q, hyre_hit* hits, uint32_t* n_hits) {
  Request r;
  r.q = &q;
  r.hits = hits;
  {
    std::lock_guard<std::mutex> lk(mu_);
    if (stop_) throw Error(HYRE_INTERNAL, "pool is shutting down");
    queue_.push_back(&r);
  }
  cv_.notify_one();
  std::unique_lock<std::mutex> lk(r.mu);
  r.cv.wait(lk, [&] { return r.done; });
  if (r.status != HYRE_OK) throw Error(static_cast<hyre_status>(r.status), r.error);
  if (n_hits) *n_hits = r.count;
}

void Pool::stats(uint64_t* batches, uint64_t* queries) const {
  std::lock_guard<std::mutex> lk(mu_);
  if (batches) *batches = batches_;
  if (queries) *queries = queries_;
}

void Pool::worker(uint32_t w) {
  Executor& ex = *execs_[w];
  std::vector<Request*> batch;
  std::vector<hyre_query> qs;
  std::vector<uint64_t> offs;
  std::vector<uint32_t> counts;
  std::vector<int32_t> statuses;
  std::vector<hyre_hit> hits;
  for (;;) {
    batch.clear();
    bool more = false;
    {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return stop_ || !queue_.empty(); });
      if (queue_.empty()) return;  // stop_ and drained
      // the batching window opens with the first queued request
      const auto deadline = std::chrono::steady_clock::now() + max_wait_;
      while (!stop_ && queue_.size() < max_batch_ &&
             cv_.wait_until(lk, deadline) != std::cv_status::timeout) {
      }
      const size_t n = std::min<size_t>(max_batch_, queue_.size());
      batch.assign(queue_.begin(), queue_.begin() + n);
      queue_.erase(queue_.begin(), queue_.begin() + n);
      ++batches_;
      queries_ += n;
      more = !queue_.empty();
    }
    if (more) cv_.notify_one();  // more work for another worker
    const uint32_t b = static_cast<uint32_t>(batch.size());
    qs.resize(b);
    offs.resize(b);
    counts.assign(b, 0);
    statuses.assign(b, 0);
    uint64_t total = 0;
    for (uint32_t i = 0; i < b; ++i) {
      qs[i] = *batch[i]->q;
      offs[i] = total;
      total += std::min<uint64_t>(qs[i].k, ex.ix->n_rows);
    }
    hits.resize(std::max<uint64_t>(total, 1));
    int32_t fail = HYRE_OK;
    std::string fail_msg;
    try {
      ex.prepare(qs.data(), b);
      ex.run();
      ex.fetch(hits.data(), offs.data(), counts.data(), statuses.data(), nullptr);
    } catch (const Error& e) {
      fail = e.code;
      fail_msg = e.what();
    } catch (const std::exception& e) {
      fail = HYRE_INTERNAL;
      fail_msg = e.what();
    }
    for (uint32_t i = 0; i < b; ++i) {
      Request& r = *batch[i];
      {
        std::lock_guard<std::mutex> lk(r.mu);
        if (fail != HYRE_OK) {
          r.status = fail;
          r.error = fail_msg;
        } else if (statuses[i] != HYRE_OK) {
          r.status = statuses[i];
          r.error = ex.slot_errors[i];
        } else {
          r.count = counts[i];
          if (r.count) std::memcpy(r.hits, hits.data() + offs[i], r.count * sizeof(hyre_hit));
        }
        r.done = true;
        r.cv.notify_one();  // under r.mu: the caller cannot return (and free r) before we let go
      }
    }
  }
}

}  // namespace hyreb
