// ShardedExecutor: one index row-sharded over G GPUs (or G shards of one GPU)
// in a single process -- SURVEY.md §8(e): contiguous row ranges
// [g N / G, (g + 1) N / G), one stream per shard, per-shard top-K merged
// exactly on the root device.  See sharded.cu.
#pragma once

#include <functional>
#include <memory>
#include <thread>
#include <vector>

#include "executor.cuh"
#include "hyre_b200.h"

namespace hyreb {

// G persistent host threads; run_all(fn) runs fn(g) on thread g and returns
// when every call has finished (rethrowing the first exception).
class ShardPool {
 public:
  explicit ShardPool(uint32_t n);
  ~ShardPool();
  void run_all(const std::function<void(uint32_t)>& fn);

 private:
  void loop(uint32_t g);
  std::mutex m_;
  std::condition_variable cv_, done_cv_;
  std::vector<std::thread> th_;
  const std::function<void(uint32_t)>* fn_ = nullptr;
  uint64_t gen_ = 0;
  uint32_t pending_ = 0;
  bool stop_ = false;
  std::vector<std::exception_ptr> err_;
};

// The device shards of one frozen index: shard g = rows
// [g N / G, (g + 1) N / G) on its device; peer access enabled between them.
struct ShardedIndex {
  ShardedIndex(const Frozen& f, const hyre_sharded_index_options& o);
  uint32_t G;
  uint64_t total_rows;
  std::vector<std::unique_ptr<DevIndex>> ix;
};

class ShardedExecutor {
 public:
  ShardedExecutor(ShardedIndex& index, uint32_t max_batch);
  ~ShardedExecutor();
  void prepare(const hyre_query* qs, uint32_t b);  // every shard (parallel host threads)
  void run();     // every shard's kernels + the root merge, enqueued without host synchronisation
  void settle();  // resolve recovery / exhaustive work on every shard, re-merge if any shard changed
  void fetch(hyre_hit* hits, const uint64_t* offsets, uint32_t* counts, int32_t* statuses, hyre_timings* t);
  void device_results(void** hits, uint64_t* n_hits, void** counts) const;
  uint32_t shards() const { return G; }
  int device_of(uint32_t g) const { return sx.ix[g]->device; }
  cudaStream_t root_stream() const { return ex[0]->st; }
  Executor& root() { return *ex[0]; }
  uint32_t recovery_rounds = 0, exhaustive_queries = 0;  // of the last settled batch, all shards
  uint32_t kernels_per_run() const;

 private:
  void merge();
  ShardedIndex& sx;
  uint32_t G;
  std::vector<std::unique_ptr<Executor>> ex;
  std::vector<ShardCtx> ctx;
  std::unique_ptr<HostBarrier> barrier;
  std::unique_ptr<ShardPool> pool;
  std::vector<cudaEvent_t> ev_done;
  cudaEvent_t ev_merged = nullptr;
  bool merged_once = false, settled = false;
  // merge buffers (root device)
  uint64_t* d_keys = nullptr;
  uint32_t* d_kcnt = nullptr;
  uint64_t* d_thr0 = nullptr;
  uint32_t* d_rerun0 = nullptr;
  uint32_t* d_out_cnt = nullptr;
  uint32_t* d_true_k = nullptr;
  hyre_hit* d_hits = nullptr;
  size_t hits_cap = 0;
  hyre_hit* h_hits = nullptr;
  std::vector<uint32_t> h_cnt;
  uint32_t cap = 0;
  uint32_t merge_kernels = 0;
};

}  // namespace hyreb
