// ShardedExecutor: the multi-GPU form of Executor.
//
// The reference runs one Executor over one FrozenIndex
// (proj/src/pipeline.cpp:95-281); rows are independent (eligibility and score
// of a row depend only on that row and the query), so the index is split into
// G contiguous row ranges, shard g resident on its own device with its own
// Executor and stream.  A batch:
//   1. every shard prepares (validation + programs; identical queries, so
//      identical statuses) and runs its kernel sequence -- G host threads, no
//      host synchronisation; k is clamped to the WHOLE index's rows;
//   2. quant pre-selection (on by default, pipeline.hpp:18) is global: the
//      shards sum their popcount histograms and offset their tie budgets by
//      reading each other's buffers in peer memory (Executor::shard_exchange),
//      so exactly the reference's quant_k survivors remain over all shards;
//   3. the root (shard 0's device) waits for every shard's stream (events)
//      and merges in one kernel pass that reads every shard's hit lists in
//      place through peer memory -- NVLink loads on a multi-GPU node, no
//      staging copy or collective library call -- then the exact K4 select
//      over the G x K keys (the global top-K is a subset of the union of the
//      shard top-Ks, and keys carry global rows, so the tie rule holds);
//      term-only lists are concatenated in shard (= row) order.
// Recovery rounds / exhaustive queries a shard needs are resolved at settle
// (fetch), after which the merge is redone.
#include <algorithm>
#include <cstring>

#include "kernels.cuh"
#include "sharded.cuh"

namespace hyreb {

// ---------------------------------------------------------------------------
ShardPool::ShardPool(uint32_t n) : err_(n) {
  for (uint32_t g = 0; g < n; ++g) th_.emplace_back([this, g] { loop(g); });
}

ShardPool::~ShardPool() {
  {
    std::lock_guard<std::mutex> lk(m_);
    stop_ = true;
  }
  cv_.notify_all();
  for (auto& t : th_) t.join();
}

void ShardPool::loop(uint32_t g) {
  uint64_t seen = 0;
  for (;;) {
    const std::function<void(uint32_t)>* fn;
    {
      std::unique_lock<std::mutex> lk(m_);
      cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      fn = fn_;
    }
    try {
      (*fn)(g);
    } catch (...) {
      err_[g] = std::current_exception();
    }
    {
      std::lock_guard<std::mutex> lk(m_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
}

void ShardPool::run_all(const std::function<void(uint32_t)>& fn) {
  {
    std::unique_lock<std::mutex> lk(m_);
    std::fill(err_.begin(), err_.end(), nullptr);
    fn_ = &fn;
    pending_ = static_cast<uint32_t>(th_.size());
    ++gen_;
  }
  cv_.notify_all();
  {
    std::unique_lock<std::mutex> lk(m_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
  }
  for (auto& e : err_)
    if (e) std::rethrow_exception(e);
}

// ---------------------------------------------------------------------------
ShardedIndex::ShardedIndex(const Frozen& f, const hyre_sharded_index_options& o) : G(o.n_shards) {
  if (G < 1 || G > kMaxShards)
    validation("n_shards must be in [1, " + std::to_string(kMaxShards) + "]");
  if (f.num_docs < G) validation("fewer rows than shards");
  int n_dev = 0;
  HYRE_CUDA(cudaGetDeviceCount(&n_dev));
  std::vector<int> dev(G);
  for (uint32_t g = 0; g < G; ++g) {
    dev[g] = o.devices ? o.devices[g] : static_cast<int>(g % std::max(1, n_dev));
    if (dev[g] < 0 || dev[g] >= n_dev) validation("shard device " + std::to_string(dev[g]) + " does not exist");
  }
  // every device reads every other shard's buffers (quant exchange, merge)
  for (uint32_t a = 0; a < G; ++a)
    for (uint32_t b = 0; b < G; ++b) {
      if (dev[a] == dev[b]) continue;
      int ok = 0;
      HYRE_CUDA(cudaDeviceCanAccessPeer(&ok, dev[a], dev[b]));
      if (!ok)
        throw Error(HYRE_CUDA_ERROR, "device " + std::to_string(dev[a]) + " cannot access device " +
                                         std::to_string(dev[b]) + " (peer access is required for sharding)");
      HYRE_CUDA(cudaSetDevice(dev[a]));
      const cudaError_t e = cudaDeviceEnablePeerAccess(dev[b], 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else HYRE_CUDA(e);
    }
  total_rows = f.num_docs;
  for (uint32_t g = 0; g < G; ++g) {
    hyre_index_options io{dev[g], o.emb_dtype, static_cast<uint32_t>(total_rows * g / G),
                          static_cast<uint32_t>(total_rows * (g + 1) / G), o.tensor_path, 0};
    ix.emplace_back(build_device_index(f, io));
  }
}

ShardedExecutor::ShardedExecutor(ShardedIndex& index, uint32_t max_batch) : sx(index), G(index.G) {
  if (max_batch < 1) validation("maxBatch must be >= 1");
  std::vector<int> dev(G);
  for (uint32_t g = 0; g < G; ++g) dev[g] = sx.ix[g]->device;
  ctx.resize(G);
  barrier = std::make_unique<HostBarrier>(G);
  for (uint32_t g = 0; g < G; ++g) ex.push_back(std::make_unique<Executor>(sx.ix[g].get(), max_batch));
  ev_done.resize(G);
  for (uint32_t g = 0; g < G; ++g) {
    ctx[g].g = g;
    ctx[g].G = G;
    ctx[g].total_rows = sx.total_rows;
    ctx[g].barrier = barrier.get();
    for (uint32_t h = 0; h < G; ++h) ctx[g].peers.push_back(ex[h].get());
    HYRE_CUDA(cudaSetDevice(dev[g]));
    for (auto& e : ctx[g].ev_x) HYRE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    HYRE_CUDA(cudaEventCreateWithFlags(&ev_done[g], cudaEventDisableTiming));
    ex[g]->shard = &ctx[g];
  }
  HYRE_CUDA(cudaSetDevice(dev[0]));
  HYRE_CUDA(cudaEventCreateWithFlags(&ev_merged, cudaEventDisableTiming));
  const size_t B = max_batch;
  cap = G * kSelectMaxK;
  d_keys = nullptr;
  HYRE_CUDA(cudaMalloc(&d_keys, B * cap * sizeof(uint64_t)));
  HYRE_CUDA(cudaMalloc(&d_kcnt, B * sizeof(uint32_t)));
  HYRE_CUDA(cudaMalloc(&d_thr0, B * sizeof(uint64_t)));
  HYRE_CUDA(cudaMemset(d_thr0, 0, B * sizeof(uint64_t)));
  HYRE_CUDA(cudaMalloc(&d_rerun0, B * sizeof(uint32_t)));
  HYRE_CUDA(cudaMalloc(&d_out_cnt, B * sizeof(uint32_t)));
  HYRE_CUDA(cudaMalloc(&d_true_k, B * sizeof(uint32_t)));
  h_cnt.resize(B);
  pool = std::make_unique<ShardPool>(G);
}

ShardedExecutor::~ShardedExecutor() {
  pool.reset();
  for (auto& e : ex) {
    cudaSetDevice(e->ix->device);
    cudaStreamSynchronize(e->st);
  }
  ex.clear();
  for (uint32_t g = 0; g < G && g < ctx.size(); ++g) {
    cudaSetDevice(sx.ix[g]->device);
    for (auto& e : ctx[g].ev_x)
      if (e) cudaEventDestroy(e);
    if (ev_done[g]) cudaEventDestroy(ev_done[g]);
  }
  cudaSetDevice(sx.ix[0]->device);
  if (ev_merged) cudaEventDestroy(ev_merged);
  for (void* p : {(void*)d_keys, (void*)d_kcnt, (void*)d_thr0, (void*)d_rerun0, (void*)d_out_cnt, (void*)d_true_k,
                  (void*)d_hits})
    cudaFree(p);
  if (h_hits) cudaFreeHost(h_hits);
}

void ShardedExecutor::prepare(const hyre_query* qs, uint32_t b) {
  pool->run_all([&](uint32_t g) { ex[g]->prepare(qs, b); });
  Executor& r = *ex[0];
  HYRE_CUDA(cudaSetDevice(r.ix->device));
  const size_t n = std::max<uint64_t>(1, r.n_hits_total);
  if (n > hits_cap) {
    HYRE_CUDA(cudaStreamSynchronize(r.st));
    cudaFree(d_hits);
    if (h_hits) cudaFreeHost(h_hits);
    hits_cap = std::max(n, hits_cap * 2);
    HYRE_CUDA(cudaMalloc(&d_hits, hits_cap * sizeof(hyre_hit)));
    HYRE_CUDA(cudaMemsetAsync(d_hits, 0, hits_cap * sizeof(hyre_hit), r.st));  // initcheck: see Executor::ensure_hits
    HYRE_CUDA(cudaMallocHost(&h_hits, hits_cap * sizeof(hyre_hit)));
  }
  HYRE_CUDA(cudaMemcpyAsync(d_true_k, r.true_k.data(), b * sizeof(uint32_t), cudaMemcpyHostToDevice, r.st));
  settled = false;
}

void ShardedExecutor::run() {
  // a shard may start overwriting its results only after the previous
  // batch's merge has read them
  pool->run_all([&](uint32_t g) {
    Executor& e = *ex[g];
    HYRE_CUDA(cudaSetDevice(e.ix->device));
    if (merged_once) HYRE_CUDA(cudaStreamWaitEvent(e.st, ev_merged, 0));
    e.run();
    HYRE_CUDA(cudaEventRecord(ev_done[g], e.st));
  });
  merge();
}

// Root-device merge over every shard's results in peer memory.
void ShardedExecutor::merge() {
  Executor& r = *ex[0];
  HYRE_CUDA(cudaSetDevice(r.ix->device));
  for (uint32_t g = 1; g < G; ++g) HYRE_CUDA(cudaStreamWaitEvent(r.st, ev_done[g], 0));
  PeerHits ph{};
  for (uint32_t g = 0; g < G; ++g) {
    ph.hits[g] = ex[g]->d_hits;
    ph.cnt[g] = ex[g]->d_counters + 3 * ex[g]->max_batch;  // out_cnt
  }
  const uint32_t B = r.B;
  merge_kernels = 0;
  if (r.any_emb) {
    launch_gather_peer_keys(ph, G, r.d_hit_off, r.d_qp, B, cap, d_keys, d_kcnt, r.st);
    SelectArgs fa{d_keys, d_kcnt, cap, r.d_qp, d_kcnt, SELECT_FINAL, d_thr0, d_rerun0, d_hits, r.d_hit_off,
                  d_out_cnt, B, QF_ACTIVE | QF_EMB, cap, nullptr, 1, 0};
    launch_select(fa, r.st);
    merge_kernels += 2;
  }
  if (r.any_term_only) {
    launch_concat_term_only(ph, G, r.d_hit_off, r.d_qp, d_true_k, B, d_hits, d_out_cnt, r.st);
    ++merge_kernels;
  }
  // hybrid k above the shared-memory select: sort the G shard lists (rare)
  for (uint32_t i : r.big_k) {
    uint32_t n = 0;
    const uint64_t n_cap = uint64_t{G} * r.true_k[i];
    r.ensure_ex(n_cap);
    launch_gather_peer_keys_one(ph, G, r.hit_off[i], i, n_cap, r.d_ex_keys, d_kcnt + i, r.st);
    HYRE_CUDA(cudaMemcpyAsync(&n, d_kcnt + i, 4, cudaMemcpyDeviceToHost, r.st));
    HYRE_CUDA(cudaStreamSynchronize(r.st));
    r.sort_desc(r.d_ex_keys, r.d_ex_sorted, n);
    launch_keys_to_hits(r.d_ex_sorted, std::min<uint64_t>(n, r.true_k[i]), d_hits + r.hit_off[i], d_out_cnt + i,
                        nullptr, r.st);
  }
  HYRE_CUDA(cudaGetLastError());
  HYRE_CUDA(cudaEventRecord(ev_merged, r.st));
  merged_once = true;
}

void ShardedExecutor::settle() {
  if (settled) return;
  std::vector<uint32_t> before(G);
  for (uint32_t g = 0; g < G; ++g) before[g] = ex[g]->finish_rounds + ex[g]->exh_count;
  pool->run_all([&](uint32_t g) {
    HYRE_CUDA(cudaSetDevice(ex[g]->ix->device));
    ex[g]->settle();
  });
  bool changed = false;
  recovery_rounds = exhaustive_queries = 0;
  for (uint32_t g = 0; g < G; ++g) {
    recovery_rounds += ex[g]->finish_rounds;
    exhaustive_queries += ex[g]->exh_count;
    changed |= ex[g]->finish_rounds + ex[g]->exh_count != before[g];
  }
  if (changed) {
    for (uint32_t g = 0; g < G; ++g) {
      HYRE_CUDA(cudaSetDevice(ex[g]->ix->device));
      HYRE_CUDA(cudaEventRecord(ev_done[g], ex[g]->st));
    }
    merge();
  }
  settled = true;
}

void ShardedExecutor::fetch(hyre_hit* hits, const uint64_t* offsets, uint32_t* counts, int32_t* st_out,
                            hyre_timings* t) {
  settle();
  Executor& r = *ex[0];
  HYRE_CUDA(cudaSetDevice(r.ix->device));
  const uint32_t B = r.B;
  HYRE_CUDA(cudaMemcpyAsync(h_cnt.data(), d_out_cnt, B * 4, cudaMemcpyDeviceToHost, r.st));
  HYRE_CUDA(cudaMemcpyAsync(h_hits, d_hits, r.n_hits_total * sizeof(hyre_hit), cudaMemcpyDeviceToHost, r.st));
  HYRE_CUDA(cudaStreamSynchronize(r.st));
  for (uint32_t i = 0; i < B; ++i) {
    if (st_out) st_out[i] = r.statuses[i];
    const uint32_t c = r.statuses[i] == HYRE_OK ? h_cnt[i] : 0u;
    if (counts) counts[i] = c;
    if (hits && c) std::memcpy(hits + offsets[i], h_hits + r.hit_off[i], c * sizeof(hyre_hit));
  }
  if (t) {
    float s6[6];
    r.stage_ms(s6);
    t->tbr_ms = s6[0];
    t->quant_ms = s6[1];
    t->ebr_ms = s6[2] + s6[3];
    t->topk_ms = s6[4];
  }
}

void ShardedExecutor::device_results(void** hits, uint64_t* n_hits, void** counts) const {
  if (hits) *hits = d_hits;
  if (n_hits) *n_hits = ex[0]->n_hits_total;
  if (counts) *counts = d_out_cnt;
}

uint32_t ShardedExecutor::kernels_per_run() const {
  uint32_t k = merge_kernels;
  for (const auto& e : ex) k += e->kernels;
  return k;
}

}  // namespace hyreb
