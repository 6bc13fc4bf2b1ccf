// Executor state (see executor.cu).
#pragma once

#include <algorithm>
#include <memory>
#include <string>
#include <vector>

#include "device.cuh"
#include "kernels.cuh"
#include "tc_score.cuh"

#include <condition_variable>
#include <mutex>

namespace hyreb {

DevIndex* build_device_index(const Frozen& f, const hyre_index_options& o);
// IndexBuilder::freeze on the GPU (freeze.cu): bit-identical host arrays.
Frozen* freeze_on_device(Builder& b, uint32_t num_bits, uint64_t seed, int device);
// Learned per-row weights of the index's own rows (n == n_rows, each in
// [0, 1]); w == nullptr restores the identity (pure cosine).  Not to be
// called while an executor of this index is running.
void set_row_weights(DevIndex& ix, const float* w, uint64_t n);

// Host barrier of the G shard threads of a ShardedExecutor.
class HostBarrier {
 public:
  explicit HostBarrier(uint32_t n) : n_(n) {}
  void arrive_and_wait() {
    std::unique_lock<std::mutex> lk(m_);
    const uint64_t gen = gen_;
    if (++count_ == n_) {
      count_ = 0;
      ++gen_;
      cv_.notify_all();
      return;
    }
    cv_.wait(lk, [&] { return gen_ != gen; });
  }

 private:
  std::mutex m_;
  std::condition_variable cv_;
  uint32_t n_, count_ = 0;
  uint64_t gen_ = 0;
};

struct Executor;
// An executor that is shard g of G row shards (ShardedExecutor, sharded.cu):
// k is clamped to the global row count, and the quant pre-selection is global
// -- the shards exchange their popcount histograms and tie counts through
// peer-memory reads (every shard's run() is driven by its own host thread).
struct ShardCtx {
  uint32_t g = 0, G = 1;
  uint64_t total_rows = 0;
  std::vector<Executor*> peers;  // [G], peers[g] = this shard
  HostBarrier* barrier = nullptr;
  cudaEvent_t ev_x[2] = {};      // this shard's exchange points (quant histogram, tie counts)
};

struct Executor {
  static constexpr uint32_t kNumCounters = 5;  // n_elig, cand_cnt, samp_cnt, out_cnt, rerun
  // K3 prefilter bound: |exact - prefilter score| for unit rows and queries.
  // bf16 RNE of row and query: |e q - hi(e) hi(q)| <= (2^-8 + 2^-18)|e q| per
  // element, summed <= 2^-8 (1 + 2^-10) |e| |q| (Cauchy-Schwarz); plus fp32
  // accumulation (measured < 2e-5 at d = 128, here allowed 2.4e-4).
  static constexpr float kPrefilterDelta = 1.0f / 256 + 1.0f / 4096;
  // the bound for this index: |e| |q| <= max_row_norm (unit queries)
  float prefilter_delta() const { return kPrefilterDelta * std::max(1.0f, ix->max_row_norm); }
  static constexpr uint32_t kSampleRows = 40 * 1024;  // dense sample slots per query (~40K sampled rows: measured optimum at c3)
  static constexpr uint32_t kFwdMinBatch = 9;          // batches above 8 queries use K1b

  DevIndex* ix;
  uint32_t max_batch;
  cudaStream_t st = nullptr;
  ShardCtx* shard = nullptr;       // set by ShardedExecutor
  uint32_t* d_qhist_sum = nullptr;  // sharded quant: the global histogram
  void shard_exchange(int point);   // record, host barrier, wait for every peer's point
  // stage events of the last kEvRing runs: start, mask, quant, pre-main,
  // post-main, end (ring slot = run counter % kEvRing); ev = the current slot
  static constexpr uint32_t kEvRing = 64;
  cudaEvent_t ev_ring[kEvRing][6] = {};
  uint8_t ev_map[kEvRing][6] = {};  // boundary -> recorded event of that slot (see mark())
  cudaEvent_t* ev = ev_ring[0];
  uint64_t n_runs = 0;
  bool stage_events = true;  // record the inner stage boundaries (hyre_batch_set_stage_events)

  // device scratch sized at construction
  uint32_t cap = 0, samp_cap = 0;
  uint32_t* d_mask = nullptr;
  uint32_t* d_chunk_cnt = nullptr;
  uint32_t* d_counters = nullptr;
  uint64_t* d_thr = nullptr;
  uint64_t* d_thr_safe = nullptr;
  uint64_t* d_cand = nullptr;
  uint32_t* d_samp = nullptr;  // dense sample scores [max_batch][samp_cap] (K2 sample pass)
  uint32_t* d_shist = nullptr;  // K3 sample pass: score histograms [max_batch][kHistBins]
  static constexpr uint32_t kHistBins = 4096;    // linear bins over [-1, 1] (width 4.9e-4)
  static constexpr uint32_t kTcSampleSegs = 100;  // K3 sample: ~100 x 1024 rows at 10M (r02 sweep 60-240 with the bias K-step: 90-120 best)
  uint32_t* d_qhist = nullptr;
  uint32_t* d_tsel = nullptr;
  uint32_t* d_eqcnt = nullptr;
  // grown on demand
  uint8_t* d_blob = nullptr;
  uint8_t* h_blob = nullptr;
  size_t blob_cap = 0;
  hyre_hit* d_hits = nullptr;
  hyre_hit* h_hits = nullptr;
  size_t hits_cap = 0;
  uint32_t* d_scratch = nullptr;
  uint32_t scratch_cap = 0;

  // prepared batch
  bool prepared = false;
  uint32_t B = 0, max_k = 1, sample_period = 1, sample_rows = 0, kernels = 0, n_scratch_used = 0;
  bool any_emb = false, any_term_only = false, any_quant = false;
  std::vector<QParam> qp;
  std::vector<uint32_t> prog;
  std::vector<std::vector<uint32_t>> prog_groups;  // term-major program per 32-query group (kernels.cu)
  std::vector<uint32_t> prog_live;
  // flat clause view of the prepared batch: query i's clauses are
  // [q_cl[i], q_cl[i+1]) with slot cl_slot[k] and index term ids
  // t_ids[cl_t[k] .. cl_t[k+1]) (term ids only on the forward/fused paths)
  std::vector<uint32_t> q_cl, cl_slot, cl_t, t_ids;
  // forward-index (K1b) program
  bool use_fwd = false, fwd_veto = false;
  struct FwdPass {
    uint32_t q0, nw, n_entries, entries, hc, live;
  };
  std::vector<FwdPass> fwd_pass;
  std::vector<uint32_t> fwd_words;
  uint32_t* d_fwd = nullptr;
  std::vector<const uint32_t*> refs;
  std::vector<ScatterItem> items;
  std::vector<uint64_t> item_prefix;
  uint64_t scatter_total = 0;
  std::vector<int32_t> statuses;
  std::vector<std::string> slot_errors;
  std::vector<uint64_t> hit_off;
  std::vector<float> qvec;
  std::vector<uint64_t> qsig;
  uint64_t n_hits_total = 0, h2d_bytes = 0, d2h_bytes = 0;
  uint64_t term_bytes = 0;  // algorithmic eligibility-input bytes of the prepared batch
  uint64_t scan_bytes = 0;  // algorithmic bytes of the K3 main stage (0 on the K2 path)
  // fused CNF in the K3 epilogue (no K1 mask pass): per query group, the
  // term-users program (TcArgs::fz) and its offsets into fz_words
  bool use_fused = false;
  bool use_small = false;  // K7 single-launch exact scorer (small index, single queries)
  bool all_match = false;  // tensor-core batch of match-all queries only: no eligibility pass
  bool k2_match_all = false;  // K2 batch of match-all queries only: no K1 mask (tail masks in K2)
  size_t o_cinit = 0;         // blob offset of the counter image of a k2_match_all run
  struct FusedGroup {
    uint32_t entries, n_entries, hc;
  };
  std::vector<FusedGroup> fz_group;
  std::vector<uint32_t> fz_words;
  std::vector<uint32_t> fz_users, fz_touched, fz_slot;  // build_fused_program scratch
  uint32_t* d_fz = nullptr;
  // tensor-core path (K3)
  bool use_tc = false;
  bool prefilter = false;  // K3 reads the hi plane only; candidates rescored exactly (final_select())
  uint32_t tc_load_ops() const { return prefilter ? 1u : ix->tc_ops; }
  uint32_t tc_q_planes() const { return prefilter ? 1u : 2u; }
  bool pf_i8 = false;  // the prefilter runs on the int8 plane (kind::i8 MMAs)
  uint32_t tc_kb() const { return ix->dp / (pf_i8 ? 128 : 64); }  // 128-byte K atoms per row
  std::vector<int8_t> qi8_h;
  std::vector<float> qscale_h, qdelta_h;  // per query: int8 score scale, prefilter bound
  float* d_qscale = nullptr;
  int8_t* d_qi8 = nullptr;
  float* d_qdelta = nullptr;
  uint32_t tc_stages = 2, tc_term_slots = 2, tc_aps = 1;  // K3 ring depths, K atoms per stage (plan_tc)
  void plan_tc();
  size_t tc_fz_bytes(uint32_t term_slots) const;
  uint32_t tc_np = 0, tc_groups = 0;
  std::vector<uint16_t> qhi_h, qlo_h;
  CUtensorMap tm_qhi{}, tm_qlo{};
  std::vector<uint32_t> h_out_cnt, h_rerun, h_cnt_rerun;
  QParam* d_qp = nullptr;
  float* d_q = nullptr;
  uint64_t* d_qsig = nullptr;
  uint64_t* d_hit_off = nullptr;
  uint32_t* d_prog = nullptr;
  const uint32_t* const* d_refs = nullptr;
  ScatterItem* d_items = nullptr;
  uint64_t* d_ipre = nullptr;

  Executor(DevIndex* index, uint32_t max_batch);
  ~Executor();

  void prepare(const hyre_query* qs, uint32_t b);
  void run();
  void fetch(hyre_hit* hits, const uint64_t* offsets, uint32_t* counts, int32_t* statuses,
             hyre_timings* t);
  float last_run_ms() const;
  // Resolves pending recovery rounds and exhaustive queries, then waits for
  // the stream: the device results are final afterwards.
  void settle();
  void eligible(uint32_t* out);  // n_elig of the last run (D2H, synchronous)
  void stage_ms(float* out) const;  // [mask, quant, sample+kth, main score, select/first-K, total]
  void stage_ms_hist(uint32_t back, float* out) const;  // the same for the run `back` runs ago

  uint64_t full_scan(const hyre_query& q, uint32_t* rows, uint64_t cap_rows);
  uint64_t batch_scan(const hyre_query* qs, uint32_t b, const uint32_t* batch_ids, hyre_messenger* out,
                      uint64_t cap);
  bool exact_scores(const float* q, uint32_t dim, const uint32_t* rows, uint64_t n, float* out);
  uint32_t top_k(const uint32_t* rows, const float* scores, uint64_t n, uint32_t k, hyre_hit* out);
  // off_stride / cnt_stride: elements between shard g's offsets / counts (0 = B)
  void merge_gathered(const hyre_hit* g_hits, const uint64_t* g_off, const uint32_t* g_cnt, uint32_t G,
                      uint64_t hits_stride, uint64_t off_stride = 0, uint64_t cnt_stride = 0);
  uint64_t preselect(const uint64_t* qwords, const uint32_t* rows, uint64_t n, uint32_t quant_k,
                     uint32_t* out);

 private:
  void ensure_blob(size_t bytes);
  void ensure_hits(size_t n);
  void ensure_scratch(uint32_t n_bitmaps);
  void finish_reruns();
  void build_term_major_program();
  void build_forward_program();
  void build_fused_program();
  void score(uint32_t mode, uint64_t* cand, uint32_t* cnt, uint32_t capacity);
  void final_select(SelectArgs fa);
  void mark(int boundary, bool stage_ran);

 public:
  uint32_t finish_rounds = 0;  // recovery rounds fetch() ran for the last batch (diagnostics)

 public:
  // ---- exhaustive exact path (kernels.cu launch_rescore_keys) -------------
  // Hybrid queries with k > kSelectMaxK (bucket_top_k returns min(k, n) for
  // any k, knn.cpp:42-95) run the threshold pipeline with k clamped to
  // kSelectMaxK and are then replaced by an exhaustive exact top-K: every
  // eligible row scored exactly, all keys sorted.  A query whose recovery
  // rounds do not converge within kMaxRecoveryRounds (more rows tied inside
  // the prefilter band than the candidate buffer holds) takes the same path.
  static constexpr int kMaxRecoveryRounds = 3;
  std::vector<uint32_t> true_k;                  // per query min(k, rows)
  std::vector<uint32_t> big_k;                   // queries with hybrid k > kSelectMaxK
  bool exh_done = false;
  uint32_t exh_count = 0;                        // exhaustive queries of the last batch (diagnostics)
  std::vector<uint32_t> raw_cl, raw_slots, raw_offs, raw_ids;  // clause copies of the prepared batch
  std::unique_ptr<Executor> aux;                 // eligibility of one query (K1 + K5 row list)
  uint64_t* d_ex_keys = nullptr;
  uint64_t* d_ex_sorted = nullptr;
  uint32_t* d_ex_rows = nullptr;
  uint8_t* d_ex_tmp = nullptr;
  size_t ex_cap = 0, ex_tmp_cap = 0;
  void finish_exhaustive();
  void exhaustive(uint32_t i);
  uint64_t scan_count(const hyre_query& q);          // prepare + run a term-only query, its eligible count
  void scan_rows(uint32_t* d_rows, uint64_t n);      // its eligible rows (ascending, global) into d_rows
  void ensure_ex(uint64_t n);
  void sort_desc(const uint64_t* in, uint64_t* out, uint64_t n);
};

}  // namespace hyreb
