// Executor: the B200 replacement for hyre::Executor (pipeline.hpp:69-96,
// pipeline.cpp:95-281).  Host work per batch is validation, query
// normalisation (double, like pipeline.cpp:19-28), term-dictionary lookups and
// one packed H2D copy; everything else is a fixed kernel sequence on the
// executor's stream:
//
//   [scatter CSR clauses] -> K1 mask -> [K6 quant] ->
//   K2 sample pass -> K4 K-th (threshold) -> K2/K3 main pass -> K4 final
//   -> K2 rerun + K4 (no-op unless a candidate buffer overflowed)
//   -> K5 first-K (term-only queries)
//
// All device scratch is sized at construction (pipeline.cpp:95-106's
// "pre-allocated" policy); only the per-batch program blob and the hit
// buffer grow, and only when a batch needs more than any earlier one.
#include <cub/cub.cuh>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <unordered_map>

#include "executor.cuh"
#include "kernels.cuh"

namespace hyreb {

namespace {
template <class T>
T* dmalloc(size_t n) {
  T* p = nullptr;
  if (n) HYRE_CUDA(cudaMalloc(&p, n * sizeof(T)));
  return p;
}
size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
uint32_t tc_debug_flags() {  // HYRE_TC_DEBUG: profiling experiments only; HYRE_TC_BIAS=0: IADD threshold compare
  static const uint32_t v = [] {
    const char* e = std::getenv("HYRE_TC_DEBUG");
    const char* b = std::getenv("HYRE_TC_BIAS");
    return (e ? static_cast<uint32_t>(std::atoi(e)) : 0u) | (b && std::string(b) == "0" ? 0x200u : 0u);
  }();
  return v;
}
// HYRE_FUSED=0 disables the fused-CNF K3 epilogue (tests, profiling).
bool fused_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("HYRE_FUSED");
    return !(e && std::string(e) == "0");
  }();
  return v;
}
// HYRE_K2_DENSE_SAMPLE=1: the K2 sample fills dense slots + a K-th selection
// (two extra kernels) instead of score histograms + hist_thr.
bool k2_hist_sample() {
  static const bool v = [] {
    const char* e = std::getenv("HYRE_K2_DENSE_SAMPLE");
    return !(e && std::string(e) == "1");
  }();
  return v;
}
// HYRE_SMALL=0 disables the K7 single-launch path for small indexes.
bool small_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("HYRE_SMALL");
    return !(e && std::string(e) == "0");
  }();
  return v;
}
// HYRE_PREFILTER=0 disables the K3 prefilter + exact rescore (the K3 pass
// then reads the full hi/lo split and scores at fp32 grade directly);
// HYRE_PREFILTER=bf16 forces the bf16 prefilter over the int8 one.
bool prefilter_enabled() {
  static const bool v = [] {
    const char* e = std::getenv("HYRE_PREFILTER");
    return !(e && std::string(e) == "0");
  }();
  return v;
}
bool k2_i8_enabled() {  // HYRE_K2_I8=0: single / small batches stream the fp32 (bf16) rows directly
  static const bool v = [] {
    const char* e = std::getenv("HYRE_K2_I8");
    return !(e && std::string(e) == "0");
  }();
  return v;
}
uint32_t tc_backoff_ns() {  // HYRE_TC_BACKOFF_NS: profiling the K3 wait back-off
  static const uint32_t v = [] {
    const char* e = std::getenv("HYRE_TC_BACKOFF_NS");
    return e ? static_cast<uint32_t>(std::atoi(e)) : 64u;
  }();
  return v;
}
bool prefilter_i8_allowed() {
  static const bool v = [] {
    const char* e = std::getenv("HYRE_PREFILTER");
    return !(e && std::string(e) == "bf16");
  }();
  return v;
}
// HYRE_MASK_PATH=bitmap|fwd forces the K1 / K1b choice (tests, profiling).
int mask_path() {
  static const int v = [] {
    const char* e = std::getenv("HYRE_MASK_PATH");
    if (!e) return 0;
    return std::string(e) == "bitmap" ? 1 : (std::string(e) == "fwd" ? 2 : 0);
  }();
  return v;
}
// HYRE_DEBUG_PREP: accumulate host prepare phase times, print at exit.
struct PrepProfile {
  double t[6] = {0, 0, 0, 0, 0, 0};
  std::vector<std::array<double, 6>> calls;
  uint64_t n = 0;
  bool on = std::getenv("HYRE_DEBUG_PREP") != nullptr;
  ~PrepProfile() {
    if (!on || calls.empty()) return;
    std::array<double, 6> med{};
    for (int i = 0; i < 6; ++i) {
      std::vector<double> v;
      for (auto& c : calls) v.push_back(c[i]);
      std::nth_element(v.begin(), v.begin() + v.size() / 2, v.end());
      med[i] = v[v.size() / 2];
    }
    std::fprintf(stderr, "[hyre] prepare median us/call (%zu calls): queries %.1f program %.1f sample %.1f qsplit %.1f "
                 "pack %.1f h2d %.1f\n", calls.size(), med[0], med[1], med[2], med[3], med[4], med[5]);
  }
};
PrepProfile g_prep;
double us_since(std::chrono::steady_clock::time_point& t0) {
  const auto t1 = std::chrono::steady_clock::now();
  const double us = std::chrono::duration<double, std::micro>(t1 - t0).count();
  t0 = t1;
  return us;
}
uint16_t bf16_rne(float f) {  // round-to-nearest-even, as __float2bfloat16_rn
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return static_cast<uint16_t>((u >> 16) | 0x40);  // NaN
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}
float bf16_to_f(uint16_t h) {
  const uint32_t u = static_cast<uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
}  // namespace

Executor::Executor(DevIndex* index, uint32_t mb) : ix(index), max_batch(mb) {
  if (max_batch < 1) validation("maxBatch must be >= 1");
  HYRE_CUDA(cudaSetDevice(ix->device));
  HYRE_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  for (auto& set : ev_ring)
    for (auto& e : set) HYRE_CUDA(cudaEventCreate(&e));
  const size_t B = max_batch;
  cap = 65536;
  samp_cap = kSampleRows;
  d_mask = dmalloc<uint32_t>(B * ix->words);
  d_chunk_cnt = dmalloc<uint32_t>(B * ix->n_chunks);
  d_counters = dmalloc<uint32_t>(B * kNumCounters);
  d_thr = dmalloc<uint64_t>(B);
  d_thr_safe = dmalloc<uint64_t>(B);
  d_cand = dmalloc<uint64_t>(B * cap);
  d_samp = dmalloc<uint32_t>(B * samp_cap);
  d_shist = dmalloc<uint32_t>(B * kHistBins);
  d_qhist = dmalloc<uint32_t>(B * (ix->num_bits + 1));
  d_tsel = dmalloc<uint32_t>(B * 4);
  d_eqcnt = dmalloc<uint32_t>(B * ix->n_chunks);
  h_out_cnt.resize(B);
  h_rerun.resize(B);
  h_cnt_rerun.resize(2 * B);
}

Executor::~Executor() {
  cudaSetDevice(ix->device);
  cudaStreamSynchronize(st);
  for (void* p : {(void*)d_mask, (void*)d_chunk_cnt, (void*)d_counters, (void*)d_thr, (void*)d_thr_safe, (void*)d_cand,
                  (void*)d_shist,
                  (void*)d_samp, (void*)d_qhist, (void*)d_tsel, (void*)d_eqcnt, (void*)d_blob,
                  (void*)d_hits, (void*)d_scratch, (void*)d_qhist_sum, (void*)d_ex_keys, (void*)d_ex_sorted, (void*)d_ex_rows,
                  (void*)d_ex_tmp})
    cudaFree(p);
  if (h_blob) cudaFreeHost(h_blob);
  if (h_hits) cudaFreeHost(h_hits);
  for (auto& set : ev_ring)
    for (auto& e : set) cudaEventDestroy(e);
  cudaStreamDestroy(st);
}

void Executor::ensure_blob(size_t bytes) {
  if (bytes <= blob_cap) return;
  HYRE_CUDA(cudaStreamSynchronize(st));
  cudaFree(d_blob);
  if (h_blob) cudaFreeHost(h_blob);
  blob_cap = std::max(bytes, blob_cap * 2);
  d_blob = dmalloc<uint8_t>(blob_cap);
  HYRE_CUDA(cudaMallocHost(&h_blob, blob_cap));
}

void Executor::ensure_hits(size_t n) {
  n = std::max<size_t>(n, 1);
  if (n <= hits_cap) return;
  HYRE_CUDA(cudaStreamSynchronize(st));
  cudaFree(d_hits);
  if (h_hits) cudaFreeHost(h_hits);
  hits_cap = std::max(n, hits_cap * 2);
  d_hits = dmalloc<hyre_hit>(hits_cap);
  // fetch copies every query's whole k-slot range; slots past a query's hit
  // count are never read, but keep them initialised (compute-sanitizer initcheck)
  HYRE_CUDA(cudaMemsetAsync(d_hits, 0, hits_cap * sizeof(hyre_hit), st));
  HYRE_CUDA(cudaMallocHost(&h_hits, hits_cap * sizeof(hyre_hit)));
}

void Executor::ensure_scratch(uint32_t n_bitmaps) {
  if (n_bitmaps <= scratch_cap) return;
  HYRE_CUDA(cudaStreamSynchronize(st));
  cudaFree(d_scratch);
  scratch_cap = std::max(n_bitmaps, scratch_cap * 2);
  d_scratch = dmalloc<uint32_t>(size_t{scratch_cap} * ix->words);
}

// ---------------------------------------------------------------------------
// prepare: validation + program construction + one packed H2D copy.
// ---------------------------------------------------------------------------
void Executor::prepare(const hyre_query* qs, uint32_t b) {
  if (b < 1) validation("batch must contain at least one query");
  if (b > max_batch)
    validation("batch size " + std::to_string(b) + " exceeds maxBatch " + std::to_string(max_batch));
  HYRE_CUDA(cudaSetDevice(ix->device));
  auto tp = std::chrono::steady_clock::now();
  B = b;
  const uint32_t dp = ix->dp, nw = ix->num_words, W = ix->words;
  const QueryShape shape{ix->num_clauses, ix->dim};
  qp.assign(b, QParam{});
  prog.clear();
  refs.clear();
  items.clear();
  item_prefix.clear();
  statuses.assign(b, HYRE_OK);
  slot_errors.assign(b, std::string());
  hit_off.assign(b, 0);
  qvec.assign(size_t{b} * dp, 0.0f);
  qsig.assign(size_t{b} * nw, 0ull);
  q_cl.assign(b + 1, 0);
  cl_slot.clear();
  cl_t.clear();
  t_ids.clear();
  any_emb = any_term_only = any_quant = false;
  max_k = 1;
  true_k.assign(b, 0);
  big_k.clear();
  raw_cl.assign(b + 1, 0);
  raw_slots.clear();
  raw_offs.clear();
  raw_ids.clear();
  uint32_t n_scratch = 0;
  std::unordered_map<uint32_t, uint32_t> bitmap_ref;  // bitmap index -> ref slot
  std::vector<std::pair<uint32_t, uint32_t>> ref_src;  // (kind 0 bitmap / 1 scratch, index)
  uint64_t total_hits = 0;
  // Batches evaluate the CNF from the forward term lists (K1b, one read of
  // the row term ids for all queries); single queries and small batches use
  // the inverted bitmaps / CSR postings of just their own terms (K1).
  use_fwd = ix->row_terms != nullptr && b >= kFwdMinBatch && mask_path() != 1 && !fwd_veto;
  fwd_veto = false;
  for (uint32_t i = 0; i < b; ++i) {
    const hyre_query& q = qs[i];
    q_cl[i] = static_cast<uint32_t>(cl_slot.size());
    raw_cl[i] = static_cast<uint32_t>(raw_slots.size());
    try {
      validate_query(shape, q);
    } catch (const Error& e) {
      statuses[i] = e.code;
      slot_errors[i] = e.what();
      continue;
    }
    for (uint32_t c = 0; c < q.n_clauses; ++c) {  // kept for the exhaustive path
      raw_slots.push_back(q.slots[c]);
      raw_offs.push_back(static_cast<uint32_t>(raw_ids.size()));
      raw_ids.insert(raw_ids.end(), q.ids + q.id_offsets[c], q.ids + q.id_offsets[c + 1]);
    }
    QParam p{};
    p.flags = QF_ACTIVE;
    // a shard clamps k to the rows of the whole index (the merged list holds
    // min(k, all rows)); a shard with fewer rows returns all it has
    const uint64_t rows_all = shard ? shard->total_rows : ix->n_rows;
    p.k = static_cast<uint32_t>(std::min<uint64_t>(q.k, rows_all));
    true_k[i] = p.k;
    if (q.embedding && p.k > kSelectMaxK) {  // the threshold pipeline runs with k clamped; exhaustive() replaces it
      big_k.push_back(i);
      p.k = kSelectMaxK;
    }
    max_k = std::max(max_k, p.k);
    p.quant_k = q.quant_k != 0 ? q.quant_k : 200u * q.k;
    if (q.embedding) {
      p.flags |= QF_EMB;
      any_emb = true;
      unit_embedding(q.embedding, ix->dim, qvec.data() + size_t{i} * dp);
      if (q.quant_enabled) {
        p.flags |= QF_QUANT;
        any_quant = true;
        encode(ix->codec, qvec.data() + size_t{i} * dp, qsig.data() + size_t{i} * nw);
      }
    } else {
      any_term_only = true;
    }
    if (q.n_clauses == 0) {
      p.flags |= QF_MATCH_ALL;
    } else {
      p.prog_off = static_cast<uint32_t>(prog.size());
      prog.push_back(q.n_clauses);
      bool empty = false;
      for (uint32_t c = 0; c < q.n_clauses && !empty; ++c) {
        const uint64_t slot = q.slots[c];
        const size_t len_at = prog.size();
        prog.push_back(0);
        uint32_t scratch_for_clause = UINT32_MAX;
        cl_slot.push_back(static_cast<uint32_t>(slot));
        cl_t.push_back(static_cast<uint32_t>(t_ids.size()));
        for (uint32_t j = q.id_offsets[c]; j < q.id_offsets[c + 1]; ++j) {
          const Term* tp = ix->terms.find((slot << 32) | q.ids[j]);
          if (!tp) continue;  // id absent from the index: matches no row
          const Term& t = *tp;
          if (use_fwd) {
            t_ids.push_back(t.id);
            prog.push_back(0);  // placeholder: the bitmap program is not used
            continue;
          }
          if (t.bitmap != UINT32_MAX) {
            auto r = bitmap_ref.find(t.bitmap);
            uint32_t ref;
            if (r == bitmap_ref.end()) {
              ref = static_cast<uint32_t>(ref_src.size());
              ref_src.push_back({0u, t.bitmap});
              bitmap_ref.emplace(t.bitmap, ref);
            } else {
              ref = r->second;
            }
            prog.push_back(ref);
          } else {
            if (scratch_for_clause == UINT32_MAX) {
              scratch_for_clause = n_scratch++;
              const uint32_t ref = static_cast<uint32_t>(ref_src.size());
              ref_src.push_back({1u, scratch_for_clause});
              prog.push_back(ref);
            }
            item_prefix.push_back(items.empty() ? 0 : item_prefix.back() + items.back().count);
            items.push_back({t.begin, t.df, scratch_for_clause});
          }
        }
        prog[len_at] = static_cast<uint32_t>(prog.size() - len_at - 1);
        if (prog[len_at] == 0) empty = true;
      }
      if (empty) p.flags |= QF_EMPTY;
    }
    qp[i] = p;
    hit_off[i] = total_hits;
    total_hits += true_k[i];
  }
  raw_cl[b] = static_cast<uint32_t>(raw_slots.size());
  if (g_prep.on) g_prep.t[0] += us_since(tp);
  q_cl[b] = static_cast<uint32_t>(cl_slot.size());
  cl_t.push_back(static_cast<uint32_t>(t_ids.size()));
  scatter_total = items.empty() ? 0 : item_prefix.back() + items.back().count;
  n_scratch_used = n_scratch;
  ensure_scratch(n_scratch);
  ensure_hits(total_hits);
  n_hits_total = total_hits;
  refs.resize(ref_src.size());
  for (size_t r = 0; r < ref_src.size(); ++r)
    refs[r] = ref_src[r].first == 0 ? ix->bitmaps + size_t{ref_src[r].second} * W
                                    : d_scratch + size_t{ref_src[r].second} * W;
  use_tc = any_emb && ix->has_tc && b >= kTcMinBatch;
  // prefilter + exact rescoring: K3 batches (int8 or bf16 prefilter), and K2
  // batches when the int8 plane exists (the int8 rows are a quarter of fp32)
  const bool i8_ok = ix->tc_i8 != nullptr && ix->dp % 128 == 0 && prefilter_i8_allowed();
  // (a weighted index keeps the prefilter on K3 batches: the weighted
  // admission and w x clamp(exact dot) rescoring live on that path)
  prefilter = any_emb && (prefilter_enabled() || (use_tc && ix->row_w)) && (use_tc || (i8_ok && k2_i8_enabled()));
  pf_i8 = prefilter && i8_ok;
  // K7: a small index answered in one scoring launch + K4 (no sample, no
  // thresholds): embedding queries only, dense-bitmap terms (no CSR scatter),
  // k <= kSmallMaxK, quant unable to cut (n <= quant_k), every segment's top k
  // fitting the candidate buffer
  use_small = false;
  if (!use_tc && any_emb && !any_term_only && !use_fwd && scatter_total == 0 && big_k.empty() && small_enabled() &&
      ix->n_rows <= kSmallMaxRows && max_k <= kSmallMaxK && ix->num_clauses <= kSmallClauses &&
      uint64_t{(ix->n_rows + kSegRows - 1) / kSegRows} * max_k <= cap &&
      small_supported(ix->dp * (ix->emb_dtype == HYRE_EMB_BF16 ? 2 : 4) / 16)) {
    use_small = true;
    for (uint32_t i = 0; i < b; ++i) {
      if ((qp[i].flags & QF_QUANT) && qp[i].quant_k < ix->n_rows) use_small = false;
      if ((qp[i].flags & QF_ACTIVE) && !(qp[i].flags & (QF_MATCH_ALL | QF_EMPTY))) {
        size_t pos = qp[i].prog_off + 1;  // program: n_clauses, {n_refs, ref...}*
        for (uint32_t c = 0; c < prog[qp[i].prog_off]; ++c) pos += 1 + prog[pos];
        if (pos - qp[i].prog_off > kSmallProg) use_small = false;  // K7 stages at most kSmallProg words
      }
    }
  }
  if (use_small) prefilter = pf_i8 = false;  // exact scores straight from the rows
  // a K2 batch whose embedding queries are all match-all needs no K1 mask:
  // K2 uses tail masks and n_elig starts at the shard's row count
  k2_match_all = !use_tc && !use_small && any_emb && !any_term_only && !any_quant && scatter_total == 0;
  for (uint32_t i = 0; i < b && k2_match_all; ++i)
    if ((qp[i].flags & QF_ACTIVE) && !(qp[i].flags & QF_MATCH_ALL)) k2_match_all = false;
  if (use_tc) {
    // one group of up to 256 queries per pass (the epilogue works in 32-column
    // chunks); a group must leave room for a >= 3-stage ring next to its
    // query tile, else groups of 128
    tc_np = std::min<uint32_t>(kTcMaxGroup, (b + 31) / 32 * 32);
    if (tc_np > 128 && tc_smem_bytes(tc_np, tc_kb(), tc_load_ops(), 3, 0, tc_q_planes(), 1) > 200 * 1024)
      tc_np = 128;
    static const uint32_t group_cap = [] {  // profiling: HYRE_TC_GROUP caps the query group (32..256)
      const char* e = std::getenv("HYRE_TC_GROUP");
      return e ? std::max(32u, std::min(kTcMaxGroup, static_cast<uint32_t>(std::atoi(e)) / 32 * 32)) : kTcMaxGroup;
    }();
    tc_np = std::min(tc_np, group_cap);
    tc_groups = (b + tc_np - 1) / tc_np;
  }
  // Fused CNF: an all-hybrid, quant-free tensor-core batch evaluates the
  // clauses in K3's epilogue from the forward term lists, when the group's
  // term tables fit next to a >= 3-stage ring.
  // A tensor-core batch whose queries are all match-all (no clauses) needs
  // no eligibility pass at all: K3 treats every row as eligible.
  all_match = use_tc && !any_quant && !any_term_only;
  for (uint32_t i = 0; i < b && all_match; ++i)
    if ((qp[i].flags & QF_ACTIVE) && !(qp[i].flags & QF_MATCH_ALL)) all_match = false;
  use_fused = false;
  if (!all_match && use_fwd && use_tc && !any_quant && !any_term_only && fused_enabled() && mask_path() == 0 &&
      ix->num_clauses <= 31 && ix->cnf_ids) {
    const size_t kb = tc_kb();
    use_fused = tc_smem_bytes(tc_np, kb, tc_load_ops(), 3, tc_fz_bytes(2), tc_q_planes()) <= 227 * 1024 - kTcStaticSmem;
  }
  if (use_tc) plan_tc();
  if (use_fused) {
    build_fused_program();
  } else if (all_match) {
    // no program
  } else if (use_fwd && mask_path() != 2) {
    // Cost model (measured on B200, c3): the term-major bitmap kernel costs
    // ~1.3 us per (32-query group x distinct ref) per 10M rows, the forward
    // kernel ~0.5 ms per pass of 64/128 queries per 10M rows.
    std::vector<std::unordered_map<uint32_t, bool>> distinct((b + 31) / 32);
    for (uint32_t i = 0; i < b; ++i)
      for (uint32_t k = q_cl[i]; k < q_cl[i + 1]; ++k)
        for (uint32_t x = cl_t[k]; x < cl_t[k + 1]; ++x) distinct[i / 32][t_ids[x]] = true;
    uint64_t ref_groups = 0;
    for (const auto& d : distinct) ref_groups += d.size();
    const uint64_t passes = (b + 127) / 128;
    if (ref_groups * 13 < passes * 5000) {
      // bitmap path is cheaper: rebuild the program with bitmap/CSR refs
      fwd_veto = true;
      return prepare(qs, b);
    }
  }
  if (!use_fused && !all_match) {
    if (use_fwd) build_forward_program(); else build_term_major_program();
  }
  if (g_prep.on) g_prep.t[1] += us_since(tp);
  // sampling period: sampled survivors ~ k * period must fit the candidate buffer
  uint32_t period = 1;
  while (period < 256 && uint64_t{period} * 2 * max_k * 4 <= cap) period *= 2;
  // the dense sample buffer holds kSampleRows rows per query
  const uint32_t n_seg = (ix->n_rows + kSegRows - 1) / kSegRows;
  period = std::max(period, (n_seg + kSampleRows / kSegRows - 1) / (kSampleRows / kSegRows));
  if (const char* e = std::getenv("HYRE_SAMPLE_PERIOD"))  // profiling: a sparser sample
    period = std::max(period, static_cast<uint32_t>(std::atoi(e)));
  if (use_tc) {
    // K3: the sample pass feeds per-query score histograms (no dense buffer),
    // so it can afford ~kTcSampleSegs segments; a denser sample tightens the
    // estimated threshold (~8 x period admitted rows per query)
    // kTcSampleSegs at c3's 10M rows, growing with the square root of the
    // index (fewer candidates per query balance more histogram increments:
    // measured optimum 60 segments at 10M rows, ~150 at 50M), at most 1/64 of
    // the index
    const double grow = std::sqrt(static_cast<double>(n_seg) / 9766.0);
    uint32_t segs = static_cast<uint32_t>(std::min(240.0, kTcSampleSegs * std::max(grow, 0.1)));
    segs = std::max<uint32_t>(8, std::min<uint32_t>(segs, n_seg / 64));
    if (const char* e = std::getenv("HYRE_TC_SAMPLE_SEGS")) segs = std::max(1, std::atoi(e));
    period = std::max<uint32_t>(1, (n_seg + segs - 1) / segs);
    if (const char* e = std::getenv("HYRE_SAMPLE_PERIOD"))
      period = std::max(period, static_cast<uint32_t>(std::atoi(e)));
  } else if (!(any_emb && ix->has_tc && b >= kTcMinBatch)) {
    // CUDA-core path (K2): its warps absorb a few thousand appends per query,
    // so a smaller sample (~16 segments, ~max(16K, 32k) rows) suffices and the
    // K-th selection over it is cheap.
    const uint32_t want_seg = std::max<uint32_t>(16, (32 * max_k + kSegRows - 1) / kSegRows);
    period = std::max(period, n_seg / want_seg);
  }
  sample_period = period;
  const uint32_t n_samp_seg = (n_seg + period - 1) / period;
  sample_rows = (n_samp_seg - 1) * kSegRows +
                std::min<uint32_t>(kSegRows, ix->n_rows - (n_samp_seg - 1) * period * kSegRows);

  if (g_prep.on) g_prep.t[2] += us_since(tp);
  // tensor-core path: bf16 (hi, lo) split of the unit queries, padded to
  // groups of tc_np rows (multiple of 16, <= kTcMaxGroup).
  qdelta_h.assign(b, prefilter ? prefilter_delta() : 0.0f);
  qscale_h.assign(b, 0.0f);
  if (pf_i8) {
    // int8 prefilter: q8 = rint(q / s_q), s_q = max|q| / 127 per query; the
    // bound: |s - s'| <= r_e |q| + (|e| + r_e) r_q + 1e-5 with
    // r_e the index's largest row residual, r_q = ||q - s_q q8||
    const size_t rows = use_tc ? size_t{tc_groups} * tc_np : size_t{b};
    qi8_h.assign(rows * dp, 0);
    const double re = ix->i8_rmax, en = std::max(1.0f, ix->max_row_norm) * 1.004;
    for (uint32_t i = 0; i < b; ++i) {
      const float* q = qvec.data() + size_t{i} * dp;
      float amax = 0.0f;
      double qn = 0.0;
      for (uint32_t e = 0; e < dp; ++e) {
        amax = std::max(amax, std::fabs(q[e]));
        qn += static_cast<double>(q[e]) * q[e];
      }
      const float sq = amax > 0.0f ? amax / 127.0f : 1.0f, inv = amax > 0.0f ? 127.0f / amax : 0.0f;
      double rq = 0.0;
      // any rounding is valid (r_q is measured on the values used); round
      // half away from zero with a plain conversion (std::nearbyint is slow)
      int8_t* q8 = qi8_h.data() + size_t{i} * dp;
      for (uint32_t e = 0; e < dp; ++e) {
        const float x = q[e] * inv;
        const int v = static_cast<int>(x + (x >= 0.0f ? 0.5f : -0.5f));
        q8[e] = static_cast<int8_t>(v > 127 ? 127 : (v < -127 ? -127 : v));
      }
      for (uint32_t e = 0; e < dp; ++e) {
        const double d = static_cast<double>(q[e]) - static_cast<double>(sq) * q8[e];
        rq += d * d;
      }
      qscale_h[i] = ix->i8_scale * sq;
      qdelta_h[i] = static_cast<float>(re * std::sqrt(qn) * (1.0 + 1e-6) + (en + re) * std::sqrt(rq) + 1e-5);
    }
  } else if (use_tc) {
    const size_t rows = size_t{tc_groups} * tc_np;
    qhi_h.assign(rows * dp, 0);
    if (prefilter) qlo_h.clear(); else qlo_h.assign(rows * dp, 0);
    for (uint32_t i = 0; i < b; ++i)
      for (uint32_t e = 0; e < dp; ++e) {
        const float x = qvec[size_t{i} * dp + e];
        const uint16_t h = bf16_rne(x);
        qhi_h[size_t{i} * dp + e] = h;
        if (!prefilter) qlo_h[size_t{i} * dp + e] = bf16_rne(x - bf16_to_f(h));  // the prefilter reads Q_hi only
      }
  }

  if (g_prep.on) g_prep.t[3] += us_since(tp);
  // ---- pack and upload ----------------------------------------------------
  size_t off = 0;
  auto place = [&](size_t bytes) {
    off = align_up(off, 256);
    const size_t at = off;
    off += bytes;
    return at;
  };
  const size_t o_qp = place(b * sizeof(QParam));
  const size_t o_q = place(qvec.size() * 4);
  const size_t o_qsig = place(qsig.size() * 8);
  const size_t o_off = place(b * 8);
  const size_t o_prog = place(std::max<size_t>(prog.size(), 1) * 4);
  const size_t o_refs = place(std::max<size_t>(refs.size(), 1) * sizeof(void*));
  const size_t o_items = place(std::max<size_t>(items.size(), 1) * sizeof(ScatterItem));
  const size_t o_ipre = place(std::max<size_t>(item_prefix.size(), 1) * 8);
  const size_t o_fwd = place(std::max<size_t>(fwd_words.size(), 1) * 4);
  const size_t o_qhi = place(std::max<size_t>(pf_i8 ? (qi8_h.size() + 1) / 2 : qhi_h.size(), 1) * 2);
  const size_t o_qlo = place(std::max<size_t>(qlo_h.size(), 1) * 2);
  const size_t o_qsc = place(b * 4);
  const size_t o_qdl = place(b * 4);
  const size_t o_fz = place(std::max<size_t>(fz_words.size(), 1) * 4);
  o_cinit = place(size_t{max_batch} * kNumCounters * 4);
  ensure_blob(off);
  {  // counter image of a k2_match_all run: n_elig = rows for the active queries, the rest 0
    uint32_t* ci = reinterpret_cast<uint32_t*>(h_blob + o_cinit);
    std::memset(ci, 0, size_t{max_batch} * kNumCounters * 4);
    for (uint32_t i = 0; i < b; ++i)
      if ((qp[i].flags & (QF_ACTIVE | QF_MATCH_ALL)) == (QF_ACTIVE | QF_MATCH_ALL)) ci[i] = ix->n_rows;
  }
  std::memcpy(h_blob + o_qp, qp.data(), b * sizeof(QParam));
  std::memcpy(h_blob + o_q, qvec.data(), qvec.size() * 4);
  std::memcpy(h_blob + o_qsig, qsig.data(), qsig.size() * 8);
  std::memcpy(h_blob + o_off, hit_off.data(), b * 8);
  if (!prog.empty()) std::memcpy(h_blob + o_prog, prog.data(), prog.size() * 4);
  if (!refs.empty()) std::memcpy(h_blob + o_refs, refs.data(), refs.size() * sizeof(void*));
  if (!items.empty()) {
    std::memcpy(h_blob + o_items, items.data(), items.size() * sizeof(ScatterItem));
    std::memcpy(h_blob + o_ipre, item_prefix.data(), item_prefix.size() * 8);
  }
  if (!fwd_words.empty()) std::memcpy(h_blob + o_fwd, fwd_words.data(), fwd_words.size() * 4);
  if (use_fused) std::memcpy(h_blob + o_fz, fz_words.data(), fz_words.size() * 4);
  if (pf_i8) {
    std::memcpy(h_blob + o_qhi, qi8_h.data(), qi8_h.size());  // int8 queries (K3 tiles or K2 rows)
  } else if (use_tc) {
    std::memcpy(h_blob + o_qhi, qhi_h.data(), qhi_h.size() * 2);
    if (!qlo_h.empty()) std::memcpy(h_blob + o_qlo, qlo_h.data(), qlo_h.size() * 2);
  }
  if (g_prep.on) g_prep.t[4] += us_since(tp);
  std::memcpy(h_blob + o_qsc, qscale_h.data(), b * 4);
  std::memcpy(h_blob + o_qdl, qdelta_h.data(), b * 4);
  HYRE_CUDA(cudaMemcpyAsync(d_blob, h_blob, off, cudaMemcpyHostToDevice, st));
  if (use_tc) {
    if (pf_i8) make_i8_map(&tm_qhi, d_blob + o_qhi, size_t{tc_groups} * tc_np, dp, tc_np);
    else make_bf16_map(&tm_qhi, d_blob + o_qhi, size_t{tc_groups} * tc_np, dp, tc_np);
    make_bf16_map(&tm_qlo, d_blob + (prefilter ? o_qhi : o_qlo), size_t{tc_groups} * tc_np, dp, tc_np);
  }
  h2d_bytes = off;
  // eligibility input bytes: distinct bitmaps W*4 each, CSR
  // postings 4 each; the forward lists N*A*2 once per pass on the fwd/fused paths
  if (use_fused)
    term_bytes = size_t{ix->n_rows} * ix->cnf_row_total() * tc_groups;  // compact CNF rows per group pass
  else if (use_fwd)
    term_bytes = size_t{ix->n_rows} * ix->row_terms_width * 2 * fwd_pass.size();
  else
    term_bytes = uint64_t{ix->words} * 4 * (ref_src.size() - n_scratch) + scatter_total * 4;
  // K3 main stage (all groups): every row's embedding operand planes the pass
  // reads (hi only for the prefilter / a bf16 index; hi + lo otherwise) plus
  // its eligibility input (compact CNF rows when fused, else the group's K1
  // mask words)
  scan_bytes = 0;
  if (use_tc) {
    const uint64_t emb = uint64_t{ix->n_rows} * ix->dp * (pf_i8 ? 1 : 2 * tc_load_ops());
    const uint64_t elig = all_match ? 0
                          : use_fused ? uint64_t{ix->n_rows} * ix->cnf_row_total()
                                      : uint64_t{ix->words} * 4 * tc_np;
    scan_bytes = (emb + elig) * tc_groups;
  }
  d_qp = reinterpret_cast<QParam*>(d_blob + o_qp);
  d_q = reinterpret_cast<float*>(d_blob + o_q);
  d_qsig = reinterpret_cast<uint64_t*>(d_blob + o_qsig);
  d_hit_off = reinterpret_cast<uint64_t*>(d_blob + o_off);
  d_prog = reinterpret_cast<uint32_t*>(d_blob + o_prog);
  d_refs = reinterpret_cast<const uint32_t* const*>(d_blob + o_refs);
  d_items = reinterpret_cast<ScatterItem*>(d_blob + o_items);
  d_ipre = reinterpret_cast<uint64_t*>(d_blob + o_ipre);
  d_fwd = reinterpret_cast<uint32_t*>(d_blob + o_fwd);
  d_fz = reinterpret_cast<uint32_t*>(d_blob + o_fz);
  d_qscale = reinterpret_cast<float*>(d_blob + o_qsc);
  d_qi8 = reinterpret_cast<int8_t*>(d_blob + o_qhi);
  d_qdelta = reinterpret_cast<float*>(d_blob + o_qdl);
  prepared = true;
  if (g_prep.on) {
    g_prep.t[5] += us_since(tp);
    std::array<double, 6> c{};
    for (int i = 0; i < 6; ++i) c[i] = g_prep.t[i];
    g_prep.calls.push_back(c);
    ++g_prep.n;
    std::fill(std::begin(g_prep.t), std::end(g_prep.t), 0.0);
  }
}

// One scorer pass (main / sample / rerun) over every embedding query: K3 on
// the tensor cores for batches above 8 queries, K2 on CUDA cores otherwise.
void Executor::score(uint32_t mode, uint64_t* cand, uint32_t* cnt, uint32_t capacity) {
  uint32_t* n_elig = d_counters;
  uint32_t* rerun = d_counters + 4 * max_batch;
  if (use_tc) {
    const uint32_t n_tiles = (ix->n_rows + 127) / 128;
    const uint32_t kb = tc_kb();
    const uint32_t n_ops = tc_load_ops();
    const uint32_t stages = tc_stages;
    const size_t fzb = use_fused ? tc_fz_bytes(tc_term_slots) : 0;
    const uint32_t cols = tc_tmem_cols(tc_np);
    uint32_t work = n_tiles;
    if (mode == SCORE_SAMPLE) {
      const uint32_t n_seg = (ix->n_rows + kSegRows - 1) / kSegRows;
      work = (n_seg + sample_period - 1) / sample_period * 8;
    }
    uint32_t grid = std::max(1u, std::min(work, 148u * tc_ctas_per_sm(use_fused, tc_np)));
    if (mode == SCORE_SAMPLE) {  // profiling: HYRE_TC_SAMPLE_GRID caps the sample pass's CTAs
      static const uint32_t sg = [] {
        const char* e = std::getenv("HYRE_TC_SAMPLE_GRID");
        return e ? static_cast<uint32_t>(std::atoi(e)) : 0u;
      }();
      if (sg) grid = std::min(grid, sg);
    }
    for (uint32_t g = 0; g < tc_groups; ++g) {
      TcArgs ta{pf_i8 ? ix->tc_i8 : ix->tc_tiles, ix->n_rows, ix->row_base, ix->words, n_tiles, B, g * tc_np, g * tc_np, tc_np, kb, stages, cols,
                n_ops == 2 ? 1u : 0u, d_mask, d_qp, n_elig, d_thr, cand, cnt, capacity, mode, sample_period, cap,
                rerun, d_samp};
      ta.debug = tc_debug_flags();
      ta.prefilter = prefilter ? 1u : 0u;
      ta.plane_bytes = ix->tc_plane_bytes;
      ta.delta = prefilter_delta();
      ta.i8 = pf_i8 ? 1u : 0u;
      ta.qscale = d_qscale;
      ta.qdelta = prefilter ? d_qdelta : nullptr;
      ta.term_slots = tc_term_slots;
      ta.shist = mode == SCORE_SAMPLE ? d_shist : nullptr;
      ta.hbins = kHistBins;
      ta.aps = tc_aps;
      ta.acc_bufs = tc_acc_bufs(tc_np);
      ta.match_all = all_match ? 1u : 0u;
      ta.sample_floor = (all_match && mode == SCORE_SAMPLE && !ix->row_w) ? 1u : 0u;
      ta.backoff_ns = tc_backoff_ns();
      ta.row_w = ix->row_w;
      if (use_fused) {
        const FusedGroup& fg = fz_group[g];
        ta.fused = 1;
        ta.cnf_ids = ix->cnf_ids;
        ta.cnf_masks = ix->cnf_masks;
        ta.slot_of = ix->slot_of;
        ta.J = ix->cnf_ids_per_row;
        ta.tb = ix->cnf_id_bytes;
        ta.wb = ix->cnf_row_bytes;
        ta.W = ix->cnf_group;
        ta.T = ix->n_terms_fwd;
        ta.C = ix->num_clauses;
        ta.fz = d_fz + fg.entries;
        ta.n_entries = fg.n_entries;
        ta.hc_off = fg.hc - fg.entries;
        ta.live_off = ta.hc_off + ix->num_clauses * tc_fused_chunks(tc_np);
      }
      launch_tc_score(tm_qhi, tm_qlo, ta, grid, tc_smem_bytes(tc_np, kb, n_ops, stages, fzb, tc_q_planes(), tc_aps),
                      st);
      ++kernels;
    }
    return;
  }
  const bool bf16 = ix->emb_dtype == HYRE_EMB_BF16;
  const void* emb = bf16 ? static_cast<const void*>(ix->emb_hi) : static_cast<const void*>(ix->emb_f32);
  const uint32_t dp_chunks = ix->dp * (bf16 ? 2 : 4) / 16;
  ScoreArgs sa{emb, ix->dp, dp_chunks, ix->n_rows, ix->row_base, ix->words, d_mask, d_qp, d_q, B, n_elig,
               d_thr, cand, cnt, capacity, mode, sample_period, cap, rerun, d_samp, 1, 1};
  sa.row_w = ix->row_w;
  sa.match_all = k2_match_all ? 1u : 0u;
  if (mode == SCORE_SAMPLE && k2_hist_sample()) {
    sa.shist = d_shist;
    sa.hbins = kHistBins;
  }
  if (pf_i8) {  // int8 prefilter rows (exact rescoring in K4p)
    sa.emb = ix->tc_i8;
    sa.qi8 = d_qi8;
    sa.qscale = d_qscale;
    sa.qdelta = d_qdelta;
  }
  // enough work items to fill the resident warp slots (148 SMs x 64 warps)
  const uint32_t n_seg = (ix->n_rows + kSegRows - 1) / kSegRows;
  const uint32_t n_samp_seg = (n_seg + sample_period - 1) / sample_period;
  while (sa.split < 32 && n_seg * sa.split < 148u * 64u) sa.split *= 2;
  while (sa.split_sample < 32 && n_samp_seg * sa.split_sample < 148u * 64u) sa.split_sample *= 2;
  if (pf_i8) launch_score_i8(sa, st);
  else launch_score(sa, bf16, st);
  ++kernels;
}

// K3 shared-memory plan: the K-atom ring depth and (fused CNF) the depth of
// the row-term ring.  The producer issues a tile's embedding stages only after
// its term block, so the bytes in flight per SM are bounded by
// min(term slots, stages / kb) tiles; the plan maximises that (Little's law:
// ~150 KB in flight per SM sustain HBM rate at ~3 us loaded latency), then
// prefers more stages.
void Executor::plan_tc() {
  const uint32_t kb = tc_kb();
  // Stage = aps K-atoms: the largest divisor of kb that still leaves a
  // >= 3-stage ring, so each tile costs few MMA commits / barrier round trips
  // (tcgen05.commit per stage was measured to pace the MMA issuer).
  auto plan = [&](uint32_t aps, uint32_t slots) {
    const size_t stage_bytes = size_t{tc_load_ops()} * aps * 128 * 128;
    const size_t fixed = tc_smem_bytes(tc_np, kb, tc_load_ops(), 0, use_fused ? tc_fz_bytes(slots) : 0, tc_q_planes(), aps);
    const size_t cap_b = tc_smem_cap(use_fused, tc_np);
    const size_t budget = cap_b > fixed ? cap_b - fixed : 0;
    return static_cast<uint32_t>(std::min<size_t>(12, budget / stage_bytes));
  };
  uint32_t aps_max = kb;
  if (const char* e = std::getenv("HYRE_TC_APS"))  // profiling: cap atoms per stage
    aps_max = std::max(1u, std::min<uint32_t>(kb, static_cast<uint32_t>(std::atoi(e))));
  tc_aps = 1;
  for (uint32_t aps = aps_max; aps >= 1; --aps)
    if (kb % aps == 0 && plan(aps, 2) >= 3) {
      tc_aps = aps;
      break;
    }
  const uint32_t spt = kb / tc_aps;  // stages per tile
  // The producer issues a tile's stages only after its term block, so the
  // tiles in flight are min(term slots, stages / spt): maximise that, then
  // prefer more stages.
  tc_term_slots = 2;
  tc_stages = plan(tc_aps, 2);
  if (use_fused) {
    uint32_t best = std::min(2u, tc_stages / spt);
    for (uint32_t slots = 3; slots <= kMaxTermSlots; ++slots) {
      const uint32_t st_n = plan(tc_aps, slots);
      const uint32_t depth = std::min(slots, st_n / spt);
      if (st_n >= 2 && depth > best) {
        best = depth;
        tc_term_slots = slots;
        tc_stages = st_n;
      }
    }
  }
  if (const char* e = std::getenv("HYRE_TC_TERM_SLOTS")) {  // profiling: fix the term ring depth
    tc_term_slots = std::max(1u, std::min<uint32_t>(kMaxTermSlots, static_cast<uint32_t>(std::atoi(e))));
    tc_stages = plan(tc_aps, tc_term_slots);
  }
  tc_stages = std::max(2u, tc_stages);
  if (const char* e = std::getenv("HYRE_TC_STAGES"))  // profiling: cap the ring depth
    tc_stages = std::max(2u, std::min<uint32_t>(tc_stages, static_cast<uint32_t>(std::atoi(e))));
}

size_t Executor::tc_fz_bytes(uint32_t slots) const {
  return tc_fused_bytes(tc_np, ix->n_terms_fwd, ix->num_clauses, static_cast<uint32_t>(ix->cnf_row_total()), slots);
}

// Final K4 after a main / rerun pass: the prefilter variant (prune, exact
// rescoring, threshold check, sort) for K3 prefilter candidates, else the
// exact select_kernel.
void Executor::final_select(SelectArgs fa) {
  if (!prefilter) {
    launch_select(fa, st);
    ++kernels;
    return;
  }
  const bool bf16 = ix->emb_dtype == HYRE_EMB_BF16;
  fa.delta = prefilter_delta();
  fa.qdelta = d_qdelta;
  PrefSelectArgs pa{fa, bf16 ? static_cast<const void*>(ix->emb_hi) : static_cast<const void*>(ix->emb_f32), ix->dp,
                    ix->dp * (bf16 ? 2 : 4) / 16, ix->row_base, d_q, ix->row_w};
  launch_select_prefilter(pa, bf16, st);
  ++kernels;
}

// Term-major form of the batch program for mask_tm_kernel: per group of 32
// queries, the slots they constrain and, per slot, each distinct ref with the
// 32-bit mask of queries whose clause contains it.
void Executor::build_term_major_program() {
  const uint32_t groups = (B + 31) / 32;
  prog_groups.assign(groups, std::vector<uint32_t>());
  prog_live.assign(groups, 0u);
  for (uint32_t g = 0; g < groups; ++g) {
    uint32_t live = 0;
    std::map<uint32_t, std::pair<uint32_t, std::map<uint32_t, uint32_t>>> slots;  // slot -> (hc, ref -> users)
    for (uint32_t j = 0; j < 32 && g * 32 + j < B; ++j) {
      const uint32_t i = g * 32 + j;
      const QParam& p = qp[i];
      if (!(p.flags & QF_ACTIVE) || (p.flags & QF_EMPTY)) continue;
      live |= 1u << j;
      if (p.flags & QF_MATCH_ALL) continue;
      uint32_t pos = p.prog_off;
      const uint32_t nc = prog[pos++];
      for (uint32_t c = 0; c < nc; ++c) {
        const uint32_t nr = prog[pos++];
        auto& e = slots[cl_slot[q_cl[i] + c]];
        e.first |= 1u << j;
        for (uint32_t r = 0; r < nr; ++r) e.second[prog[pos + r]] |= 1u << j;
        pos += nr;
      }
    }
    prog_live[g] = live;
    auto& w = prog_groups[g];
    w.push_back(static_cast<uint32_t>(slots.size()));
    for (auto& [slot, e] : slots) {
      w.push_back(e.first);
      w.push_back(static_cast<uint32_t>(e.second.size()));
      for (auto& [ref, users] : e.second) {
        const uint64_t ptr = reinterpret_cast<uint64_t>(refs[ref]);
        w.push_back(static_cast<uint32_t>(ptr));
        w.push_back(static_cast<uint32_t>(ptr >> 32));
        w.push_back(users);
      }
    }
  }
}

// K1b program: per pass of 64 * nw queries, the sparse users table (term id
// -> 64-bit query masks), the per-slot constrained-query masks and the live
// mask, all in one u32 array (fwd_words); fwd_pass holds each pass's offsets.
void Executor::build_forward_program() {
  fwd_words.clear();
  fwd_pass.clear();
  const uint32_t nwp = B > 64 ? 2 : 1, per = 64 * nwp, C = ix->num_clauses;
  for (uint32_t q0 = 0; q0 < B; q0 += per) {
    std::map<uint32_t, std::vector<uint64_t>> users;
    std::vector<uint64_t> hc(size_t{C} * nwp, 0ull), live(nwp, 0ull);
    for (uint32_t i = q0; i < std::min(B, q0 + per); ++i) {
      const QParam& p = qp[i];
      if (!(p.flags & QF_ACTIVE) || (p.flags & QF_EMPTY)) continue;
      const uint32_t w = (i - q0) >> 6;
      const uint64_t bit = 1ull << ((i - q0) & 63);
      live[w] |= bit;
      for (uint32_t k = q_cl[i]; k < q_cl[i + 1]; ++k) {
        hc[size_t{cl_slot[k]} * nwp + w] |= bit;
        for (uint32_t x = cl_t[k]; x < cl_t[k + 1]; ++x) {
          const uint32_t t = t_ids[x];
          auto& u = users[t];
          if (u.empty()) u.assign(nwp, 0ull);
          u[w] |= bit;
        }
      }
    }
    FwdPass fp{};
    fp.q0 = q0;
    fp.nw = nwp;
    fp.n_entries = static_cast<uint32_t>(users.size());
    fp.entries = static_cast<uint32_t>(fwd_words.size());
    for (auto& [t, u] : users) {
      fwd_words.push_back(t);
      for (uint32_t w = 0; w < nwp; ++w) {
        fwd_words.push_back(static_cast<uint32_t>(u[w]));
        fwd_words.push_back(static_cast<uint32_t>(u[w] >> 32));
      }
    }
    while (fwd_words.size() % 2) fwd_words.push_back(0);  // 8-byte align the masks
    fp.hc = static_cast<uint32_t>(fwd_words.size());
    for (uint64_t v : hc) {
      fwd_words.push_back(static_cast<uint32_t>(v));
      fwd_words.push_back(static_cast<uint32_t>(v >> 32));
    }
    fp.live = static_cast<uint32_t>(fwd_words.size());
    for (uint64_t v : live) {
      fwd_words.push_back(static_cast<uint32_t>(v));
      fwd_words.push_back(static_cast<uint32_t>(v >> 32));
    }
    fwd_pass.push_back(fp);
  }
}

// Fused-CNF program per K3 query group (TcArgs::fz): for every term any
// query of the group lists, v = hc(slot) & ~users (the queries constraining
// the term's slot that do not list it); per slot, the queries that
// constrain it; the live (active, satisfiable) queries; the constrained-slot
// mask.  Word w holds query chunk w (queries 32w .. 32w + 31).
void Executor::build_fused_program() {
  fz_words.clear();
  fz_group.clear();
  const uint32_t C = ix->num_clauses, fw = tc_fused_chunks(tc_np), T = ix->n_terms_fwd;
  // dense per-term users scratch (T <= kForwardMaxTerms), reset via the touched list
  if (fz_users.size() < size_t{T} * fw) fz_users.assign(size_t{T} * fw, 0u);
  if (fz_slot.size() < T) fz_slot.assign(T, 0u);
  for (uint32_t g = 0; g < tc_groups; ++g) {
    fz_touched.clear();
    std::vector<uint32_t> hc(size_t{C} * fw, 0u), live(fw, 0u);
    uint32_t cslots = 0;
    for (uint32_t i = g * tc_np; i < std::min(B, (g + 1) * tc_np); ++i) {
      const QParam& p = qp[i];
      if (!(p.flags & QF_ACTIVE) || (p.flags & QF_EMPTY)) continue;
      const uint32_t j = i - g * tc_np, w = j / 32, bit = 1u << (j & 31);
      live[w] |= bit;
      for (uint32_t k = q_cl[i]; k < q_cl[i + 1]; ++k) {
        hc[size_t{cl_slot[k]} * fw + w] |= bit;
        cslots |= 1u << cl_slot[k];
        for (uint32_t x = cl_t[k]; x < cl_t[k + 1]; ++x) {
          uint32_t* u = fz_users.data() + size_t{t_ids[x]} * fw;
          bool fresh = true;
          for (uint32_t v = 0; v < fw; ++v) fresh &= u[v] == 0u;
          if (fresh) {
            fz_touched.push_back(t_ids[x]);
            fz_slot[t_ids[x]] = cl_slot[k];
          }
          u[w] |= bit;
        }
      }
    }
    FusedGroup fg{};
    fg.entries = static_cast<uint32_t>(fz_words.size());
    fg.n_entries = static_cast<uint32_t>(fz_touched.size());
    for (uint32_t t : fz_touched) {  // v(t) = hc(slot(t)) & ~users(t)
      uint32_t* u = fz_users.data() + size_t{t} * fw;
      const uint32_t* h = hc.data() + size_t{fz_slot[t]} * fw;
      fz_words.push_back(t);
      for (uint32_t v = 0; v < fw; ++v) fz_words.push_back(h[v] & ~u[v]);
      std::fill(u, u + fw, 0u);
    }
    fg.hc = static_cast<uint32_t>(fz_words.size());
    fz_words.insert(fz_words.end(), hc.begin(), hc.end());
    fz_words.insert(fz_words.end(), live.begin(), live.end());
    fz_words.push_back(cslots);
    fz_group.push_back(fg);
  }
}

// ---------------------------------------------------------------------------
// run: the fixed kernel sequence, no host synchronisation.
// ---------------------------------------------------------------------------
void Executor::run() {
  if (!prepared) throw Error(HYRE_INTERNAL, "hyre_batch_run before hyre_batch_prepare");
  HYRE_CUDA(cudaSetDevice(ix->device));
  kernels = 0;
  finish_rounds = 0;
  exh_done = false;
  exh_count = 0;
  ev = ev_ring[n_runs++ % kEvRing];
  const uint32_t W = ix->words;
  uint32_t* n_elig = d_counters;
  uint32_t* cand_cnt = d_counters + max_batch;
  uint32_t* samp_cnt = d_counters + 2 * max_batch;
  uint32_t* out_cnt = d_counters + 3 * max_batch;
  uint32_t* rerun = d_counters + 4 * max_batch;
  mark(0, true);
  // sampled thresholds through per-query score histograms (K3, and K2 unless
  // HYRE_K2_DENSE_SAMPLE=1 keeps the dense sample + K-th selection)
  const bool hist_sample = any_emb && ix->n_rows > cap && (use_tc || k2_hist_sample());
  if (use_fused || all_match) {
    // One init kernel instead of three memsets: counters zeroed; eligible
    // counts unknown (all-ones: eligibility is evaluated inside K3, or every
    // row is eligible), which K4's rerun logic treats as "at least K"; the
    // sample histograms zeroed.
    launch_run_init(d_counters, max_batch * kNumCounters, B, hist_sample ? d_shist : nullptr,
                    size_t{B} * kHistBins, st);
    ++kernels;
  } else if (k2_match_all) {
    HYRE_CUDA(cudaMemcpyAsync(d_counters, d_blob + o_cinit, sizeof(uint32_t) * max_batch * kNumCounters,
                              cudaMemcpyDeviceToDevice, st));
    if (hist_sample) HYRE_CUDA(cudaMemsetAsync(d_shist, 0, sizeof(uint32_t) * B * kHistBins, st));
  } else {
    HYRE_CUDA(cudaMemsetAsync(d_counters, 0, sizeof(uint32_t) * max_batch * kNumCounters, st));
    if (hist_sample) HYRE_CUDA(cudaMemsetAsync(d_shist, 0, sizeof(uint32_t) * B * kHistBins, st));
  }
  if (use_small) {
    // K7: CNF words + exact scores + per-segment top k in one launch, then K4
    mark(1, false);
    mark(2, false);
    mark(3, false);
    const bool bf16 = ix->emb_dtype == HYRE_EMB_BF16;
    SmallArgs sa{bf16 ? static_cast<const void*>(ix->emb_hi) : static_cast<const void*>(ix->emb_f32), ix->dp,
                 ix->dp * (bf16 ? 2 : 4) / 16, ix->n_rows, ix->row_base, W, d_refs, d_prog,
                 static_cast<uint32_t>(prog.size()), static_cast<uint32_t>(refs.size()), d_qp, B, d_q,
                 ix->row_w, d_cand, cand_cnt, cap, n_elig};
    launch_small(sa, bf16, st);
    ++kernels;
    mark(4, true);
    SelectArgs fa{d_cand, cand_cnt, cap, d_qp, n_elig, SELECT_FINAL, d_thr, rerun, d_hits, d_hit_off,
                  out_cnt, B, QF_ACTIVE | QF_EMB, cap, nullptr, 1, 0};
    final_select(fa);
    mark(5, true);
    HYRE_CUDA(cudaGetLastError());
    return;
  }
  if (use_fused || all_match) {
  } else if (use_fwd) {
    for (const FwdPass& fp : fwd_pass) {
      FwdArgs fa{ix->row_terms, ix->slot_of, ix->row_terms_width, ix->n_rows, W, ix->n_chunks, B, ix->num_clauses,
                 ix->n_terms_fwd, d_fwd + fp.entries, fp.n_entries,
                 reinterpret_cast<const uint64_t*>(d_fwd + fp.hc), reinterpret_cast<const uint64_t*>(d_fwd + fp.live),
                 fp.q0, fp.nw, d_mask, d_chunk_cnt, n_elig};
      launch_fwd_mask(fa, st);
      ++kernels;
    }
  } else if (scatter_total) {
    HYRE_CUDA(cudaMemsetAsync(d_scratch, 0, size_t{n_scratch_used} * W * 4, st));
    launch_scatter(d_items, d_ipre, static_cast<uint32_t>(items.size()), scatter_total, ix->post_rows,
                   d_scratch, W, st);
    ++kernels;
  }
  if (!use_fwd && !use_fused && !all_match && !k2_match_all) {
    MaskArgs ma{d_refs, static_cast<uint32_t>(refs.size()), d_prog, d_qp, B, W, ix->n_chunks, ix->n_rows,
                d_mask, d_chunk_cnt, n_elig};
    const uint32_t ml = launch_mask_tm(ma, prog_groups, prog_live, st);
    if (ml & 0x80000000u) {
      launch_mask(ma, st);  // a single 32-query group's program exceeds the parameter limit
      ++kernels;
    }
    kernels += ml & 0x7fffffffu;
  }
  mark(1, !use_fused && !all_match && !k2_match_all);  // K1/K1b mask pass (the K3 init kernel is attributed to the sample stage)
  if (any_quant) {
    HYRE_CUDA(cudaMemsetAsync(d_qhist, 0, sizeof(uint32_t) * B * (ix->num_bits + 1), st));
    QuantArgs qa{ix->sigs, ix->num_words, ix->num_bits, d_qsig, d_qp, B, W, ix->n_chunks, ix->n_rows,
                 d_mask, d_chunk_cnt, n_elig, d_qhist, d_tsel, d_eqcnt};
    if (!shard || shard->G == 1) {
      launch_quant(qa, st);
      kernels += 5;
    } else {
      // global quant_k over every shard (pipeline.cpp:126-130 on the whole
      // index): sum the histograms, pick the global threshold, keep the ties
      // of the lowest global rows first
      const size_t nh = size_t{B} * (ix->num_bits + 1);
      if (!d_qhist_sum) d_qhist_sum = dmalloc<uint32_t>(size_t{max_batch} * (ix->num_bits + 1));
      qa.shard_mode = 1;
      qa.hist_total = d_qhist_sum;
      launch_quant_hist(qa, st);
      shard_exchange(0);
      PeerPtrs hp{}, tp{};
      for (uint32_t g = 0; g < shard->G; ++g) {
        hp.p[g] = shard->peers[g]->d_qhist;
        tp.p[g] = shard->peers[g]->d_tsel;
      }
      launch_sum_peers(hp, shard->G, nh, d_qhist_sum, st);
      launch_quant_select(qa, st);
      shard_exchange(1);
      launch_quant_offset(tp, shard->g, B, d_tsel, st);
      launch_quant_apply(qa, st);
      kernels += 7;
    }
  }
  mark(2, any_quant);
  if (any_emb) {
    if (hist_sample) {
      // K3 / K2 sample pass into per-query score histograms (zeroed above) -> thresholds
      score(SCORE_SAMPLE, nullptr, samp_cnt, samp_cap);
      HistThrArgs ha{d_shist, kHistBins, d_qp, n_elig, cap, sample_period, B, QF_ACTIVE | QF_EMB, d_thr, d_thr_safe,
                     prefilter ? prefilter_delta() : 0.0f, prefilter ? d_qdelta : nullptr};
      launch_hist_thr(ha, st);
      ++kernels;
    } else if (ix->n_rows > cap) {
      HYRE_CUDA(cudaMemset2DAsync(d_samp, sizeof(uint32_t) * samp_cap, 0, sizeof(uint32_t) * sample_rows, B, st));
      score(SCORE_SAMPLE, nullptr, samp_cnt, samp_cap);
      SelectArgs ka{nullptr, samp_cnt, samp_cap, d_qp, n_elig, SELECT_KTH, d_thr, nullptr, nullptr,
                    nullptr, nullptr, B, QF_ACTIVE | QF_EMB, cap, d_thr_safe, sample_period, sample_rows,
                    d_samp, ix->row_base, d_cand, cap, prefilter ? prefilter_delta() : 0.0f,
                    prefilter ? d_qdelta : nullptr};
      launch_sample_kth(ka, samp_cnt, st);
      ++kernels;
    } else {
      HYRE_CUDA(cudaMemsetAsync(d_thr, 0, sizeof(uint64_t) * B, st));
      HYRE_CUDA(cudaMemsetAsync(d_thr_safe, 0, sizeof(uint64_t) * B, st));
    }
    mark(3, true);
    score(SCORE_MAIN, d_cand, cand_cnt, cap);
    mark(4, true);
    SelectArgs fa{d_cand, cand_cnt, cap, d_qp, n_elig, SELECT_FINAL, d_thr, rerun, d_hits, d_hit_off,
                  out_cnt, B, QF_ACTIVE | QF_EMB, cap, d_thr_safe, sample_period, 0};
    final_select(fa);
    // Recovery (a query whose estimated threshold admitted too few rows, or
    // whose candidate buffer overflowed) is rare: fetch() sees the rerun
    // flags with the results and runs it then, so the common batch costs no
    // speculative kernels.
  } else {
    mark(3, false);
    mark(4, false);
  }
  if (any_term_only) {
    FirstKArgs fk{d_mask, d_chunk_cnt, n_elig, d_qp, B, W, ix->n_chunks, ix->row_base, d_hit_off, d_hits,
                  out_cnt, nullptr, 0, 0};
    launch_first_k(fk, st);
    ++kernels;
  }
  mark(5, true);
  HYRE_CUDA(cudaGetLastError());
}

// Resolve any candidate-buffer overflow left after the speculative round.
void Executor::finish_reruns() {
  uint32_t* n_elig = d_counters;
  uint32_t* cand_cnt = d_counters + max_batch;
  uint32_t* out_cnt = d_counters + 3 * max_batch;
  uint32_t* rerun = d_counters + 4 * max_batch;
  for (int round = 0; round < 64; ++round) {
    HYRE_CUDA(cudaMemcpyAsync(h_rerun.data(), rerun, B * 4, cudaMemcpyDeviceToHost, st));
    HYRE_CUDA(cudaStreamSynchronize(st));
    bool any = false;
    for (uint32_t i = 0; i < B; ++i) any |= h_rerun[i] != 0;
    if (!any) return;
    if (round >= kMaxRecoveryRounds) {
      // not converging (rows tied inside the prefilter band exceed the
      // candidate buffer): exact exhaustive top-K for those queries
      for (uint32_t i = 0; i < B; ++i)
        if (h_rerun[i]) exhaustive(i);
      continue;
    }
    ++finish_rounds;
    if (std::getenv("HYRE_DEBUG_COUNTS") && round < 4) {  // diagnostics: the recovery state of query 0
      uint64_t t[2];
      uint32_t c[2];
      HYRE_CUDA(cudaMemcpy(&t[0], d_thr, 8, cudaMemcpyDeviceToHost));
      HYRE_CUDA(cudaMemcpy(&t[1], d_thr_safe, 8, cudaMemcpyDeviceToHost));
      HYRE_CUDA(cudaMemcpy(&c[0], cand_cnt, 4, cudaMemcpyDeviceToHost));
      HYRE_CUDA(cudaMemcpy(&c[1], n_elig, 4, cudaMemcpyDeviceToHost));
      std::fprintf(stderr, "[hyre] rerun round %d: q0 rerun %u thr %.6f thr_safe %.6f cand %u elig %u\n", round,
                   h_rerun[0], key_score(t[0]), key_score(t[1]), c[0], c[1]);
    }
    HYRE_CUDA(cudaMemsetAsync(cand_cnt, 0, sizeof(uint32_t) * max_batch, st));
    score(SCORE_RERUN, d_cand, cand_cnt, cap);
    SelectArgs fa{d_cand, cand_cnt, cap, d_qp, n_elig, SELECT_FINAL_RERUN, d_thr, rerun, d_hits, d_hit_off,
                  out_cnt, B, QF_ACTIVE | QF_EMB, cap, d_thr_safe, sample_period, 0};
    final_select(fa);
  }
  throw Error(HYRE_INTERNAL, "top-K candidate selection did not converge");
}

void Executor::fetch(hyre_hit* hits, const uint64_t* offsets, uint32_t* counts, int32_t* st_out,
                     hyre_timings* t) {
  if (!prepared) throw Error(HYRE_INTERNAL, "hyre_batch_fetch before hyre_batch_prepare");
  uint32_t* out_cnt = d_counters + 3 * max_batch;
  uint32_t* rerun = d_counters + 4 * max_batch;
  if (!big_k.empty() && !exh_done) {
    finish_reruns();
    finish_exhaustive();
  }
  // one round trip in the common case: results and the recovery flags
  // together; a pending recovery (candidate overflow) reruns and re-copies
  for (int pass = 0;; ++pass) {
    // out counts and rerun flags are adjacent counter rows: one copy for both
    HYRE_CUDA(cudaMemcpyAsync(h_cnt_rerun.data(), out_cnt, sizeof(uint32_t) * (max_batch + B), cudaMemcpyDeviceToHost,
                              st));
    HYRE_CUDA(cudaMemcpyAsync(h_hits, d_hits, n_hits_total * sizeof(hyre_hit), cudaMemcpyDeviceToHost, st));
    HYRE_CUDA(cudaStreamSynchronize(st));
    std::memcpy(h_out_cnt.data(), h_cnt_rerun.data(), B * 4);
    std::memcpy(h_rerun.data(), h_cnt_rerun.data() + max_batch, B * 4);
    bool pending = false;
    for (uint32_t i = 0; any_emb && i < B; ++i) pending |= h_rerun[i] != 0;
    if (!pending) break;
    if (pass > 0) throw Error(HYRE_INTERNAL, "top-K candidate selection did not converge");
    finish_reruns();
  }
  d2h_bytes = B * 4 + n_hits_total * sizeof(hyre_hit);
  if (std::getenv("HYRE_DEBUG_COUNTS")) {  // diagnostics: candidate / admitted counts per query
    std::vector<uint32_t> c(size_t{max_batch} * kNumCounters);
    HYRE_CUDA(cudaMemcpy(c.data(), d_counters, c.size() * 4, cudaMemcpyDeviceToHost));
    uint64_t sc = 0, mx = 0;
    for (uint32_t i = 0; i < B; ++i) {
      sc += c[max_batch + i];
      mx = std::max<uint64_t>(mx, c[max_batch + i]);
    }
    std::fprintf(stderr, "[hyre] B=%u candidates mean %.1f max %lu, sample period %u, reruns %d\n", B,
                 double(sc) / B, static_cast<unsigned long>(mx), sample_period, int(finish_rounds));
  }
  for (uint32_t i = 0; i < B; ++i) {
    if (st_out) st_out[i] = statuses[i];
    const uint32_t c = statuses[i] == HYRE_OK ? h_out_cnt[i] : 0u;
    if (counts) counts[i] = c;
    if (hits && c) std::memcpy(hits + offsets[i], h_hits + hit_off[i], c * sizeof(hyre_hit));
  }
  if (t) {
    float s6[6];
    stage_ms(s6);
    t->tbr_ms = s6[0];
    t->quant_ms = s6[1];
    t->ebr_ms = s6[2] + s6[3];
    t->topk_ms = s6[4];
  }
}

void Executor::shard_exchange(int point) {
  HYRE_CUDA(cudaEventRecord(shard->ev_x[point], st));
  shard->barrier->arrive_and_wait();  // every shard has recorded this point
  for (uint32_t g = 0; g < shard->G; ++g)
    if (g != shard->g) HYRE_CUDA(cudaStreamWaitEvent(st, shard->peers[g]->shard->ev_x[point], 0));
}

void Executor::settle() {
  if (!prepared) throw Error(HYRE_INTERNAL, "hyre_batch_settle before hyre_batch_prepare");
  if (any_emb) finish_reruns();
  finish_exhaustive();
  HYRE_CUDA(cudaStreamSynchronize(st));
}

void Executor::finish_exhaustive() {
  if (exh_done) return;
  exh_done = true;
  for (uint32_t i : big_k) exhaustive(i);
}

void Executor::ensure_ex(uint64_t n) {
  n = std::max<uint64_t>(n, 1);
  if (n > ex_cap) {
    HYRE_CUDA(cudaStreamSynchronize(st));
    for (void* p : {(void*)d_ex_keys, (void*)d_ex_sorted, (void*)d_ex_rows}) cudaFree(p);
    ex_cap = std::max<uint64_t>(n, ex_cap * 2);
    d_ex_keys = dmalloc<uint64_t>(ex_cap);
    d_ex_sorted = dmalloc<uint64_t>(ex_cap);
    d_ex_rows = dmalloc<uint32_t>(ex_cap);
  }
  size_t tmp = 0;
  HYRE_CUDA(cub::DeviceRadixSort::SortKeysDescending(nullptr, tmp, d_ex_keys, d_ex_sorted, static_cast<int>(ex_cap),
                                                     0, 64, st));
  if (tmp > ex_tmp_cap) {
    HYRE_CUDA(cudaStreamSynchronize(st));
    cudaFree(d_ex_tmp);
    ex_tmp_cap = tmp;
    d_ex_tmp = dmalloc<uint8_t>(ex_tmp_cap);
  }
}

void Executor::sort_desc(const uint64_t* in, uint64_t* out, uint64_t n) {
  if (!n) return;
  size_t tmp = ex_tmp_cap;
  HYRE_CUDA(cub::DeviceRadixSort::SortKeysDescending(d_ex_tmp, tmp, in, out, static_cast<int>(n), 0, 64, st));
}

uint64_t Executor::scan_count(const hyre_query& q) {
  hyre_query t = q;
  t.embedding = nullptr;
  t.embedding_dim = 0;
  t.k = 1;
  t.quant_enabled = 0;
  t.granularity = 100;
  prepare(&t, 1);
  if (statuses[0] != HYRE_OK) throw Error(static_cast<hyre_status>(statuses[0]), slot_errors[0]);
  run();
  uint32_t ne = 0;
  HYRE_CUDA(cudaMemcpyAsync(&ne, d_counters, 4, cudaMemcpyDeviceToHost, st));
  HYRE_CUDA(cudaStreamSynchronize(st));
  return ne;
}

void Executor::scan_rows(uint32_t* d_rows, uint64_t n) {
  if (!n) return;
  FirstKArgs fk{d_mask, d_chunk_cnt, d_counters, d_qp, 1, ix->words, ix->n_chunks, ix->row_base, d_hit_off,
                nullptr, nullptr, d_rows, n, 1};
  launch_first_k(fk, st);
  HYRE_CUDA(cudaStreamSynchronize(st));
}

// Exact exhaustive top-K of prepared query i (synchronous; see executor.cuh):
// its eligible rows -> exact rescoring of every row -> sort (score desc, row
// asc) -> first min(k, n) as the query's hits.  The rows come from this
// batch's K1 mask when it has one -- then already narrowed by the quant
// pre-selection (quantizer.cpp:100-138; global over the shards of a sharded
// index) -- else (fused CNF or match-all batches, never quant) from the
// query's clauses on the aux executor (K1 mask + K5).
void Executor::exhaustive(uint32_t i) {
  HYRE_CUDA(cudaSetDevice(ix->device));
  // the previous exhaustive query's kernels on this stream still read the
  // shared d_ex_* buffers, which the aux executor's scan (its own stream)
  // is about to overwrite
  HYRE_CUDA(cudaStreamSynchronize(st));
  ++exh_count;
  uint32_t* out_cnt = d_counters + 3 * max_batch;
  uint32_t* rerun = d_counters + 4 * max_batch;
  uint64_t n = 0;
  if (!use_fused && !all_match && !k2_match_all) {
    uint32_t ne = 0;
    HYRE_CUDA(cudaMemcpyAsync(&ne, d_counters + i, 4, cudaMemcpyDeviceToHost, st));
    HYRE_CUDA(cudaStreamSynchronize(st));
    n = ne;
    ensure_ex(n);
    if (n) {
      FirstKArgs fk{d_mask + size_t{i} * ix->words, d_chunk_cnt + size_t{i} * ix->n_chunks, d_counters + i, d_qp + i,
                    1, ix->words, ix->n_chunks, ix->row_base, d_hit_off, nullptr, nullptr, d_ex_rows, n, 1};
      launch_first_k(fk, st);
    }
  } else {
    if (!aux) aux = std::make_unique<Executor>(ix, 1);
    hyre_query t{};
    t.n_clauses = raw_cl[i + 1] - raw_cl[i];
    std::vector<uint32_t> offs(t.n_clauses + 1, 0);
    for (uint32_t c = 0; c < t.n_clauses; ++c) offs[c] = raw_offs[raw_cl[i] + c];
    offs[t.n_clauses] =
        raw_cl[i + 1] < raw_offs.size() ? raw_offs[raw_cl[i + 1]] : static_cast<uint32_t>(raw_ids.size());
    t.slots = raw_slots.data() + raw_cl[i];
    t.id_offsets = offs.data();
    t.ids = raw_ids.data();
    n = aux->scan_count(t);
    ensure_ex(n);
    aux->scan_rows(d_ex_rows, n);
  }
  launch_rows_to_keys(d_ex_rows, n, d_ex_keys, st);
  const bool bf16 = ix->emb_dtype == HYRE_EMB_BF16;
  PrefSelectArgs pa{SelectArgs{}, bf16 ? static_cast<const void*>(ix->emb_hi) : static_cast<const void*>(ix->emb_f32),
                    ix->dp, ix->dp * (bf16 ? 2 : 4) / 16, ix->row_base, d_q, ix->row_w};
  launch_rescore_keys(pa, bf16, i, d_ex_keys, n, st);
  sort_desc(d_ex_keys, d_ex_sorted, n);
  launch_keys_to_hits(d_ex_sorted, std::min<uint64_t>(n, true_k[i]), d_hits + hit_off[i], out_cnt + i, rerun + i, st);
  HYRE_CUDA(cudaGetLastError());
}

void Executor::eligible(uint32_t* out) {
  HYRE_CUDA(cudaMemcpyAsync(out, d_counters, sizeof(uint32_t) * B, cudaMemcpyDeviceToHost, st));
  HYRE_CUDA(cudaStreamSynchronize(st));
}

float Executor::last_run_ms() const {
  float ms = 0;
  cudaEventSynchronize(ev[5]);
  const uint8_t* map = ev_map[(n_runs - 1) % kEvRing];
  cudaEventSynchronize(ev[map[5]]);
  cudaEventElapsedTime(&ms, ev[map[0]], ev[map[5]]);
  return ms;
}

// Stage times of one ring slot: boundary i is the event ev_map[slot][i] (an
// empty stage records no event and reuses the previous boundary: 0 ms).
static void slot_stage_ms(const cudaEvent_t* e, const uint8_t* map, float* out) {
  cudaEventSynchronize(e[map[5]]);
  for (int i = 0; i < 5; ++i) {
    out[i] = 0;
    if (map[i] != map[i + 1]) cudaEventElapsedTime(out + i, e[map[i]], e[map[i + 1]]);
  }
  out[5] = 0;
  cudaEventElapsedTime(out + 5, e[map[0]], e[map[5]]);
}

void Executor::stage_ms_hist(uint32_t back, float* out) const {
  if (back >= kEvRing || back >= n_runs) throw Error(HYRE_INVALID_ARGUMENT, "no such run in the timing ring");
  const uint64_t slot = (n_runs - 1 - back) % kEvRing;
  slot_stage_ms(ev_ring[slot], ev_map[slot], out);
}

void Executor::stage_ms(float* out) const {
  if (n_runs == 0) throw Error(HYRE_INVALID_ARGUMENT, "no run to time");
  const uint64_t slot = (n_runs - 1) % kEvRing;
  slot_stage_ms(ev_ring[slot], ev_map[slot], out);
}

// Boundary i of the current run: an event when its stage did work, else an
// alias of boundary i - 1 (each event record costs ~1-2 us of stream time).
void Executor::mark(int i, bool stage_ran) {
  uint8_t* map = ev_map[(n_runs - 1) % kEvRing];
  if (i == 0 || i == 5 || (stage_ran && stage_events)) {
    HYRE_CUDA(cudaEventRecord(ev[i], st));
    map[i] = static_cast<uint8_t>(i);
  } else {
    map[i] = map[i - 1];
  }
}

// ---------------------------------------------------------------------------
// Stage functions
// ---------------------------------------------------------------------------
uint64_t Executor::full_scan(const hyre_query& q, uint32_t* rows, uint64_t cap_rows) {
  hyre_query t = q;
  t.embedding = nullptr;
  t.k = 1;
  t.granularity = 100;
  prepare(&t, 1);
  if (statuses[0] != HYRE_OK) throw Error(static_cast<hyre_status>(statuses[0]), slot_errors[0]);
  run();
  uint32_t ne = 0;
  HYRE_CUDA(cudaMemcpyAsync(&ne, d_counters, 4, cudaMemcpyDeviceToHost, st));
  HYRE_CUDA(cudaStreamSynchronize(st));
  const uint64_t take = std::min<uint64_t>(ne, cap_rows);
  if (take) {
    uint32_t* d_rows = dmalloc<uint32_t>(take);
    FirstKArgs fk{d_mask, d_chunk_cnt, d_counters, d_qp, 1, ix->words, ix->n_chunks, ix->row_base, d_hit_off,
                  nullptr, nullptr, d_rows, take, 1};
    launch_first_k(fk, st);
    HYRE_CUDA(cudaMemcpyAsync(rows, d_rows, take * 4, cudaMemcpyDeviceToHost, st));
    HYRE_CUDA(cudaStreamSynchronize(st));
    cudaFree(d_rows);
  }
  return ne;
}

// batch_scan_tbr (pipeline.cpp:75-93): the batch's eligibility masks (K1 /
// K1b, one pass over the rows for all b queries) -> per-word counts -> scan
// -> messengers in (row, query position) order.
uint64_t Executor::batch_scan(const hyre_query* qs, uint32_t b, const uint32_t* batch_ids, hyre_messenger* out,
                              uint64_t cap) {
  if (b == 0) return 0;
  std::vector<hyre_query> t(qs, qs + b);
  for (hyre_query& q : t) {
    q.embedding = nullptr;
    q.embedding_dim = 0;
    q.k = 1;
    q.quant_enabled = 0;
    q.granularity = 100;
  }
  prepare(t.data(), b);
  for (uint32_t i = 0; i < b; ++i)
    if (statuses[i] != HYRE_OK) throw Error(static_cast<hyre_status>(statuses[i]), slot_errors[i]);
  run();
  const uint32_t W = ix->words;
  uint64_t* d_cnt = dmalloc<uint64_t>(W + 1);
  uint64_t* d_off = dmalloc<uint64_t>(W + 1);
  uint32_t* d_bid = dmalloc<uint32_t>(b);
  HYRE_CUDA(cudaMemcpyAsync(d_bid, batch_ids, b * 4, cudaMemcpyHostToDevice, st));
  launch_scan_count(d_mask, d_qp, b, W, d_cnt, st);
  size_t tmp = 0;
  HYRE_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, d_cnt, d_off, W + 1, st));
  uint8_t* d_tmp = dmalloc<uint8_t>(std::max<size_t>(tmp, 1));
  HYRE_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp, tmp, d_cnt, d_off, W + 1, st));
  uint64_t total = 0;
  HYRE_CUDA(cudaMemcpyAsync(&total, d_off + W, 8, cudaMemcpyDeviceToHost, st));
  HYRE_CUDA(cudaStreamSynchronize(st));
  const uint64_t take = std::min(total, cap);
  if (take) {
    hyre_messenger* d_out = dmalloc<hyre_messenger>(take);
    launch_scan_emit(d_mask, d_qp, b, W, ix->row_base, d_off, d_bid, d_out, take, st);
    HYRE_CUDA(cudaMemcpyAsync(out, d_out, take * sizeof(hyre_messenger), cudaMemcpyDeviceToHost, st));
    HYRE_CUDA(cudaStreamSynchronize(st));
    cudaFree(d_out);
  }
  HYRE_CUDA(cudaGetLastError());
  for (void* p : {(void*)d_cnt, (void*)d_off, (void*)d_bid, (void*)d_tmp}) cudaFree(p);
  return total;
}

bool Executor::exact_scores(const float* q, uint32_t dim, const uint32_t* rows, uint64_t n, float* out) {
  if (dim != ix->dim)
    validation("query embedding dim " + std::to_string(dim) + " != index dim " + std::to_string(ix->dim));
  for (uint64_t i = 0; i < n; ++i)
    if (rows[i] < ix->row_base || rows[i] >= ix->row_base + ix->n_rows)
      validation("row " + std::to_string(rows[i]) + " outside this index shard");
  HYRE_CUDA(cudaSetDevice(ix->device));
  std::vector<float> unit(ix->dp, 0.0f);
  const bool ren = unit_embedding(q, dim, unit.data());
  float* d_qv = dmalloc<float>(ix->dp);
  uint32_t* d_rows = dmalloc<uint32_t>(std::max<uint64_t>(n, 1));
  float* d_out = dmalloc<float>(std::max<uint64_t>(n, 1));
  HYRE_CUDA(cudaMemcpyAsync(d_qv, unit.data(), ix->dp * 4, cudaMemcpyHostToDevice, st));
  if (n) HYRE_CUDA(cudaMemcpyAsync(d_rows, rows, n * 4, cudaMemcpyHostToDevice, st));
  const bool bf16 = ix->emb_dtype == HYRE_EMB_BF16;
  launch_gather_scores(bf16 ? static_cast<const void*>(ix->emb_hi) : ix->emb_f32, bf16, ix->dp, ix->row_base,
                       d_qv, d_rows, n, d_out, st);
  if (n) HYRE_CUDA(cudaMemcpyAsync(out, d_out, n * 4, cudaMemcpyDeviceToHost, st));
  HYRE_CUDA(cudaStreamSynchronize(st));
  cudaFree(d_qv);
  cudaFree(d_rows);
  cudaFree(d_out);
  return ren;
}

uint32_t Executor::top_k(const uint32_t* rows, const float* scores, uint64_t n, uint32_t k, hyre_hit* out) {
  if (n == 0) return 0;
  HYRE_CUDA(cudaSetDevice(ix->device));
  const uint32_t kk = static_cast<uint32_t>(std::min<uint64_t>(k, n));
  if (kk > kSelectMaxK) {  // beyond the shared-memory select: sort every key (bucket_top_k takes any k)
    ensure_ex(n);
    uint32_t* d_rows = dmalloc<uint32_t>(n);
    float* d_sc = dmalloc<float>(n);
    hyre_hit* d_out = dmalloc<hyre_hit>(kk);
    HYRE_CUDA(cudaMemcpyAsync(d_rows, rows, n * 4, cudaMemcpyHostToDevice, st));
    HYRE_CUDA(cudaMemcpyAsync(d_sc, scores, n * 4, cudaMemcpyHostToDevice, st));
    launch_make_keys(d_rows, d_sc, n, d_ex_keys, st);
    sort_desc(d_ex_keys, d_ex_sorted, n);
    launch_keys_to_hits(d_ex_sorted, kk, d_out, nullptr, nullptr, st);
    HYRE_CUDA(cudaMemcpyAsync(out, d_out, kk * sizeof(hyre_hit), cudaMemcpyDeviceToHost, st));
    HYRE_CUDA(cudaStreamSynchronize(st));
    for (void* p2 : {(void*)d_rows, (void*)d_sc, (void*)d_out}) cudaFree(p2);
    return kk;
  }
  uint32_t* d_rows = dmalloc<uint32_t>(n);
  float* d_sc = dmalloc<float>(n);
  uint64_t* d_keys = dmalloc<uint64_t>(n);
  hyre_hit* d_out = dmalloc<hyre_hit>(kk);
  uint32_t* d_misc = dmalloc<uint32_t>(8);
  uint64_t* d_off = dmalloc<uint64_t>(1);
  QParam p{QF_ACTIVE | QF_EMB, kk, 0, 0};
  QParam* d_p = dmalloc<QParam>(1);
  HYRE_CUDA(cudaMemcpyAsync(d_rows, rows, n * 4, cudaMemcpyHostToDevice, st));
  HYRE_CUDA(cudaMemcpyAsync(d_sc, scores, n * 4, cudaMemcpyHostToDevice, st));
  HYRE_CUDA(cudaMemcpyAsync(d_p, &p, sizeof p, cudaMemcpyHostToDevice, st));
  const uint32_t n32 = static_cast<uint32_t>(n);
  uint32_t misc[8] = {n32, n32, 0, 0, 0, 0, 0, 0};  // cnt, n_elig, rerun, out_cnt
  HYRE_CUDA(cudaMemcpyAsync(d_misc, misc, sizeof misc, cudaMemcpyHostToDevice, st));
  HYRE_CUDA(cudaMemsetAsync(d_off, 0, 8, st));
  launch_make_keys(d_rows, d_sc, n, d_keys, st);
  uint64_t* d_t = dmalloc<uint64_t>(1);
  SelectArgs fa{d_keys, d_misc, n32, d_p, d_misc + 1, SELECT_FINAL, d_t, d_misc + 2, d_out, d_off, d_misc + 3,
                1, QF_ACTIVE | QF_EMB, n32, nullptr, 1, 0};
  launch_select(fa, st);
  uint32_t cnt = 0;
  HYRE_CUDA(cudaMemcpyAsync(&cnt, d_misc + 3, 4, cudaMemcpyDeviceToHost, st));
  HYRE_CUDA(cudaStreamSynchronize(st));
  HYRE_CUDA(cudaMemcpy(out, d_out, cnt * sizeof(hyre_hit), cudaMemcpyDeviceToHost));
  for (void* p2 : {(void*)d_rows, (void*)d_sc, (void*)d_keys, (void*)d_out, (void*)d_misc, (void*)d_off,
                   (void*)d_p, (void*)d_t})
    cudaFree(p2);
  return cnt;
}

// Replaces this executor's results with the exact merge of G gathered shard
// result sets (device pointers, e.g. filled by an NCCL all-gather).
void Executor::merge_gathered(const hyre_hit* g_hits, const uint64_t* g_off, const uint32_t* g_cnt, uint32_t G,
                              uint64_t hits_stride, uint64_t off_stride, uint64_t cnt_stride) {
  if (!prepared) throw Error(HYRE_INTERNAL, "merge before hyre_batch_prepare");
  if (uint64_t{G} * max_k > cap) validation("merge needs G*k <= candidate capacity");
  HYRE_CUDA(cudaSetDevice(ix->device));
  uint32_t* cand_cnt = d_counters + max_batch;
  uint32_t* out_cnt = d_counters + 3 * max_batch;
  uint32_t* rerun = d_counters + 4 * max_batch;
  launch_gather_keys(g_hits, hits_stride, g_off, off_stride ? off_stride : B, g_cnt, cnt_stride ? cnt_stride : B, G, B,
                     cap, d_cand, cand_cnt, st);
  // term-only hits carry score 0, so key order is row order: the merged
  // first-K equals concatenating shard first-K lists in row order.
  SelectArgs fa{d_cand, cand_cnt, cap, d_qp, cand_cnt, SELECT_FINAL, d_thr, rerun, d_hits, d_hit_off,
                out_cnt, B, QF_ACTIVE, cap, nullptr, 1, 0};
  launch_select(fa, st);
  HYRE_CUDA(cudaGetLastError());
}

uint64_t Executor::preselect(const uint64_t* qwords, const uint32_t* rows, uint64_t n, uint32_t quant_k,
                             uint32_t* out) {
  if (quant_k < 1) validation("quantK must be >= 1");
  if (n <= quant_k) {
    std::memcpy(out, rows, n * 4);
    return n;
  }
  HYRE_CUDA(cudaSetDevice(ix->device));
  const uint32_t nw = ix->num_words;
  uint32_t* d_rows = dmalloc<uint32_t>(n);
  uint64_t* d_q = dmalloc<uint64_t>(nw);
  uint64_t* d_keys = dmalloc<uint64_t>(n);
  uint64_t* d_sorted = dmalloc<uint64_t>(n);
  HYRE_CUDA(cudaMemcpyAsync(d_rows, rows, n * 4, cudaMemcpyHostToDevice, st));
  HYRE_CUDA(cudaMemcpyAsync(d_q, qwords, nw * 8, cudaMemcpyHostToDevice, st));
  launch_quant_keys(ix->sigs, nw, ix->num_bits, ix->row_base, d_q, d_rows, n, d_keys, st);
  size_t tmp = 0;
  cub::DeviceRadixSort::SortKeysDescending(nullptr, tmp, d_keys, d_sorted, static_cast<int>(n), 0, 64, st);
  uint8_t* d_tmp = dmalloc<uint8_t>(tmp);
  cub::DeviceRadixSort::SortKeysDescending(d_tmp, tmp, d_keys, d_sorted, static_cast<int>(n), 0, 64, st);
  std::vector<uint64_t> top(quant_k);
  HYRE_CUDA(cudaMemcpyAsync(top.data(), d_sorted, quant_k * 8ull, cudaMemcpyDeviceToHost, st));
  HYRE_CUDA(cudaStreamSynchronize(st));
  for (uint32_t i = 0; i < quant_k; ++i) out[i] = ~static_cast<uint32_t>(top[i]);
  std::sort(out, out + quant_k);
  for (void* p : {(void*)d_rows, (void*)d_q, (void*)d_keys, (void*)d_sorted, (void*)d_tmp}) cudaFree(p);
  return quant_k;
}

}  // namespace hyreb
