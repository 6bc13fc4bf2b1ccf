// Launch interfaces of the hot-path kernels (K1, K2, K4, K5, K6 in
// SURVEY.md §2 / DESIGN.md §4).  All launches are asynchronous on `st`.
#pragma once

#include <vector>

#include "device.cuh"

namespace hyreb {

// ---- K1: CNF eligibility mask (term_match.cpp:56-78, pipeline.cpp:75-93) ----
struct MaskArgs {
  const uint32_t* const* refs;  // batch ref table: bitmap base pointers (W words each)
  uint32_t n_refs;
  const uint32_t* prog;  // per query: n_clauses, {n_refs, ref...}*
  const QParam* qp;
  uint32_t B, words, n_chunks, n_rows;
  uint32_t* mask;        // [B][W]
  uint32_t* chunk_cnt;   // [B][n_chunks]
  uint32_t* n_elig;      // [B] (zeroed by caller)
};
void launch_mask(const MaskArgs& a, cudaStream_t st);

// Term-major K1: the batch program (per 32-query group: slots, refs and the
// 32-bit mask of queries using each ref) is a __grid_constant__ parameter so the
// per-ref query masks are warp-uniform; each thread keeps 32 query
// accumulators in registers.  Returns false if the program does not fit (the
// generic launch_mask is used instead).
constexpr uint32_t kMaskProgWords = 7936;  // fits the 32 KB kernel-parameter limit
// Returns the number of launches; bit 31 set if a group's program alone is too
// large (the caller then uses the generic launch_mask).
uint32_t launch_mask_tm(const MaskArgs& a, const std::vector<std::vector<uint32_t>>& groups,
                        const std::vector<uint32_t>& live, cudaStream_t st);

// K1b: forward-index CNF evaluation for batches (see kernels.cu).  One pass
// evaluates up to 64 * NW queries; `entries` lists (term id, NW x 64-bit
// users mask) for every term referenced by the pass's clauses.
struct FwdArgs {
  const uint16_t* row_terms;
  const uint8_t* slot_of;
  uint32_t A, n_rows, words, n_chunks, B, C, T;
  const uint32_t* entries;  // n_entries x (1 + 2 * NW) u32
  uint32_t n_entries;
  const uint64_t* hc;       // [C][NW] queries constraining each slot
  const uint64_t* live;     // [NW] active, non-empty queries
  uint32_t q0;              // first query of this pass
  uint32_t nw;              // 1 or 2
  uint32_t* mask;
  uint32_t* chunk_cnt;
  uint32_t* n_elig;
};
size_t fwd_mask_smem(uint32_t T, uint32_t C, uint32_t nw);
void launch_fwd_mask(const FwdArgs& a, cudaStream_t st);

// CSR postings scattered into per-clause scratch bitmaps.
struct ScatterItem {
  uint64_t begin;   // first posting in post_rows
  uint32_t count;   // df
  uint32_t target;  // scratch bitmap index
};
void launch_scatter(const ScatterItem* items, const uint64_t* item_prefix, uint32_t n_items,
                    uint64_t total, const uint32_t* post_rows, uint32_t* scratch, uint32_t words,
                    cudaStream_t st);

// ---- K2: CUDA-core streaming scorer with threshold candidate filter ----
enum ScoreMode : uint32_t { SCORE_MAIN = 0, SCORE_SAMPLE = 1, SCORE_RERUN = 2 };
struct ScoreArgs {
  const void* emb;  // float or bf16 rows, stride dp elements
  uint32_t dp, dp_chunks, n_rows, row_base, words;
  const uint32_t* mask;
  const QParam* qp;
  const float* q;  // [B][dp]
  uint32_t B;
  const uint32_t* n_elig;
  const uint64_t* thr;  // [B]
  uint64_t* cand;       // [B][cap]
  uint32_t* cand_cnt;   // [B]
  uint32_t cap;
  uint32_t mode, period;
  uint32_t gate;          // queries with n_elig > gate are sampled (= candidate cap)
  const uint32_t* rerun;  // [B]
  uint32_t* samp;         // SCORE_SAMPLE: dense [B][cap] orderable scores (0 = ineligible)
  uint32_t split;         // main/rerun: parts per 1024-row segment (power of two <= 32)
  uint32_t split_sample;  // the same for the sample pass
  // int8 prefilter (emb = DevIndex::tc_i8, the swizzled 128-row tiles): the
  // int8 query qi8 [B][dp], score s' = acc x qscale[q]; rows are admitted
  // when s' >= score(thr) - qdelta[q] (exact rescoring follows in K4p)
  const int8_t* qi8;
  const float* qscale;
  const float* qdelta;
  // learned per-row weights (local rows; nullptr = identity): every score and
  // prefilter score is w[r] x clamp(s).  w <= 1 keeps the prefilter bound.
  const float* row_w;
  uint32_t match_all;  // every active query is match-all: tail masks, no K1 mask
  // SCORE_SAMPLE into per-query score histograms [B][hbins] (linear bins over
  // [-1, 1]) instead of the dense slots; thresholds then come from hist_thr
  uint32_t* shist;
  uint32_t hbins;
};
void launch_score(const ScoreArgs& a, bool bf16, cudaStream_t st);
void launch_score_i8(const ScoreArgs& a, cudaStream_t st);

// Largest key whose score is <= s - delta: a lower bound, in key space, for
// every exact score of a row whose prefilter score was s (delta = the bound).
__host__ __device__ __forceinline__ uint64_t key_minus_delta(uint64_t key, float delta) {
  return key == 0ull ? 0ull : (static_cast<uint64_t>(f2ord(key_score(key) - delta)) << 32);
}

// ---- K4: per-query exact selection over candidate keys ----
enum SelectMode : uint32_t { SELECT_KTH = 0, SELECT_FINAL = 1, SELECT_FINAL_RERUN = 2 };
struct SelectArgs {
  const uint64_t* buf;
  const uint32_t* cnt;
  uint32_t cap;
  const QParam* qp;
  const uint32_t* n_elig;
  uint32_t mode;
  uint64_t* thr;       // KTH: out; FINAL: out on overflow
  uint32_t* rerun;     // FINAL: set on overflow; FINAL_RERUN: consumed
  hyre_hit* hits;      // FINAL: out
  const uint64_t* hit_off;
  uint32_t* out_cnt;
  uint32_t B;
  uint32_t require_flags;  // queries must have these flags (QF_ACTIVE|QF_EMB)
  uint32_t gate;           // KTH: only queries with n_elig > gate were sampled
  // KTH also writes thr_safe = K-th sampled key (a guaranteed lower bound on
  // the global K-th key) and sets thr to the m-th sampled key, m =
  // min(K, max(8, 4K/period)): an estimate admitting ~m*period rows.  FINAL
  // falls back to thr_safe (rerun) if the estimate admitted fewer than K rows.
  uint64_t* thr_safe;
  uint32_t period;
  uint32_t dense_n;  // KTH over a dense sample buffer: slots [0, dense_n) (0 = ineligible)
  // dense sample (KTH with dense_n): [B][cap] orderable scores f2ord(score);
  // slot s holds local row (s / 1024) * period * 1024 + s % 1024
  const uint32_t* samp;
  uint32_t row_base;
  uint64_t* fb;     // KTH fallback scratch ([B][fb_cap] keys; the candidate buffer)
  uint32_t fb_cap;
  // K3 prefilter bound: KTH lowers thr_safe by delta (the sample holds
  // prefilter scores); select_prefilter_kernel prunes and checks with it.
  float delta;
  const float* qdelta;  // per-query bounds (replace delta when given)
};
void launch_select(const SelectArgs& a, cudaStream_t st);
// K4 for K3 prefilter candidates (SELECT_FINAL / SELECT_FINAL_RERUN; see
// kernels.cu): prunes to the rows that can still reach the exact top K,
// rescores them exactly with K2's arithmetic over the resident row-major rows
// (fp32, or the bf16 rows of a bf16 index) and the fp32 unit queries, checks
// the threshold, sorts.  s.delta = the prefilter bound.
struct PrefSelectArgs {
  SelectArgs s;
  const void* emb;
  uint32_t dp, dp_chunks, row_base;
  const float* q;  // [B][dp]
  const float* row_w;  // learned per-row weights (local rows) or nullptr
};
void launch_select_prefilter(const PrefSelectArgs& a, bool bf16, cudaStream_t st);
// SELECT_KTH over the dense sample: per-slice top keys gathered into fb
// (ucnt [B] zeroed by the caller), then one sort per query.
void launch_sample_kth(const SelectArgs& a, uint32_t* ucnt, cudaStream_t st);

// Thresholds from per-query sample histograms (K3 sample pass with shist):
// thr = lower edge of the bin holding the sample's m-th score (the same m as
// SELECT_KTH), thr_safe = lower edge of the K-th's bin (a lower bound on the
// global K-th score: K sampled rows lie at or above it), lowered by delta for
// prefilter scores.  Queries not sampled get 0 (no threshold).
struct HistThrArgs {
  const uint32_t* hist;  // [B][nb]
  uint32_t nb;
  const QParam* qp;
  const uint32_t* n_elig;
  uint32_t gate, period, B, require_flags;
  uint64_t* thr;
  uint64_t* thr_safe;
  float delta;
  const float* qdelta;  // per-query bounds (replace delta when given)
};
void launch_hist_thr(const HistThrArgs& a, cudaStream_t st);
// Run prologue of a K3 batch: counters[0 .. n_counters) = 0 except the first
// B (eligible counts) = ~0 (unknown), and hist[0 .. hist_words) = 0.
void launch_run_init(uint32_t* counters, uint32_t n_counters, uint32_t B, uint32_t* hist, size_t hist_words,
                     cudaStream_t st);

// ---- K5: term-only first-K rows (pipeline.cpp:30-40) ----
struct FirstKArgs {
  const uint32_t* mask;
  const uint32_t* chunk_cnt;
  const uint32_t* n_elig;
  const QParam* qp;
  uint32_t B, words, n_chunks, row_base;
  const uint64_t* hit_off;
  hyre_hit* hits;
  uint32_t* out_cnt;
  uint32_t* rows_out;   // optional: plain rows (full_scan_tbr), capacity rows_cap
  uint64_t rows_cap;
  uint32_t all_rows;    // 1: ignore k (full scan)
};
void launch_first_k(const FirstKArgs& a, cudaStream_t st);

// ---- K6: sign-quant pre-selection narrowing the mask (quantizer.cpp:100-138) ----
struct QuantArgs {
  const uint64_t* sigs;  // [n_rows][nw]
  uint32_t nw, num_bits;
  const uint64_t* qsig;  // [B][nw]
  const QParam* qp;
  uint32_t B, words, n_chunks, n_rows;
  uint32_t* mask;
  uint32_t* chunk_cnt;
  uint32_t* n_elig;
  uint32_t* hist;       // [B][num_bits + 1]
  uint32_t* tsel;       // [B][4]: threshold score t, ==t rows to keep, active, local ==t rows
  uint32_t* eq_cnt;     // [B][n_chunks] ==t rows per chunk
  // Row shard of a sharded index (global quant, ShardCtx): hist counts every
  // QF_QUANT query's rows; the threshold comes from hist_total (the sum of
  // every shard's histogram), the ==t rows to keep from the global budget
  // minus the ties of lower shards (quant_offset); n_elig = local survivors.
  uint32_t shard_mode;
  const uint32_t* hist_total;  // [B][num_bits + 1] (nullptr: hist)
};
void launch_quant(const QuantArgs& a, cudaStream_t st);
// The same in three phases for a sharded index: hist | thresh + eq + scan | apply.
void launch_quant_hist(const QuantArgs& a, cudaStream_t st);
void launch_quant_select(const QuantArgs& a, cudaStream_t st);
void launch_quant_apply(const QuantArgs& a, cudaStream_t st);
// Peer-memory exchanges of a sharded batch (pointers of every shard's buffer,
// readable from this device: same device or peer access enabled).
constexpr uint32_t kMaxShards = 16;
struct PeerPtrs {
  const uint32_t* p[kMaxShards];
};
// dst[i] = sum over shards of src_g[i]
void launch_sum_peers(const PeerPtrs& src, uint32_t G, size_t n, uint32_t* dst, cudaStream_t st);
// shard g: tsel[q][1] = max(0, global ==t budget - sum of the ==t rows of shards < g)
void launch_quant_offset(const PeerPtrs& tsel, uint32_t g, uint32_t B, uint32_t* my_tsel, cudaStream_t st);
// Sharded merge: per query, keys of every shard's hits (emb queries) and the
// concatenated row lists of term-only queries (k unlimited).
struct PeerHits {
  const hyre_hit* hits[kMaxShards];
  const uint32_t* cnt[kMaxShards];
};
void launch_gather_peer_keys(const PeerHits& ph, uint32_t G, const uint64_t* hit_off, const QParam* qp, uint32_t B,
                             uint32_t cap, uint64_t* keys, uint32_t* cnt, cudaStream_t st);
void launch_concat_term_only(const PeerHits& ph, uint32_t G, const uint64_t* hit_off, const QParam* qp,
                             const uint32_t* true_k, uint32_t B, hyre_hit* out, uint32_t* out_cnt, cudaStream_t st);
// one query's keys from every shard into keys (count -> *cnt)
void launch_gather_peer_keys_one(const PeerHits& ph, uint32_t G, uint64_t off, uint32_t q, uint64_t cap,
                                 uint64_t* keys, uint32_t* cnt, cudaStream_t st);

// ---- stage helpers ----
void launch_gather_scores(const void* emb, bool bf16, uint32_t dp, uint32_t row_base,
                          const float* q, const uint32_t* rows, uint64_t n, float* out,
                          cudaStream_t st);
void launch_make_keys(const uint32_t* rows, const float* scores, uint64_t n, uint64_t* keys,
                      cudaStream_t st);
void launch_quant_keys(const uint64_t* sigs, uint32_t nw, uint32_t num_bits, uint32_t row_base,
                       const uint64_t* qsig, const uint32_t* rows, uint64_t n, uint64_t* keys,
                       cudaStream_t st);
// Exhaustive exact top-K of one query (Executor::exhaustive): rows -> keys
// (score 0), quant keys -> keys, exact rescoring of every key in place with
// K4p's arithmetic (many CTAs), sorted keys -> hits (+ count, rerun flag).
void launch_rows_to_keys(const uint32_t* rows, uint64_t n, uint64_t* keys, cudaStream_t st);
void launch_quant_to_keys(const uint64_t* qkeys, uint64_t n, uint64_t* keys, cudaStream_t st);
void launch_rescore_keys(const PrefSelectArgs& a, bool bf16, uint32_t q, uint64_t* keys, uint64_t n,
                         cudaStream_t st);
void launch_keys_to_hits(const uint64_t* keys, uint64_t n, hyre_hit* out, uint32_t* out_cnt, uint32_t* rerun,
                         cudaStream_t st);
// Multi-GPU merge: per query, keys of the hits of G gathered shard lists
// (shard g's arrays at g x stride elements: separate [G][...] arrays, or
// one packed record per shard).
void launch_gather_keys(const hyre_hit* g_hits, uint64_t hits_stride, const uint64_t* g_off, uint64_t off_stride,
                        const uint32_t* g_cnt, uint64_t cnt_stride, uint32_t G, uint32_t B, uint32_t cap,
                        uint64_t* keys, uint32_t* cnt, cudaStream_t st);

// batch_scan_tbr (pipeline.cpp:75-93): per 32-row word, matches over the
// active queries of a [B][W] mask (cnt has W + 1 slots; cnt[W] = 0), then --
// with off = exclusive scan of cnt -- the messengers in (row, query) order.
void launch_scan_count(const uint32_t* mask, const QParam* qp, uint32_t B, uint32_t W, uint64_t* cnt,
                       cudaStream_t st);
void launch_scan_emit(const uint32_t* mask, const QParam* qp, uint32_t B, uint32_t W, uint32_t row_base,
                      const uint64_t* off, const uint32_t* batch_ids, hyre_messenger* out, uint64_t cap,
                      cudaStream_t st);

// ---- K7: single-launch exact scorer for small indexes (single queries) ----
struct SmallArgs {
  const void* emb;  // fp32 or bf16 rows, stride dp
  uint32_t dp, dp_chunks, n_rows, row_base, words;
  const uint32_t* const* refs;  // K1 program refs (dense bitmaps)
  const uint32_t* prog;
  uint32_t prog_words, n_refs;  // program length (all queries), refs in the table
  const QParam* qp;
  uint32_t B;
  const float* q;       // [B][dp] unit queries
  const float* row_w;   // learned per-row weights or nullptr
  uint64_t* cand;       // [B][cap] candidate keys (per-segment top k)
  uint32_t* cand_cnt;   // [B] (zeroed)
  uint32_t cap;
  uint32_t* n_elig;     // [B] (zeroed)
};
constexpr uint32_t kSmallMaxRows = 262144;  // K7 indexes: n_seg x k candidates fit the buffer
constexpr uint32_t kSmallMaxK = 256;
constexpr uint32_t kSmallProg = 1024;   // program words staged per query (K7 requires a shorter program)
constexpr uint32_t kSmallRefs = 512;    // ref pointers staged in shared memory
constexpr uint32_t kSmallClauses = 32;  // clause slots (hyre_index num_clauses <= 32)
bool small_supported(uint32_t dp_chunks);
void launch_small(const SmallArgs& a, bool bf16, cudaStream_t st);

}  // namespace hyreb
