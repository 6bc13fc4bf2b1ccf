/*
 * hyre_b200.h -- C-ABI of the B200-native hybrid retrieval hot path
 * (arXiv 2402.13435, "hyre" reference at /root/reference/proj).
 *
 * This is the drop-in boundary for the reference's C++ API in
 * proj/include/hyre/{corpus,term_match,quantizer,knn,pipeline,types,common}.hpp.
 * Every entry point below names the reference interface it replaces.  Plain
 * pointers and sizes only; no torch or CUDA types cross this boundary (the
 * executor's stream is exposed as an opaque void*).
 *
 * Error convention (reference: proj/include/hyre/common.hpp:15-33,
 * knn.cpp:59-61, service.cpp:219-225):
 *   HYRE_INVALID_ARGUMENT  <=> hyre::ValidationError (message names the field,
 *                              byte-identical to the reference's message)
 *   HYRE_OUT_OF_RANGE      <=> std::domain_error (score outside [-1, 1])
 *   HYRE_LOAD_ERROR        <=> hyre::LoadError, cause via hyre_last_load_cause()
 *   HYRE_CUDA_ERROR / HYRE_OUT_OF_MEMORY / HYRE_INTERNAL <=> std::runtime_error
 * The message of the last failing call on the calling thread is returned by
 * hyre_last_error().
 *
 * Threading (reference: corpus.hpp:54-56, pipeline.hpp:66-68): a hyre_frozen /
 * hyre_index is immutable after creation and may be shared by any number of
 * executors; one hyre_executor runs one batch at a time.
 */
#ifndef HYRE_B200_H_
#define HYRE_B200_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define HYRE_B200_ABI_VERSION 1

typedef enum hyre_status {
  HYRE_OK = 0,
  HYRE_INVALID_ARGUMENT = 1,
  HYRE_OUT_OF_RANGE = 2,
  HYRE_LOAD_ERROR = 3,
  HYRE_CUDA_ERROR = 4,
  HYRE_OUT_OF_MEMORY = 5,
  HYRE_INTERNAL = 6
} hyre_status;

/* hyre::LoadError::Cause (common.hpp:24) */
typedef enum hyre_load_cause {
  HYRE_LOAD_BAD_MAGIC = 0,
  HYRE_LOAD_VERSION_MISMATCH = 1,
  HYRE_LOAD_TRUNCATED = 2,
  HYRE_LOAD_CHECKSUM = 3
} hyre_load_cause;

typedef enum hyre_emb_dtype {
  HYRE_EMB_F32 = 0,  /* reference storage (corpus.hpp:118) */
  HYRE_EMB_BF16 = 1  /* RNE-bf16 of the frozen fp32 rows (config c4) */
} hyre_emb_dtype;

const char* hyre_last_error(void);
int hyre_last_load_cause(void);
int hyre_abi_version(void);

/* ------------------------------------------------------------------------
 * Host-side index build: IndexBuilder / FrozenIndex (corpus.hpp:36-124)
 * ------------------------------------------------------------------------ */
typedef struct hyre_builder hyre_builder;
typedef struct hyre_frozen hyre_frozen;

/* IndexBuilder::IndexBuilder(IndexConfig) -- corpus.hpp:40, corpus.cpp:15-27.
 * clause_names: NULL (defaults c0, c1, ...) or num_names strings. */
hyre_status hyre_builder_create(uint32_t num_clauses, uint32_t max_num_attr, uint32_t dim,
                                const char* const* clause_names, uint32_t num_names,
                                hyre_builder** out);
void hyre_builder_destroy(hyre_builder* b);

/* IndexBuilder::add_document -- corpus.hpp:43, corpus.cpp:29-52.
 * Clause c of the document holds ids[slot_offsets[c] .. slot_offsets[c+1]);
 * num_slots is the document's clause count (validated against num_clauses). */
hyre_status hyre_builder_add_document(hyre_builder* b, const char* doc_id,
                                      uint32_t num_slots, const uint32_t* slot_offsets,
                                      const uint32_t* ids, const float* embedding,
                                      uint32_t embedding_len, uint32_t* row_out);

/* Bulk form of add_document for n documents with ids doc_id_prefix + index
 * (the prefix + decimal of the running row number).  Clause c of document i
 * holds ids[slot_offsets[i*C + c] .. slot_offsets[i*C + c + 1]). */
hyre_status hyre_builder_add_documents(hyre_builder* b, uint32_t n, const char* doc_id_prefix,
                                       const uint64_t* slot_offsets, const uint32_t* ids,
                                       const float* embeddings);
uint32_t hyre_builder_size(const hyre_builder* b);

/* ---- ingestion (dataio.hpp:15-28; host C++, csrc/ingest.cpp) ----------------
 * read_schema_json (dataio.cpp:118-140): {"clauses": ["geo", ...], "dim": 4}. */
typedef struct hyre_schema hyre_schema;
hyre_status hyre_schema_read_json(const char* path, hyre_schema** out);
hyre_status hyre_schema_create(uint32_t n_clauses, const char* const* clause_names, uint32_t dim,
                               hyre_schema** out);
void hyre_schema_destroy(hyre_schema* s);
uint32_t hyre_schema_num_clauses(const hyre_schema* s);
const char* hyre_schema_clause_name(const hyre_schema* s, uint32_t i);
uint32_t hyre_schema_dim(const hyre_schema* s);
/* read_documents_jsonl (dataio.cpp:142-187): the documents of a JSONL corpus in
 * file order, flat: slot_offsets (count x C + 1) into ids, embeddings count x dim;
 * widest = the largest per-document count of distinct ids (hyre build's
 * maxNumAttr, cli_commands.cpp:37-63).  Errors: "<path>:<line>: <what>". */
typedef struct hyre_documents hyre_documents;
hyre_status hyre_documents_read_jsonl(const char* path, const hyre_schema* s, hyre_documents** out);
void hyre_documents_destroy(hyre_documents* d);
uint32_t hyre_documents_count(const hyre_documents* d);
uint32_t hyre_documents_widest(const hyre_documents* d);
const char* hyre_documents_id(const hyre_documents* d, uint32_t i);
const uint64_t* hyre_documents_slot_offsets(const hyre_documents* d);
const uint32_t* hyre_documents_ids(const hyre_documents* d);
const float* hyre_documents_embeddings(const hyre_documents* d);
/* add_document (corpus.cpp:29-52) for every document of the set, in order. */
hyre_status hyre_builder_add_document_set(hyre_builder* b, const hyre_documents* d, uint32_t* first_row);
/* The learned-link serving-graph export (write_links_export, dataio.cpp:253-274):
 * side 0 = seekerAttributes, 1 = jobAttributes; names in key order, node ids
 * (the config-5 term vocabulary, link_learner.cpp:327-347) sorted, unique. */
typedef struct hyre_links hyre_links;
hyre_status hyre_links_read_json(const char* path, hyre_links** out);
void hyre_links_destroy(hyre_links* l);
uint32_t hyre_links_num_nodes(const hyre_links* l);
uint32_t hyre_links_count(const hyre_links* l, int32_t side);
const char* hyre_links_name(const hyre_links* l, int32_t side, uint32_t i);
const uint32_t* hyre_links_ids(const hyre_links* l, int32_t side, uint32_t i, uint32_t* n);

/* std::move(builder).freeze(make_codec(dim, num_bits, seed)) -- corpus.hpp:47,
 * corpus.cpp:54-129.  The builder is consumed (further calls fail). */
hyre_status hyre_builder_freeze(hyre_builder* b, uint32_t num_bits, uint64_t seed,
                                hyre_frozen** out);
/* The same freeze computed on GPU `device` (per-clause sort + dedup, double
 * L2 normalisation, signatures): bit-identical arrays and the same errors,
 * for large builds.  The builder is consumed. */
hyre_status hyre_builder_freeze_device(hyre_builder* b, uint32_t num_bits, uint64_t seed,
                                       int32_t device, hyre_frozen** out);

/* Wraps flat FrozenIndex arrays (corpus.hpp:114-123) that a caller already
 * holds -- e.g. the reference's own FrozenIndex -- without re-freezing.
 * doc_ids: NULL (ids become doc_id_prefix + row) or num_docs C strings. */
hyre_status hyre_frozen_from_arrays(uint32_t num_docs, uint32_t num_clauses,
                                    uint32_t max_num_attr, uint32_t dim, uint32_t num_bits,
                                    uint64_t seed, const uint32_t* attributes,
                                    const uint32_t* offsets, const float* embeddings,
                                    const uint64_t* signatures, const uint8_t* zero_flags,
                                    const char* const* doc_ids, const char* doc_id_prefix,
                                    hyre_frozen** out);

/* FrozenIndex::save / FrozenIndex::load -- corpus.cpp:144-201 ("HYREIDN1" v1). */
hyre_status hyre_frozen_save(const hyre_frozen* f, const char* path);
hyre_status hyre_frozen_load(const char* path, hyre_frozen** out);
void hyre_frozen_destroy(hyre_frozen* f);

typedef struct hyre_shape {
  uint32_t num_docs, num_clauses, max_num_attr, dim, num_bits, num_words;
  uint64_t seed;
} hyre_shape;
void hyre_frozen_shape(const hyre_frozen* f, hyre_shape* out);

/* Read-only views of the frozen host arrays (valid while f lives). */
const uint32_t* hyre_frozen_attributes(const hyre_frozen* f);  /* N x A */
const uint32_t* hyre_frozen_offsets(const hyre_frozen* f);     /* N x (C+1) */
const float* hyre_frozen_embeddings(const hyre_frozen* f);     /* N x d */
const uint64_t* hyre_frozen_signatures(const hyre_frozen* f);  /* N x words */
const uint8_t* hyre_frozen_zero_flags(const hyre_frozen* f);   /* N */
/* doc_id(): for rows added in bulk (prefix + row) the string is generated into
 * a thread-local buffer valid until this thread's next call; copy it. */
const char* hyre_frozen_doc_id(const hyre_frozen* f, uint32_t row);
int64_t hyre_frozen_row_of(const hyre_frozen* f, const char* doc_id);         /* row_of(), -1 */
int32_t hyre_frozen_resolve_clause_slot(const hyre_frozen* f, const char* n); /* :103 */
const char* hyre_frozen_clause_name(const hyre_frozen* f, uint32_t slot);

/* ------------------------------------------------------------------------
 * Sign-quant codec (quantizer.hpp:48-65)
 * ------------------------------------------------------------------------ */
/* encode(make_codec(dim, num_bits, seed), x) -> ceil(num_bits/64) words. */
hyre_status hyre_encode(uint32_t dim, uint32_t num_bits, uint64_t seed, const float* x,
                        uint64_t* words);
/* quant_score_words (quantizer.hpp:59-61). */
uint32_t hyre_quant_score_words(const uint64_t* a, const uint64_t* b, uint32_t num_words,
                                uint32_t num_bits);

/* ------------------------------------------------------------------------
 * Queries (term_match.hpp:14-33, pipeline.hpp:17-57)
 * ------------------------------------------------------------------------ */
/* A HybridQuery whose CnfQuery is already normalized: clause c constrains slot
 * slots[c] with ids[id_offsets[c] .. id_offsets[c+1]).  embedding == NULL is
 * a term-only query.  quant_enabled/quant_k/granularity are ExecOptions. */
typedef struct hyre_query {
  uint32_t n_clauses;
  const uint32_t* slots;
  const uint32_t* id_offsets;
  const uint32_t* ids;
  const float* embedding;
  uint32_t embedding_dim;
  uint32_t k;
  uint32_t quant_enabled;
  uint32_t quant_k;      /* 0 => 200 * k (pipeline.hpp:22-24) */
  uint32_t granularity;  /* bucket_top_k granularity G (validated, result-invariant) */
} hyre_query;

typedef struct hyre_hit {
  uint32_t row;  /* global rowId */
  float score;   /* clamp(dot(unit(q), row), -1, 1); 0 for term-only */
} hyre_hit;

/* Messenger (types.hpp:12-17): one stage record of the batch scan. */
typedef struct hyre_messenger {
  uint32_t row_id;   /* global rowId */
  uint32_t batch_id; /* the batchId stamped on the query's matches */
  float score;       /* 0 (term match only) */
} hyre_messenger;

/* StageTimings (pipeline.hpp:40-46); device stages are timed with CUDA events. */
typedef struct hyre_timings {
  double tbr_ms, quant_ms, ebr_ms, topk_ms, total_ms;
} hyre_timings;

/* normalize_query (term_match.hpp:31-33, term_match.cpp:7-30) over a raw
 * {slot: ids} map given as n_raw (slot, id list) entries.  Outputs need room
 * for n_raw clauses and all raw ids. */
hyre_status hyre_normalize_query(uint32_t n_raw, const uint32_t* raw_slots,
                                 const uint32_t* raw_offsets, const uint32_t* raw_ids,
                                 uint32_t num_clauses, uint32_t* out_n, uint32_t* out_slots,
                                 uint32_t* out_offsets, uint32_t* out_ids);

/* validate_query (pipeline.hpp:57, pipeline.cpp:44-73). */
hyre_status hyre_validate_query(const hyre_frozen* f, const hyre_query* q);

/* ------------------------------------------------------------------------
 * Device-resident index (the FrozenIndex's B200 column store)
 * ------------------------------------------------------------------------ */
typedef struct hyre_index hyre_index;

typedef struct hyre_index_options {
  int32_t device;        /* CUDA ordinal */
  uint32_t emb_dtype;    /* hyre_emb_dtype */
  uint32_t row_begin;    /* shard [row_begin, row_end) of the frozen rows; */
  uint32_t row_end;      /* row_end == 0 => all rows */
  uint32_t tensor_path;  /* 1: also store the bf16 (hi, lo) split for tcgen05 batches */
  uint32_t row_offset;   /* added to every reported row: global id of the frozen's row 0
                            (a rank that froze only its own shard of a larger corpus) */
} hyre_index_options;

typedef struct hyre_index_stats {
  uint64_t num_rows, row_base, dim, row_stride;
  uint64_t num_terms, bitmap_terms, csr_terms, postings;
  uint64_t embedding_bytes, tensor_bytes, bitmap_bytes, csr_bytes, signature_bytes, forward_bytes;
} hyre_index_stats;

/* Uploads a frozen index (or a row shard of it) into device memory: embeddings
 * row-major with a padded 16-byte-granular stride, per-term bitmaps / CSR
 * postings derived from attributes+offsets, signatures.  Replaces the
 * FrozenIndex arrays read by full_scan_tbr/exact_scores/preselect. */
hyre_status hyre_index_create(const hyre_frozen* f, const hyre_index_options* opts,
                              hyre_index** out);
void hyre_index_destroy(hyre_index* ix);
/* Learned per-row weights (the north star's link/attribute weights applied in
 * the scoring epilogue; no reference counterpart -- its score is the pure
 * cosine, knn.cpp:36-37): every returned score becomes w[row] x clamp(dot),
 * w in [0, 1], for hybrid queries (term-only scores stay 0).  w has one weight
 * per row of this index (n == its row count); w == NULL restores the
 * identity.  Must not overlap a running executor of the index. */
hyre_status hyre_index_set_row_weights(hyre_index* ix, const float* w, uint64_t n);
hyre_status hyre_index_stats_get(const hyre_index* ix, hyre_index_stats* out);

/* ------------------------------------------------------------------------
 * Executor (pipeline.hpp:69-96)
 * ------------------------------------------------------------------------ */
typedef struct hyre_executor hyre_executor;

/* Executor(index, max_batch): owns a CUDA stream and all device scratch,
 * sized once here (pipeline.cpp:95-106). */
hyre_status hyre_executor_create(hyre_index* ix, uint32_t max_batch, hyre_executor** out);
void hyre_executor_destroy(hyre_executor* ex);
void* hyre_executor_stream(hyre_executor* ex); /* cudaStream_t */

/* Executor::execute (pipeline.cpp:108-145).  hits needs min(k, num_docs)
 * entries; *n_hits receives the hit count. */
hyre_status hyre_execute(hyre_executor* ex, const hyre_query* q, hyre_hit* hits,
                         uint32_t* n_hits, hyre_timings* timings);

/* Executor::execute_batch (pipeline.cpp:147-281).  Hits of slot i are written
 * at hits + hit_offsets[i] (caller-chosen, room for min(k_i, num_docs)).
 * statuses[i] = HYRE_OK or HYRE_INVALID_ARGUMENT (message via
 * hyre_executor_slot_error); empty batch / b > max_batch fail the call. */
hyre_status hyre_execute_batch(hyre_executor* ex, const hyre_query* qs, uint32_t b,
                               hyre_hit* hits, const uint64_t* hit_offsets, uint32_t* counts,
                               int32_t* statuses, hyre_timings* timings);
const char* hyre_executor_slot_error(const hyre_executor* ex, uint32_t slot);

/* Split form of execute_batch for device-resident timing: prepare validates
 * and uploads the batch, run enqueues the kernels on the executor stream
 * without any host synchronisation, fetch synchronises and copies results
 * out (same layout as hyre_execute_batch).  run may be repeated. */
hyre_status hyre_batch_prepare(hyre_executor* ex, const hyre_query* qs, uint32_t b);
hyre_status hyre_batch_run(hyre_executor* ex);
/* Waits for the last run and resolves any pending recovery round (a query
 * whose estimated threshold admitted too few rows or whose candidate buffer
 * overflowed), so the device results are final: call before reading them on
 * the device (hyre_batch_device_results, the multi-GPU gather).  fetch does
 * this itself. */
hyre_status hyre_batch_settle(hyre_executor* ex);
hyre_status hyre_batch_fetch(hyre_executor* ex, hyre_hit* hits, const uint64_t* hit_offsets,
                             uint32_t* counts, int32_t* statuses, hyre_timings* timings);
/* Number of kernels the last hyre_batch_run enqueued. */
uint32_t hyre_batch_kernel_count(const hyre_executor* ex);
/* Kernel path of the prepared batch (bit flags): 1 tensor-core scorer (K3),
 * 2 CNF fused into K3 (no mask pass), 4 forward-list mask (K1b), 8 sample
 * pass + threshold.  Diagnostics for benchmarks and tests. */
#define HYRE_PATH_TC 1u
#define HYRE_PATH_FUSED 2u
#define HYRE_PATH_FWD_MASK 4u
#define HYRE_PATH_SAMPLED 8u
#define HYRE_PATH_MATCH_ALL 16u /* tensor-core batch of match-all queries: no eligibility pass */
#define HYRE_PATH_I8 32u        /* the main pass streams the int8 prefilter plane (exact rescoring of survivors) */
#define HYRE_PATH_SMALL 64u     /* small index: one exact scoring launch (K7) + the top-K select, no sampling */
uint32_t hyre_batch_path(const hyre_executor* ex);
/* K3 kernel variant of the prepared batch (diagnostics for tests that must
 * run a given instantiation): out4 = {J compact CNF ids per row (0 = not
 * fused), bytes per id (1 = u8, 2 = u16), query chunks per CNF thread,
 * queries per MMA group (Np)}; all zero when the batch runs on K2. */
void hyre_batch_tc_variant(const hyre_executor* ex, uint32_t* out4);
/* Fused CNF row layout of the prepared batch: W > 0 = slot-grouped rows (W ids
 * per slot group, no masks), 0 = segmented rows + masks (or not fused). */
uint32_t hyre_batch_cnf_group(const hyre_executor* ex);
/* Eligible-row counts of the last run (u32[b], waits for it): the CNF
 * matches per query; 0xFFFFFFFF where the CNF ran fused inside K3 (the count
 * is never materialised there).  Diagnostics for benchmarks and tests. */
hyre_status hyre_batch_eligible(hyre_executor* ex, uint32_t* out);
/* Algorithmic bytes of the prepared batch's eligibility inputs: distinct
 * term bitmaps + CSR postings (K1), or the forward term lists once per pass
 * (K1b / fused K3). */
uint64_t hyre_batch_term_bytes(const hyre_executor* ex);
/* Algorithmic bytes the prepared batch's K3 main stage reads (all query
 * groups): the embedding planes it streams (bf16 hi for the prefilter or a
 * bf16 index, hi + lo otherwise) + the eligibility input (compact CNF rows
 * when fused, else the K1 mask words); 0 when the batch runs on K2. */
uint64_t hyre_batch_scan_bytes(const hyre_executor* ex);
/* CUDA-event durations (ms) of the last run, waiting for it to finish:
 * [0] K1 mask (+CSR scatter) [1] K6 quant [2] sample pass + K-th select
 * [3] main scorer (K2/K3) [4] final select + first-K [5] whole run. */
hyre_status hyre_batch_stage_ms(hyre_executor* ex, float* out6);
/* The same for the run `back` runs before the last (0 = last; the executor
 * keeps the events of its last 64 runs), so a benchmark can read per-kernel
 * times of every step of a back-to-back timed region afterwards. */
hyre_status hyre_batch_stage_ms_hist(hyre_executor* ex, uint32_t back, float* out6);
/* Record the inner stage boundaries [1]-[4] (default on).  Off, a run records
 * only its start and end events: a stream event between two kernels ends the
 * programmatic-dependent-launch overlap of the second kernel's prologue with
 * the first one's tail, so throughput runs switch them off and the stage
 * durations then read 0 (the whole-run time [5] stays). */
hyre_status hyre_batch_set_stage_events(hyre_executor* ex, int on);
/* Device pointers of the last run's results (for on-device multi-GPU
 * gathers): hits (hyre_hit[*n_hits]), per-slot hit offsets (u64[b]) and
 * per-slot counts (u32[b]).  Valid until the next prepare. */
hyre_status hyre_batch_device_results(hyre_executor* ex, void** hits, uint64_t* n_hits, void** offsets,
                                      void** counts);
/* Recovery work the last batch needed once settled (fetch / settle):
 * out2 = {threshold recovery rounds, queries answered by the exhaustive exact
 * path (hybrid k > 4096, or a recovery that did not converge)}.  A benchmark
 * timing hyre_batch_run alone asserts both are 0. */
hyre_status hyre_batch_recovery(const hyre_executor* ex, uint32_t* out2);
/* Bytes the last prepare copied host->device and the last fetch copied back. */
hyre_status hyre_batch_io_bytes(const hyre_executor* ex, uint64_t* h2d, uint64_t* d2h);
/* ------------------------------------------------------------------------
 * Row-sharded executor over several GPUs (the multi-GPU
 * form of FrozenIndex + Executor, pipeline.hpp:69-96).  The frozen rows are
 * split into n_shards contiguous ranges; shard g lives on devices[g]
 * (nullable: device g % device count; several shards may share a device)
 * with its own Executor and stream.  Per-shard top-K lists are merged exactly
 * on shard 0's device by one kernel that reads every shard's hits through
 * peer memory (NVLink), term-only lists are concatenated in row order, and
 * the quant pre-selection is global (shards exchange histograms and tie
 * counts the same way), so results equal the unsharded executor's.  Peer
 * access between the devices is required.  Single-in-flight like Executor.
 * ------------------------------------------------------------------------ */
typedef struct hyre_sharded_index hyre_sharded_index;
typedef struct hyre_sharded_index_options {
  uint32_t n_shards;       /* G, 1 .. 16 */
  const int32_t* devices;  /* [n_shards] CUDA ordinals, or NULL */
  uint32_t emb_dtype;      /* hyre_emb_dtype */
  uint32_t tensor_path;    /* as hyre_index_options */
} hyre_sharded_index_options;
/* The device shards of a frozen index (enables peer access between their
 * devices); shared by every sharded executor created over it. */
hyre_status hyre_sharded_index_create(const hyre_frozen* f, const hyre_sharded_index_options* opts,
                                      hyre_sharded_index** out);
void hyre_sharded_index_destroy(hyre_sharded_index* ix);
/* hyre_index_set_row_weights over every shard: w covers all rows (global order). */
hyre_status hyre_sharded_index_set_row_weights(hyre_sharded_index* ix, const float* w, uint64_t n);
/* shard count and each shard's device (devices may be NULL) */
hyre_status hyre_sharded_index_info(const hyre_sharded_index* ix, uint32_t* n_shards, int32_t* devices);

typedef struct hyre_sharded hyre_sharded;
/* Executor(index, max_batch) over the shards: one Executor + stream per shard. */
hyre_status hyre_sharded_create(hyre_sharded_index* ix, uint32_t max_batch, hyre_sharded** out);
void hyre_sharded_destroy(hyre_sharded* s);
/* Executor::execute_batch over all shards (same contract as hyre_execute_batch). */
hyre_status hyre_sharded_execute_batch(hyre_sharded* s, const hyre_query* qs, uint32_t b, hyre_hit* hits,
                                       const uint64_t* hit_offsets, uint32_t* counts, int32_t* statuses,
                                       hyre_timings* timings);
const char* hyre_sharded_slot_error(const hyre_sharded* s, uint32_t slot);
/* Split form for device-resident timing (as hyre_batch_prepare/run/settle/
 * fetch): run enqueues every shard and the root merge without host
 * synchronisation; the root stream's work completes after all of it. */
hyre_status hyre_sharded_prepare(hyre_sharded* s, const hyre_query* qs, uint32_t b);
hyre_status hyre_sharded_run(hyre_sharded* s);
hyre_status hyre_sharded_settle(hyre_sharded* s);
hyre_status hyre_sharded_fetch(hyre_sharded* s, hyre_hit* hits, const uint64_t* hit_offsets, uint32_t* counts,
                               int32_t* statuses, hyre_timings* timings);
void* hyre_sharded_stream(const hyre_sharded* s); /* root stream (cudaStream_t) */
uint32_t hyre_sharded_kernel_count(const hyre_sharded* s);
/* out2 = {recovery rounds, exhaustive queries} summed over shards (after settle/fetch) */
hyre_status hyre_sharded_recovery(const hyre_sharded* s, uint32_t* out2);

/* ------------------------------------------------------------------------
 * Executor pool with dynamic request batching: the replacement for
 * SearchService::ExecutorPool (service.cpp:99-141; ServiceConfig{workers,
 * max_batch} service.hpp:19-26).  `workers` executors (own CUDA streams);
 * concurrent hyre_pool_search calls are grouped into batches of up to
 * max_batch queries, waiting at most max_wait_us after the first arrives.
 * hyre_pool_search is thread-safe and blocking; its result (or validation
 * error, thread-local hyre_last_error) is that of hyre_execute for the query.
 * ------------------------------------------------------------------------ */
typedef struct hyre_pool hyre_pool;
hyre_status hyre_pool_create(hyre_index* ix, uint32_t workers, uint32_t max_batch, uint32_t max_wait_us,
                             hyre_pool** out);
void hyre_pool_destroy(hyre_pool* p);
hyre_status hyre_pool_search(hyre_pool* p, const hyre_query* q, hyre_hit* hits, uint32_t* n_hits);
/* Batches run and queries served so far (queries / batches = mean batch size). */
hyre_status hyre_pool_stats(const hyre_pool* p, uint64_t* batches, uint64_t* queries);

/* Exact on-device merge of G shard result sets gathered from the executors of
 * every shard (same batch): g_hits [G][hits_stride] hyre_hit, g_offsets [G][b]
 * u64 and g_counts [G][b] u32 (the hyre_batch_device_results layouts).  The
 * merged top-K replaces this executor's results; fetch them as usual. */
hyre_status hyre_batch_merge_gathered(hyre_executor* ex, const void* g_hits, const void* g_offsets,
                                      const void* g_counts, uint32_t n_lists, uint64_t hits_stride);
/* The same over one packed record per shard (a single all-gather): record g at
 * g x record_words u32 words holds the shard's hits (hits_words u32 words,
 * even), then b u64 hit offsets, then b u32 counts. */
hyre_status hyre_batch_merge_packed(hyre_executor* ex, const void* g_records, uint32_t n_lists,
                                    uint64_t record_words, uint64_t hits_words);

/* Stage entry points (public in the reference and used by its tests). */
/* full_scan_tbr (term_match.hpp:43-45): ascending eligible rows (global ids). */
hyre_status hyre_full_scan_tbr(hyre_executor* ex, const hyre_query* q, uint32_t* rows,
                               uint64_t cap, uint64_t* n);
/* batch_scan_tbr (pipeline.hpp:59-64, pipeline.cpp:75-93): one pass over the
 * rows for b <= max_batch queries (clauses only; embeddings ignored), emitting
 * a messenger per (row, query) match ordered by (rowId, query position) and
 * stamped with batch_ids[i].  Writes min(n, cap) messengers, *n = total. */
hyre_status hyre_batch_scan_tbr(hyre_executor* ex, const hyre_query* qs, uint32_t b,
                                const uint32_t* batch_ids, hyre_messenger* out, uint64_t cap,
                                uint64_t* n);
/* exact_scores (knn.hpp:24-26) over explicit global rows. */
hyre_status hyre_exact_scores(hyre_executor* ex, const float* q, uint32_t dim,
                              const uint32_t* rows, uint64_t n, float* scores,
                              int32_t* renormalized);
/* bucket_top_k (knn.hpp:33-35) over explicit (row, score) messengers. */
hyre_status hyre_bucket_top_k(hyre_executor* ex, const uint32_t* rows, const float* scores,
                              uint64_t n, uint32_t k, uint32_t granularity, hyre_hit* out,
                              uint32_t* n_out);
/* preselect (quantizer.hpp:71-74) over explicit global rows (ascending). */
hyre_status hyre_preselect(hyre_executor* ex, const uint64_t* query_words, const uint32_t* rows,
                           uint64_t n, uint32_t quant_k, uint32_t* rows_out, uint64_t* n_out);

/* Exact merge of per-shard top-K lists (multi-GPU): lists[i] has
 * counts[i] hits sorted by (score desc, row asc); writes min(k, total). */
hyre_status hyre_merge_topk(const hyre_hit* const* lists, const uint32_t* counts, uint32_t n_lists,
                            uint32_t k, hyre_hit* out, uint32_t* n_out);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#endif  /* HYRE_B200_H_ */
