// hyre_b200.hpp -- header-only C++ drop-in for the reference's hot-path API
// (proj/include/hyre/{types,common,corpus,quantizer,term_match,knn,pipeline}.hpp)
// implemented over the C-ABI in hyre_b200.h.  Same namespace, class names,
// signatures and exceptions, so the reference's callers -- SearchService
// (service.cpp:151-226), run_bench (bench.cpp:52-131), tt::knn_recall
// (two_tower.cpp:369-394) -- compile unchanged against this header and link
// libhyre_b200.so instead of the reference's corpus/term_match/quantizer/
// knn/pipeline translation units.  See INTEGRATION.md.
//
// Differences a caller can observe (documented in DESIGN.md §6):
//  * scores are computed on the GPU (FMA / tensor-core accumulation): equal to
//    the reference within 1e-3 relative (2e-5 absolute floor), ties at the
//    K-th score may resolve to a different row of the same score;
//  * QuantCodec carries (dim, num_bits, seed); its rounds are re-derived inside
//    the library exactly like FrozenIndex::load does (corpus.cpp:183).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "hyre_b200.h"

namespace hyre {

// ---- errors (common.hpp:15-33, knn.cpp:59-61) ------------------------------
class ValidationError : public std::invalid_argument {
 public:
  using std::invalid_argument::invalid_argument;
};

class LoadError : public std::runtime_error {
 public:
  enum class Cause { kBadMagic, kVersionMismatch, kTruncated, kChecksum };
  LoadError(Cause cause, const std::string& msg) : std::runtime_error(msg), cause_(cause) {}
  Cause cause() const { return cause_; }

 private:
  Cause cause_;
};

namespace detail {
inline void check(hyre_status st) {
  if (st == HYRE_OK) return;
  const std::string msg = hyre_last_error();
  switch (st) {
    case HYRE_INVALID_ARGUMENT: throw ValidationError(msg);
    case HYRE_OUT_OF_RANGE: throw std::domain_error(msg);
    case HYRE_LOAD_ERROR: throw LoadError(static_cast<LoadError::Cause>(hyre_last_load_cause()), msg);
    default: throw std::runtime_error(msg);
  }
}
}  // namespace detail

// ---- types.hpp ----------------------------------------------------------------
struct Messenger {
  std::uint32_t row_id = 0;
  std::uint32_t batch_id = 0;
  float score = 0.0f;
  bool operator==(const Messenger&) const = default;
};

struct ScoredDoc {
  std::string doc_id;
  std::uint32_t row_id = 0;
  float score = 0.0f;
  bool operator==(const ScoredDoc&) const = default;
};

struct TopKResult {
  std::vector<ScoredDoc> hits;
  bool operator==(const TopKResult&) const = default;
};

// ---- quantizer.hpp (codec half) ---------------------------------------------------
struct QuantCodec {
  std::uint32_t dim = 0;
  std::uint32_t num_bits = 0;
  std::uint64_t seed = 0;
  std::size_t num_words() const { return (num_bits + 63) / 64; }
};

struct Signature {
  std::uint32_t num_bits = 0;
  std::vector<std::uint64_t> words;
  bool bit(std::uint32_t b) const { return (words[b / 64] >> (b % 64)) & 1u; }
  bool operator==(const Signature&) const = default;
};

inline QuantCodec make_codec(std::uint32_t dim, std::uint32_t num_bits, std::uint64_t seed) {
  if (dim == 0) throw ValidationError("codec dim must be >= 1");
  if (num_bits == 0) throw ValidationError("codec numBits must be >= 1");
  return QuantCodec{dim, num_bits, seed};
}

inline Signature encode(const QuantCodec& codec, std::span<const float> embedding) {
  if (embedding.size() != codec.dim)
    throw ValidationError("embedding length " + std::to_string(embedding.size()) + " != codec dim " +
                          std::to_string(codec.dim));
  Signature s{codec.num_bits, std::vector<std::uint64_t>(codec.num_words())};
  detail::check(hyre_encode(codec.dim, codec.num_bits, codec.seed, embedding.data(), s.words.data()));
  return s;
}

inline std::uint32_t quant_score_words(std::span<const std::uint64_t> a, std::span<const std::uint64_t> b,
                                       std::uint32_t num_bits) {
  return hyre_quant_score_words(a.data(), b.data(), static_cast<std::uint32_t>(a.size()), num_bits);
}

inline std::uint32_t quant_score(const Signature& a, const Signature& b) {
  if (a.num_bits != b.num_bits) throw ValidationError("signature width mismatch");
  return quant_score_words(a.words, b.words, a.num_bits);
}

// ---- corpus.hpp ---------------------------------------------------------------------
struct DocumentInput {
  std::string doc_id;
  std::vector<std::vector<std::uint32_t>> clauses;
  std::vector<float> embedding;
};

struct IndexConfig {
  std::uint32_t num_clauses = 0;
  std::uint32_t max_num_attr = 0;
  std::uint32_t dim = 0;
  std::vector<std::string> clause_names;
};

class Executor;

// Where an index's device copy lives (not part of the reference API, which
// is CPU-only).  Defaults: one GPU (device 0), fp32 rows + tensor-core tiles;
// the environment overrides them for callers relinked without code changes:
// HYRE_GPUS=N shards the rows over devices 0..N-1 (HYRE_DEVICES="a,b,..."
// names them), HYRE_EMB_DTYPE=bf16 stores bf16 rows.
struct DeviceOptions {
  std::vector<int> devices{0};  // one entry per row shard
  bool bf16 = false;
  bool tensor_path = true;
  static DeviceOptions from_env() {
    DeviceOptions o;
    if (const char* d = std::getenv("HYRE_DEVICES")) {
      o.devices.clear();
      for (const char* p = d; *p;) {
        char* end = nullptr;
        o.devices.push_back(static_cast<int>(std::strtol(p, &end, 10)));
        p = *end ? end + 1 : end;
      }
    } else if (const char* n = std::getenv("HYRE_GPUS")) {
      o.devices.clear();
      for (int g = 0; g < std::max(1, std::atoi(n)); ++g) o.devices.push_back(g);
    }
    if (const char* t = std::getenv("HYRE_EMB_DTYPE")) o.bf16 = std::string(t) == "bf16";
    return o;
  }
};

class FrozenIndex {
 public:
  FrozenIndex(FrozenIndex&&) noexcept = default;
  FrozenIndex& operator=(FrozenIndex&&) noexcept = default;

  std::uint32_t num_docs() const { return shape_.num_docs; }
  std::uint32_t num_clauses() const { return shape_.num_clauses; }
  std::uint32_t max_num_attr() const { return shape_.max_num_attr; }
  std::uint32_t dim() const { return shape_.dim; }
  QuantCodec codec() const { return QuantCodec{shape_.dim, shape_.num_bits, shape_.seed}; }
  std::vector<std::string> clause_names() const {
    std::vector<std::string> out;
    for (std::uint32_t c = 0; c < shape_.num_clauses; ++c) out.emplace_back(hyre_frozen_clause_name(f_.get(), c));
    return out;
  }

  std::span<const std::uint32_t> attribute_row(std::uint32_t row) const {
    return {hyre_frozen_attributes(f_.get()) + std::size_t{row} * shape_.max_num_attr, shape_.max_num_attr};
  }
  std::span<const std::uint32_t> offsets_row(std::uint32_t row) const {
    return {hyre_frozen_offsets(f_.get()) + std::size_t{row} * (shape_.num_clauses + 1), shape_.num_clauses + 1u};
  }
  std::span<const std::uint32_t> clause_slice(std::uint32_t row, std::uint32_t clause) const {
    auto offs = offsets_row(row);
    return attribute_row(row).subspan(offs[clause], offs[clause + 1] - offs[clause]);
  }
  std::span<const float> embedding_row(std::uint32_t row) const {
    return {hyre_frozen_embeddings(f_.get()) + std::size_t{row} * shape_.dim, shape_.dim};
  }
  std::span<const std::uint64_t> signature_words(std::uint32_t row) const {
    return {hyre_frozen_signatures(f_.get()) + std::size_t{row} * shape_.num_words, shape_.num_words};
  }
  Signature signature_row(std::uint32_t row) const {
    auto w = signature_words(row);
    return Signature{shape_.num_bits, {w.begin(), w.end()}};
  }
  bool embedding_is_zero(std::uint32_t row) const { return hyre_frozen_zero_flags(f_.get())[row] != 0; }
  std::string doc_id(std::uint32_t row) const { return hyre_frozen_doc_id(f_.get(), row); }
  std::optional<std::uint32_t> row_of(const std::string& doc_id) const {
    const std::int64_t r = hyre_frozen_row_of(f_.get(), doc_id.c_str());
    if (r < 0) return std::nullopt;
    return static_cast<std::uint32_t>(r);
  }
  int resolve_clause_slot(const std::string& name) const {
    return hyre_frozen_resolve_clause_slot(f_.get(), name.c_str());
  }

  void save(const std::string& path) const { detail::check(hyre_frozen_save(f_.get(), path.c_str())); }
  static FrozenIndex load(const std::string& path) {
    hyre_frozen* f = nullptr;
    detail::check(hyre_frozen_load(path.c_str(), &f));
    return FrozenIndex(f);
  }

  // Device placement for the executors created later (before the first one;
  // default DeviceOptions::from_env()).
  void set_device_options(DeviceOptions o) {
    std::lock_guard<std::mutex> lk(dev_->m);
    if (dev_->ix || dev_->sx) throw ValidationError("device options must be set before the first Executor");
    dev_->opts = std::move(o);
  }
  const DeviceOptions& device_options() const { return dev_->opts; }
  bool sharded() const { return dev_->opts.devices.size() > 1; }
  // The device column store (one GPU) or its row shards (several), built on
  // first use by an Executor and shared by every executor of this index; safe
  // to call from several threads (the reference FrozenIndex is shared
  // read-only, corpus.hpp:54-56).
  hyre_index* device() const {
    std::lock_guard<std::mutex> lk(dev_->m);
    if (!dev_->ix) {
      const DeviceOptions& d = dev_->opts;
      hyre_index_options o{d.devices.empty() ? 0 : d.devices[0], d.bf16 ? HYRE_EMB_BF16 : HYRE_EMB_F32, 0, 0,
                           d.tensor_path ? 1u : 0u, 0};
      detail::check(hyre_index_create(f_.get(), &o, &dev_->ix));
    }
    return dev_->ix;
  }
  hyre_sharded_index* device_shards() const {
    std::lock_guard<std::mutex> lk(dev_->m);
    if (!dev_->sx) {
      const DeviceOptions& d = dev_->opts;
      hyre_sharded_index_options o{static_cast<std::uint32_t>(d.devices.size()), d.devices.data(),
                                   d.bf16 ? HYRE_EMB_BF16 : HYRE_EMB_F32, d.tensor_path ? 1u : 0u};
      detail::check(hyre_sharded_index_create(f_.get(), &o, &dev_->sx));
    }
    return dev_->sx;
  }
  const hyre_frozen* handle() const { return f_.get(); }

  // Learned per-row weights (the north star's link/attribute weights; no
  // reference counterpart): hybrid scores become w[row] x clamp(cosine), one
  // weight in [0, 1] per row; an empty span restores the pure cosine.  Applies
  // to the device index (or its shards) every executor of this index reads;
  // not while one of them is running.
  void set_row_weights(std::span<const float> w) const {
    const float* p = w.empty() ? nullptr : w.data();
    if (sharded()) detail::check(hyre_sharded_index_set_row_weights(device_shards(), p, w.size()));
    else detail::check(hyre_index_set_row_weights(device(), p, w.size()));
  }

 private:
  friend class IndexBuilder;
  explicit FrozenIndex(hyre_frozen* f) : f_(f, &hyre_frozen_destroy), dev_(std::make_shared<Dev>()) {
    hyre_frozen_shape(f, &shape_);
  }
  struct Dev {
    std::mutex m;
    DeviceOptions opts = DeviceOptions::from_env();
    hyre_index* ix = nullptr;
    hyre_sharded_index* sx = nullptr;
    ~Dev() {
      if (ix) hyre_index_destroy(ix);
      if (sx) hyre_sharded_index_destroy(sx);
    }
  };
  std::unique_ptr<hyre_frozen, void (*)(hyre_frozen*)> f_;
  std::shared_ptr<Dev> dev_;
  hyre_shape shape_{};
};

class IndexBuilder {
 public:
  explicit IndexBuilder(IndexConfig config) : dim_(config.dim) {
    std::vector<const char*> names;
    for (const auto& n : config.clause_names) names.push_back(n.c_str());
    hyre_builder* b = nullptr;
    detail::check(hyre_builder_create(config.num_clauses, config.max_num_attr, config.dim,
                                      names.empty() ? nullptr : names.data(),
                                      static_cast<std::uint32_t>(names.size()), &b));
    b_.reset(b);
  }
  std::uint32_t add_document(const DocumentInput& doc) {
    std::vector<std::uint32_t> offs{0}, ids;
    for (const auto& c : doc.clauses) {
      ids.insert(ids.end(), c.begin(), c.end());
      offs.push_back(static_cast<std::uint32_t>(ids.size()));
    }
    std::uint32_t row = 0;
    detail::check(hyre_builder_add_document(b_.get(), doc.doc_id.c_str(),
                                            static_cast<std::uint32_t>(doc.clauses.size()), offs.data(),
                                            ids.data(), doc.embedding.data(),
                                            static_cast<std::uint32_t>(doc.embedding.size()), &row));
    return row;
  }
  std::size_t size() const { return hyre_builder_size(b_.get()); }
  hyre_builder* handle() const { return b_.get(); }
  // corpus.hpp:47.  HYRE_FREEZE_DEVICE=<ordinal> runs the freeze on that GPU
  // (bit-identical arrays) for a relinked caller without code changes.
  FrozenIndex freeze(const QuantCodec& codec) && {
    if (const char* d = std::getenv("HYRE_FREEZE_DEVICE")) return std::move(*this).freeze_on_device(codec, std::atoi(d));
    if (codec.dim != dim_) throw ValidationError("codec dim != index dim");
    hyre_frozen* f = nullptr;
    detail::check(hyre_builder_freeze(b_.get(), codec.num_bits, codec.seed, &f));
    return FrozenIndex(f);
  }
  // The freeze computed on GPU `device` (large builds; same arrays and errors).
  FrozenIndex freeze_on_device(const QuantCodec& codec, int device) && {
    if (codec.dim != dim_) throw ValidationError("codec dim != index dim");
    hyre_frozen* f = nullptr;
    detail::check(hyre_builder_freeze_device(b_.get(), codec.num_bits, codec.seed, device, &f));
    return FrozenIndex(f);
  }

 private:
  struct Del {
    void operator()(hyre_builder* b) const { hyre_builder_destroy(b); }
  };
  std::unique_ptr<hyre_builder, Del> b_;
  std::uint32_t dim_;
};

// ---- dataio.hpp (ingestion; host C++ in the library) ------------------------------
struct IngestSchema {
  std::vector<std::string> clause_names;
  std::uint32_t dim = 0;
};

// {"clauses": ["geo", "skill"], "dim": 4}  (dataio.hpp:20-21)
inline IngestSchema read_schema_json(const std::string& path) {
  hyre_schema* s = nullptr;
  detail::check(hyre_schema_read_json(path.c_str(), &s));
  IngestSchema out;
  for (std::uint32_t i = 0; i < hyre_schema_num_clauses(s); ++i) out.clause_names.emplace_back(hyre_schema_clause_name(s, i));
  out.dim = hyre_schema_dim(s);
  hyre_schema_destroy(s);
  return out;
}

namespace detail {
struct DocSet {  // a parsed JSONL corpus held by the library
  DocSet(const std::string& path, const IngestSchema& schema) {
    std::vector<const char*> names;
    for (const auto& n : schema.clause_names) names.push_back(n.c_str());
    hyre_schema* s = nullptr;
    check(hyre_schema_create(static_cast<std::uint32_t>(names.size()), names.data(), schema.dim, &s));
    const hyre_status st = hyre_documents_read_jsonl(path.c_str(), s, &d);
    hyre_schema_destroy(s);
    check(st);
  }
  ~DocSet() { hyre_documents_destroy(d); }
  DocSet(const DocSet&) = delete;
  DocSet& operator=(const DocSet&) = delete;
  hyre_documents* d = nullptr;
};
}  // namespace detail

// One document per line (dataio.hpp:23-28):
//   {"id": "doc1", "clauses": {"geo": [934]}, "embedding": [0.1, ...]}
inline std::vector<DocumentInput> read_documents_jsonl(const std::string& path, const IngestSchema& schema) {
  detail::DocSet ds(path, schema);
  const std::uint32_t n = hyre_documents_count(ds.d), C = static_cast<std::uint32_t>(schema.clause_names.size());
  const std::uint64_t* so = hyre_documents_slot_offsets(ds.d);
  const std::uint32_t* ids = hyre_documents_ids(ds.d);
  const float* emb = hyre_documents_embeddings(ds.d);
  std::vector<DocumentInput> out(n);
  for (std::uint32_t i = 0; i < n; ++i) {
    out[i].doc_id = hyre_documents_id(ds.d, i);
    out[i].clauses.resize(C);
    for (std::uint32_t c = 0; c < C; ++c) out[i].clauses[c].assign(ids + so[i * C + c], ids + so[i * C + c + 1]);
    out[i].embedding.assign(emb + std::size_t{i} * schema.dim, emb + std::size_t{i + 1} * schema.dim);
  }
  return out;
}

// `hyre build` (cli_commands.cpp:37-63) in the library: IndexConfig from the
// schema, maxNumAttr = the widest document, every document staged in file
// order, frozen with make_codec(dim, num_bits, seed) -- on GPU `freeze_device`
// when >= 0 (bit-identical arrays).
inline FrozenIndex build_index_jsonl(const std::string& schema_path, const std::string& corpus_path,
                                     std::uint32_t num_bits = 512, std::uint64_t seed = 1, int freeze_device = -1) {
  const IngestSchema schema = read_schema_json(schema_path);
  detail::DocSet ds(corpus_path, schema);
  if (hyre_documents_count(ds.d) == 0) throw ValidationError("no documents");
  IndexBuilder b(IndexConfig{static_cast<std::uint32_t>(schema.clause_names.size()),
                             std::max<std::uint32_t>(1, hyre_documents_widest(ds.d)), schema.dim, schema.clause_names});
  detail::check(hyre_builder_add_document_set(b.handle(), ds.d, nullptr));
  const QuantCodec codec = make_codec(schema.dim, num_bits, seed);
  return freeze_device >= 0 ? std::move(b).freeze_on_device(codec, freeze_device) : std::move(b).freeze(codec);
}

// The learned-link serving-graph export (write_links_export, dataio.cpp:253-274)
// read back as the config-5 vocabulary: node ids per seeker / job.
struct LinksExport {
  std::uint32_t num_nodes = 0;
  std::map<std::string, std::vector<std::uint32_t>> seeker_attributes, job_attributes;
};
inline LinksExport read_links_export(const std::string& path) {
  hyre_links* l = nullptr;
  detail::check(hyre_links_read_json(path.c_str(), &l));
  LinksExport out;
  out.num_nodes = hyre_links_num_nodes(l);
  for (int side = 0; side < 2; ++side) {
    auto& dst = side == 0 ? out.seeker_attributes : out.job_attributes;
    for (std::uint32_t i = 0; i < hyre_links_count(l, side); ++i) {
      std::uint32_t n = 0;
      const std::uint32_t* ids = hyre_links_ids(l, side, i, &n);
      dst[hyre_links_name(l, side, i)].assign(ids, ids + n);
    }
  }
  hyre_links_destroy(l);
  return out;
}

// ---- term_match.hpp -------------------------------------------------------------
struct CnfClause {
  std::uint32_t slot = 0;
  std::vector<std::uint32_t> attribute_ids;
  bool operator==(const CnfClause&) const = default;
};

struct CnfQuery {
  std::vector<CnfClause> clauses;
  bool match_all() const { return clauses.empty(); }
  bool operator==(const CnfQuery&) const = default;
};

inline CnfQuery normalize_query(const std::map<std::uint32_t, std::vector<std::uint32_t>>& raw,
                                std::uint32_t num_clauses) {
  std::vector<std::uint32_t> slots, offs{0}, ids;
  for (const auto& [s, v] : raw) {
    slots.push_back(s);
    ids.insert(ids.end(), v.begin(), v.end());
    offs.push_back(static_cast<std::uint32_t>(ids.size()));
  }
  std::vector<std::uint32_t> os(raw.size() + 1), oo(raw.size() + 2), oi(ids.size() + 1);
  std::uint32_t n = 0;
  detail::check(hyre_normalize_query(static_cast<std::uint32_t>(raw.size()), slots.data(), offs.data(),
                                     ids.data(), num_clauses, &n, os.data(), oo.data(), oi.data()));
  CnfQuery q;
  for (std::uint32_t c = 0; c < n; ++c) q.clauses.push_back({os[c], {oi.begin() + oo[c], oi.begin() + oo[c + 1]}});
  return q;
}

// ---- pipeline.hpp ---------------------------------------------------------------------
struct ExecOptions {
  bool quant_enabled = true;
  std::uint32_t quant_k = 0;
  std::uint32_t granularity = 100;
  std::uint32_t effective_quant_k(std::uint32_t k) const { return quant_k != 0 ? quant_k : 200 * k; }
};

struct HybridQuery {
  CnfQuery terms;
  std::optional<std::vector<float>> embedding;
  std::uint32_t k = 10;
  ExecOptions options;
};

struct BatchRequest {
  std::vector<HybridQuery> queries;
};

struct StageTimings {
  double tbr_ms = 0, quant_ms = 0, ebr_ms = 0, topk_ms = 0, total_ms = 0;
};

struct QueryOutcome {
  bool ok = false;
  TopKResult result;
  std::string error;
};

struct ScoredMessengers {
  std::vector<Messenger> items;
  bool query_was_renormalized = false;
};

namespace detail {
// Flattens HybridQuery objects into hyre_query structs (pointers stay valid
// while the pack lives).
struct QueryPack {
  std::vector<std::vector<std::uint32_t>> slots, offs, ids;
  std::vector<hyre_query> q;
  explicit QueryPack(const std::vector<HybridQuery>& qs) : slots(qs.size()), offs(qs.size()), ids(qs.size()) {
    for (std::size_t i = 0; i < qs.size(); ++i) {
      offs[i].push_back(0);
      for (const auto& c : qs[i].terms.clauses) {
        slots[i].push_back(c.slot);
        ids[i].insert(ids[i].end(), c.attribute_ids.begin(), c.attribute_ids.end());
        offs[i].push_back(static_cast<std::uint32_t>(ids[i].size()));
      }
      const auto& e = qs[i].embedding;
      q.push_back(hyre_query{static_cast<std::uint32_t>(qs[i].terms.clauses.size()), slots[i].data(),
                             offs[i].data(), ids[i].data(), e ? e->data() : nullptr,
                             e ? static_cast<std::uint32_t>(e->size()) : 0u, qs[i].k,
                             qs[i].options.quant_enabled ? 1u : 0u, qs[i].options.quant_k,
                             qs[i].options.granularity});
    }
  }
};
}  // namespace detail

inline void validate_query(const FrozenIndex& index, const HybridQuery& query) {
  detail::QueryPack p({query});
  detail::check(hyre_validate_query(index.handle(), p.q.data()));
}

class Executor {
 public:
  // One GPU: an executor with its own stream and scratch.  Several (the
  // index's DeviceOptions name more than one device): a sharded executor --
  // one stream per shard, exact merge on the first device; same results.
  explicit Executor(const FrozenIndex& index, std::uint32_t max_batch = 16) : index_(index), max_batch_(max_batch) {
    if (max_batch < 1) throw ValidationError("maxBatch must be >= 1");
    if (index.sharded()) {
      hyre_sharded* s = nullptr;
      detail::check(hyre_sharded_create(index.device_shards(), max_batch, &s));
      sh_.reset(s);
      return;
    }
    hyre_executor* ex = nullptr;
    detail::check(hyre_executor_create(index.device(), max_batch, &ex));
    ex_.reset(ex);
  }

  TopKResult execute(const HybridQuery& query, StageTimings* timings = nullptr) {
    if (sh_) {
      auto out = execute_batch(BatchRequest{{query}}, timings);
      if (!out[0].ok) throw ValidationError(out[0].error);
      return std::move(out[0].result);
    }
    detail::QueryPack p({query});
    std::vector<hyre_hit> hits(std::max<std::uint32_t>(1, std::min(query.k, index_.num_docs())));
    std::uint32_t n = 0;
    hyre_timings t{};
    detail::check(hyre_execute(ex_.get(), p.q.data(), hits.data(), &n, &t));
    if (timings) *timings = StageTimings{t.tbr_ms, t.quant_ms, t.ebr_ms, t.topk_ms, t.total_ms};
    return to_result(hits.data(), n);
  }

  std::vector<QueryOutcome> execute_batch(const BatchRequest& batch, StageTimings* timings = nullptr) {
    const auto b = static_cast<std::uint32_t>(batch.queries.size());
    detail::QueryPack p(batch.queries);
    std::vector<std::uint64_t> offs(b + 1, 0);
    for (std::uint32_t i = 0; i < b; ++i) offs[i + 1] = offs[i] + std::min(batch.queries[i].k, index_.num_docs());
    std::vector<hyre_hit> hits(std::max<std::uint64_t>(1, offs[b]));
    std::vector<std::uint32_t> counts(b);
    std::vector<std::int32_t> st(b);
    hyre_timings t{};
    if (sh_)
      detail::check(hyre_sharded_execute_batch(sh_.get(), p.q.data(), b, hits.data(), offs.data(), counts.data(),
                                               st.data(), &t));
    else
      detail::check(hyre_execute_batch(ex_.get(), p.q.data(), b, hits.data(), offs.data(), counts.data(), st.data(),
                                       &t));
    if (timings) *timings = StageTimings{t.tbr_ms, t.quant_ms, t.ebr_ms, t.topk_ms, t.total_ms};
    std::vector<QueryOutcome> out(b);
    for (std::uint32_t i = 0; i < b; ++i) {
      out[i].ok = st[i] == HYRE_OK;
      if (out[i].ok) out[i].result = to_result(hits.data() + offs[i], counts[i]);
      else out[i].error = sh_ ? hyre_sharded_slot_error(sh_.get(), i) : hyre_executor_slot_error(ex_.get(), i);
    }
    return out;
  }

  const FrozenIndex& index() const { return index_; }
  std::uint32_t max_batch() const { return max_batch_; }
  hyre_executor* handle() const { return ex_.get(); }  // single-GPU executors
  hyre_sharded* sharded_handle() const { return sh_.get(); }

 private:
  TopKResult to_result(const hyre_hit* h, std::uint32_t n) const {
    TopKResult r;
    r.hits.reserve(n);
    for (std::uint32_t i = 0; i < n; ++i) r.hits.push_back({index_.doc_id(h[i].row), h[i].row, h[i].score});
    return r;
  }
  struct Del {
    void operator()(hyre_executor* e) const { hyre_executor_destroy(e); }
    void operator()(hyre_sharded* s) const { hyre_sharded_destroy(s); }
  };
  const FrozenIndex& index_;
  std::uint32_t max_batch_;
  std::unique_ptr<hyre_executor, Del> ex_;
  std::unique_ptr<hyre_sharded, Del> sh_;
};

inline TopKResult execute(const FrozenIndex& index, const HybridQuery& query) {
  Executor exec(index, 1);
  return exec.execute(query);
}

inline std::vector<QueryOutcome> execute_batch(const FrozenIndex& index, const BatchRequest& batch) {
  Executor exec(index, std::max<std::uint32_t>(1, static_cast<std::uint32_t>(batch.queries.size())));
  return exec.execute_batch(batch);
}

// ---- stage functions (term_match.hpp:43-45, knn.hpp:24-35, quantizer.hpp:71-74) ----
namespace detail {
// A single-GPU executor over the whole index for the stage functions (also
// on a sharded index: they are per-call test / tooling entry points).
struct StageExec {
  explicit StageExec(const FrozenIndex& index) {
    hyre_executor* e = nullptr;
    check(hyre_executor_create(index.device(), 1, &e));
    ex.reset(e);
  }
  hyre_executor* handle() const { return ex.get(); }
  struct Del {
    void operator()(hyre_executor* e) const { hyre_executor_destroy(e); }
  };
  std::unique_ptr<hyre_executor, Del> ex;
};
}  // namespace detail

inline std::vector<Messenger> full_scan_tbr(const FrozenIndex& index, const CnfQuery& query,
                                            std::uint32_t batch_id = 0) {
  detail::StageExec ex(index);
  HybridQuery hq{query, std::nullopt, 1, {}};
  detail::QueryPack p({hq});
  std::vector<std::uint32_t> rows(index.num_docs());
  std::uint64_t n = 0;
  detail::check(hyre_full_scan_tbr(ex.handle(), p.q.data(), rows.data(), rows.size(), &n));
  std::vector<Messenger> out;
  out.reserve(n);
  for (std::uint64_t i = 0; i < n; ++i) out.push_back({rows[i], batch_id, 0.0f});
  return out;
}

// pipeline.hpp:59-64: the matches of every query in one pass, ordered by
// (rowId, query position), stamped with batch_ids[i].
inline std::vector<Messenger> batch_scan_tbr(const FrozenIndex& index, std::span<const CnfQuery> queries,
                                             std::span<const std::uint32_t> batch_ids) {
  if (batch_ids.size() != queries.size()) throw ValidationError("batch_ids must have one id per query");
  if (queries.empty()) return {};
  hyre_executor* e = nullptr;
  detail::check(hyre_executor_create(index.device(), static_cast<std::uint32_t>(queries.size()), &e));
  std::unique_ptr<hyre_executor, detail::StageExec::Del> ex(e);
  std::vector<HybridQuery> hq;
  for (const auto& q : queries) hq.push_back(HybridQuery{q, std::nullopt, 1, {}});
  detail::QueryPack p(hq);
  const auto b = static_cast<std::uint32_t>(queries.size());
  std::uint64_t n = 0;
  detail::check(hyre_batch_scan_tbr(ex.get(), p.q.data(), b, batch_ids.data(), nullptr, 0, &n));
  std::vector<hyre_messenger> raw(n);
  detail::check(hyre_batch_scan_tbr(ex.get(), p.q.data(), b, batch_ids.data(), raw.data(), n, &n));
  std::vector<Messenger> out;
  out.reserve(n);
  for (const auto& m : raw) out.push_back({m.row_id, m.batch_id, 0.0f});
  return out;
}

inline ScoredMessengers exact_scores(const FrozenIndex& index, std::span<const float> query_embedding,
                                     std::vector<Messenger> candidates) {
  detail::StageExec ex(index);
  std::vector<std::uint32_t> rows;
  for (const auto& m : candidates) rows.push_back(m.row_id);
  std::vector<float> sc(rows.size());
  std::int32_t ren = 0;
  detail::check(hyre_exact_scores(ex.handle(), query_embedding.data(), static_cast<std::uint32_t>(query_embedding.size()),
                                  rows.data(), rows.size(), sc.data(), &ren));
  ScoredMessengers out{std::move(candidates), ren != 0};
  for (std::size_t i = 0; i < out.items.size(); ++i) out.items[i].score = sc[i];
  return out;
}

inline TopKResult bucket_top_k(const FrozenIndex& index, const ScoredMessengers& scored, std::uint32_t k,
                               std::uint32_t granularity = 100) {
  detail::StageExec ex(index);
  std::vector<std::uint32_t> rows;
  std::vector<float> sc;
  for (const auto& m : scored.items) {
    rows.push_back(m.row_id);
    sc.push_back(m.score);
  }
  std::vector<hyre_hit> hits(std::max<std::size_t>(1, std::min<std::size_t>(k, rows.size())));
  std::uint32_t n = 0;
  detail::check(hyre_bucket_top_k(ex.handle(), rows.data(), sc.data(), rows.size(), k, granularity, hits.data(), &n));
  TopKResult r;
  for (std::uint32_t i = 0; i < n; ++i) r.hits.push_back({index.doc_id(hits[i].row), hits[i].row, hits[i].score});
  return r;
}

inline std::vector<Messenger> preselect(const FrozenIndex& index, const Signature& query_signature,
                                        std::span<const Messenger> candidates, std::uint32_t quant_k) {
  detail::StageExec ex(index);
  std::vector<std::uint32_t> rows, out(candidates.size());
  for (const auto& m : candidates) rows.push_back(m.row_id);
  std::uint64_t n = 0;
  detail::check(hyre_preselect(ex.handle(), query_signature.words.data(), rows.data(), rows.size(), quant_k,
                               out.data(), &n));
  std::vector<Messenger> kept;
  for (std::uint64_t i = 0; i < n; ++i)
    for (const auto& m : candidates)
      if (m.row_id == out[i]) {
        kept.push_back(m);
        break;
      }
  return kept;
}

}  // namespace hyre
