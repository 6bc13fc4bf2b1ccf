// Host-side internals shared by the C-ABI, the device index builder and the
// executor.  Everything here is plain C++ (no CUDA types).
#pragma once

#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "hyre_b200.h"

namespace hyreb {

// Carries a hyre_status across the C++ layers; the C-ABI turns it into the
// return code + thread-local message (hyre_last_error).
struct Error : std::runtime_error {
  hyre_status code;
  int load_cause;
  Error(hyre_status c, const std::string& m, int cause = -1)
      : std::runtime_error(m), code(c), load_cause(cause) {}
};

[[noreturn]] inline void validation(const std::string& m) {
  throw Error(HYRE_INVALID_ARGUMENT, m);
}

// ---------------------------------------------------------------------------
// Sign-quant codec: quantizer.hpp:17-30 / quantizer.cpp:12-70.
// ---------------------------------------------------------------------------
struct Codec {
  struct Round {
    std::vector<uint32_t> perm;
    std::vector<float> signs;
    std::vector<uint32_t> bounds;
  };
  uint32_t dim = 0, num_bits = 0;
  uint64_t seed = 0;
  std::vector<Round> rounds;
  size_t num_words() const { return (num_bits + 63) / 64; }
};

Codec make_codec(uint32_t dim, uint32_t num_bits, uint64_t seed);
void encode(const Codec& c, const float* x, uint64_t* words);
uint32_t quant_score_words(const uint64_t* a, const uint64_t* b, size_t words,
                           uint32_t num_bits);

// ---------------------------------------------------------------------------
// Row -> docId (corpus.hpp:100-101).  Explicitly added ids are stored as
// strings; a bulk add (prefix + decimal row number, the synthetic and
// `hyre build --prefix` case) is one range whose ids are generated on demand,
// so a 50M-row build keeps no 50M strings and no 50M-entry hash map.
// ---------------------------------------------------------------------------
class DocIds {
 public:
  uint32_t size() const { return n_; }
  bool empty() const { return n_ == 0; }
  void push(std::string id);                           // explicit id of row size()
  void push_range(const std::string& prefix, uint32_t count);  // rows size() ..: prefix + row
  std::string at(uint32_t row) const;
  const char* c_str(uint32_t row) const;  // thread-local copy for range rows
  int64_t find(const std::string& id) const;  // row or -1
  // smallest row r in [row0, row0 + count) whose id prefix + r already exists, or -1
  int64_t first_collision(const std::string& prefix, uint32_t row0, uint32_t count) const;
  void clear();

 private:
  struct Seg {
    uint32_t row0, count;
    bool range;
    std::string prefix;  // range
    size_t first;        // explicit: index of row0's id in explicit_
  };
  const Seg& seg_of(uint32_t row) const;
  std::vector<Seg> segs_;
  std::vector<std::string> explicit_;
  std::vector<uint32_t> explicit_rows_;  // row of explicit_[i]
  uint32_t n_ = 0;
  mutable std::unordered_map<std::string, uint32_t> map_;  // explicit ids, built lazily
  mutable size_t mapped_ = 0;                              // explicit ids already in map_
};

// ---------------------------------------------------------------------------
// FrozenIndex host arrays: corpus.hpp:57-124.
// ---------------------------------------------------------------------------
struct Frozen {
  uint32_t num_docs = 0, num_clauses = 0, max_num_attr = 0, dim = 0, num_bits = 0;
  uint64_t seed = 0;
  std::vector<std::string> clause_names;
  std::vector<uint32_t> attributes;   // N x A
  std::vector<uint32_t> offsets;      // N x (C+1)
  std::vector<float> embeddings;      // N x d
  std::vector<uint64_t> signatures;   // N x words
  std::vector<uint8_t> zero;          // N
  DocIds doc_ids;                     // N

  size_t num_words() const { return (num_bits + 63) / 64; }
  int64_t row_of(const std::string& id) const;
};

struct Builder {
  uint32_t num_clauses = 0, max_num_attr = 0, dim = 0;
  std::vector<std::string> clause_names;
  std::vector<uint64_t> slot_offsets{0};  // (docs * C) + 1
  std::vector<uint32_t> ids;
  std::vector<float> embeddings;
  DocIds doc_ids;
  bool frozen = false;

  Builder(uint32_t c, uint32_t a, uint32_t d, std::vector<std::string> names);
  uint32_t add(const std::string& doc_id, uint32_t num_slots, const uint32_t* slot_offsets,
               const uint32_t* ids, const float* emb, uint32_t emb_len);
  void add_bulk(uint32_t n, const std::string& prefix, const uint64_t* slot_offsets,
                const uint32_t* ids, const float* embs);
  Frozen* freeze(uint32_t num_bits, uint64_t seed);
  uint32_t size() const { return doc_ids.size(); }
};

// ---------------------------------------------------------------------------
// Ingestion (ingest.cpp): dataio.hpp:15-28 and the links export.
// ---------------------------------------------------------------------------
struct Schema {  // IngestSchema (dataio.hpp:15-18)
  std::vector<std::string> clause_names;
  uint32_t dim = 0;
};
struct DocumentSet {  // read_documents_jsonl's documents, flat (file order)
  uint32_t num_clauses = 0, dim = 0, widest = 0;  // widest: max distinct ids of a document
  std::vector<std::string> doc_ids;
  std::vector<uint64_t> slot_offsets;  // docs x C + 1
  std::vector<uint32_t> ids;
  std::vector<float> embeddings;  // docs x dim
};
struct LinksExport {  // serving-graph export (dataio.cpp:253-274)
  uint32_t num_nodes = 0;
  std::vector<std::string> names[2];           // [0] seekers, [1] jobs (key order)
  std::vector<std::vector<uint32_t>> ids[2];  // node ids, sorted unique
};
Schema read_schema_json(const std::string& path);
DocumentSet read_documents_jsonl(const std::string& path, const Schema& schema);
LinksExport read_links_export(const std::string& path);

void save(const Frozen& f, const std::string& path);
Frozen* load(const std::string& path);

// ---------------------------------------------------------------------------
// Queries: term_match.cpp:7-30, pipeline.cpp:19-73.
// ---------------------------------------------------------------------------
struct QueryShape {
  uint32_t num_clauses, dim;
};
void validate_query(const QueryShape& s, const hyre_query& q);
// unit_embedding (pipeline.cpp:19-28); returns true if renormalized.
bool unit_embedding(const float* raw, uint32_t n, float* out);

// Parallel-for over [0, n) on up to hardware_concurrency threads.
void parallel_for(size_t n, size_t grain, const std::function<void(size_t, size_t)>& fn);

}  // namespace hyreb
