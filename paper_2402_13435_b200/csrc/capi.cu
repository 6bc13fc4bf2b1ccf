// extern "C" entry points declared in include/hyre_b200.h.  Each wraps the
// C++ layer, maps exceptions to hyre_status and records the message in a
// thread-local buffer (hyre_last_error).
#include <chrono>
#include <cstdio>
#include <map>
#include <memory>
#include <string>

#include "executor.cuh"
#include "service.cuh"
#include "sharded.cuh"
#include "hyre_b200.h"

using namespace hyreb;

struct hyre_builder {
  Builder b;
};
struct hyre_frozen {
  std::unique_ptr<Frozen> f;
};
struct hyre_index {
  std::unique_ptr<DevIndex> ix;
};
struct hyre_executor {
  std::unique_ptr<Executor> ex;
};
struct hyre_schema {
  Schema s;
};
struct hyre_documents {
  DocumentSet d;
};
struct hyre_links {
  LinksExport l;
};
struct hyre_pool {
  std::unique_ptr<Pool> p;
};
struct hyre_sharded_index {
  std::unique_ptr<ShardedIndex> ix;
};
struct hyre_sharded {
  std::unique_ptr<ShardedExecutor> s;
};

namespace {
thread_local std::string g_err;
thread_local int g_cause = -1;

template <class F>
hyre_status guard(F&& fn) {
  try {
    fn();
    return HYRE_OK;
  } catch (const Error& e) {
    g_err = e.what();
    g_cause = e.load_cause;
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_err = "host allocation failed";
    return HYRE_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HYRE_INTERNAL;
  }
}
void need(const void* p, const char* what) {
  if (!p) throw Error(HYRE_INVALID_ARGUMENT, std::string(what) + " must not be null");
}
}  // namespace

extern "C" {

const char* hyre_last_error(void) { return g_err.c_str(); }
int hyre_last_load_cause(void) { return g_cause; }
int hyre_abi_version(void) { return HYRE_B200_ABI_VERSION; }

// ---- builder / frozen ------------------------------------------------------
hyre_status hyre_builder_create(uint32_t num_clauses, uint32_t max_num_attr, uint32_t dim,
                                const char* const* clause_names, uint32_t num_names,
                                hyre_builder** out) {
  return guard([&] {
    need(out, "out");
    std::vector<std::string> names;
    if (clause_names)
      for (uint32_t i = 0; i < num_names; ++i) names.emplace_back(clause_names[i]);
    *out = new hyre_builder{Builder(num_clauses, max_num_attr, dim, std::move(names))};
  });
}

void hyre_builder_destroy(hyre_builder* b) { delete b; }

hyre_status hyre_builder_add_document(hyre_builder* b, const char* doc_id, uint32_t num_slots,
                                      const uint32_t* slot_offsets, const uint32_t* ids,
                                      const float* embedding, uint32_t embedding_len,
                                      uint32_t* row_out) {
  return guard([&] {
    need(b, "builder");
    need(doc_id, "doc_id");
    const uint32_t r = b->b.add(doc_id, num_slots, slot_offsets, ids, embedding, embedding_len);
    if (row_out) *row_out = r;
  });
}

hyre_status hyre_builder_add_documents(hyre_builder* b, uint32_t n, const char* prefix,
                                       const uint64_t* slot_offsets, const uint32_t* ids,
                                       const float* embeddings) {
  return guard([&] {
    need(b, "builder");
    if (n == 0) return;
    need(slot_offsets, "slot_offsets");
    need(embeddings, "embeddings");
    b->b.add_bulk(n, prefix ? prefix : "", slot_offsets, ids, embeddings);
  });
}

uint32_t hyre_builder_size(const hyre_builder* b) { return b ? b->b.size() : 0; }

// ---- ingestion (ingest.cpp; dataio.hpp:15-28) -----------------------------------
hyre_status hyre_schema_read_json(const char* path, hyre_schema** out) {
  return guard([&] {
    need(path, "path");
    need(out, "out");
    *out = new hyre_schema{read_schema_json(path)};
  });
}
hyre_status hyre_schema_create(uint32_t n, const char* const* names, uint32_t dim, hyre_schema** out) {
  return guard([&] {
    need(out, "out");
    if (n && !names) validation("schema: clause names required");
    Schema s;
    for (uint32_t i = 0; i < n; ++i) s.clause_names.emplace_back(names[i]);
    s.dim = dim;
    *out = new hyre_schema{std::move(s)};
  });
}
void hyre_schema_destroy(hyre_schema* s) { delete s; }
uint32_t hyre_schema_num_clauses(const hyre_schema* s) { return s ? static_cast<uint32_t>(s->s.clause_names.size()) : 0; }
const char* hyre_schema_clause_name(const hyre_schema* s, uint32_t i) {
  return s && i < s->s.clause_names.size() ? s->s.clause_names[i].c_str() : nullptr;
}
uint32_t hyre_schema_dim(const hyre_schema* s) { return s ? s->s.dim : 0; }

hyre_status hyre_documents_read_jsonl(const char* path, const hyre_schema* s, hyre_documents** out) {
  return guard([&] {
    need(path, "path");
    need(s, "schema");
    need(out, "out");
    *out = new hyre_documents{read_documents_jsonl(path, s->s)};
  });
}
void hyre_documents_destroy(hyre_documents* d) { delete d; }
uint32_t hyre_documents_count(const hyre_documents* d) { return d ? static_cast<uint32_t>(d->d.doc_ids.size()) : 0; }
uint32_t hyre_documents_widest(const hyre_documents* d) { return d ? d->d.widest : 0; }
const char* hyre_documents_id(const hyre_documents* d, uint32_t i) {
  return d && i < d->d.doc_ids.size() ? d->d.doc_ids[i].c_str() : nullptr;
}
const uint64_t* hyre_documents_slot_offsets(const hyre_documents* d) { return d ? d->d.slot_offsets.data() : nullptr; }
const uint32_t* hyre_documents_ids(const hyre_documents* d) { return d ? d->d.ids.data() : nullptr; }
const float* hyre_documents_embeddings(const hyre_documents* d) { return d ? d->d.embeddings.data() : nullptr; }

hyre_status hyre_builder_add_document_set(hyre_builder* b, const hyre_documents* ds, uint32_t* first_row) {
  return guard([&] {
    need(b, "builder");
    need(ds, "documents");
    const DocumentSet& d = ds->d;
    if (first_row) *first_row = b->b.size();
    std::vector<uint32_t> so(d.num_clauses + 1);
    for (size_t i = 0; i < d.doc_ids.size(); ++i) {  // add_document semantics and messages, file order
      const uint64_t base = d.slot_offsets[i * d.num_clauses];
      for (uint32_t c = 0; c <= d.num_clauses; ++c)
        so[c] = static_cast<uint32_t>(d.slot_offsets[i * d.num_clauses + c] - base);
      b->b.add(d.doc_ids[i], d.num_clauses, so.data(), d.ids.data() + base, d.embeddings.data() + i * d.dim, d.dim);
    }
  });
}

hyre_status hyre_links_read_json(const char* path, hyre_links** out) {
  return guard([&] {
    need(path, "path");
    need(out, "out");
    *out = new hyre_links{read_links_export(path)};
  });
}
void hyre_links_destroy(hyre_links* l) { delete l; }
uint32_t hyre_links_num_nodes(const hyre_links* l) { return l ? l->l.num_nodes : 0; }
uint32_t hyre_links_count(const hyre_links* l, int32_t side) {
  return l && (side == 0 || side == 1) ? static_cast<uint32_t>(l->l.names[side].size()) : 0;
}
const char* hyre_links_name(const hyre_links* l, int32_t side, uint32_t i) {
  return hyre_links_count(l, side) > i ? l->l.names[side][i].c_str() : nullptr;
}
const uint32_t* hyre_links_ids(const hyre_links* l, int32_t side, uint32_t i, uint32_t* n) {
  if (hyre_links_count(l, side) <= i) {
    if (n) *n = 0;
    return nullptr;
  }
  if (n) *n = static_cast<uint32_t>(l->l.ids[side][i].size());
  return l->l.ids[side][i].data();
}

hyre_status hyre_builder_freeze(hyre_builder* b, uint32_t num_bits, uint64_t seed, hyre_frozen** out) {
  return guard([&] {
    need(b, "builder");
    need(out, "out");
    *out = new hyre_frozen{std::unique_ptr<Frozen>(b->b.freeze(num_bits, seed))};
  });
}

hyre_status hyre_builder_freeze_device(hyre_builder* b, uint32_t num_bits, uint64_t seed, int32_t device,
                                       hyre_frozen** out) {
  return guard([&] {
    need(b, "builder");
    need(out, "out");
    *out = new hyre_frozen{std::unique_ptr<Frozen>(freeze_on_device(b->b, num_bits, seed, device))};
  });
}

hyre_status hyre_frozen_from_arrays(uint32_t num_docs, uint32_t num_clauses, uint32_t max_num_attr,
                                    uint32_t dim, uint32_t num_bits, uint64_t seed,
                                    const uint32_t* attributes, const uint32_t* offsets,
                                    const float* embeddings, const uint64_t* signatures,
                                    const uint8_t* zero_flags, const char* const* doc_ids,
                                    const char* doc_id_prefix, hyre_frozen** out) {
  return guard([&] {
    need(out, "out");
    need(attributes, "attributes");
    need(offsets, "offsets");
    need(embeddings, "embeddings");
    if (num_docs == 0) validation("no documents staged");
    if (num_clauses == 0) validation("numClauses must be >= 1");
    if (dim == 0) validation("dim must be >= 1");
    if (max_num_attr == 0) validation("maxNumAttr must be >= 1");
    std::unique_ptr<Frozen> f(new Frozen);
    f->num_docs = num_docs;
    f->num_clauses = num_clauses;
    f->max_num_attr = max_num_attr;
    f->dim = dim;
    f->num_bits = num_bits;
    f->seed = seed;
    Codec codec = make_codec(dim, num_bits, seed);
    const size_t n = num_docs, nw = codec.num_words();
    f->attributes.assign(attributes, attributes + n * max_num_attr);
    f->offsets.assign(offsets, offsets + n * (num_clauses + 1));
    f->embeddings.assign(embeddings, embeddings + n * dim);
    if (signatures) {
      f->signatures.assign(signatures, signatures + n * nw);
    } else {
      f->signatures.assign(n * nw, 0);
      parallel_for(n, 4096, [&](size_t b0, size_t e0) {
        for (size_t r = b0; r < e0; ++r)
          encode(codec, f->embeddings.data() + r * dim, f->signatures.data() + r * nw);
      });
    }
    if (zero_flags) {
      f->zero.assign(zero_flags, zero_flags + n);
    } else {
      f->zero.assign(n, 0);
      for (size_t r = 0; r < n; ++r) {
        bool z = true;
        for (uint32_t d = 0; d < dim && z; ++d) z = f->embeddings[r * dim + d] == 0.0f;
        f->zero[r] = z;
      }
    }
    if (doc_ids) {
      for (size_t r = 0; r < n; ++r) f->doc_ids.push(doc_ids[r]);
    } else {
      f->doc_ids.push_range(doc_id_prefix ? doc_id_prefix : "", static_cast<uint32_t>(n));
    }
    for (uint32_t c = 0; c < num_clauses; ++c) f->clause_names.push_back("c" + std::to_string(c));
    *out = new hyre_frozen{std::move(f)};
  });
}

hyre_status hyre_frozen_save(const hyre_frozen* f, const char* path) {
  return guard([&] {
    need(f, "frozen");
    need(path, "path");
    save(*f->f, path);
  });
}

hyre_status hyre_frozen_load(const char* path, hyre_frozen** out) {
  return guard([&] {
    need(path, "path");
    need(out, "out");
    *out = new hyre_frozen{std::unique_ptr<Frozen>(load(path))};
  });
}

void hyre_frozen_destroy(hyre_frozen* f) { delete f; }

void hyre_frozen_shape(const hyre_frozen* f, hyre_shape* s) {
  s->num_docs = f->f->num_docs;
  s->num_clauses = f->f->num_clauses;
  s->max_num_attr = f->f->max_num_attr;
  s->dim = f->f->dim;
  s->num_bits = f->f->num_bits;
  s->num_words = static_cast<uint32_t>(f->f->num_words());
  s->seed = f->f->seed;
}

const uint32_t* hyre_frozen_attributes(const hyre_frozen* f) { return f->f->attributes.data(); }
const uint32_t* hyre_frozen_offsets(const hyre_frozen* f) { return f->f->offsets.data(); }
const float* hyre_frozen_embeddings(const hyre_frozen* f) { return f->f->embeddings.data(); }
const uint64_t* hyre_frozen_signatures(const hyre_frozen* f) { return f->f->signatures.data(); }
const uint8_t* hyre_frozen_zero_flags(const hyre_frozen* f) { return f->f->zero.data(); }
const char* hyre_frozen_doc_id(const hyre_frozen* f, uint32_t row) {
  return row < f->f->doc_ids.size() ? f->f->doc_ids.c_str(row) : nullptr;
}
int64_t hyre_frozen_row_of(const hyre_frozen* f, const char* doc_id) { return f->f->row_of(doc_id); }
int32_t hyre_frozen_resolve_clause_slot(const hyre_frozen* f, const char* name) {
  for (uint32_t c = 0; c < f->f->num_clauses; ++c)
    if (f->f->clause_names[c] == name) return static_cast<int32_t>(c);
  return -1;
}
const char* hyre_frozen_clause_name(const hyre_frozen* f, uint32_t slot) {
  return slot < f->f->clause_names.size() ? f->f->clause_names[slot].c_str() : nullptr;
}

// ---- codec -------------------------------------------------------------------
hyre_status hyre_encode(uint32_t dim, uint32_t num_bits, uint64_t seed, const float* x, uint64_t* words) {
  return guard([&] {
    need(x, "x");
    need(words, "words");
    Codec c = make_codec(dim, num_bits, seed);
    encode(c, x, words);
  });
}

uint32_t hyre_quant_score_words(const uint64_t* a, const uint64_t* b, uint32_t num_words, uint32_t num_bits) {
  return quant_score_words(a, b, num_words, num_bits);
}

// ---- queries -------------------------------------------------------------------
hyre_status hyre_normalize_query(uint32_t n_raw, const uint32_t* raw_slots, const uint32_t* raw_offsets,
                                 const uint32_t* raw_ids, uint32_t num_clauses, uint32_t* out_n,
                                 uint32_t* out_slots, uint32_t* out_offsets, uint32_t* out_ids) {
  return guard([&] {
    // std::map iteration = ascending slot, as term_match.cpp:10 walks the map.
    std::map<uint32_t, std::vector<uint32_t>> raw;
    for (uint32_t i = 0; i < n_raw; ++i)
      raw[raw_slots[i]].assign(raw_ids + raw_offsets[i], raw_ids + raw_offsets[i + 1]);
    uint32_t n = 0, pos = 0;
    out_offsets[0] = 0;
    for (auto& [slot, ids] : raw) {
      if (slot >= num_clauses)
        validation("unknown clause slot " + std::to_string(slot) + " (index has " +
                   std::to_string(num_clauses) + ")");
      for (auto id : ids)
        if (id == 0) validation("attribute id 0 is reserved for padding");
      std::sort(ids.begin(), ids.end());
      ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
      if (ids.empty()) continue;  // no constraint on this slot (term_match.cpp:26)
      out_slots[n] = slot;
      for (auto id : ids) out_ids[pos++] = id;
      out_offsets[++n] = pos;
    }
    *out_n = n;
  });
}

hyre_status hyre_validate_query(const hyre_frozen* f, const hyre_query* q) {
  return guard([&] {
    need(f, "frozen");
    need(q, "query");
    validate_query(QueryShape{f->f->num_clauses, f->f->dim}, *q);
  });
}

// ---- device index ----------------------------------------------------------------
hyre_status hyre_index_create(const hyre_frozen* f, const hyre_index_options* opts, hyre_index** out) {
  return guard([&] {
    need(f, "frozen");
    need(out, "out");
    hyre_index_options o{};
    if (opts) o = *opts;
    *out = new hyre_index{std::unique_ptr<DevIndex>(build_device_index(*f->f, o))};
  });
}

void hyre_index_destroy(hyre_index* ix) { delete ix; }

hyre_status hyre_index_set_row_weights(hyre_index* ix, const float* w, uint64_t n) {
  return guard([&] {
    need(ix, "index");
    set_row_weights(*ix->ix, w, n);
  });
}

hyre_status hyre_index_stats_get(const hyre_index* ix, hyre_index_stats* out) {
  return guard([&] {
    need(ix, "index");
    need(out, "out");
    *out = ix->ix->stats;
  });
}

// ---- executor ------------------------------------------------------------------
hyre_status hyre_executor_create(hyre_index* ix, uint32_t max_batch, hyre_executor** out) {
  return guard([&] {
    need(ix, "index");
    need(out, "out");
    *out = new hyre_executor{std::unique_ptr<Executor>(new Executor(ix->ix.get(), max_batch))};
  });
}

void hyre_executor_destroy(hyre_executor* ex) { delete ex; }

hyre_status hyre_pool_create(hyre_index* ix, uint32_t workers, uint32_t max_batch, uint32_t max_wait_us,
                             hyre_pool** out) {
  return guard([&] {
    need(ix, "index");
    need(out, "out");
    *out = new hyre_pool{std::unique_ptr<Pool>(new Pool(ix->ix.get(), workers, max_batch, max_wait_us))};
  });
}

void hyre_pool_destroy(hyre_pool* p) { delete p; }

hyre_status hyre_pool_search(hyre_pool* p, const hyre_query* q, hyre_hit* hits, uint32_t* n_hits) {
  return guard([&] {
    need(p, "pool");
    need(q, "query");
    p->p->search(*q, hits, n_hits);
  });
}

hyre_status hyre_pool_stats(const hyre_pool* p, uint64_t* batches, uint64_t* queries) {
  return guard([&] {
    need(p, "pool");
    p->p->stats(batches, queries);
  });
}
void* hyre_executor_stream(hyre_executor* ex) { return ex ? ex->ex->st : nullptr; }

hyre_status hyre_execute(hyre_executor* ex, const hyre_query* q, hyre_hit* hits, uint32_t* n_hits,
                         hyre_timings* timings) {
  return guard([&] {
    need(ex, "executor");
    need(q, "query");
    const auto t0 = std::chrono::steady_clock::now();
    ex->ex->prepare(q, 1);
    if (ex->ex->statuses[0] != HYRE_OK)
      throw Error(static_cast<hyre_status>(ex->ex->statuses[0]), ex->ex->slot_errors[0]);
    ex->ex->run();
    const uint64_t off = 0;
    uint32_t cnt = 0;
    int32_t stt = 0;
    ex->ex->fetch(hits, &off, &cnt, &stt, timings);
    if (n_hits) *n_hits = cnt;
    if (timings)
      timings->total_ms =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  });
}

hyre_status hyre_execute_batch(hyre_executor* ex, const hyre_query* qs, uint32_t b, hyre_hit* hits,
                               const uint64_t* hit_offsets, uint32_t* counts, int32_t* statuses,
                               hyre_timings* timings) {
  return guard([&] {
    need(ex, "executor");
    const auto t0 = std::chrono::steady_clock::now();
    ex->ex->prepare(qs, b);
    const auto t1 = std::chrono::steady_clock::now();
    ex->ex->run();
    const auto t2 = std::chrono::steady_clock::now();
    ex->ex->fetch(hits, hit_offsets, counts, statuses, timings);
    if (std::getenv("HYRE_DEBUG_E2E")) {  // diagnostics: host phases of one call
      const auto t3 = std::chrono::steady_clock::now();
      auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
      std::fprintf(stderr, "[hyre] execute_batch us: prepare %.1f run(launch) %.1f fetch(wait+copy) %.1f\n",
                   us(t0, t1), us(t1, t2), us(t2, t3));
    }
    if (timings)
      timings->total_ms =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  });
}

// ---- sharded executor --------------------------------------------------------
hyre_status hyre_sharded_index_create(const hyre_frozen* f, const hyre_sharded_index_options* o,
                                      hyre_sharded_index** out) {
  return guard([&] {
    need(f, "frozen");
    need(o, "options");
    need(out, "out");
    *out = new hyre_sharded_index{std::make_unique<ShardedIndex>(*f->f, *o)};
  });
}

void hyre_sharded_index_destroy(hyre_sharded_index* ix) { delete ix; }

hyre_status hyre_sharded_index_set_row_weights(hyre_sharded_index* ix, const float* w, uint64_t n) {
  return guard([&] {
    need(ix, "index");
    ShardedIndex& si = *ix->ix;
    if (w && n != si.total_rows)
      validation("row weights: expected " + std::to_string(si.total_rows) + " weights, got " + std::to_string(n));
    const uint32_t base0 = si.ix.front()->row_base;
    for (auto& d : si.ix) set_row_weights(*d, w ? w + (d->row_base - base0) : nullptr, d->n_rows);
  });
}

hyre_status hyre_sharded_index_info(const hyre_sharded_index* ix, uint32_t* n_shards, int32_t* devices) {
  return guard([&] {
    need(ix, "sharded index");
    if (n_shards) *n_shards = ix->ix->G;
    if (devices)
      for (uint32_t g = 0; g < ix->ix->G; ++g) devices[g] = ix->ix->ix[g]->device;
  });
}

hyre_status hyre_sharded_create(hyre_sharded_index* ix, uint32_t max_batch, hyre_sharded** out) {
  return guard([&] {
    need(ix, "sharded index");
    need(out, "out");
    *out = new hyre_sharded{std::make_unique<ShardedExecutor>(*ix->ix, max_batch)};
  });
}

void hyre_sharded_destroy(hyre_sharded* s) { delete s; }

hyre_status hyre_sharded_execute_batch(hyre_sharded* s, const hyre_query* qs, uint32_t b, hyre_hit* hits,
                                       const uint64_t* hit_offsets, uint32_t* counts, int32_t* statuses,
                                       hyre_timings* timings) {
  return guard([&] {
    need(s, "sharded executor");
    const auto t0 = std::chrono::steady_clock::now();
    s->s->prepare(qs, b);
    s->s->run();
    s->s->fetch(hits, hit_offsets, counts, statuses, timings);
    if (timings)
      timings->total_ms =
          std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  });
}

const char* hyre_sharded_slot_error(const hyre_sharded* s, uint32_t slot) {
  if (!s || slot >= s->s->root().slot_errors.size()) return "";
  return s->s->root().slot_errors[slot].c_str();
}

hyre_status hyre_sharded_prepare(hyre_sharded* s, const hyre_query* qs, uint32_t b) {
  return guard([&] {
    need(s, "sharded executor");
    s->s->prepare(qs, b);
  });
}

hyre_status hyre_sharded_run(hyre_sharded* s) {
  return guard([&] {
    need(s, "sharded executor");
    s->s->run();
  });
}

hyre_status hyre_sharded_settle(hyre_sharded* s) {
  return guard([&] {
    need(s, "sharded executor");
    s->s->settle();
  });
}

hyre_status hyre_sharded_fetch(hyre_sharded* s, hyre_hit* hits, const uint64_t* hit_offsets, uint32_t* counts,
                               int32_t* statuses, hyre_timings* timings) {
  return guard([&] {
    need(s, "sharded executor");
    s->s->fetch(hits, hit_offsets, counts, statuses, timings);
  });
}

void* hyre_sharded_stream(const hyre_sharded* s) { return s ? s->s->root_stream() : nullptr; }

uint32_t hyre_sharded_kernel_count(const hyre_sharded* s) { return s ? s->s->kernels_per_run() : 0; }

hyre_status hyre_sharded_recovery(const hyre_sharded* s, uint32_t* out2) {
  return guard([&] {
    need(s, "sharded executor");
    need(out2, "out");
    out2[0] = s->s->recovery_rounds;
    out2[1] = s->s->exhaustive_queries;
  });
}

const char* hyre_executor_slot_error(const hyre_executor* ex, uint32_t slot) {
  if (!ex || slot >= ex->ex->slot_errors.size()) return "";
  return ex->ex->slot_errors[slot].c_str();
}

hyre_status hyre_batch_settle(hyre_executor* ex) {
  return guard([&] {
    need(ex, "executor");
    ex->ex->settle();
  });
}

hyre_status hyre_batch_prepare(hyre_executor* ex, const hyre_query* qs, uint32_t b) {
  return guard([&] {
    need(ex, "executor");
    ex->ex->prepare(qs, b);
  });
}

hyre_status hyre_batch_run(hyre_executor* ex) {
  return guard([&] {
    need(ex, "executor");
    ex->ex->run();
  });
}

hyre_status hyre_batch_fetch(hyre_executor* ex, hyre_hit* hits, const uint64_t* hit_offsets, uint32_t* counts,
                             int32_t* statuses, hyre_timings* timings) {
  return guard([&] {
    need(ex, "executor");
    ex->ex->fetch(hits, hit_offsets, counts, statuses, timings);
  });
}

uint32_t hyre_batch_kernel_count(const hyre_executor* ex) { return ex ? ex->ex->kernels : 0; }

uint64_t hyre_batch_term_bytes(const hyre_executor* ex) { return ex ? ex->ex->term_bytes : 0; }
uint64_t hyre_batch_scan_bytes(const hyre_executor* ex) { return ex ? ex->ex->scan_bytes : 0; }

hyre_status hyre_batch_eligible(hyre_executor* ex, uint32_t* out) {
  return guard([&] {
    need(ex, "executor");
    need(out, "out");
    ex->ex->eligible(out);
  });
}

uint32_t hyre_batch_path(const hyre_executor* ex) {
  if (!ex) return 0;
  const Executor* e = ex->ex.get();
  return (e->use_tc ? HYRE_PATH_TC : 0u) | (e->use_fused ? HYRE_PATH_FUSED : 0u) |
         (e->use_fwd && !e->use_fused && !e->all_match ? HYRE_PATH_FWD_MASK : 0u) |
         (e->all_match ? HYRE_PATH_MATCH_ALL : 0u) | (e->pf_i8 ? HYRE_PATH_I8 : 0u) |
         (e->any_emb && e->ix->n_rows > e->cap && !e->use_small ? HYRE_PATH_SAMPLED : 0u) |
         (e->use_small ? HYRE_PATH_SMALL : 0u);
}

uint32_t hyre_batch_cnf_group(const hyre_executor* ex) {
  return ex && ex->ex->use_fused ? ex->ex->ix->cnf_group : 0u;
}

void hyre_batch_tc_variant(const hyre_executor* ex, uint32_t* out4) {
  if (!out4) return;
  out4[0] = out4[1] = out4[2] = out4[3] = 0;
  if (!ex || !ex->ex->use_tc) return;
  const Executor* e = ex->ex.get();
  if (e->use_fused) {
    out4[0] = e->ix->cnf_ids_per_row;
    out4[1] = e->ix->cnf_id_bytes;
    out4[2] = tc_fused_chunks(e->tc_np);
  }
  out4[3] = e->tc_np;
}

hyre_status hyre_batch_stage_ms(hyre_executor* ex, float* out6) {
  return guard([&] {
    need(ex, "executor");
    need(out6, "out");
    ex->ex->stage_ms(out6);
  });
}

hyre_status hyre_batch_stage_ms_hist(hyre_executor* ex, uint32_t back, float* out6) {
  return guard([&] {
    need(ex, "executor");
    need(out6, "out");
    ex->ex->stage_ms_hist(back, out6);
  });
}

hyre_status hyre_batch_set_stage_events(hyre_executor* ex, int on) {
  return guard([&] {
    need(ex, "executor");
    ex->ex->stage_events = on != 0;
  });
}

hyre_status hyre_batch_recovery(const hyre_executor* ex, uint32_t* out2) {
  return guard([&] {
    need(ex, "executor");
    need(out2, "out");
    out2[0] = ex->ex->finish_rounds;
    out2[1] = ex->ex->exh_count;
  });
}

hyre_status hyre_batch_io_bytes(const hyre_executor* ex, uint64_t* h2d, uint64_t* d2h) {
  return guard([&] {
    need(ex, "executor");
    if (h2d) *h2d = ex->ex->h2d_bytes;
    if (d2h) *d2h = ex->ex->d2h_bytes;
  });
}

hyre_status hyre_batch_merge_gathered(hyre_executor* ex, const void* g_hits, const void* g_offsets,
                                      const void* g_counts, uint32_t n_lists, uint64_t hits_stride) {
  return guard([&] {
    need(ex, "executor");
    ex->ex->merge_gathered(static_cast<const hyre_hit*>(g_hits), static_cast<const uint64_t*>(g_offsets),
                           static_cast<const uint32_t*>(g_counts), n_lists, hits_stride);
  });
}

hyre_status hyre_batch_merge_packed(hyre_executor* ex, const void* g_records, uint32_t n_lists,
                                    uint64_t record_words, uint64_t hits_words) {
  return guard([&] {
    need(ex, "executor");
    need(g_records, "records");
    const uint32_t B = ex->ex->B;
    if (hits_words % 2 || record_words % 2 || record_words < hits_words + 3ull * B)
      validation("packed merge: record must hold hits (even words), then b u64 offsets, then b u32 counts");
    const uint32_t* r = static_cast<const uint32_t*>(g_records);
    ex->ex->merge_gathered(reinterpret_cast<const hyre_hit*>(r), reinterpret_cast<const uint64_t*>(r + hits_words),
                           r + hits_words + 2ull * B, n_lists, record_words / 2, record_words / 2, record_words);
  });
}

hyre_status hyre_batch_device_results(hyre_executor* ex, void** hits, uint64_t* n_hits, void** offsets,
                                      void** counts) {
  return guard([&] {
    need(ex, "executor");
    Executor& e = *ex->ex;
    if (hits) *hits = e.d_hits;
    if (n_hits) *n_hits = e.n_hits_total;
    if (offsets) *offsets = e.d_hit_off;
    if (counts) *counts = e.d_counters + 3 * e.max_batch;
  });
}

hyre_status hyre_full_scan_tbr(hyre_executor* ex, const hyre_query* q, uint32_t* rows, uint64_t cap,
                               uint64_t* n) {
  return guard([&] {
    need(ex, "executor");
    need(q, "query");
    *n = ex->ex->full_scan(*q, rows, cap);
  });
}

hyre_status hyre_batch_scan_tbr(hyre_executor* ex, const hyre_query* qs, uint32_t b, const uint32_t* batch_ids,
                                hyre_messenger* out, uint64_t cap, uint64_t* n) {
  return guard([&] {
    need(ex, "executor");
    need(n, "n");
    if (b && (!qs || !batch_ids)) validation("batch_scan_tbr: queries and batch_ids are required");
    if (b > ex->ex->max_batch)
      validation("batch of " + std::to_string(b) + " exceeds maxBatch " + std::to_string(ex->ex->max_batch));
    *n = ex->ex->batch_scan(qs, b, batch_ids, out, out ? cap : 0);
  });
}

hyre_status hyre_exact_scores(hyre_executor* ex, const float* q, uint32_t dim, const uint32_t* rows,
                              uint64_t n, float* scores, int32_t* renormalized) {
  return guard([&] {
    need(ex, "executor");
    need(q, "query");
    const bool r = ex->ex->exact_scores(q, dim, rows, n, scores);
    if (renormalized) *renormalized = r;
  });
}

hyre_status hyre_bucket_top_k(hyre_executor* ex, const uint32_t* rows, const float* scores, uint64_t n,
                              uint32_t k, uint32_t granularity, hyre_hit* out, uint32_t* n_out) {
  return guard([&] {
    need(ex, "executor");
    if (k < 1) validation("k must be >= 1");
    if (granularity < 1) validation("granularity must be >= 1");
    for (uint64_t i = 0; i < n; ++i)  // knn.cpp:59-61
      if (scores[i] < -1.0f || scores[i] > 1.0f)
        throw Error(HYRE_OUT_OF_RANGE,
                    "score " + std::to_string(scores[i]) + " outside the documented [-1, 1] bounds");
    *n_out = ex->ex->top_k(rows, scores, n, k, out);
  });
}

hyre_status hyre_preselect(hyre_executor* ex, const uint64_t* query_words, const uint32_t* rows, uint64_t n,
                           uint32_t quant_k, uint32_t* rows_out, uint64_t* n_out) {
  return guard([&] {
    need(ex, "executor");
    *n_out = ex->ex->preselect(query_words, rows, n, quant_k, rows_out);
  });
}

hyre_status hyre_merge_topk(const hyre_hit* const* lists, const uint32_t* counts, uint32_t n_lists, uint32_t k,
                            hyre_hit* out, uint32_t* n_out) {
  return guard([&] {
    // K-way merge by the orderable key (score desc, row asc); lists are short.
    std::vector<uint32_t> pos(n_lists, 0);
    uint32_t m = 0;
    while (m < k) {
      int best = -1;
      uint64_t bk = 0;
      for (uint32_t l = 0; l < n_lists; ++l) {
        if (pos[l] >= counts[l]) continue;
        const hyre_hit& h = lists[l][pos[l]];
        const uint64_t key = make_key(h.score + 0.0f, h.row);
        if (best < 0 || key > bk) {
          best = static_cast<int>(l);
          bk = key;
        }
      }
      if (best < 0) break;
      out[m++] = lists[best][pos[best]++];
    }
    *n_out = m;
  });
}

}  // extern "C"
