// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the *unmodified* reference engine
// (/root/reference/proj/src/{corpus,term_match,quantizer,knn,pipeline,bench}.cpp),
// compiled together with those sources by oracle/Makefile into
// oracle/_ref/libhyre_ref.so.  Only tests/, bench.py's cpu_baseline /
// --impl reference leg and __graft_entry__.smoke() may load it, and only as
// the checker or the timed CPU baseline -- never as part of the product path.
//
// No reference source is copied here: this file only *calls* the reference's
// public API (proj/include/hyre/*.hpp) and marshals plain arrays.
//
// Error convention mirrors the product C-ABI (include/hyre_b200.h):
//   0 ok, 1 ValidationError, 2 std::domain_error, 3 LoadError, 6 other.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "hyre/bench.hpp"
#include "hyre/common.hpp"
#include "hyre/corpus.hpp"
#include "hyre/knn.hpp"
#include "hyre/pipeline.hpp"
#include "hyre/quantizer.hpp"
#include "hyre/term_match.hpp"

namespace {

// Same field layout as hyre_query in include/hyre_b200.h (kept separate so
// the oracle does not depend on product headers).
struct RefQuery {
  uint32_t n_clauses;
  const uint32_t* slots;
  const uint32_t* id_offsets;
  const uint32_t* ids;
  const float* embedding;  // nullable -> term-only
  uint32_t embedding_dim;
  uint32_t k;
  uint32_t quant_enabled;
  uint32_t quant_k;
  uint32_t granularity;
};

thread_local std::string g_err;

int set_err(int code, const char* what) {
  g_err = what ? what : "";
  return code;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const hyre::ValidationError& e) {
    return set_err(1, e.what());
  } catch (const std::domain_error& e) {
    return set_err(2, e.what());
  } catch (const hyre::LoadError& e) {
    return set_err(3, e.what());
  } catch (const std::exception& e) {
    return set_err(6, e.what());
  }
}

hyre::HybridQuery to_hybrid(const RefQuery& rq) {
  hyre::HybridQuery q;
  for (uint32_t c = 0; c < rq.n_clauses; ++c) {
    hyre::CnfClause clause;
    clause.slot = rq.slots[c];
    clause.attribute_ids.assign(rq.ids + rq.id_offsets[c],
                                rq.ids + rq.id_offsets[c + 1]);
    q.terms.clauses.push_back(std::move(clause));
  }
  if (rq.embedding)
    q.embedding = std::vector<float>(rq.embedding, rq.embedding + rq.embedding_dim);
  q.k = rq.k;
  q.options.quant_enabled = rq.quant_enabled != 0;
  q.options.quant_k = rq.quant_k;
  q.options.granularity = rq.granularity;
  return q;
}

void write_hits(const hyre::TopKResult& r, uint32_t* rows, float* scores,
                uint32_t cap, uint32_t* n) {
  const uint32_t take = std::min<uint32_t>(cap, static_cast<uint32_t>(r.hits.size()));
  for (uint32_t i = 0; i < take; ++i) {
    rows[i] = r.hits[i].row_id;
    scores[i] = r.hits[i].score;
  }
  *n = static_cast<uint32_t>(r.hits.size());
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// IndexBuilder(config) + add_document per doc + freeze(make_codec(dim,num_bits,seed)).
// Raw clause ids of doc i, slot c live in ids[slot_offsets[i*C+c] .. slot_offsets[i*C+c+1]).
// doc ids are "doc_prefix" + i unless doc_ids (NUL-separated blob) is given.
int ref_build(uint32_t n_docs, uint32_t num_clauses, uint32_t max_num_attr,
              uint32_t dim, const uint32_t* slot_offsets, const uint32_t* ids,
              const float* embeddings, uint32_t num_bits, uint64_t seed,
              const char* doc_prefix, void** out) {
  return guarded([&] {
    hyre::IndexConfig cfg;
    cfg.num_clauses = num_clauses;
    cfg.max_num_attr = max_num_attr;
    cfg.dim = dim;
    hyre::IndexBuilder b(cfg);
    for (uint32_t i = 0; i < n_docs; ++i) {
      hyre::DocumentInput d;
      d.doc_id = std::string(doc_prefix ? doc_prefix : "doc") + std::to_string(i);
      d.clauses.resize(num_clauses);
      for (uint32_t c = 0; c < num_clauses; ++c) {
        const size_t s = std::size_t{i} * num_clauses + c;
        d.clauses[c].assign(ids + slot_offsets[s], ids + slot_offsets[s + 1]);
      }
      d.embedding.assign(embeddings + std::size_t{i} * dim,
                         embeddings + std::size_t{i + 1} * dim);
      b.add_document(d);
    }
    auto* idx = new hyre::FrozenIndex(
        std::move(b).freeze(hyre::make_codec(dim, num_bits, seed)));
    *out = idx;
  });
}

int ref_load(const char* path, void** out) {
  return guarded([&] { *out = new hyre::FrozenIndex(hyre::FrozenIndex::load(path)); });
}

int ref_save(void* h, const char* path) {
  return guarded([&] { static_cast<hyre::FrozenIndex*>(h)->save(path); });
}

void ref_free(void* h) { delete static_cast<hyre::FrozenIndex*>(h); }

void ref_shape(void* h, uint32_t* shape /* n, C, A, d, num_bits, words */) {
  auto* idx = static_cast<hyre::FrozenIndex*>(h);
  shape[0] = idx->num_docs();
  shape[1] = idx->num_clauses();
  shape[2] = idx->max_num_attr();
  shape[3] = idx->dim();
  shape[4] = idx->codec().num_bits;
  shape[5] = static_cast<uint32_t>(idx->codec().num_words());
}

// Copies the frozen flat arrays out (any pointer may be null).
void ref_export(void* h, uint32_t* attributes, uint32_t* offsets,
                float* embeddings, uint64_t* signatures, uint8_t* zero_flags) {
  auto* idx = static_cast<hyre::FrozenIndex*>(h);
  const uint32_t n = idx->num_docs();
  const uint32_t a = idx->max_num_attr(), c1 = idx->num_clauses() + 1, d = idx->dim();
  const size_t w = idx->codec().num_words();
  for (uint32_t r = 0; r < n; ++r) {
    if (attributes) {
      auto s = idx->attribute_row(r);
      std::copy(s.begin(), s.end(), attributes + std::size_t{r} * a);
    }
    if (offsets) {
      auto s = idx->offsets_row(r);
      std::copy(s.begin(), s.end(), offsets + std::size_t{r} * c1);
    }
    if (embeddings) {
      auto s = idx->embedding_row(r);
      std::copy(s.begin(), s.end(), embeddings + std::size_t{r} * d);
    }
    if (signatures) {
      auto s = idx->signature_words(r);
      std::copy(s.begin(), s.end(), signatures + std::size_t{r} * w);
    }
    if (zero_flags) zero_flags[r] = idx->embedding_is_zero(r) ? 1 : 0;
  }
}

// Copies doc_id(row) into buf (NUL-terminated, truncated to cap).
void ref_doc_id(void* h, uint32_t row, char* buf, uint32_t cap) {
  const auto& s = static_cast<hyre::FrozenIndex*>(h)->doc_id(row);
  std::snprintf(buf, cap, "%s", s.c_str());
}

// normalize_query over a raw {slot: ids} map given as parallel arrays
// (slots may repeat -> later entries overwrite like std::map assignment).
// Output: normalized clauses (slots, id_offsets, ids) with capacity checks.
int ref_normalize_query(uint32_t n_raw, const uint32_t* raw_slots,
                        const uint32_t* raw_offsets, const uint32_t* raw_ids,
                        uint32_t num_clauses, uint32_t* out_n, uint32_t* out_slots,
                        uint32_t* out_offsets, uint32_t* out_ids) {
  return guarded([&] {
    std::map<std::uint32_t, std::vector<std::uint32_t>> raw;
    for (uint32_t i = 0; i < n_raw; ++i)
      raw[raw_slots[i]].assign(raw_ids + raw_offsets[i], raw_ids + raw_offsets[i + 1]);
    auto q = hyre::normalize_query(raw, num_clauses);
    *out_n = static_cast<uint32_t>(q.clauses.size());
    uint32_t pos = 0;
    out_offsets[0] = 0;
    for (size_t c = 0; c < q.clauses.size(); ++c) {
      out_slots[c] = q.clauses[c].slot;
      for (auto id : q.clauses[c].attribute_ids) out_ids[pos++] = id;
      out_offsets[c + 1] = pos;
    }
  });
}

// full_scan_tbr -> ascending rows. Returns the match count in *n (rows
// written up to cap).
int ref_full_scan_tbr(void* h, const RefQuery* rq, uint32_t* rows, uint64_t cap,
                      uint64_t* n) {
  return guarded([&] {
    auto q = to_hybrid(*rq);
    auto ms = hyre::full_scan_tbr(*static_cast<hyre::FrozenIndex*>(h), q.terms, 0);
    *n = ms.size();
    for (uint64_t i = 0; i < ms.size() && i < cap; ++i) rows[i] = ms[i].row_id;
  });
}

// batch_scan_tbr (pipeline.cpp:75-93) -> (row, batch) pairs interleaved in
// out[2i], out[2i+1]; total in *n (pairs written up to cap).
int ref_batch_scan_tbr(void* h, const RefQuery* qs, uint32_t b, const uint32_t* batch_ids, uint32_t* out,
                       uint64_t cap, uint64_t* n) {
  return guarded([&] {
    std::vector<hyre::CnfQuery> terms;
    for (uint32_t i = 0; i < b; ++i) terms.push_back(to_hybrid(qs[i]).terms);
    auto ms = hyre::batch_scan_tbr(*static_cast<hyre::FrozenIndex*>(h), terms,
                                   std::span<const std::uint32_t>(batch_ids, b));
    *n = ms.size();
    for (uint64_t i = 0; i < ms.size() && i < cap; ++i) {
      out[2 * i] = ms[i].row_id;
      out[2 * i + 1] = ms[i].batch_id;
    }
  });
}

int ref_validate_query(void* h, const RefQuery* rq) {
  return guarded([&] {
    hyre::validate_query(*static_cast<hyre::FrozenIndex*>(h), to_hybrid(*rq));
  });
}

int ref_execute(void* h, const RefQuery* rq, uint32_t* rows, float* scores,
                uint32_t cap, uint32_t* n, double* timings /* 5, nullable */) {
  return guarded([&] {
    hyre::Executor ex(*static_cast<hyre::FrozenIndex*>(h), 1);
    hyre::StageTimings t;
    auto r = ex.execute(to_hybrid(*rq), &t);
    write_hits(r, rows, scores, cap, n);
    if (timings) {
      timings[0] = t.tbr_ms; timings[1] = t.quant_ms; timings[2] = t.ebr_ms;
      timings[3] = t.topk_ms; timings[4] = t.total_ms;
    }
  });
}

// execute_batch; per-slot status in statuses (0 ok / 1 validation error),
// hits of slot i at rows/scores + i*cap_per_query.
int ref_execute_batch(void* h, const RefQuery* qs, uint32_t b, uint32_t max_batch,
                      uint32_t* rows, float* scores, uint32_t cap_per_query,
                      uint32_t* counts, int32_t* statuses) {
  return guarded([&] {
    hyre::Executor ex(*static_cast<hyre::FrozenIndex*>(h), max_batch);
    hyre::BatchRequest br;
    for (uint32_t i = 0; i < b; ++i) br.queries.push_back(to_hybrid(qs[i]));
    auto outs = ex.execute_batch(br);
    for (uint32_t i = 0; i < b; ++i) {
      statuses[i] = outs[i].ok ? 0 : 1;
      counts[i] = 0;
      if (outs[i].ok)
        write_hits(outs[i].result, rows + std::size_t{i} * cap_per_query,
                   scores + std::size_t{i} * cap_per_query, cap_per_query, &counts[i]);
    }
  });
}

// ---------------------------------------------------------------------------
// Sharded oracle ("c4/c5 (50M) use the sharded oracle").
// The reference is single-threaded per query, so a 10M-50M index is built as
// G FrozenIndex shards of one corpus (shard s = global rows
// [s*n/G, (s+1)*n/G), built concurrently, each by the reference's own
// IndexBuilder + freeze) and every (query, shard) pair runs the reference
// Executor::execute.  Per query the shard results are merged:
//  - hybrid: by (score desc, global row asc) -- the order bucket_top_k
//    returns (proj/src/knn.cpp:79-92), so with quant off the merge equals the
//    unsharded result exactly (the global top-K is a subset of the union of
//    the shard top-Ks; per-row eligibility and scores do not depend on the
//    shard);
//  - term-only: shard lists concatenated in shard order, first k
//    (term_only_result, proj/src/pipeline.cpp:30-40: ascending global rows).
// Quant pre-selection is NOT exact under sharding (preselect ranks within
// the shard), so quant-on parity uses an unsharded index.
// ---------------------------------------------------------------------------
namespace {
hyre::FrozenIndex* build_rows(uint64_t begin, uint64_t end, uint32_t num_clauses,
                              uint32_t max_num_attr, uint32_t dim,
                              const uint64_t* slot_offsets, const uint32_t* ids,
                              const float* embeddings, uint32_t num_bits, uint64_t seed,
                              const char* doc_prefix) {
  hyre::IndexConfig cfg;
  cfg.num_clauses = num_clauses;
  cfg.max_num_attr = max_num_attr;
  cfg.dim = dim;
  hyre::IndexBuilder b(cfg);
  for (uint64_t i = begin; i < end; ++i) {
    hyre::DocumentInput d;
    d.doc_id = std::string(doc_prefix ? doc_prefix : "doc") + std::to_string(i);
    d.clauses.resize(num_clauses);
    for (uint32_t c = 0; c < num_clauses; ++c) {
      const size_t s = i * num_clauses + c;
      d.clauses[c].assign(ids + slot_offsets[s], ids + slot_offsets[s + 1]);
    }
    d.embedding.assign(embeddings + i * dim, embeddings + (i + 1) * dim);
    b.add_document(d);
  }
  return new hyre::FrozenIndex(std::move(b).freeze(hyre::make_codec(dim, num_bits, seed)));
}
}  // namespace

// Builds g shards concurrently (one thread per shard, at most `threads` at a
// time); out[s] = shard handle, bases[s] = its first global row.  Doc ids are
// doc_prefix + global row.  slot_offsets are u64 (50M-row corpora).
int ref_build_shards(uint64_t n_docs, uint32_t num_clauses, uint32_t max_num_attr,
                     uint32_t dim, const uint64_t* slot_offsets, const uint32_t* ids,
                     const float* embeddings, uint32_t num_bits, uint64_t seed,
                     const char* doc_prefix, uint32_t g, uint32_t threads, void** out,
                     uint64_t* bases) {
  return guarded([&] {
    std::vector<std::string> errs(g);
    std::atomic<uint32_t> next{0};
    std::vector<std::thread> pool;
    for (uint32_t s = 0; s < g; ++s) out[s] = nullptr;
    for (uint32_t t = 0; t < std::max<uint32_t>(1, std::min(threads, g)); ++t)
      pool.emplace_back([&] {
        for (uint32_t s = next++; s < g; s = next++) {
          const uint64_t b = n_docs * s / g, e = n_docs * (s + 1) / g;
          bases[s] = b;
          try {
            out[s] = build_rows(b, e, num_clauses, max_num_attr, dim, slot_offsets, ids,
                                embeddings, num_bits, seed, doc_prefix);
          } catch (const std::exception& ex) {
            errs[s] = ex.what();
          }
        }
      });
    for (auto& th : pool) th.join();
    for (uint32_t s = 0; s < g; ++s)
      if (!errs[s].empty()) {
        for (uint32_t r = 0; r < g; ++r) delete static_cast<hyre::FrozenIndex*>(out[r]);
        throw std::runtime_error(errs[s]);
      }
  });
}

// Runs b queries over g shards on `threads` workers (each worker keeps one
// reference Executor per shard it touches, like an ExecutorPool lease) and
// merges per query as described above.  Rows written are GLOBAL rows.
// *seconds = wall time of the whole call (executes + merges).
int ref_execute_sharded(void* const* hs, const uint64_t* bases, uint32_t g,
                        const RefQuery* qs, uint32_t b, uint32_t threads, uint32_t* rows,
                        float* scores, uint32_t cap_per_query, uint32_t* counts,
                        int32_t* statuses, double* seconds) {
  return guarded([&] {
    std::vector<hyre::HybridQuery> hq;
    for (uint32_t i = 0; i < b; ++i) hq.push_back(to_hybrid(qs[i]));
    const uint64_t items = uint64_t{b} * g;
    std::vector<hyre::TopKResult> res(items);
    std::vector<int> st(items, 0);
    std::vector<std::string> msg(items);
    std::atomic<uint64_t> next{0};
    const uint32_t nt = std::max<uint32_t>(1, threads);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (uint32_t t = 0; t < nt; ++t)
      pool.emplace_back([&] {
        std::vector<std::unique_ptr<hyre::Executor>> ex(g);
        for (uint64_t it = next++; it < items; it = next++) {
          const uint32_t qi = static_cast<uint32_t>(it / g), s = static_cast<uint32_t>(it % g);
          if (!ex[s]) ex[s] = std::make_unique<hyre::Executor>(*static_cast<hyre::FrozenIndex*>(hs[s]), 1);
          try {
            res[it] = ex[s]->execute(hq[qi]);
          } catch (const hyre::ValidationError& e) {
            st[it] = 1;
            msg[it] = e.what();
          } catch (const std::domain_error& e) {
            st[it] = 2;
            msg[it] = e.what();
          }
        }
      });
    for (auto& th : pool) th.join();
    for (uint32_t qi = 0; qi < b; ++qi) {
      statuses[qi] = 0;
      counts[qi] = 0;
      for (uint32_t s = 0; s < g; ++s)
        if (st[uint64_t{qi} * g + s]) statuses[qi] = st[uint64_t{qi} * g + s];
      if (statuses[qi]) continue;
      std::vector<std::pair<float, uint32_t>> all;
      for (uint32_t s = 0; s < g; ++s)
        for (const auto& h : res[uint64_t{qi} * g + s].hits)
          all.emplace_back(h.score, static_cast<uint32_t>(bases[s] + h.row_id));
      if (hq[qi].embedding)
        std::sort(all.begin(), all.end(), [](const auto& x, const auto& y) {
          return x.first != y.first ? x.first > y.first : x.second < y.second;
        });
      const uint32_t take = std::min<uint32_t>(
          {cap_per_query, hq[qi].k, static_cast<uint32_t>(all.size())});
      for (uint32_t j = 0; j < take; ++j) {
        rows[std::size_t{qi} * cap_per_query + j] = all[j].second;
        scores[std::size_t{qi} * cap_per_query + j] = all[j].first;
      }
      counts[qi] = take;
    }
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}

// Throughput harness mirroring SearchService's ExecutorPool
// (proj/src/service.cpp:99-141): `threads` workers, one Executor each over
// the shared FrozenIndex, pulling single queries from a shared counter.
// Returns wall seconds for all b queries in *seconds; hits as in
// ref_execute_batch.
int ref_execute_parallel(void* h, const RefQuery* qs, uint32_t b, uint32_t threads,
                         uint32_t* rows, float* scores, uint32_t cap_per_query,
                         uint32_t* counts, double* seconds) {
  return guarded([&] {
    auto& idx = *static_cast<hyre::FrozenIndex*>(h);
    std::vector<hyre::HybridQuery> hq;
    for (uint32_t i = 0; i < b; ++i) hq.push_back(to_hybrid(qs[i]));
    std::atomic<uint32_t> next{0};
    std::vector<std::string> errs(threads);
    const uint32_t nt = std::max<uint32_t>(1, threads);
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (uint32_t t = 0; t < nt; ++t) {
      pool.emplace_back([&, t] {
        try {
          hyre::Executor ex(idx, 1);
          for (uint32_t i = next++; i < b; i = next++) {
            auto r = ex.execute(hq[i]);
            if (rows)
              write_hits(r, rows + std::size_t{i} * cap_per_query,
                         scores + std::size_t{i} * cap_per_query, cap_per_query,
                         &counts[i]);
          }
        } catch (const std::exception& e) {
          errs[t] = e.what();
        }
      });
    }
    for (auto& th : pool) th.join();
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (auto& e : errs)
      if (!e.empty()) throw std::runtime_error(e);
  });
}

// exact_scores over explicit candidate rows.
int ref_exact_scores(void* h, const float* q, uint32_t dim, const uint32_t* rows,
                     uint64_t n, float* scores_out, int32_t* renormalized) {
  return guarded([&] {
    std::vector<hyre::Messenger> ms(n);
    for (uint64_t i = 0; i < n; ++i) ms[i] = {rows[i], 0, 0.0f};
    auto s = hyre::exact_scores(*static_cast<hyre::FrozenIndex*>(h),
                                std::span<const float>(q, dim), std::move(ms));
    for (uint64_t i = 0; i < n; ++i) scores_out[i] = s.items[i].score;
    *renormalized = s.query_was_renormalized ? 1 : 0;
  });
}

// bucket_top_k over explicit (row, score) messengers.
int ref_bucket_top_k(void* h, const uint32_t* rows, const float* scores, uint64_t n,
                     uint32_t k, uint32_t granularity, uint32_t* rows_out,
                     float* scores_out, uint32_t* n_out) {
  return guarded([&] {
    hyre::ScoredMessengers s;
    s.items.resize(n);
    for (uint64_t i = 0; i < n; ++i) s.items[i] = {rows[i], 0, scores[i]};
    auto r = hyre::bucket_top_k(*static_cast<hyre::FrozenIndex*>(h), s, k, granularity);
    write_hits(r, rows_out, scores_out, k, n_out);
  });
}

// encode(make_codec(dim, num_bits, seed), x) -> words (ceil(num_bits/64)).
int ref_encode(uint32_t dim, uint32_t num_bits, uint64_t seed, const float* x,
               uint64_t* words) {
  return guarded([&] {
    auto codec = hyre::make_codec(dim, num_bits, seed);
    auto sig = hyre::encode(codec, std::span<const float>(x, dim));
    std::copy(sig.words.begin(), sig.words.end(), words);
  });
}

// Codec structure: rounds, then per round perm/signs/bounds flattened.
int ref_codec(uint32_t dim, uint32_t num_bits, uint64_t seed, uint32_t* n_rounds,
              uint32_t* perm, float* signs, uint32_t* bounds, uint32_t* n_bounds) {
  return guarded([&] {
    auto codec = hyre::make_codec(dim, num_bits, seed);
    *n_rounds = static_cast<uint32_t>(codec.rounds.size());
    uint32_t bpos = 0;
    for (size_t r = 0; r < codec.rounds.size(); ++r) {
      const auto& rd = codec.rounds[r];
      if (perm) std::copy(rd.perm.begin(), rd.perm.end(), perm + r * dim);
      if (signs) std::copy(rd.signs.begin(), rd.signs.end(), signs + r * dim);
      n_bounds[r] = static_cast<uint32_t>(rd.bounds.size());
      if (bounds) std::copy(rd.bounds.begin(), rd.bounds.end(), bounds + bpos);
      bpos += static_cast<uint32_t>(rd.bounds.size());
    }
  });
}

// preselect over explicit candidate rows (ascending) with a query signature.
int ref_preselect(void* h, const uint64_t* qwords, const uint32_t* rows, uint64_t n,
                  uint32_t quant_k, uint32_t* rows_out, uint64_t* n_out) {
  return guarded([&] {
    auto& idx = *static_cast<hyre::FrozenIndex*>(h);
    hyre::Signature sig;
    sig.num_bits = idx.codec().num_bits;
    sig.words.assign(qwords, qwords + idx.codec().num_words());
    std::vector<hyre::Messenger> ms(n);
    for (uint64_t i = 0; i < n; ++i) ms[i] = {rows[i], 0, 0.0f};
    auto kept = hyre::preselect(idx, sig, ms, quant_k);
    *n_out = kept.size();
    for (size_t i = 0; i < kept.size(); ++i) rows_out[i] = kept[i].row_id;
  });
}

}  // extern "C"
