// Synthetic workloads of SURVEY.md §8(d) -- bench / test infrastructure
// (libhyre_synth.so), not part of the query path.  RNG conventions follow
// the reference exactly (std::mt19937_64, uniform = (rng() >> 11) * 2^-53,
// random_unit as proj/src/bench.cpp:16-32), so the Python generators in
// oracle/hyre_oracle.py produce identical arrays for small n.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

namespace {

inline double unit_uniform(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

void random_unit(uint32_t dim, std::mt19937_64& rng, float* v) {
  double norm_sq = 0.0;
  for (uint32_t i = 0; i < dim; ++i) {
    v[i] = static_cast<float>(2.0 * unit_uniform(rng) - 1.0);
    norm_sq += static_cast<double>(v[i]) * v[i];
  }
  if (norm_sq == 0.0) {
    v[0] = 1.0f;
    return;
  }
  const double inv = 1.0 / std::sqrt(norm_sq);
  for (uint32_t i = 0; i < dim; ++i) v[i] = static_cast<float>(v[i] * inv);
}

}  // namespace

extern "C" {

__attribute__((visibility("default")))
// CNF workload docs (c1/c3): per doc, per slot c: a = 1 + rng()%max_ids ids,
// each 1 + c*V + rng()%V; then random_unit(dim).  Only docs in
// [row_begin, row_end) are stored (the stream is still drawn for all rows
// before row_end, so shards of one corpus are consistent).
// slot_offsets: (rows*C + 1) u64, relative to the stored range;
// ids: capacity rows*C*max_ids; emb: rows*dim.  Returns the id count.
uint64_t synth_cnf_docs(uint32_t row_begin, uint32_t row_end, uint32_t dim, uint32_t C, uint32_t V,
                        uint32_t max_ids, uint64_t seed, uint64_t* slot_offsets, uint32_t* ids, float* emb) {
  std::mt19937_64 rng(seed);
  std::vector<float> scratch(dim);
  uint64_t n_ids = 0, s = 0;
  if (slot_offsets) slot_offsets[0] = 0;
  for (uint32_t i = 0; i < row_end; ++i) {
    const bool keep = i >= row_begin;
    for (uint32_t c = 0; c < C; ++c) {
      const uint32_t a = 1 + static_cast<uint32_t>(rng() % max_ids);
      for (uint32_t j = 0; j < a; ++j) {
        const uint32_t id = 1 + c * V + static_cast<uint32_t>(rng() % V);
        if (keep) ids[n_ids++] = id;
      }
      if (keep) slot_offsets[++s] = n_ids;
    }
    random_unit(dim, rng, keep ? emb + static_cast<size_t>(i - row_begin) * dim : scratch.data());
  }
  return n_ids;
}

__attribute__((visibility("default")))
// CNF workload queries: per query, per slot `draws` ids with replacement
// (raw, un-normalized: ids[(q*C + c)*draws + j]), then random_unit(dim).
void synth_cnf_queries(uint32_t b, uint32_t dim, uint32_t C, uint32_t V, uint32_t draws, uint64_t seed,
                       uint32_t* ids, float* emb) {
  std::mt19937_64 rng(seed);
  for (uint32_t q = 0; q < b; ++q) {
    for (uint32_t c = 0; c < C; ++c)
      for (uint32_t j = 0; j < draws; ++j)
        ids[(static_cast<size_t>(q) * C + c) * draws + j] = 1 + c * V + static_cast<uint32_t>(rng() % V);
    random_unit(dim, rng, emb + static_cast<size_t>(q) * dim);
  }
}

__attribute__((visibility("default")))
// n random_unit vectors from one stream (c2/c4 corpora and queries).
void synth_unit_vectors(uint32_t row_begin, uint32_t row_end, uint32_t dim, uint64_t seed, float* out) {
  std::mt19937_64 rng(seed);
  std::vector<float> scratch(dim);
  for (uint32_t i = 0; i < row_end; ++i)
    random_unit(dim, rng, i >= row_begin ? out + static_cast<size_t>(i - row_begin) * dim : scratch.data());
}

__attribute__((visibility("default")))
// Zipf(s) "learned link" ids (c5): per doc 1 + rng()%max_ids ids drawn by
// inverse CDF over ranks 1..vocab; one clause slot; embeddings all
// random_unit(dim) from a second stream (seed + 1).
uint64_t synth_zipf_docs(uint32_t row_begin, uint32_t row_end, uint32_t dim, uint32_t vocab, double s,
                         uint32_t max_ids, uint64_t seed, uint64_t* slot_offsets, uint32_t* ids, float* emb) {
  std::vector<double> cdf(vocab);
  double acc = 0.0;
  for (uint32_t k = 0; k < vocab; ++k) cdf[k] = (acc += std::pow(static_cast<double>(k + 1), -s));
  for (auto& c : cdf) c /= acc;
  std::mt19937_64 rng(seed), erng(seed + 1);
  std::vector<float> scratch(dim);
  uint64_t n_ids = 0, sl = 0;
  slot_offsets[0] = 0;
  for (uint32_t i = 0; i < row_end; ++i) {
    const bool keep = i >= row_begin;
    const uint32_t a = 1 + static_cast<uint32_t>(rng() % max_ids);
    for (uint32_t j = 0; j < a; ++j) {
      const double u = unit_uniform(rng);
      const uint32_t id = 1 + static_cast<uint32_t>(std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
      if (keep) ids[n_ids++] = std::min(id, vocab);
    }
    if (keep) slot_offsets[++sl] = n_ids;
    random_unit(dim, erng, keep ? emb + static_cast<size_t>(i - row_begin) * dim : scratch.data());
  }
  return n_ids;
}

}  // extern "C"
