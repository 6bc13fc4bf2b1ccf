// Host side of the drop-in boundary: index staging/freeze, the sign-quant
// codec, the HYREIDN1 index file, query normalisation and validation.
//
// Semantics follow the reference exactly (messages included) so the C-ABI is
// a drop-in for proj/include/hyre/{corpus,quantizer,term_match,pipeline}.hpp;
// the implementation is our own (flat staging arrays instead of per-document
// vectors, multithreaded freeze).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <map>
#include <numeric>
#include <random>
#include <thread>

#include "host.hpp"

namespace hyreb {

void parallel_for(size_t n, size_t grain, const std::function<void(size_t, size_t)>& fn) {
  if (n == 0) return;
  size_t hw = std::max(1u, std::thread::hardware_concurrency());
  size_t chunks = std::min(hw, (n + grain - 1) / grain);
  if (chunks <= 1) {
    fn(0, n);
    return;
  }
  std::vector<std::thread> ts;
  size_t per = (n + chunks - 1) / chunks;
  for (size_t t = 0; t < chunks; ++t) {
    size_t b = t * per, e = std::min(n, b + per);
    if (b >= e) break;
    ts.emplace_back([&fn, b, e] { fn(b, e); });
  }
  for (auto& t : ts) t.join();
}

// ---------------------------------------------------------------------------
// Codec -- quantizer.cpp:12-84.  Draws come straight from mt19937_64's output
// (Fisher-Yates as common.hpp:166-172) so permutations match bit for bit.
// ---------------------------------------------------------------------------
Codec make_codec(uint32_t dim, uint32_t num_bits, uint64_t seed) {
  if (dim == 0) validation("codec dim must be >= 1");
  if (num_bits == 0) validation("codec numBits must be >= 1");
  Codec c;
  c.dim = dim;
  c.num_bits = num_bits;
  c.seed = seed;
  std::mt19937_64 rng(seed);
  uint32_t emitted = 0;
  while (emitted < num_bits) {
    Codec::Round r;
    r.perm.resize(dim);
    std::iota(r.perm.begin(), r.perm.end(), 0u);
    for (size_t i = dim; i > 1; --i) std::swap(r.perm[i - 1], r.perm[rng() % i]);
    r.signs.resize(dim);
    for (auto& s : r.signs) s = (rng() & 1u) ? 1.0f : -1.0f;
    const uint32_t bins = std::min(num_bits - emitted, dim);
    const uint32_t base = dim / bins, extra = dim % bins;
    r.bounds.resize(bins + 1);
    r.bounds[0] = 0;
    for (uint32_t b = 0; b < bins; ++b) r.bounds[b + 1] = r.bounds[b] + base + (b < extra ? 1u : 0u);
    emitted += bins;
    c.rounds.push_back(std::move(r));
  }
  return c;
}

void encode(const Codec& c, const float* x, uint64_t* words) {
  std::fill(words, words + c.num_words(), 0ull);
  uint32_t bit = 0;
  for (const auto& r : c.rounds) {
    const uint32_t bins = static_cast<uint32_t>(r.bounds.size() - 1);
    for (uint32_t b = 0; b < bins && bit < c.num_bits; ++b, ++bit) {
      double agg = 0.0;
      for (uint32_t i = r.bounds[b]; i < r.bounds[b + 1]; ++i)
        agg += static_cast<double>(r.signs[i]) * x[r.perm[i]];
      if (agg >= 0.0) words[bit / 64] |= uint64_t{1} << (bit % 64);  // sign(0) = +1
    }
  }
}

uint32_t quant_score_words(const uint64_t* a, const uint64_t* b, size_t words, uint32_t num_bits) {
  uint32_t s = 0;
  for (size_t w = 0; w < words; ++w) {
    uint64_t same = ~(a[w] ^ b[w]);
    if (w + 1 == words && num_bits % 64 != 0) same &= (uint64_t{1} << (num_bits % 64)) - 1;
    s += static_cast<uint32_t>(__builtin_popcountll(same));
  }
  return s;
}

// ---------------------------------------------------------------------------
// Builder -- corpus.cpp:15-129.
// ---------------------------------------------------------------------------
Builder::Builder(uint32_t c, uint32_t a, uint32_t d, std::vector<std::string> names)
    : num_clauses(c), max_num_attr(a), dim(d), clause_names(std::move(names)) {
  if (num_clauses == 0) validation("numClauses must be >= 1");
  if (dim == 0) validation("dim must be >= 1");
  if (max_num_attr == 0) validation("maxNumAttr must be >= 1");
  if (clause_names.empty())
    for (uint32_t i = 0; i < num_clauses; ++i) clause_names.push_back("c" + std::to_string(i));
  if (clause_names.size() != num_clauses) validation("clause_names size != numClauses");
}

uint32_t Builder::add(const std::string& doc_id, uint32_t num_slots, const uint32_t* so,
                      const uint32_t* in_ids, const float* emb, uint32_t emb_len) {
  if (frozen) validation("builder already frozen");
  if (doc_ids.find(doc_id) >= 0) validation("duplicate docId: " + doc_id);
  if (num_slots != num_clauses)
    validation("clauses: expected " + std::to_string(num_clauses) + " clause slots, got " +
               std::to_string(num_slots));
  if (emb_len != dim)
    validation("embedding: expected dim " + std::to_string(dim) + ", got " + std::to_string(emb_len));
  for (uint32_t c = 0; c < num_slots; ++c)
    for (uint32_t i = so[c]; i < so[c + 1]; ++i)
      if (in_ids[i] == 0)
        validation("attribute id 0 is reserved for padding (docId " + doc_id + ")");
  const auto row = doc_ids.size();
  doc_ids.push(doc_id);
  for (uint32_t c = 0; c < num_slots; ++c) {
    ids.insert(ids.end(), in_ids + so[c], in_ids + so[c + 1]);
    slot_offsets.push_back(ids.size());
  }
  embeddings.insert(embeddings.end(), emb, emb + dim);
  return row;
}

void Builder::add_bulk(uint32_t n, const std::string& prefix, const uint64_t* so,
                       const uint32_t* in_ids, const float* embs) {
  if (frozen) validation("builder already frozen");
  const uint64_t base = so[0];
  // Validate everything before staging anything (all-or-nothing), reporting
  // the first offending row as the per-document loop would.
  const uint32_t row0 = doc_ids.size();
  const int64_t dup = doc_ids.first_collision(prefix, row0, n);
  for (uint32_t i = 0; i < n; ++i) {
    if (dup == int64_t{row0} + i) validation("duplicate docId: " + prefix + std::to_string(row0 + i));
    for (uint64_t j = so[size_t{i} * num_clauses]; j < so[size_t{i + 1} * num_clauses]; ++j)
      if (in_ids[j - base] == 0)
        validation("attribute id 0 is reserved for padding (docId " + prefix + std::to_string(row0 + i) + ")");
  }
  const uint64_t shift = ids.size() - base;
  ids.insert(ids.end(), in_ids, in_ids + (so[size_t{n} * num_clauses] - base));
  slot_offsets.reserve(slot_offsets.size() + size_t{n} * num_clauses);
  for (size_t s = 1; s <= size_t{n} * num_clauses; ++s) slot_offsets.push_back(so[s] + shift);
  embeddings.insert(embeddings.end(), embs, embs + size_t{n} * dim);
  doc_ids.push_range(prefix, n);
}

Frozen* Builder::freeze(uint32_t num_bits, uint64_t seed) {
  if (frozen) validation("builder already frozen");
  if (doc_ids.empty()) validation("no documents staged");
  Codec codec = make_codec(dim, num_bits, seed);  // codec.dim == dim by construction
  frozen = true;
  const uint32_t n = static_cast<uint32_t>(doc_ids.size());
  const uint32_t C = num_clauses, A = max_num_attr;

  auto* f = new Frozen;
  f->num_docs = n;
  f->num_clauses = C;
  f->max_num_attr = A;
  f->dim = dim;
  f->num_bits = num_bits;
  f->seed = seed;
  f->clause_names = clause_names;
  f->attributes.assign(size_t{n} * A, 0);
  f->offsets.assign(size_t{n} * (C + 1), 0);
  f->embeddings.assign(size_t{n} * dim, 0.0f);
  f->signatures.assign(size_t{n} * codec.num_words(), 0);
  f->zero.assign(n, 0);

  // Canonicalize per clause (sort + dedup) before the width check
  // (corpus.cpp:61-81); widths are checked on the de-duplicated size.
  std::vector<uint8_t> wide(n, 0);
  parallel_for(n, 4096, [&](size_t b, size_t e) {
    std::vector<uint32_t> tmp;
    for (size_t r = b; r < e; ++r) {
      uint32_t* attr = f->attributes.data() + r * A;
      uint32_t* offs = f->offsets.data() + r * (C + 1);
      uint32_t pos = 0;
      bool too_wide = false;
      for (uint32_t c = 0; c < C; ++c) {
        const uint64_t s0 = slot_offsets[r * C + c], s1 = slot_offsets[r * C + c + 1];
        tmp.assign(ids.begin() + s0, ids.begin() + s1);
        std::sort(tmp.begin(), tmp.end());
        tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
        offs[c] = pos;
        for (auto id : tmp) {
          if (pos < A) attr[pos] = id;
          ++pos;
        }
        if (pos > A) too_wide = true;
      }
      offs[C] = std::min(pos, A);
      wide[r] = too_wide;
      // L2-normalize in double (corpus.cpp:109-119).
      const float* emb = embeddings.data() + r * dim;
      double norm_sq = 0.0;
      for (uint32_t d = 0; d < dim; ++d) norm_sq += static_cast<double>(emb[d]) * emb[d];
      float* out = f->embeddings.data() + r * dim;
      if (norm_sq == 0.0) {
        f->zero[r] = 1;
      } else {
        const double inv = 1.0 / std::sqrt(norm_sq);
        for (uint32_t d = 0; d < dim; ++d) out[d] = static_cast<float>(emb[d] * inv);
      }
      encode(codec, out, f->signatures.data() + r * codec.num_words());
    }
  });
  std::string too;
  for (uint32_t r = 0; r < n; ++r)
    if (wide[r]) too += " " + doc_ids.at(r);
  if (!too.empty()) {
    delete f;
    validation("documents wider than maxNumAttr=" + std::to_string(A) + ":" + too);
  }
  f->doc_ids = std::move(doc_ids);
  // Staging memory is released (the builder is consumed, corpus.hpp:47 `&&`).
  std::vector<uint32_t>().swap(ids);
  std::vector<float>().swap(embeddings);
  std::vector<uint64_t>().swap(slot_offsets);
  return f;
}

int64_t Frozen::row_of(const std::string& id) const { return doc_ids.find(id); }

// ---------------------------------------------------------------------------
// DocIds
// ---------------------------------------------------------------------------
namespace {
// value of a canonical decimal (no sign, no leading zero unless "0"), or -1
int64_t parse_row(const std::string& s, size_t from) {
  if (from >= s.size() || s.size() - from > 10) return -1;
  if (s[from] == '0' && s.size() - from > 1) return -1;
  int64_t v = 0;
  for (size_t i = from; i < s.size(); ++i) {
    if (s[i] < '0' || s[i] > '9') return -1;
    v = v * 10 + (s[i] - '0');
  }
  return v <= 0xFFFFFFFFll ? v : -1;
}
}  // namespace

void DocIds::push(std::string id) {
  if (segs_.empty() || segs_.back().range) segs_.push_back(Seg{n_, 0, false, {}, explicit_.size()});
  explicit_.push_back(std::move(id));
  explicit_rows_.push_back(n_);
  ++segs_.back().count;
  ++n_;
}

void DocIds::push_range(const std::string& prefix, uint32_t count) {
  if (count == 0) return;
  segs_.push_back(Seg{n_, count, true, prefix, 0});
  n_ += count;
}

const DocIds::Seg& DocIds::seg_of(uint32_t row) const {
  auto it = std::upper_bound(segs_.begin(), segs_.end(), row, [](uint32_t r, const Seg& s) { return r < s.row0; });
  return *(it - 1);
}

std::string DocIds::at(uint32_t row) const {
  const Seg& s = seg_of(row);
  return s.range ? s.prefix + std::to_string(row) : explicit_[s.first + (row - s.row0)];
}

const char* DocIds::c_str(uint32_t row) const {
  const Seg& s = seg_of(row);
  if (!s.range) return explicit_[s.first + (row - s.row0)].c_str();
  thread_local std::string buf;
  buf = s.prefix + std::to_string(row);
  return buf.c_str();
}

int64_t DocIds::find(const std::string& id) const {
  for (const Seg& s : segs_) {  // ranges: prefix + canonical decimal row inside the range
    if (!s.range || id.compare(0, s.prefix.size(), s.prefix) != 0) continue;
    const int64_t r = parse_row(id, s.prefix.size());
    if (r >= s.row0 && r < int64_t{s.row0} + s.count) return r;
  }
  if (explicit_.empty()) return -1;
  for (; mapped_ < explicit_.size(); ++mapped_)  // index the explicit ids added since the last lookup
    map_.emplace(explicit_[mapped_], explicit_rows_[mapped_]);
  auto it = map_.find(id);
  return it == map_.end() ? -1 : static_cast<int64_t>(it->second);
}

int64_t DocIds::first_collision(const std::string& prefix, uint32_t row0, uint32_t count) const {
  int64_t best = -1;
  auto consider = [&](int64_t r) {
    if (r >= row0 && r < int64_t{row0} + count && (best < 0 || r < best)) best = r;
  };
  for (const std::string& e : explicit_)  // explicit ids of the form prefix + row
    if (e.compare(0, prefix.size(), prefix) == 0) consider(parse_row(e, prefix.size()));
  for (const Seg& s : segs_) {
    if (!s.range) continue;
    // ids prefix + r (new) vs s.prefix + r' (existing): equal only if one
    // prefix extends the other by digits.  Same prefix: rows differ.
    if (s.prefix == prefix) continue;
    const bool new_longer = prefix.size() > s.prefix.size();
    const std::string& lo = new_longer ? s.prefix : prefix;
    const std::string& hi = new_longer ? prefix : s.prefix;
    if (hi.compare(0, lo.size(), lo) != 0) continue;
    const std::string extra = hi.substr(lo.size());
    if (extra.find_first_not_of("0123456789") != std::string::npos || extra[0] == '0') continue;
    if (new_longer) {  // new id = lo + extra + r; an existing row r' = extra + r
      for (uint32_t i = 0; i < count; ++i) {
        const int64_t rp = parse_row(extra + std::to_string(row0 + i), 0);
        if (rp >= s.row0 && rp < int64_t{s.row0} + s.count) {
          consider(row0 + i);
          break;
        }
      }
    } else {  // existing id = lo + extra + r'; a new row r = extra + r'
      for (uint32_t i = 0; i < s.count; ++i) consider(parse_row(extra + std::to_string(s.row0 + i), 0));
    }
  }
  return best;
}

void DocIds::clear() {
  segs_.clear();
  explicit_.clear();
  explicit_rows_.clear();
  map_.clear();
  mapped_ = 0;
  n_ = 0;
}

// ---------------------------------------------------------------------------
// HYREIDN1 index file -- corpus.cpp:144-201, checksummed IO common.hpp:35-162.
// Layout: magic u64, version u32, C, A, d, num_bits u32, seed u64, N u32,
// attributes, offsets, embeddings, signatures, zero flags, N doc-id strings,
// C clause-name strings (u32 length + bytes), then FNV-1a-64 of all of it.
// ---------------------------------------------------------------------------
namespace {
constexpr uint64_t kMagic = 0x314e444945525948ull;  // "HYREIDN1" little-endian
constexpr uint32_t kVersion = 1;
constexpr uint64_t kFnvBasis = 0xcbf29ce484222325ull;

uint64_t fnv(const void* p, size_t n, uint64_t h) {
  auto* b = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < n; ++i) {
    h ^= b[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

struct Writer {
  std::ofstream out;
  uint64_t sum = kFnvBasis;
  explicit Writer(const std::string& p) : out(p, std::ios::binary) {
    if (!out) throw Error(HYRE_INTERNAL, "cannot open for write: " + p);
  }
  void bytes(const void* d, size_t n) {
    if (!n) return;
    out.write(static_cast<const char*>(d), static_cast<std::streamsize>(n));
    sum = fnv(d, n, sum);
  }
  template <class T> void pod(T v) { bytes(&v, sizeof v); }
  template <class T> void vec(const std::vector<T>& v) { bytes(v.data(), v.size() * sizeof(T)); }
  void str(const std::string& s) {
    pod<uint32_t>(static_cast<uint32_t>(s.size()));
    bytes(s.data(), s.size());
  }
  void finish() {
    uint64_t s = sum;
    out.write(reinterpret_cast<const char*>(&s), sizeof s);
    out.close();
    if (!out) throw Error(HYRE_INTERNAL, "write failed on close");
  }
};

struct Reader {
  std::ifstream in;
  uint64_t remaining = 0, sum = kFnvBasis;
  explicit Reader(const std::string& p) : in(p, std::ios::binary) {
    if (!in) throw Error(HYRE_LOAD_ERROR, "cannot open for read: " + p, HYRE_LOAD_TRUNCATED);
    in.seekg(0, std::ios::end);
    remaining = static_cast<uint64_t>(in.tellg());
    in.seekg(0, std::ios::beg);
    if (remaining < 8)
      throw Error(HYRE_LOAD_ERROR, "file shorter than its checksum: " + p, HYRE_LOAD_TRUNCATED);
    remaining -= 8;
  }
  void bytes(void* d, size_t n) {
    if (n > remaining)
      throw Error(HYRE_LOAD_ERROR,
                  "truncated file: need " + std::to_string(n) + " more bytes, have " +
                      std::to_string(remaining),
                  HYRE_LOAD_TRUNCATED);
    if (!n) return;
    in.read(static_cast<char*>(d), static_cast<std::streamsize>(n));
    if (!in) throw Error(HYRE_LOAD_ERROR, "read failed mid-file", HYRE_LOAD_TRUNCATED);
    remaining -= n;
    sum = fnv(d, n, sum);
  }
  template <class T> T pod() {
    T v{};
    bytes(&v, sizeof v);
    return v;
  }
  template <class T> void vec(std::vector<T>& v, size_t n) {
    v.resize(n);
    bytes(v.data(), n * sizeof(T));
  }
  std::string str() {
    auto n = pod<uint32_t>();
    std::string s(n, '\0');
    bytes(s.data(), n);
    return s;
  }
  void verify() {
    if (remaining != 0)
      throw Error(HYRE_LOAD_ERROR, "trailing bytes before checksum", HYRE_LOAD_TRUNCATED);
    uint64_t stored = 0;
    in.read(reinterpret_cast<char*>(&stored), sizeof stored);
    if (!in) throw Error(HYRE_LOAD_ERROR, "missing checksum", HYRE_LOAD_TRUNCATED);
    if (stored != sum) throw Error(HYRE_LOAD_ERROR, "checksum mismatch", HYRE_LOAD_CHECKSUM);
  }
};
}  // namespace

void save(const Frozen& f, const std::string& path) {
  Writer w(path);
  w.pod(kMagic);
  w.pod(kVersion);
  w.pod(f.num_clauses);
  w.pod(f.max_num_attr);
  w.pod(f.dim);
  w.pod(f.num_bits);
  w.pod(f.seed);
  w.pod(f.num_docs);
  w.vec(f.attributes);
  w.vec(f.offsets);
  w.vec(f.embeddings);
  w.vec(f.signatures);
  w.vec(f.zero);
  for (uint32_t r = 0; r < f.num_docs; ++r) w.str(f.doc_ids.at(r));
  for (const auto& s : f.clause_names) w.str(s);
  w.finish();
}

Frozen* load(const std::string& path) {
  Reader r(path);
  if (r.pod<uint64_t>() != kMagic)
    throw Error(HYRE_LOAD_ERROR, "not an index file: " + path, HYRE_LOAD_BAD_MAGIC);
  const auto version = r.pod<uint32_t>();
  if (version != kVersion)
    throw Error(HYRE_LOAD_ERROR,
                "index version " + std::to_string(version) + " unsupported (expected " +
                    std::to_string(kVersion) + ")",
                HYRE_LOAD_VERSION_MISMATCH);
  std::unique_ptr<Frozen> f(new Frozen);
  f->num_clauses = r.pod<uint32_t>();
  f->max_num_attr = r.pod<uint32_t>();
  f->dim = r.pod<uint32_t>();
  f->num_bits = r.pod<uint32_t>();
  f->seed = r.pod<uint64_t>();
  f->num_docs = r.pod<uint32_t>();
  make_codec(f->dim, f->num_bits, f->seed);  // the reference re-derives (and validates) it
  const size_t n = f->num_docs;
  r.vec(f->attributes, n * f->max_num_attr);
  r.vec(f->offsets, n * (f->num_clauses + 1));
  r.vec(f->embeddings, n * f->dim);
  r.vec(f->signatures, n * f->num_words());
  r.vec(f->zero, n);
  for (size_t i = 0; i < n; ++i) f->doc_ids.push(r.str());
  for (uint32_t c = 0; c < f->num_clauses; ++c) f->clause_names.push_back(r.str());
  r.verify();
  return f.release();
}

// ---------------------------------------------------------------------------
// Queries
// ---------------------------------------------------------------------------
void validate_query(const QueryShape& s, const hyre_query& q) {
  if (q.k < 1) validation("k must be >= 1");
  if (q.granularity < 1) validation("granularity must be >= 1");
  if (q.embedding && q.embedding_dim != s.dim)
    validation("embedding: expected dim " + std::to_string(s.dim) + ", got " +
               std::to_string(q.embedding_dim));
  for (uint32_t c = 0; c < q.n_clauses; ++c) {
    const uint32_t slot = q.slots[c];
    if (slot >= s.num_clauses) validation("unknown clause slot " + std::to_string(slot));
    if (c > 0 && slot <= q.slots[c - 1]) validation("clause slots must be ascending and unique");
    const uint32_t b = q.id_offsets[c], e = q.id_offsets[c + 1];
    if (e <= b) validation("clause " + std::to_string(slot) + " has no attribute ids");
    for (uint32_t i = b; i < e; ++i) {
      if (q.ids[i] == 0) validation("attribute id 0 is reserved for padding");
      if (i > b && q.ids[i] <= q.ids[i - 1])
        validation("clause attribute ids must be strictly increasing (use normalize_query)");
    }
  }
}

bool unit_embedding(const float* raw, uint32_t n, float* out) {
  double norm_sq = 0.0;
  for (uint32_t i = 0; i < n; ++i) norm_sq += static_cast<double>(raw[i]) * raw[i];
  if (norm_sq != 0.0 && std::abs(norm_sq - 1.0) > 1e-6) {
    const double inv = 1.0 / std::sqrt(norm_sq);
    for (uint32_t i = 0; i < n; ++i) out[i] = static_cast<float>(raw[i] * inv);
    return true;
  }
  std::copy(raw, raw + n, out);
  return false;
}

}  // namespace hyreb
