// C++ drop-in check: the reference's own test patterns (proj/tests/
// test_corpus.cpp, test_term_match.cpp, test_pipeline.cpp) written against
// include/hyre_b200.hpp -- i.e. what the reference's callers see after
// relinking.  Prints one [PASS]/[FAIL] line per check (acceptance.cpp style);
// exit code = failures.  `--host-only` skips the checks that need a GPU.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>

#include "hyre_b200.hpp"

using namespace hyre;

static int failures = 0;
#define CHECK(name, cond)                                                         \
  do {                                                                            \
    const bool ok_ = (cond);                                                      \
    std::printf("[%s] %s\n", ok_ ? "PASS" : "FAIL", name);                      \
    failures += ok_ ? 0 : 1;                                                      \
  } while (0)

template <class E, class F>
static bool throws_with(F&& f, const std::string& msg) {
  try {
    f();
  } catch (const E& e) {
    return msg.empty() || msg == e.what();
  }
  return false;
}

static FrozenIndex appendix_index() {
  IndexBuilder b({2, 5, 2, {"geo", "skill"}});
  b.add_document({"doc1", {{934, 2934}, {945, 342, 3112}}, {1.0f, 0.0f}});
  b.add_document({"doc2", {{129}, {9342, 234}}, {0.0f, 1.0f}});
  return std::move(b).freeze(make_codec(2, 16, 7));
}

// row r carries attribute r + 1 (test_pipeline.cpp:24-45)
static FrozenIndex addressable(std::uint32_t n, std::uint32_t dim = 8) {
  std::mt19937_64 rng(3);
  IndexBuilder b({1, 1, dim, {}});
  for (std::uint32_t r = 0; r < n; ++r) {
    std::vector<float> e(dim);
    double ss = 0;
    for (auto& x : e) {
      x = static_cast<float>(2.0 * (static_cast<double>(rng() >> 11) * 0x1.0p-53) - 1.0);
      ss += double(x) * x;
    }
    for (auto& x : e) x = static_cast<float>(x / std::sqrt(ss));
    b.add_document({"doc" + std::to_string(r), {{r + 1}}, e});
  }
  return std::move(b).freeze(make_codec(dim, 64, 503));
}

int main(int argc, char** argv) {
  const bool host_only = argc > 1 && std::strcmp(argv[1], "--host-only") == 0;
  const FrozenIndex idx = appendix_index();
  auto a0 = idx.attribute_row(0), a1 = idx.attribute_row(1);
  CHECK("appendix layout (test_corpus.cpp:50-69)",
        std::vector<std::uint32_t>(a0.begin(), a0.end()) == std::vector<std::uint32_t>({934, 2934, 342, 945, 3112}) &&
            std::vector<std::uint32_t>(a1.begin(), a1.end()) == std::vector<std::uint32_t>({129, 234, 9342, 0, 0}));
  CHECK("doc id mapping", idx.doc_id(1) == "doc2" && idx.row_of("doc1") == 0u && !idx.row_of("nope"));
  CHECK("clause slots by name", idx.resolve_clause_slot("skill") == 1 && idx.resolve_clause_slot("x") == -1);
  CHECK("duplicate docId message", throws_with<ValidationError>(
                                       [] {
                                         IndexBuilder b({2, 5, 4, {}});
                                         b.add_document({"dup", {{1}, {2}}, {1, 0, 0, 0}});
                                         b.add_document({"dup", {{3}, {4}}, {1, 0, 0, 0}});
                                       },
                                       "duplicate docId: dup"));
  CHECK("no documents staged", throws_with<ValidationError>(
                                   [] { IndexBuilder b({2, 5, 4, {}}); (void)std::move(b).freeze(make_codec(4, 64, 7)); },
                                   "no documents staged"));
  {  // ingestion (dataio.hpp:15-28) -> the appendix index, through the library's C++ parser
    const std::string dir = std::string(std::getenv("TMPDIR") ? std::getenv("TMPDIR") : "/tmp");
    const std::string sp = dir + "/hyre_api_schema.json", cp = dir + "/hyre_api_docs.jsonl";
    std::FILE* f = std::fopen(sp.c_str(), "w");
    std::fputs("{\"clauses\": [\"geo\", \"skill\"], \"dim\": 2}", f);
    std::fclose(f);
    f = std::fopen(cp.c_str(), "w");
    std::fputs("{\"id\": \"doc1\", \"clauses\": {\"geo\": [934, 2934], \"skill\": [945, 342, 3112]}, "
               "\"embedding\": [1, 0]}\n\n{\"id\": \"doc2\", \"clauses\": {\"skill\": [9342, 234], \"geo\": [129]}, "
               "\"embedding\": [0.0, 1e0]}\n", f);
    std::fclose(f);
    const IngestSchema schema = read_schema_json(sp);
    const auto docs = read_documents_jsonl(cp, schema);
    CHECK("read_schema_json / read_documents_jsonl (dataio.hpp:20-28)",
          schema.clause_names == std::vector<std::string>({"geo", "skill"}) && schema.dim == 2 && docs.size() == 2 &&
              docs[1].doc_id == "doc2" && docs[1].clauses[0] == std::vector<std::uint32_t>({129}) &&
              docs[1].embedding == std::vector<float>({0.0f, 1.0f}));
    const FrozenIndex built = build_index_jsonl(sp, cp, 16, 7);
    auto b0 = built.attribute_row(0);
    CHECK("hyre build from JSONL = the appendix layout",
          built.max_num_attr() == 5 &&
              std::vector<std::uint32_t>(b0.begin(), b0.end()) == std::vector<std::uint32_t>({934, 2934, 342, 945, 3112}) &&
              built.resolve_clause_slot("skill") == 1);
    f = std::fopen(cp.c_str(), "w");
    std::fputs("{\"id\": \"a\"}\n{\"id\": \"b\", \"clauses\": {\"salary\": [1]}}\n", f);
    std::fclose(f);
    CHECK("ingest errors name file and line",
          throws_with<ValidationError>([&] { read_documents_jsonl(cp, schema); }, cp + ":2: unknown clause 'salary'"));
  }
  const CnfQuery q = normalize_query({{1, {9, 3, 9, 1}}}, 2);
  CHECK("normalize_query sorts + dedups", q.clauses.size() == 1 && q.clauses[0].attribute_ids ==
                                                                       std::vector<std::uint32_t>({1, 3, 9}));
  CHECK("normalize_query unknown slot", throws_with<ValidationError>([] { normalize_query({{2, {1}}}, 2); },
                                                                     "unknown clause slot 2 (index has 2)"));
  HybridQuery bad;
  bad.embedding = std::vector<float>{1.0f};
  const FrozenIndex addr = addressable(10);
  CHECK("validate_query names the field",
        throws_with<ValidationError>([&] { validate_query(addr, bad); }, "embedding: expected dim 8, got 1"));
  const std::string path = "/tmp/hyre_api_parity.bin";
  idx.save(path);
  const FrozenIndex back = FrozenIndex::load(path);
  CHECK("save/load round trip", back.num_docs() == 2 && back.doc_id(0) == "doc1");
  if (host_only) return failures;

  // ---- device path ----
  auto rows = [](const std::vector<Messenger>& ms) {
    std::vector<std::uint32_t> r;
    for (auto& m : ms) r.push_back(m.row_id);
    return r;
  };
  CHECK("conjunctive scan (test_term_match.cpp:71-89)",
        rows(full_scan_tbr(idx, normalize_query({{0, {129}}, {1, {234}}}, 2))) == std::vector<std::uint32_t>({1}) &&
            full_scan_tbr(idx, normalize_query({{0, {129}}, {1, {945}}}, 2)).empty() &&
            rows(full_scan_tbr(idx, normalize_query({{1, {234, 342}}}, 2))) == std::vector<std::uint32_t>({0, 1}));
  {
    const std::vector<CnfQuery> bq{normalize_query({{0u, {2, 3, 6}}}, 1), normalize_query({{0u, {4, 6, 10}}}, 1)};
    const std::vector<std::uint32_t> bid{0, 1};
    const auto ms = batch_scan_tbr(addr, bq, bid);
    std::vector<std::pair<std::uint32_t, std::uint32_t>> got;
    for (const auto& m : ms) got.emplace_back(m.row_id, m.batch_id);
    CHECK("batch scan stream (test_pipeline.cpp:221-235)",
          got == (std::vector<std::pair<std::uint32_t, std::uint32_t>>{{1, 0}, {2, 0}, {3, 1}, {5, 0}, {5, 1}, {9, 1}}));
  }
  HybridQuery term_only;
  term_only.terms = normalize_query({{0u, {8, 3, 6}}}, 1);
  term_only.k = 2;
  const TopKResult r = execute(addr, term_only);
  CHECK("term-only rows ascending (test_pipeline.cpp:100-112)",
        r.hits.size() == 2 && r.hits[0].row_id == 2 && r.hits[1].row_id == 5 && r.hits[0].score == 0.0f &&
            r.hits[0].doc_id == "doc2");
  Executor ex(addr, 4);
  BatchRequest batch;
  batch.queries.push_back(term_only);
  HybridQuery k0;
  k0.k = 0;
  batch.queries.push_back(k0);
  HybridQuery hybrid;
  hybrid.embedding = std::vector<float>(addr.embedding_row(7).begin(), addr.embedding_row(7).end());
  hybrid.k = 3;
  hybrid.options.quant_enabled = false;
  batch.queries.push_back(hybrid);
  const auto outs = ex.execute_batch(batch);
  CHECK("malformed query fails its slot (test_pipeline.cpp:277-298)",
        outs[0].ok && !outs[1].ok && outs[1].error == "k must be >= 1" && outs[2].ok);
  CHECK("self-similarity ranks first", outs[2].result.hits.size() == 3 && outs[2].result.hits[0].row_id == 7 &&
                                           outs[2].result.hits[0].score >= 0.999999f);
  StageTimings t;
  (void)ex.execute(hybrid, &t);
  CHECK("stage timings populated", t.total_ms > 0.0 && t.total_ms >= t.tbr_ms);

  // ---- the same index row-sharded (DeviceOptions: 3 shards, here all on
  // device 0; HYRE_GPUS=N picks devices 0..N-1): identical results ----
  FrozenIndex shard3 = addressable(10);
  DeviceOptions three;
  three.devices = {0, 0, 0};
  shard3.set_device_options(three);
  Executor sex(shard3, 4);
  const auto souts = sex.execute_batch(batch);
  bool same = souts.size() == outs.size();
  for (std::size_t i = 0; same && i < outs.size(); ++i) {
    same = souts[i].ok == outs[i].ok && souts[i].error == outs[i].error &&
           souts[i].result.hits.size() == outs[i].result.hits.size();
    for (std::size_t j = 0; same && j < outs[i].result.hits.size(); ++j)
      same = souts[i].result.hits[j].row_id == outs[i].result.hits[j].row_id &&
             souts[i].result.hits[j].score == outs[i].result.hits[j].score &&
             souts[i].result.hits[j].doc_id == outs[i].result.hits[j].doc_id;
  }
  CHECK("sharded executor == single-GPU executor (SURVEY 8e)", same && sex.sharded_handle() != nullptr);
  CHECK("device options fixed after the first executor",
        throws_with<ValidationError>([&] { shard3.set_device_options(DeviceOptions{}); }, ""));
  return failures;
}
