"""CPU: pins the numpy oracle (oracle/hyre_oracle.py) before it is trusted.

Every check compares against golden vectors produced by the compiled
reference itself (tests/golden/reference_fixtures.json, written by
tests/golden/make_golden.py from oracle/_ref) or against the reference's own
hand-written known-answer tests (proj/tests/*.cpp, cited per test).  The
oracle restates the reference's arithmetic, so agreement is bit-exact.
"""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

from oracle import hyre_oracle as O

FIX = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_fixtures.json")))


def unhex(xs):
    return np.asarray([int(x, 16) for x in xs], np.uint32).view(np.float32)


def digest(*arrays):
    import hashlib
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def test_mt19937_64_known_answer():
    r = O.MT19937_64(5489)
    assert r() == 14514284786278117030  # std::mt19937_64 default-seed first output
    r = O.MT19937_64(5489)
    for _ in range(9999):
        r()
    assert r() == 9981545732273789042  # [rand.predef]: 10000th output


@pytest.mark.parametrize("case", range(3))
def test_freeze_layout_matches_reference(case):
    fx = FIX["freeze"][case]
    spec = O.CorpusSpec(**fx["spec"])
    docs, fr = O.make_corpus(spec)
    assert fr.max_num_attr == fx["widest"]
    assert digest(fr.attributes, fr.offsets, fr.embeddings.view(np.uint32), fr.signatures, fr.zero) == fx["sha256"]
    assert [fr.doc_ids[0], fr.doc_ids[-1]] == fx["doc_ids"]


def test_appendix_fixture_layout():
    # test_corpus.cpp:50-69 / PAPER.md appendix table
    docs = [O.Doc("doc1", [[934, 2934], [945, 342, 3112]], np.array([1, 0, 0, 0], np.float32)),
            O.Doc("doc2", [[129], [9342, 234]], np.array([1, 0, 0, 0], np.float32))]
    fr = O.freeze(docs, 2, 5, 4, 64, 7)
    assert fr.attributes.tolist() == [[934, 2934, 342, 945, 3112], [129, 234, 9342, 0, 0]]
    assert fr.offsets.tolist() == [[0, 2, 5], [0, 1, 3]]


def test_normalization_and_zero_rows():
    # test_corpus.cpp:80-96
    docs = [O.Doc("a", [[1], [2]], np.array([3, 4, 0, 0], np.float32)),
            O.Doc("z", [[1], [2]], np.zeros(4, np.float32))]
    fr = O.freeze(docs, 2, 5, 4, 64, 7)
    assert fr.embeddings[0].tolist() == [np.float32(0.6), np.float32(0.8), 0.0, 0.0]
    assert fr.zero.tolist() == [0, 1] and not fr.embeddings[1].any()


def test_tbr_matches_reference():
    spec = O.CorpusSpec(num_docs=60, num_clauses=3, attr_universe=12)
    for fx in FIX["tbr"]:
        spec.seed = fx["seed"]
        docs, fr = O.make_corpus(spec)
        q = [(s, ids) for s, ids in fx["query"]]
        assert O.full_scan_tbr(fr, q).tolist() == fx["rows"]
        assert O.reference_tbr(docs, q).tolist() == fx["rows"]  # test_util.hpp hash-set oracle


def test_tbr_known_answers():
    # test_term_match.cpp:71-107
    docs = [O.Doc("doc1", [[934, 2934], [945, 342, 3112]], np.array([1, 0], np.float32)),
            O.Doc("doc2", [[129], [9342, 234]], np.array([0, 1], np.float32))]
    fr = O.freeze(docs, 2, 5, 2, 16, 7)
    nq = O.normalize_query
    assert O.full_scan_tbr(fr, nq({0: [129], 1: [234]}, 2)).tolist() == [1]
    assert O.full_scan_tbr(fr, nq({0: [129], 1: [945]}, 2)).tolist() == []
    assert O.full_scan_tbr(fr, nq({1: [234, 342]}, 2)).tolist() == [0, 1]
    assert O.full_scan_tbr(fr, nq({}, 2)).tolist() == [0, 1]
    sparse = O.freeze([O.Doc("sparse", [[7], []], np.array([1, 0], np.float32))], 2, 2, 2, 16, 7)
    assert O.full_scan_tbr(sparse, nq({1: [7]}, 2)).tolist() == []
    assert O.full_scan_tbr(sparse, nq({0: [7]}, 2)).tolist() == [0]


def test_batch_scan_stream_matches_reference():
    # pipeline.cpp:75-93 against streams the compiled reference produced
    spec = O.CorpusSpec(num_docs=60, num_clauses=3, attr_universe=12)
    for fx in FIX["batch_scan"]:
        spec.seed = fx["seed"]
        _, fr = O.make_corpus(spec)
        qs = [[(s, ids) for s, ids in q] for q in fx["queries"]]
        assert [list(p) for p in O.batch_scan_tbr(fr, qs, fx["batch_ids"])] == fx["stream"]


def test_batch_scan_known_answer():
    # test_pipeline.cpp:221-235: addressable corpus (row r holds id r + 1)
    docs = [O.Doc(f"doc{r}", [[r + 1]], np.ones(2, np.float32)) for r in range(10)]
    fr = O.freeze(docs, 1, 1, 2, 16, 3)
    qs = [O.normalize_query({0: [2, 3, 6]}, 1), O.normalize_query({0: [4, 6, 10]}, 1)]
    assert O.batch_scan_tbr(fr, qs, [0, 1]) == [(1, 0), (2, 0), (3, 1), (5, 0), (5, 1), (9, 1)]


def test_hybrid_and_quant_match_reference_bit_exactly():
    spec = O.CorpusSpec(num_docs=300, dim=12, num_clauses=2, attr_universe=10)
    for fx in FIX["hybrid"]:
        spec.seed = fx["seed"]
        docs, fr = O.make_corpus(spec)
        terms = [(s, ids) for s, ids in fx["terms"]]
        rows, sc = O.execute(fr, terms, unhex(fx["raw"]), fx["k"], fx["quant"], fx["quant_k"])
        assert rows.tolist() == fx["rows"]
        assert np.array_equal(sc.view(np.uint32), unhex(fx["scores"]).view(np.uint32))


def test_quant_preselection_matches_reference():
    q = FIX["quant"]
    docs, fr = O.make_corpus(O.CorpusSpec(**q["spec"]))
    for fx in q["cases"]:
        terms = [(s, ids) for s, ids in fx["terms"]]
        rows, sc = O.execute(fr, terms, unhex(fx["raw"]), fx["k"], True, fx["quant_k"])
        assert rows.tolist() == fx["rows"]
        assert np.array_equal(sc.view(np.uint32), unhex(fx["scores"]).view(np.uint32))


def test_codec_structure_matches_reference():
    for key, fx in FIX["codec"].items():
        d, b, s = map(int, key.split("_"))
        c = O.make_codec(d, b, s)
        assert len(c.rounds) == fx["n_rounds"]
        assert c.rounds[0][0].tolist() == fx["first_perm"]
        assert c.rounds[0][1].tolist() == fx["first_signs"]
        assert [r[2].tolist() for r in c.rounds[-2:]] == fx["bounds"]
    # test_quantizer.cpp:335-369
    assert len(O.make_codec(4, 512, 3).rounds) == 128
    assert O.make_codec(8, 12, 3).rounds[1][2].tolist() == [0, 2, 4, 6, 8]
    assert O.make_codec(10, 13, 3).rounds[1][2].tolist() == [0, 4, 7, 10]


def test_encode_matches_reference():
    for fx in FIX["encode"]:
        c = O.make_codec(fx["dim"], fx["bits"], fx["seed"])
        w = O.encode_rows(c, unhex(fx["x"]))[0]
        assert [f"{int(x):016x}" for x in w] == fx["words"]


def test_quant_score_known_answers():
    # test_quantizer.cpp:155-187
    a = np.asarray([0b0101], np.uint64)  # bits (1,0,1,0)
    b = np.asarray([0b1001], np.uint64)  # bits (1,0,0,1)
    assert O.quant_score_words(a, b[None, :], 4)[0] == 2
    assert O.quant_score_words(a, a[None, :], 4)[0] == 4


def test_top_k_matches_reference_bucket_selection():
    for fx in FIX["topk"]:
        rows, _ = O.top_k(np.arange(500), unhex(fx["scores"]), fx["k"], fx["g"])
        assert rows.tolist() == fx["rows"]
    # test_knn.cpp:94-143
    r, _ = O.top_k(np.arange(6), np.array([0.5, 0.7, 0.5, 0.7, 0.5, -0.2], np.float32), 4)
    assert r.tolist() == [1, 3, 0, 2]
    r, s = O.top_k(np.arange(4), np.array([1.0, -1.0, 0.0, 1.0], np.float32), 4)
    assert r.tolist() == [0, 3, 2, 1]
    with pytest.raises(O.DomainError):
        O.top_k(np.arange(2), np.array([0.5, 1.5], np.float32), 1)
    with pytest.raises(O.ValidationError):
        O.top_k(np.arange(2), np.array([0.5, 0.1], np.float32), 0)


def test_c1_workload_slice_matches_reference():
    fx = FIX["c1_slice"]
    offs, ids, emb = O.cnf_workload_docs(fx["n"], fx["dim"], fx["clauses"], fx["vocab"], fx["seed"])
    docs = []
    C = fx["clauses"]
    for i in range(fx["n"]):
        cl = [ids[offs[i * C + c]:offs[i * C + c + 1]].tolist() for c in range(C)]
        docs.append(O.Doc(f"d{i}", cl, emb[i]))
    fr = O.freeze(docs, C, 3 * C, fx["dim"], 512, 42)
    assert digest(fr.attributes, fr.offsets, fr.embeddings.view(np.uint32), fr.signatures, fr.zero) == fx["sha256"]
    for q in fx["queries"]:
        clauses = [(s, ids) for s, ids in q["query"]]
        assert len(O.full_scan_tbr(fr, clauses)) == q["n_tbr"]
        rows, sc = O.execute(fr, clauses, unhex(q["emb"]), 100, quant_enabled=False)
        assert rows.tolist() == q["rows"]
        assert np.array_equal(sc.view(np.uint32), unhex(q["scores"]).view(np.uint32))


def test_normalize_query_messages_match_reference():
    for name, raw, nc in [("unknown_slot", {2: [1]}, 2), ("zero_id", {0: [0]}, 2)]:
        with pytest.raises(O.ValidationError) as e:
            O.normalize_query(raw, nc)
        assert str(e.value) == FIX["messages"][name]
