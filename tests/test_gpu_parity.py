"""GPU parity: the CUDA path (through the C-ABI) against the oracle.

Mirrors the reference's hot-path suites (proj/tests/test_term_match.cpp,
test_knn.cpp, test_pipeline.cpp, acceptance.cpp #1/#2/#4/#5) with the
tolerance policy of tests/parity.py for floating-point scores and bit-exact
checks for eligibility sets, term-only row lists and quant survivor sets.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import hyre_oracle as O
from tests.helpers import corpus_pair, hits, product_index, to_cnf
from tests.parity import assert_topk_match

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hy():
    import paper_2402_13435_b200 as hy
    return hy


def appendix_index(hy):
    b = hy.IndexBuilder(hy.IndexConfig(2, 5, 2, ["geo", "skill"]))
    b.add_document(hy.DocumentInput("doc1", [[934, 2934], [945, 342, 3112]], [1.0, 0.0]))
    b.add_document(hy.DocumentInput("doc2", [[129], [9342, 234]], [0.0, 1.0]))
    return b.freeze(hy.make_codec(2, 16, 7))


def rows_of(ms):
    return [m.row_id for m in ms]


# ---------------------------------------------------------------- term match
def test_conjunctive_scan_on_the_two_document_fixture(hy):
    # test_term_match.cpp:71-89
    index = appendix_index(hy)
    assert rows_of(hy.full_scan_tbr(index, hy.normalize_query({0: [129], 1: [234]}, 2))) == [1]
    assert hy.full_scan_tbr(index, hy.normalize_query({0: [129], 1: [945]}, 2)) == []
    assert rows_of(hy.full_scan_tbr(index, hy.normalize_query({1: [234, 342]}, 2))) == [0, 1]
    assert rows_of(hy.full_scan_tbr(index, hy.normalize_query({}, 2))) == [0, 1]


def test_a_clause_over_an_empty_slot_cannot_match(hy):
    # test_term_match.cpp:91-107
    b = hy.IndexBuilder(hy.IndexConfig(2, 2, 2))
    b.add_document(hy.DocumentInput("sparse", [[7], []], [1.0, 0.0]))
    index = b.freeze(hy.make_codec(2, 16, 7))
    assert hy.full_scan_tbr(index, hy.normalize_query({1: [7]}, 2)) == []
    assert rows_of(hy.full_scan_tbr(index, hy.normalize_query({0: [7]}, 2))) == [0]


def test_messengers_carry_the_requested_batch_id(hy):
    index = appendix_index(hy)
    ms = hy.full_scan_tbr(index, hy.normalize_query({}, 2), 3)
    assert len(ms) == 2 and all(m.batch_id == 3 and m.score == 0.0 for m in ms)


def test_full_scan_agrees_with_hash_set_reference_on_random_corpora(hy):
    # test_term_match.cpp:119-132 (200 corpora, bit-exact row sets)
    spec = O.CorpusSpec(num_docs=60, num_clauses=3, attr_universe=12)
    rng = O.MT19937_64(99)
    for trial in range(200):
        spec.seed = 1000 + trial
        docs, ref, prod = corpus_pair(spec)
        q = O.random_query(spec, rng)
        got = rows_of(hy.full_scan_tbr(prod, to_cnf(q)))
        assert got == O.reference_tbr(docs, q).tolist(), trial


def test_tbr_bitexact_large_mixed_bitmap_and_csr_terms(hy):
    # 200K rows, Zipf-like id popularity so both dense (bitmap) and sparse (CSR) terms occur.
    n, C = 200_000, 3
    rs = np.random.default_rng(5)
    docs = []
    for i in range(n):
        cl = []
        for c in range(C):
            k = rs.integers(0, 4)
            cl.append((1 + np.minimum(rs.zipf(1.3, size=k), 5000)).tolist())
        docs.append(O.Doc(f"d{i}", cl, np.ones(4, np.float32)))
    width = max(sum(len(set(c)) for c in d.clauses) for d in docs)
    prod = product_index(docs, C, width, 4, 64, 1)
    ref = O.freeze(docs, C, width, 4, 64, 1)
    st = prod.device().stats()
    assert st["bitmap_terms"] > 0 and st["csr_terms"] > 0, st
    for t in range(12):
        raw = {c: (1 + np.minimum(rs.zipf(1.3, size=rs.integers(1, 6)), 5000)).tolist()
               for c in range(C) if rs.random() < 0.7}
        q = O.normalize_query(raw, C)
        got = prod.device() and hy.Executor(prod, 4).full_scan_rows(to_cnf(q))
        assert np.array_equal(got, O.full_scan_tbr(ref, q)), t


# ---------------------------------------------------------------- scoring / selection
def test_exact_scores_within_tolerance_and_renorm_flag(hy):
    spec = O.CorpusSpec(num_docs=40, dim=8, num_clauses=1, seed=9)
    docs, ref, prod = corpus_pair(spec)
    raw = np.zeros(8, np.float32)
    raw[0], raw[1] = 3.0, 4.0
    all_ = [hy.Messenger(r, 0) for r in range(40)]
    s = hy.exact_scores(prod, raw, all_)
    assert s.query_was_renormalized
    want, _ = O.exact_scores(ref, raw, np.arange(40))
    got = np.asarray([m.score for m in s.items], np.float32)
    assert np.all(np.abs(got - want) <= np.maximum(1e-3 * np.abs(want), 2e-5))
    u = O.random_unit_vector(8, O.MT19937_64(2))
    assert not hy.exact_scores(prod, u, all_).query_was_renormalized
    with pytest.raises(hy.ValidationError, match="query embedding dim 2 != index dim 8"):
        hy.exact_scores(prod, [1.0, 0.0], [])


def test_scores_stay_inside_unit_interval_for_self_similarity(hy):
    spec = O.CorpusSpec(num_docs=40, dim=8, num_clauses=1, seed=9)
    docs, ref, prod = corpus_pair(spec)
    all_ = [hy.Messenger(r, 0) for r in range(40)]
    for r in range(40):
        s = hy.exact_scores(prod, prod.embedding_row(r), all_)
        sc = np.asarray([m.score for m in s.items])
        assert (sc <= 1.0).all() and (sc >= -1.0).all()
        assert s.items[r].score >= 0.999999


def _scored(hy, scores):
    return hy.ScoredMessengers([hy.Messenger(r, 0, float(np.float32(s))) for r, s in enumerate(scores)])


def test_bucket_selection_known_answers(hy):
    # test_knn.cpp:94-143
    spec = O.CorpusSpec(num_docs=8, dim=8, num_clauses=1)
    _, _, prod = corpus_pair(spec)
    top = hy.bucket_top_k(prod, _scored(hy, [0.9, 0.1, 0.5]), 2)
    assert [h.row_id for h in top.hits] == [0, 2]
    assert [h.score for h in top.hits] == [np.float32(0.9), np.float32(0.5)]
    assert top.hits[0].doc_id == prod.doc_id(0)
    assert [h.row_id for h in hy.bucket_top_k(prod, _scored(hy, [0.5, 0.7, 0.5, 0.7, 0.5, -0.2]), 4).hits] == [1, 3, 0, 2]
    assert [h.row_id for h in hy.bucket_top_k(prod, _scored(hy, [0.1, 0.9, 0.4]), 10).hits] == [1, 2, 0]
    assert hy.bucket_top_k(prod, hy.ScoredMessengers(), 5).hits == []
    with pytest.raises(hy.ValidationError):
        hy.bucket_top_k(prod, _scored(hy, [0.1, 0.2, 0.3]), 0)
    with pytest.raises(hy.ValidationError):
        hy.bucket_top_k(prod, _scored(hy, [0.1, 0.2, 0.3]), 2, 0)
    with pytest.raises(hy.ScoreDomainError):
        hy.bucket_top_k(prod, _scored(hy, [0.5, 1.5]), 1)
    with pytest.raises(hy.ScoreDomainError):
        hy.bucket_top_k(prod, _scored(hy, [-1.01, 0.0]), 1)
    top = hy.bucket_top_k(prod, _scored(hy, [1.0, -1.0, 0.0, 1.0]), 4)
    assert [h.row_id for h in top.hits] == [0, 3, 2, 1]
    assert [h.score for h in top.hits] == [1.0, 1.0, 0.0, -1.0]


def test_bucket_selection_matches_full_sort_with_planted_ties(hy):
    # test_knn.cpp:145-171 -- selection is exact integer/float work: bit-exact.
    spec = O.CorpusSpec(num_docs=500, dim=8, num_clauses=1, seed=77)
    _, _, prod = corpus_pair(spec)
    rng = O.MT19937_64(123)
    for g in (1, 2, 100):
        for k in (1, 7, 100, 499, 500):
            s = np.asarray([np.float32(2.0 * O.unit_uniform(rng) - 1.0) for _ in range(500)], np.float32)
            s[17] = s[401] = s[88]
            top = hy.bucket_top_k(prod, _scored(hy, s), k, g)
            er, es = O.top_k(np.arange(500), s, k, g)
            assert [h.row_id for h in top.hits] == er.tolist()
            assert np.array_equal(np.asarray([h.score for h in top.hits], np.float32), es)


def test_bucket_selection_million_scores_k2000(hy):
    # acceptance.cpp:271-319 (#4): top-2000 of 1M random scores == full sort.
    spec = O.CorpusSpec(num_docs=8, dim=8, num_clauses=1)
    _, _, prod = corpus_pair(spec)
    ex = hy.Executor(prod, 1)
    rs = np.random.default_rng(555)
    n, k = 1_000_000, 2000
    s = (2.0 * rs.random(n) - 1.0).astype(np.float32)
    rows = np.arange(n, dtype=np.uint32)
    import ctypes as C
    from paper_2402_13435_b200 import _lib as L
    out = (L.hyre_hit * k)()
    cnt = C.c_uint32()
    rc = L.lib().hyre_bucket_top_k(ex._h, rows.ctypes.data_as(L.u32p), s.ctypes.data_as(L.f32p), n, k, 100, out,
                                   C.byref(cnt))
    assert rc == 0
    er, es = O.top_k(rows, s, k)
    assert [out[i].row for i in range(cnt.value)] == er.tolist()


# ---------------------------------------------------------------- pipeline
def addressable_corpus(hy, n, dim=8, seed=3):
    rng = O.MT19937_64(seed)
    docs = [O.Doc(f"doc{r}", [[r + 1]], O.random_unit_vector(dim, rng)) for r in range(n)]
    return docs, product_index(docs, 1, 1, dim, 64, seed + 500), O.freeze(docs, 1, 1, dim, 64, seed + 500)


def rows_query(hy, rows):
    return hy.normalize_query({0: [r + 1 for r in rows]}, 1)


def test_batch_scan_interleaves_by_row_then_batch_id(hy):
    # test_pipeline.cpp:221-235
    _, prod, _ = addressable_corpus(hy, 10)
    ms = hy.batch_scan_tbr(prod, [rows_query(hy, [1, 2, 5]), rows_query(hy, [3, 5, 9])], [0, 1])
    assert [(m.row_id, m.batch_id) for m in ms] == [(1, 0), (2, 0), (3, 1), (5, 0), (5, 1), (9, 1)]
    assert all(m.score == 0.0 for m in ms)


def test_batch_scan_matches_reference_streams(hy):
    # golden streams of the compiled reference's batch_scan_tbr
    import json
    fx_all = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_fixtures.json")))
    spec = O.CorpusSpec(num_docs=60, num_clauses=3, attr_universe=12)
    for fx in fx_all["batch_scan"]:
        spec.seed = fx["seed"]
        _, _, prod = corpus_pair(spec)
        qs = [to_cnf(q) for q in fx["queries"]]
        ms = hy.batch_scan_tbr(prod, qs, fx["batch_ids"])
        assert [[m.row_id, m.batch_id] for m in ms] == fx["stream"], fx["seed"]


@pytest.mark.parametrize("B", [3, 20, 130])
def test_batch_scan_large_batches_match_oracle(hy, B):
    # K1 (B <= 8) and the forward-list K1b (B > 8, two passes at 130) masks
    # feed the same stream; match-all and absent-id queries included
    n, C = 20_000, 3
    rs = np.random.default_rng(17)
    docs = [O.Doc(f"d{i}", [(1 + np.minimum(rs.zipf(1.4, size=rs.integers(0, 4)), 500)).tolist() for _ in range(C)],
                  np.ones(4, np.float32)) for i in range(n)]
    width = max(sum(len(set(c)) for c in d.clauses) for d in docs)
    prod = product_index(docs, C, width, 4, 64, 1)
    ref = O.freeze(docs, C, width, 4, 64, 1)
    qs = []
    for i in range(B):
        raw = {} if i % 11 == 5 else ({0: [99_999]} if i % 13 == 7 else
                                        {c: (1 + np.minimum(rs.zipf(1.4, size=rs.integers(1, 4)), 500)).tolist()
                                         for c in range(C) if rs.random() < 0.6})
        qs.append(O.normalize_query(raw, C))
    ids = [1000 + 3 * i for i in range(B)]
    got = hy.Executor(prod, max_batch=B).batch_scan_tbr([to_cnf(q) for q in qs], ids)
    expect = O.batch_scan_tbr(ref, qs, ids)
    assert len(got) == len(expect)
    assert [(m.row_id, m.batch_id) for m in got] == expect


def test_term_only_queries_return_matches_in_row_order_with_zero_scores(hy):
    _, prod, _ = addressable_corpus(hy, 10)
    q = hy.HybridQuery(rows_query(hy, [7, 2, 5]), None, 2)
    r = hy.execute(prod, q)
    assert [h.row_id for h in r.hits] == [2, 5] and all(h.score == 0.0 for h in r.hits)
    q.k = 10
    assert [h.row_id for h in hy.execute(prod, q).hits] == [2, 5, 7]


def test_no_term_matches_yields_an_empty_result(hy):
    _, prod, _ = addressable_corpus(hy, 4)
    q = hy.HybridQuery(hy.normalize_query({0: [999]}, 1), O.random_unit_vector(8, O.MT19937_64(1)), 3)
    assert hy.execute(prod, q).hits == []


def test_hybrid_execution_equals_filter_score_full_sort(hy):
    # test_pipeline.cpp:124-150 (40 trials)
    spec = O.CorpusSpec(num_docs=300, dim=12, num_clauses=2, attr_universe=10)
    rng = O.MT19937_64(41)
    for trial in range(40):
        spec.seed = 500 + trial
        docs, ref, prod = corpus_pair(spec)
        terms = O.random_query(spec, rng)
        raw = np.asarray([np.float32(4.0 * O.unit_uniform(rng) - 2.0) for _ in range(spec.dim)], np.float32)
        q = hy.HybridQuery(to_cnf(terms), raw, 10, hy.ExecOptions(quant_enabled=False))
        gr, gs = hits(hy.execute(prod, q))
        er, es = O.execute(ref, terms, raw, 10, quant_enabled=False)
        assert_topk_match(ref, raw, gr, gs, er, es)


def test_exact_retrieval_acceptance_1(hy):
    # acceptance.cpp:78-119: 200 queries on a 10k x 64 index, k in [1, 20], some raw-scaled.
    spec = O.CorpusSpec(num_docs=10000, dim=64, num_clauses=2, max_attrs_per_clause=4, attr_universe=50,
                        num_bits=64, seed=11)
    docs, ref, prod = corpus_pair(spec)
    ex = hy.Executor(prod, 16)
    rng = O.MT19937_64(123)
    for t in range(200):
        terms = O.random_query(spec, rng)
        raw = O.random_unit_vector(spec.dim, rng)
        if t % 3 == 0:
            raw = raw * np.float32(1.75)
        k = 1 + rng() % 20
        q = hy.HybridQuery(to_cnf(terms), raw, k, hy.ExecOptions(quant_enabled=False))
        gr, gs = hits(ex.execute(q))
        er, es = O.execute(ref, terms, raw, k, quant_enabled=False)
        assert_topk_match(ref, raw, gr, gs, er, es)
        res = ex.execute(q)
        assert all(h.doc_id == prod.doc_id(h.row_id) for h in res.hits)


def test_quantized_preselection_is_bit_exact_with_the_reference(hy):
    # Quant survivors are integer work: the GPU survivor set must equal the
    # reference's nth_element selection, so hybrid results agree as usual.
    spec = O.CorpusSpec(num_docs=4000, dim=16, num_bits=256, num_clauses=1, max_attrs_per_clause=1,
                        attr_universe=2, seed=7)
    docs, ref, prod = corpus_pair(spec)
    rng = O.MT19937_64(13)
    for t in range(20):
        raw = O.random_unit_vector(spec.dim, rng)
        terms = O.normalize_query({0: [1]}, 1) if t % 2 else []
        qk = [60, 200, 1000, 0][t % 4]
        k = 1 + t
        q = hy.HybridQuery(to_cnf(terms), raw, k, hy.ExecOptions(quant_enabled=True, quant_k=qk))
        gr, gs = hits(hy.execute(prod, q))
        er, es = O.execute(ref, terms, raw, k, quant_enabled=True, quant_k=qk)
        assert_topk_match(ref, raw, gr, gs, er, es)


def test_preselect_keeps_exactly_the_top_quant_k(hy):
    # test_quantizer.cpp:220-277
    spec = O.CorpusSpec(num_docs=120, dim=16, num_bits=64, seed=31)
    docs, ref, prod = corpus_pair(spec)
    qvec = O.random_unit_vector(spec.dim, O.MT19937_64(8))
    qsig = hy.encode(prod.codec(), qvec)
    cands = [hy.Messenger(r, 0) for r in range(120)]
    kept = hy.preselect(prod, qsig, cands, 200)
    assert [m.row_id for m in kept] == list(range(120))
    for qk in (1, 7, 40, 119):
        kept = hy.preselect(prod, qsig, cands, qk)
        assert [m.row_id for m in kept] == O.preselect(ref, qsig.words, np.arange(120), qk).tolist()
    with pytest.raises(hy.ValidationError):
        hy.preselect(prod, qsig, cands, 0)


def test_batch_execution_matches_single_execution(hy):
    # test_pipeline.cpp:237-275 -- batch transparency is exact on the GPU too
    # (the same kernels score a row whatever batch it is in).
    spec = O.CorpusSpec(num_docs=250, dim=12, num_clauses=2, attr_universe=8)
    rng = O.MT19937_64(71)
    for trial in range(50):
        spec.seed = 900 + trial
        docs, ref, prod = corpus_pair(spec)
        ex = hy.Executor(prod, 8)
        b = 1 + rng() % 8
        batch = hy.BatchRequest()
        for _ in range(b):
            terms = O.random_query(spec, rng)
            emb = None
            if rng() % 4 != 0:
                emb = np.asarray([np.float32(2.0 * O.unit_uniform(rng) - 1.0) for _ in range(spec.dim)],
                                 np.float32)
            k = 1 + rng() % 12
            qe = rng() % 2 == 0
            qk = 20 + rng() % 100
            batch.queries.append(hy.HybridQuery(to_cnf(terms), emb, k, hy.ExecOptions(qe, qk)))
        outs = ex.execute_batch(batch)
        for q, o in zip(batch.queries, outs):
            assert o.ok
            single = ex.execute(q)
            assert [(h.row_id, h.score) for h in o.result.hits] == [(h.row_id, h.score) for h in single.hits]
            terms = [(c.slot, c.attribute_ids) for c in q.terms.clauses]
            er, es = O.execute(ref, terms, q.embedding, q.k, q.options.quant_enabled, q.options.quant_k)
            gr, gs = hits(o.result)
            if q.embedding is None:
                assert gr.tolist() == er.tolist()
            else:
                assert_topk_match(ref, q.embedding, gr, gs, er, es)


def test_a_malformed_query_fails_its_slot_not_the_batch(hy):
    _, prod, _ = addressable_corpus(hy, 10)
    ex = hy.Executor(prod, 4)
    batch = hy.BatchRequest([hy.HybridQuery(rows_query(hy, [1, 2]), None, 2), hy.HybridQuery(k=0),
                             hy.HybridQuery(rows_query(hy, [3]), None, 1)])
    outs = ex.execute_batch(batch)
    assert outs[0].ok and [h.row_id for h in outs[0].result.hits] == [1, 2]
    assert not outs[1].ok and outs[1].error == "k must be >= 1"
    assert outs[2].ok and [h.row_id for h in outs[2].result.hits] == [3]


def test_batch_size_limits_are_enforced(hy):
    _, prod, _ = addressable_corpus(hy, 4)
    ex = hy.Executor(prod, 2)
    with pytest.raises(hy.ValidationError):
        ex.execute_batch(hy.BatchRequest())
    with pytest.raises(hy.ValidationError, match="batch size 3 exceeds maxBatch 2"):
        ex.execute_batch(hy.BatchRequest([hy.HybridQuery(rows_query(hy, [1]), None, 1)] * 3))


def test_executor_scratch_does_not_leak_state_across_calls(hy):
    docs, prod, ref = addressable_corpus(hy, 60, 8, 21)
    reused = hy.Executor(prod, 4)
    rng = O.MT19937_64(17)
    for rnd in range(10):
        rows = [r for r in range(60) if rng() % 3 == 0] or [0]
        q = hy.HybridQuery(rows_query(hy, rows), O.random_unit_vector(8, rng), 5,
                           hy.ExecOptions(quant_enabled=(rnd % 2 == 0), quant_k=10))
        fresh = hy.Executor(prod, 4)
        assert reused.execute(q) == fresh.execute(q)
        a = reused.execute_batch(hy.BatchRequest([q, q, q]))
        b = fresh.execute_batch(hy.BatchRequest([q, q, q]))
        assert [(x.ok, x.result) for x in a] == [(x.ok, x.result) for x in b]


def test_zero_query_scores_everything_zero_rows_ascending(hy):
    _, prod, _ = addressable_corpus(hy, 50)
    q = hy.HybridQuery(hy.CnfQuery(), np.zeros(8, np.float32), 7, hy.ExecOptions(quant_enabled=False))
    r = hy.execute(prod, q)
    assert [h.row_id for h in r.hits] == list(range(7)) and all(h.score == 0.0 for h in r.hits)


def test_k_larger_than_corpus_returns_everything(hy):
    spec = O.CorpusSpec(num_docs=400, dim=16, num_bits=256, num_clauses=1, max_attrs_per_clause=1, attr_universe=2,
                        seed=7)
    docs, ref, prod = corpus_pair(spec)
    raw = O.random_unit_vector(16, O.MT19937_64(13))
    q = hy.HybridQuery(hy.CnfQuery(), raw, 1000, hy.ExecOptions(quant_enabled=False))
    gr, gs = hits(hy.execute(prod, q))
    er, es = O.execute(ref, [], raw, 1000, quant_enabled=False)
    assert len(gr) == 400
    assert_topk_match(ref, raw, gr, gs, er, es)


# ---------------------------------------------------------------- tensor-core batched scorer (K3)
def _cnf_index(hy, n, dim, C, V, max_ids, seed, dtype="f32"):
    from paper_2402_13435_b200 import workloads as W
    w = W.Workload("t", n, dim, C, V, 7, max_ids, 10, 16, "cnf", seed=seed, qseed=seed + 1)
    so, ids, emb = W.cnf_docs(w)
    b = hy.IndexBuilder(hy.IndexConfig(C, C * max_ids, dim))
    b.add_documents(so, ids, emb)
    prod = b.freeze(hy.make_codec(dim, 64, seed))
    ref = O.Frozen(n, C, C * max_ids, dim, 64, seed, np.array(prod.attributes), np.array(prod.offsets),
                   np.array(prod.embeddings), np.array(prod.signatures), np.array(prod.zero_flags))
    return w, prod, ref


@pytest.mark.parametrize("B,dim,dtype", [(16, 64, "f32"), (64, 128, "f32"), (200, 128, "f32"), (64, 128, "bf16"),
                                         (9, 256, "f32"), (256, 128, "bf16"), (300, 64, "f32")])
def test_tensor_core_batch_matches_oracle(hy, B, dim, dtype):
    from paper_2402_13435_b200 import workloads as W
    w, prod, ref = _cnf_index(hy, 70_000, dim, 4, 6, 3, 5)
    ex = hy.Executor(prod.device(0, dtype), max_batch=B)
    raws, qemb = W.queries(W.Workload("q", 0, dim, 4, 6, 2, 3, 10, B, "cnf", qseed=9), B)
    emb_scored = ref.embeddings
    if dtype == "bf16":
        import torch
        emb_scored = torch.from_numpy(ref.embeddings).to(torch.bfloat16).float().numpy()
    batch = hy.BatchRequest()
    for i, raw in enumerate(raws):
        clauses = [] if i % 5 == 0 else O.normalize_query(raw, 4)  # mix match-all + CNF
        k = [10, 100, 1, 257][i % 4]
        batch.queries.append(hy.HybridQuery(to_cnf(clauses), qemb[i] * (1.0 + (i % 3)), k,
                                            hy.ExecOptions(quant_enabled=False)))
    outs = ex.execute_batch(batch)
    for q, o in zip(batch.queries, outs):
        assert o.ok
        clauses = [(c.slot, c.attribute_ids) for c in q.terms.clauses]
        rows = O.full_scan_tbr(ref, clauses)
        qq, _ = O.unit_embedding(q.embedding)
        sc = O.scores_rows(emb_scored, qq, rows)
        er, es = O.top_k(rows, sc, q.k)
        gr, gs = hits(o.result)
        assert_topk_match(ref, q.embedding, gr, gs, er, es, emb_override=emb_scored)


@pytest.mark.parametrize("B,dtype", [(64, "f32"), (256, "bf16")])
def test_match_all_tensor_core_batch(hy, B, dtype):
    # A batch of match-all queries runs K3 with no eligibility pass at all
    # (every row of the shard eligible, the tail tile masked): exact against
    # the oracle's full scan and identical to single-query execution.
    from paper_2402_13435_b200 import workloads as W
    w, prod, ref = _cnf_index(hy, 50_003, 64, 4, 6, 3, 5)
    dev = prod.device(0, dtype)
    ex = hy.Executor(dev, max_batch=B)
    _, qemb = W.queries(W.Workload("q", 0, 64, 4, 6, 2, 3, 10, B, "cnf", qseed=33), B)
    emb_scored = ref.embeddings
    if dtype == "bf16":
        import torch
        emb_scored = torch.from_numpy(ref.embeddings).to(torch.bfloat16).float().numpy()
    batch = hy.BatchRequest([hy.HybridQuery(hy.CnfQuery(), qemb[i], [100, 7, 1000][i % 3],
                                            hy.ExecOptions(quant_enabled=False)) for i in range(B)])
    outs = ex.execute_batch(batch)
    rows = np.arange(ref.num_docs)
    single = hy.Executor(dev, max_batch=1)
    for i, (q, o) in enumerate(zip(batch.queries, outs)):
        assert o.ok
        qq, _ = O.unit_embedding(q.embedding)
        er, es = O.top_k(rows, O.scores_rows(emb_scored, qq, rows), q.k)
        gr, gs = hits(o.result)
        assert_topk_match(ref, q.embedding, gr, gs, er, es, emb_override=emb_scored)
        if i % 16 == 0 and os.environ.get("HYRE_PREFILTER") != "0":  # exact K2 rescoring only with a prefilter
            assert [(h.row_id, h.score) for h in o.result.hits] == [(h.row_id, h.score) for h in single.execute(q).hits]


@pytest.mark.parametrize("B", [1, 16])
def test_candidate_overflow_recovers(hy, B):
    # Scores increase with the row id, so the strided sample (early rows)
    # yields a weak threshold and the main pass overflows the candidate
    # buffer; the recovery rounds must still return exactly the last rows.
    n, dim = 1_000_000, 64
    emb = np.zeros((n, dim), np.float32)
    emb[:, 0] = np.arange(n, dtype=np.float32) / n
    emb[:, 1] = 1.0
    b = hy.IndexBuilder(hy.IndexConfig(1, 1, dim))
    b.add_documents(np.arange(n + 1, dtype=np.uint64), np.ones(n, np.uint32), emb)
    prod = b.freeze(hy.make_codec(dim, 64, 1))
    ex = hy.Executor(prod, max_batch=B)
    q = np.zeros(dim, np.float32)
    q[0] = 1.0
    outs = ex.execute_batch(hy.BatchRequest([hy.HybridQuery(hy.CnfQuery(), q, 50, hy.ExecOptions(False))] * B))
    ref = O.Frozen(n, 1, 1, dim, 64, 1, np.array(prod.attributes), np.array(prod.offsets),
                   np.array(prod.embeddings), np.array(prod.signatures), np.array(prod.zero_flags))
    rows = np.arange(n)
    sc = O.scores_rows(ref.embeddings, q, rows)
    er, es = O.top_k(rows, sc, 50)
    assert er.min() > 900_000  # the answer lives at the end of the index
    for o in outs:
        gr, gs = hits(o.result)
        assert_topk_match(ref, q, gr, gs, er, es)


@pytest.mark.parametrize("B", [9, 64, 130])
def test_batched_tbr_bitexact(hy, B):
    # Batches > 8 evaluate the CNF from the forward term lists (K1b); the row
    # sets must equal the oracle's full_scan_tbr bit for bit, including sparse
    # (CSR) terms, absent ids (empty clause), match-all and 2-pass batches.
    n, C = 60_000, 3
    rs = np.random.default_rng(11)
    docs = []
    for i in range(n):
        cl = [(1 + np.minimum(rs.zipf(1.3, size=rs.integers(0, 4)), 3000)).tolist() for _ in range(C)]
        docs.append(O.Doc(f"d{i}", cl, np.ones(4, np.float32)))
    width = max(sum(len(set(c)) for c in d.clauses) for d in docs)
    prod = product_index(docs, C, width, 4, 64, 1)
    ref = O.freeze(docs, C, width, 4, 64, 1)
    ex = hy.Executor(prod, max_batch=B)
    batch, expect = hy.BatchRequest(), []
    for i in range(B):
        if i % 17 == 0:
            raw = {}
        elif i % 23 == 0:
            raw = {1: [999_999]}  # id absent from the index
        else:
            raw = {c: (1 + np.minimum(rs.zipf(1.3, size=rs.integers(1, 5)), 3000)).tolist()
                   for c in range(C) if rs.random() < 0.7}
        q = O.normalize_query(raw, C)
        batch.queries.append(hy.HybridQuery(to_cnf(q), None, n))
        expect.append(O.full_scan_tbr(ref, q))
    outs = ex.execute_batch(batch)
    for o, e in zip(outs, expect):
        assert o.ok
        assert np.array_equal(np.asarray([h.row_id for h in o.result.hits], np.int64), e)


@pytest.mark.parametrize("B", [9, 64, 130])
def test_fused_cnf_eligibility_bitexact(hy, B):
    # Hybrid batches on the tensor-core path evaluate the CNF inside K3's
    # epilogue (fused, no mask pass).  With identical embeddings every
    # eligible row scores the same, so each query's top-k is exactly its
    # first k eligible rows (tie rule: row ascending) -- a bit-exact check of
    # the fused eligibility against full_scan_tbr, covering sparse terms,
    # rows with empty slots, absent ids, match-all and 2-group (B=130) batches.
    n, C, dim = 12_000, 3, 64
    rs = np.random.default_rng(5)
    e0 = np.zeros(dim, np.float32)
    e0[0], e0[1] = 0.6, 0.8
    docs = []
    for i in range(n):
        cl = [(1 + np.minimum(rs.zipf(1.3, size=rs.integers(0, 4)), 400)).tolist() for _ in range(C)]
        docs.append(O.Doc(f"d{i}", cl, e0))
    width = max(sum(len(set(c)) for c in d.clauses) for d in docs)
    prod = product_index(docs, C, width, dim, 64, 1)
    ref = O.freeze(docs, C, width, dim, 64, 1)
    ex = hy.Executor(prod, max_batch=B)
    batch, expect = hy.BatchRequest(), []
    q = np.zeros(dim, np.float32)
    q[1] = 1.0
    for i in range(B):
        if i % 17 == 0:
            raw = {}
        elif i % 23 == 0:
            raw = {1: [999_999]}  # id absent from the index
        else:
            raw = {c: (1 + np.minimum(rs.zipf(1.3, size=rs.integers(1, 5)), 400)).tolist()
                   for c in range(C) if rs.random() < 0.7}
        clauses = O.normalize_query(raw, C)
        k = 4096 if i % 3 else 1 + i
        batch.queries.append(hy.HybridQuery(to_cnf(clauses), q, k, hy.ExecOptions(quant_enabled=False)))
        expect.append(O.full_scan_tbr(ref, clauses)[:k])
    outs = ex.execute_batch(batch)
    for o, e in zip(outs, expect):
        assert o.ok
        gr, gs = hits(o.result)
        assert np.array_equal(gr, e), (len(gr), len(e))
        assert np.all(gs == gs[0]) if len(gs) else True


def test_executor_pool_batches_concurrent_requests(hy):
    # the ExecutorPool replacement groups concurrent single-query
    # requests into batches; every caller gets the oracle's answer for its own
    # query, and a malformed request fails alone (service.cpp:219-225).
    import threading
    from paper_2402_13435_b200 import workloads as W
    w, prod, ref = _cnf_index(hy, 70_000, 128, 4, 6, 3, 5)
    raws, qemb = W.queries(W.Workload("q", 0, 128, 4, 6, 2, 3, 10, 40, "cnf", qseed=19), 40)
    pool = hy.ExecutorPool(prod, workers=2, max_batch=16, max_wait_us=5000)
    queries = []
    for i, raw in enumerate(raws):
        clauses = [] if i % 7 == 0 else O.normalize_query(raw, 4)
        queries.append(hy.HybridQuery(to_cnf(clauses), qemb[i], [10, 100, 3][i % 3],
                                      hy.ExecOptions(quant_enabled=False)))
    bad = hy.HybridQuery(to_cnf([]), qemb[0], 0)  # k = 0
    results, errors = [None] * len(queries), []
    barrier = threading.Barrier(len(queries) + 1)

    def worker(i):
        barrier.wait()
        results[i] = pool.search(queries[i])

    def bad_worker():
        barrier.wait()
        try:
            pool.search(bad)
        except hy.ValidationError as e:
            errors.append(str(e))

    threads = [threading.Thread(target=worker, args=(i,)) for i in range(len(queries))]
    threads.append(threading.Thread(target=bad_worker))
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert errors == ["k must be >= 1"]
    batches, served = pool.stats()
    assert served == len(queries) + 1 and batches < served  # requests were batched
    for q, r in zip(queries, results):
        clauses = [(c.slot, c.attribute_ids) for c in q.terms.clauses]
        er, es = O.execute(ref, clauses, q.embedding, q.k, quant_enabled=False)
        gr, gs = hits(r)
        assert_topk_match(ref, q.embedding, gr, gs, er, es)
    pool.close()


# ---------------------------------------------------------------- K3 prefilter + exact rescore
def _singles(hy, ex, batch):
    return [[(h.row_id, h.score) for h in ex.execute(q).hits] for q in batch.queries]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_tensor_core_batch_equals_single_queries_exactly(hy, dtype):
    # Batches > 8 run K3, which admits rows on a bf16 prefilter score and
    # rescores the admitted rows with K2's exact arithmetic; single queries
    # run K2.  Batch transparency (test_pipeline.cpp:237-275) is therefore
    # exact -- identical rows AND scores -- for tensor-core batches too.
    from paper_2402_13435_b200 import workloads as W
    w, prod, ref = _cnf_index(hy, 70_000, 128, 4, 6, 3, 5)
    ex = hy.Executor(prod.device(0, dtype), max_batch=64)
    raws, qemb = W.queries(W.Workload("q", 0, 128, 4, 6, 2, 3, 10, 64, "cnf", qseed=21), 64)
    batch = hy.BatchRequest()
    for i, raw in enumerate(raws):
        clauses = [] if i % 5 == 0 else O.normalize_query(raw, 4)
        batch.queries.append(hy.HybridQuery(to_cnf(clauses), qemb[i], [10, 100, 1, 257][i % 4],
                                            hy.ExecOptions(quant_enabled=False)))
    outs = ex.execute_batch(batch)
    for o, s in zip(outs, _singles(hy, ex, batch)):
        assert o.ok
        assert [(h.row_id, h.score) for h in o.result.hits] == s


@pytest.mark.parametrize("dim", [64, 128])  # bf16 prefilter (dp % 128 != 0) / int8 prefilter
def test_prefilter_keeps_exact_order_among_bf16_indistinguishable_rows(hy, dim):
    # Rows differ from a common direction by ~1e-3, so their exact scores are
    # distinct while most bf16 prefilter scores coincide: the K-th exact
    # score sits inside a band of thousands of prefilter ties.  The admitted
    # set (prefilter >= threshold - delta) must still contain the exact top-K,
    # and the rescored result must equal the exact single-query (K2) answer
    # and the oracle's.
    n = 60_000
    rs = np.random.default_rng(3)
    base = rs.standard_normal(dim).astype(np.float32)
    emb = (base[None, :] + 1e-3 * rs.standard_normal((n, dim))).astype(np.float32)
    b = hy.IndexBuilder(hy.IndexConfig(1, 1, dim))
    b.add_documents(np.arange(n + 1, dtype=np.uint64), np.ones(n, np.uint32), emb)
    prod = b.freeze(hy.make_codec(dim, 64, 1))
    ref = O.Frozen(n, 1, 1, dim, 64, 1, np.array(prod.attributes), np.array(prod.offsets),
                   np.array(prod.embeddings), np.array(prod.signatures), np.array(prod.zero_flags))
    ex = hy.Executor(prod, max_batch=16)
    batch = hy.BatchRequest()
    for i in range(16):
        q = (base + 0.02 * rs.standard_normal(dim)).astype(np.float32)
        batch.queries.append(hy.HybridQuery(hy.CnfQuery(), q, [100, 7, 1000, 1][i % 4],
                                            hy.ExecOptions(quant_enabled=False)))
    outs = ex.execute_batch(batch)
    rows = np.arange(n)
    for q, o, s in zip(batch.queries, outs, _singles(hy, ex, batch)):
        assert o.ok
        assert [(h.row_id, h.score) for h in o.result.hits] == s
        qq, _ = O.unit_embedding(q.embedding)
        er, es = O.top_k(rows, O.scores_rows(ref.embeddings, qq, rows), q.k)
        gr, gs = hits(o.result)
        assert_topk_match(ref, q.embedding, gr, gs, er, es)


@pytest.mark.parametrize("mode", ["bf16", "0"])
def test_prefilter_modes_in_a_fresh_process(mode):
    # The prefilter kind is fixed per process (HYRE_PREFILTER): rerun the
    # exactness tests with the bf16 prefilter, and the oracle-tolerance tests
    # with no prefilter (the K3 hi/lo split then scores directly, so its
    # scores match K2's only within the fp32 tolerance), in a child process.
    import os
    import subprocess
    import sys
    env = dict(os.environ, HYRE_PREFILTER=mode)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", os.path.join(root, "tests",
                        "test_gpu_parity.py"), "-k", ("equals_single or indistinguishable or tensor_core_batch_matches"
                                                      if mode != "0" else "tensor_core_batch_matches or match_all")],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
