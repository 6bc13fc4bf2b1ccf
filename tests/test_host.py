"""CPU: the drop-in boundary's host side (no GPU needed).

* libhyre_b200.so loads and exports every symbol include/hyre_b200.h declares;
* IndexBuilder / freeze produce the reference's FrozenIndex arrays bit for bit
  (golden digests from the compiled reference);
* validation / normalisation messages, the codec, the HYREIDN1 index file and
  the shard merge behave like the reference (test_corpus.cpp, test_term_match.cpp,
  test_quantizer.cpp, test_pipeline.cpp cited per test).
"""

from __future__ import annotations

import ctypes as C
import hashlib
import json
import os
import re

import numpy as np
import pytest

import paper_2402_13435_b200 as hy
from oracle import hyre_oracle as O
from paper_2402_13435_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIX = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_fixtures.json")))


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def unhex(xs):
    return np.asarray([int(x, 16) for x in xs], np.uint32).view(np.float32)


def build(docs, num_clauses, max_num_attr, dim, num_bits, seed, names=()):
    b = hy.IndexBuilder(hy.IndexConfig(num_clauses, max_num_attr, dim, list(names)))
    for d in docs:
        b.add_document(hy.DocumentInput(d.doc_id, d.clauses, d.embedding))
    return b.freeze(hy.make_codec(dim, num_bits, seed))


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "hyre_b200.h")).read()
    declared = set(re.findall(r"\b(hyre_[a-z0-9_]+)\s*\(", header))
    assert len(declared) > 40
    lib = C.CDLL(L.LIB_PATH)
    missing = [s for s in sorted(declared) if not hasattr(lib, s)]
    assert not missing, missing
    assert declared == set(L.SIGNATURES), declared ^ set(L.SIGNATURES)
    assert L.lib().hyre_abi_version() == 1


@pytest.mark.parametrize("case", range(3))
def test_freeze_is_bit_identical_to_the_reference(case):
    fx = FIX["freeze"][case]
    spec = O.CorpusSpec(**fx["spec"])
    docs, widest = O.make_corpus_docs(spec)
    f = build(docs, spec.num_clauses, widest, spec.dim, spec.num_bits, spec.seed + 1000)
    assert digest(f.attributes, f.offsets, f.embeddings.view(np.uint32), f.signatures, f.zero_flags) == fx["sha256"]
    assert [f.doc_id(0), f.doc_id(spec.num_docs - 1)] == fx["doc_ids"]


def test_bulk_builder_matches_reference_c1_slice():
    fx = FIX["c1_slice"]
    from paper_2402_13435_b200 import workloads as W
    w = W.Workload("c1", fx["n"], fx["dim"], fx["clauses"], fx["vocab"], fx["draws"], 3, 100, 1, "cnf", seed=fx["seed"],
                   qseed=fx["qseed"])
    so, ids, emb = W.cnf_docs(w)
    b = hy.IndexBuilder(hy.IndexConfig(w.num_clauses, w.max_num_attr, w.dim))
    b.add_documents(so, ids, emb)
    f = b.freeze(hy.make_codec(w.dim, 512, 42))
    assert digest(f.attributes, f.offsets, f.embeddings.view(np.uint32), f.signatures, f.zero_flags) == fx["sha256"]
    assert f.doc_id(5) == "d5" and f.row_of("d19999") == 19999


def test_native_generator_matches_python_generator():
    from paper_2402_13435_b200 import workloads as W
    w = W.Workload("t", 300, 16, 4, 20, 7, 3, 10, 4, "cnf", seed=11, qseed=7)
    so, ids, emb = W.cnf_docs(w)
    po, pids, pemb = O.cnf_workload_docs(300, 16, 4, 20, 11)
    assert np.array_equal(so, po) and np.array_equal(ids, pids)
    assert np.array_equal(emb.view(np.uint32), pemb.view(np.uint32))
    so2, ids2, emb2 = W.cnf_docs(w, 100, 200)  # shard consistency
    assert np.array_equal(emb2, emb[100:200]) and np.array_equal(ids2, ids[so[400]:so[800]])
    raws, qe = W.queries(w)
    pq, pqe = O.cnf_workload_queries(4, 16, 4, 20, 7, 7)
    assert [O.normalize_query(r, 4) for r in raws] == pq and np.array_equal(qe, pqe)


def test_layout_of_the_appendix_fixture():
    # test_corpus.cpp:50-69
    f = build([O.Doc("doc1", [[934, 2934], [945, 342, 3112]], [1, 0, 0, 0]),
               O.Doc("doc2", [[129], [9342, 234]], [1, 0, 0, 0])], 2, 5, 4, 64, 7, ["geo", "skill"])
    assert f.attribute_row(0).tolist() == [934, 2934, 342, 945, 3112]
    assert f.offsets_row(1).tolist() == [0, 1, 3]
    assert f.clause_slice(0, 1).tolist() == [342, 945, 3112]
    assert f.doc_id(1) == "doc2" and f.row_of("doc1") == 0 and f.row_of("nope") is None
    assert f.resolve_clause_slot("skill") == 1 and f.resolve_clause_slot("salary") == -1
    assert f.clause_names() == ["geo", "skill"]


def test_normalization_zero_rows_and_signatures():
    # test_corpus.cpp:80-96, 196-204
    f = build([O.Doc("a", [[1], [2]], [3, 4, 0, 0]), O.Doc("z", [[1], [2]], [0, 0, 0, 0])], 2, 5, 4, 64, 7)
    assert f.embedding_row(0).tolist() == [np.float32(0.6), np.float32(0.8), 0.0, 0.0]
    assert f.embedding_is_zero(1) and not f.embedding_row(1).any()
    for r in range(2):
        assert f.signature_row(r) == hy.encode(f.codec(), f.embedding_row(r))


def test_default_clause_names():
    f = build([O.Doc("a", [[1], [2], [3]], [1, 0])], 3, 3, 2, 16, 7)
    assert f.clause_names() == ["c0", "c1", "c2"]


def test_builder_rejects_malformed_input():
    # test_corpus.cpp:114-179 (messages verbatim)
    with pytest.raises(hy.ValidationError, match="numClauses must be >= 1"):
        hy.IndexBuilder(hy.IndexConfig(0, 1, 1))
    with pytest.raises(hy.ValidationError, match="dim must be >= 1"):
        hy.IndexBuilder(hy.IndexConfig(1, 1, 0))
    with pytest.raises(hy.ValidationError, match="maxNumAttr must be >= 1"):
        hy.IndexBuilder(hy.IndexConfig(1, 0, 1))
    with pytest.raises(hy.ValidationError, match="clause_names size != numClauses"):
        hy.IndexBuilder(hy.IndexConfig(1, 1, 1, ["a", "b"]))
    b = hy.IndexBuilder(hy.IndexConfig(2, 5, 4))
    b.add_document(hy.DocumentInput("dup", [[1], [2]], [1, 0, 0, 0]))
    with pytest.raises(hy.ValidationError) as e:
        b.add_document(hy.DocumentInput("dup", [[3], [4]], [1, 0, 0, 0]))
    assert str(e.value) == "duplicate docId: dup"
    with pytest.raises(hy.ValidationError, match=r"attribute id 0 is reserved for padding \(docId a\)"):
        b.add_document(hy.DocumentInput("a", [[0], [2]], [1, 0, 0, 0]))
    with pytest.raises(hy.ValidationError, match="clauses: expected 2 clause slots, got 1"):
        b.add_document(hy.DocumentInput("b", [[1]], [1, 0, 0, 0]))
    with pytest.raises(hy.ValidationError, match="embedding: expected dim 4, got 1"):
        b.add_document(hy.DocumentInput("c", [[1], [2]], [1]))
    wide = hy.IndexBuilder(hy.IndexConfig(2, 5, 4))
    wide.add_document(hy.DocumentInput("wide", [[1, 2, 3], [4, 5, 6]], [1, 0, 0, 0]))
    with pytest.raises(hy.ValidationError) as e:
        wide.freeze(hy.make_codec(4, 64, 7))
    assert str(e.value) == "documents wider than maxNumAttr=5: wide"
    ok = hy.IndexBuilder(hy.IndexConfig(2, 5, 4))
    ok.add_document(hy.DocumentInput("ok", [[1, 1, 1, 2, 3], [4, 4, 5]], [1, 0, 0, 0]))
    ok.freeze(hy.make_codec(4, 64, 7))  # duplicates collapse before the width check
    with pytest.raises(hy.ValidationError, match="no documents staged"):
        hy.IndexBuilder(hy.IndexConfig(2, 5, 4)).freeze(hy.make_codec(4, 64, 7))
    b2 = hy.IndexBuilder(hy.IndexConfig(2, 5, 4))
    b2.add_document(hy.DocumentInput("a", [[1], [2]], [1, 0, 0, 0]))
    with pytest.raises(hy.ValidationError, match="codec dim != index dim"):
        b2.freeze(hy.make_codec(8, 64, 7))


def test_normalize_query_rules():
    # test_term_match.cpp:42-69
    q = hy.normalize_query({1: [9, 3, 9, 1]}, 2)
    assert q.clauses[0].slot == 1 and q.clauses[0].attribute_ids == [1, 3, 9]
    assert hy.normalize_query({}, 3).match_all()
    assert [c.slot for c in hy.normalize_query({0: [], 1: [5]}, 2).clauses] == [1]
    assert [c.slot for c in hy.normalize_query({1: [4], 0: [2]}, 2).clauses] == [0, 1]
    for name, raw, nc in [("unknown_slot", {2: [1]}, 2), ("zero_id", {0: [0]}, 2)]:
        with pytest.raises(hy.ValidationError) as e:
            hy.normalize_query(raw, nc)
        assert str(e.value) == FIX["messages"][name]


def test_validate_query_names_the_field():
    # test_pipeline.cpp:72-98
    f = build([O.Doc(f"doc{r}", [[r + 1]], O.random_unit_vector(8, O.MT19937_64(r))) for r in range(4)], 1, 1, 8,
              64, 3)
    cases = [
        (hy.HybridQuery(k=0), "k must be >= 1"),
        (hy.HybridQuery(options=hy.ExecOptions(granularity=0)), "granularity must be >= 1"),
        (hy.HybridQuery(embedding=[1.0]), "embedding: expected dim 8, got 1"),
        (hy.HybridQuery(hy.CnfQuery([hy.CnfClause(5, [1])])), "unknown clause slot 5"),
        (hy.HybridQuery(hy.CnfQuery([hy.CnfClause(0, [0])])), "attribute id 0 is reserved for padding"),
        (hy.HybridQuery(hy.CnfQuery([hy.CnfClause(0, [])])), "clause 0 has no attribute ids"),
        (hy.HybridQuery(hy.CnfQuery([hy.CnfClause(0, [3, 2])])),
         "clause attribute ids must be strictly increasing (use normalize_query)"),
    ]
    for q, msg in cases:
        with pytest.raises(hy.ValidationError) as e:
            hy.validate_query(f, q)
        assert str(e.value) == msg
    hy.validate_query(f, hy.HybridQuery())
    assert hy.ExecOptions().effective_quant_k(10) == 2000 and hy.ExecOptions(quant_k=50).effective_quant_k(10) == 50


def test_codec_and_encode_match_reference():
    for fx in FIX["encode"]:
        sig = hy.encode(hy.make_codec(fx["dim"], fx["bits"], fx["seed"]), unhex(fx["x"]))
        assert [f"{int(w):016x}" for w in sig.words] == fx["words"]
    # test_quantizer.cpp:403-465
    c = hy.make_codec(8, 40, 5)
    assert all(hy.encode(c, np.zeros(8, np.float32)).bit(b) for b in range(40))
    x = O.random_unit_vector(16, O.MT19937_64(4))
    c16 = hy.make_codec(16, 64, 9)
    assert hy.encode(c16, x) == hy.encode(c16, x * np.float32(2.5))
    a = hy.Signature(4, np.asarray([0b0101], np.uint64))
    b = hy.Signature(4, np.asarray([0b1001], np.uint64))
    assert hy.quant_score(a, b) == 2 and hy.quant_score(a, a) == 4
    with pytest.raises(hy.ValidationError):
        hy.make_codec(0, 8, 1)


def test_save_load_round_trip_and_corruption_classes(tmp_path):
    # test_corpus.cpp:206-264
    docs, widest = O.make_corpus_docs(O.CorpusSpec(num_docs=37, dim=6, num_bits=96))
    f = build(docs, 2, widest, 6, 96, 1001)
    path = str(tmp_path / "idx.bin")
    f.save(path)
    g = hy.FrozenIndex.load(path)
    assert g == f
    raw = open(path, "rb").read()

    def expect(mutate, cause):
        bad = str(tmp_path / "bad.bin")
        open(bad, "wb").write(mutate(bytearray(raw)))
        with pytest.raises(hy.LoadError) as e:
            hy.FrozenIndex.load(bad)
        assert e.value.cause() == cause

    def flip(i, m):
        def f_(b):
            b[i] ^= m
            return bytes(b)
        return f_

    expect(flip(0, 0xFF), hy.LoadError.Cause.kBadMagic)
    expect(flip(8, 0x01), hy.LoadError.Cause.kVersionMismatch)
    expect(lambda b: bytes(b[: len(b) // 2]), hy.LoadError.Cause.kTruncated)
    expect(flip(len(raw) - 9, 0x10), hy.LoadError.Cause.kChecksum)


def test_index_file_is_byte_identical_to_the_reference_writer(tmp_path):
    # The HYREIDN1 format written by the product must be what the reference's
    # FrozenIndex::save writes for the same index (corpus.cpp:144-162).
    from oracle import ref as R
    if not R.available():
        pytest.skip("oracle/_ref not built")
    spec = O.CorpusSpec(num_docs=37, dim=6, num_bits=96)
    docs, widest = O.make_corpus_docs(spec)
    f = build(docs, 2, widest, 6, 96, 1001)
    mine = str(tmp_path / "mine.bin")
    f.save(mine)
    r = R.RefIndex.load(mine)  # the reference reads it ...
    theirs = str(tmp_path / "theirs.bin")
    r.save(theirs)  # ... and writes back the same bytes
    assert open(mine, "rb").read() == open(theirs, "rb").read()


def test_merge_topk_is_exact():
    rs = np.random.default_rng(0)
    dt = np.dtype([("row", np.uint32), ("score", np.float32)])
    lists, allrows, allsc = [], [], []
    for g in range(4):
        rows = np.arange(g * 1000, g * 1000 + 1000, dtype=np.uint32)
        sc = np.round(rs.random(1000), 2).astype(np.float32)  # many ties
        order = np.lexsort((rows, -sc.astype(np.float64)))[:50]
        lists.append(np.array(list(zip(rows[order], sc[order])), dtype=dt))
        allrows.append(rows)
        allsc.append(sc)
    merged = hy.merge_topk(lists, 50)
    er, es = O.top_k(np.concatenate(allrows), np.concatenate(allsc), 50)
    assert merged["row"].tolist() == er.tolist()


def _bulk(b, n, prefix, dim=2):
    so = np.arange(n + 1, dtype=np.uint64)  # one slot, one id per row
    b.add_documents(so, np.ones(n, np.uint32), np.ones((n, dim), np.float32), doc_id_prefix=prefix)


def test_bulk_doc_ids_are_ranges_with_reference_duplicate_semantics(tmp_path):
    # corpus.cpp:29-52: a docId may appear once; bulk rows carry prefix + row
    b = hy.IndexBuilder(hy.IndexConfig(1, 1, 2))
    _bulk(b, 5, "d")                                   # d0 .. d4
    with pytest.raises(hy.ValidationError, match="duplicate docId: d3"):
        b.add_document(hy.DocumentInput("d3", [[1]], [1.0, 0.0]))
    b.add_document(hy.DocumentInput("d03", [[1]], [1.0, 0.0]))  # not canonical: a distinct id (row 5)
    b.add_document(hy.DocumentInput("x9", [[1]], [1.0, 0.0]))   # row 6
    with pytest.raises(hy.ValidationError, match="duplicate docId: x9"):
        _bulk(b, 5, "x")                               # x7 .. x11 would repeat x9
    _bulk(b, 4, "d1")                                  # d17 .. d110 (rows 7 .. 10)
    with pytest.raises(hy.ValidationError, match="duplicate docId: d17"):
        _bulk(b, 10, "d")                              # rows 11 .. 20: d17? no -- d11 .. d20 vs d1+7 = d17
    f = b.freeze(hy.make_codec(2, 16, 1))
    assert [f.doc_id(r) for r in (0, 4, 5, 6, 7, 10)] == ["d0", "d4", "d03", "x9", "d17", "d110"]
    assert f.row_of("d110") == 10 and f.row_of("d03") == 5 and f.row_of("x9") == 6 and f.row_of("d5") is None
    p = str(tmp_path / "ids.bin")
    f.save(p)
    g = hy.FrozenIndex.load(p)
    assert [g.doc_id(r) for r in range(11)] == [f.doc_id(r) for r in range(11)] and g.row_of("d17") == 7
