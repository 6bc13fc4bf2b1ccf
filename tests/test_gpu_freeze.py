"""GPU-side freeze (corpus.cpp:54-129 on the device,
csrc/freeze.cu): the frozen arrays must be bit-identical to the host freeze,
which tests/test_host.py pins to the compiled reference's digests -- so the
device freeze is pinned to the reference too."""

from __future__ import annotations

import dataclasses
import json
import os

import numpy as np
import pytest

from oracle import hyre_oracle as O

pytestmark = [pytest.mark.gpu]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIX = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_fixtures.json")))


@pytest.fixture(scope="module")
def hy():
    import paper_2402_13435_b200 as hy
    return hy


def _arrays(f):
    return [np.array(f.attributes), np.array(f.offsets), np.array(f.embeddings).view(np.uint32),
            np.array(f.signatures), np.array(f.zero_flags)]


def _builder(hy, docs, C, A, dim, names=()):
    b = hy.IndexBuilder(hy.IndexConfig(C, A, dim, list(names)))
    for d in docs:
        b.add_document(hy.DocumentInput(d.doc_id, d.clauses, d.embedding))
    return b


@pytest.mark.parametrize("case", range(3))
def test_device_freeze_matches_the_reference_digests(hy, case):
    fx = FIX["freeze"][case]
    spec = O.CorpusSpec(**fx["spec"])
    docs, widest = O.make_corpus_docs(spec)
    f = _builder(hy, docs, spec.num_clauses, widest, spec.dim).freeze(
        hy.make_codec(spec.dim, spec.num_bits, spec.seed + 1000), device=0)
    from tests.test_host import digest  # the digest the host-freeze test pins
    assert digest(f.attributes, f.offsets, f.embeddings.view(np.uint32), f.signatures, f.zero_flags) == fx["sha256"]
    assert [f.doc_id(0), f.doc_id(spec.num_docs - 1)] == fx["doc_ids"]


def test_device_freeze_equals_host_freeze_on_the_c3_generator(hy):
    from paper_2402_13435_b200 import workloads as W
    w = dataclasses.replace(W.WORKLOADS["c3"], n=300_000)
    so, ids, emb = W.docs(w)
    emb[7] = 0.0  # a zero row
    out = []
    for dev in (None, 0):
        b = hy.IndexBuilder(hy.IndexConfig(w.num_clauses, w.max_num_attr, w.dim))
        b.add_documents(so, ids, emb, doc_id_prefix="d")
        out.append(b.freeze(hy.make_codec(w.dim, w.num_bits, w.seed), device=dev))
    for a, b in zip(_arrays(out[0]), _arrays(out[1])):
        assert np.array_equal(a, b)
    assert out[1].zero_flags[7] == 1 and out[1].doc_id(299_999) == "d299999"


def test_device_freeze_edge_rows_and_errors(hy):
    rs = np.random.default_rng(4)
    docs = []
    for i in range(500):
        cl = [rs.integers(1, 40, rs.integers(0, 6)).tolist(), rs.integers(1, 9, rs.integers(0, 5)).tolist()]
        if i == 3:
            cl[0] = [5] * 60 + [2] * 7  # > 48 staged ids in a slot: host canonicalisation, dedups to 2
        if i == 4:
            cl = [[], []]
        e = rs.standard_normal(24).astype(np.float32)
        if i % 50 == 0:
            e[:] = 0.0
        docs.append(O.Doc(f"r{i}", cl, e))
    widest = max(len(set(d.clauses[0])) + len(set(d.clauses[1])) for d in docs)
    f_host = _builder(hy, docs, 2, widest, 24).freeze(hy.make_codec(24, 100, 9))
    f_dev = _builder(hy, docs, 2, widest, 24).freeze(hy.make_codec(24, 100, 9), device=0)
    for a, b in zip(_arrays(f_host), _arrays(f_dev)):
        assert np.array_equal(a, b)
    # too wide: the same message (documents listed in row order)
    msgs = []
    for dev in (None, 0):
        with pytest.raises(hy.ValidationError) as e:
            _builder(hy, docs, 2, 3, 24).freeze(hy.make_codec(24, 100, 9), device=dev)
        msgs.append(str(e.value))
    assert msgs[0] == msgs[1] and msgs[0].startswith("documents wider than maxNumAttr=3:")
    b = _builder(hy, docs[:3], 2, widest, 24)
    b.freeze(hy.make_codec(24, 100, 9), device=0)
    with pytest.raises(hy.ValidationError, match="builder already frozen"):
        b.freeze(hy.make_codec(24, 100, 9), device=0)
