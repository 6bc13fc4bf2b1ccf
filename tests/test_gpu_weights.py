"""Learned per-row weights applied in the scoring epilogue (north star:
"the term mask and the learned link/attribute weights are applied in the
epilogue").  The reference has no counterpart -- its score is the pure cosine
(proj/src/knn.cpp:36-37) -- so:
  * identity weights must reproduce the unweighted results bit for bit (the
    reference-parity default);
  * arbitrary weights w in [0, 1] are checked against the oracle's weighted
    epilogue (oracle/hyre_oracle.py weighted_scores: w[row] x the reference's
    exact score, one fp32 multiply) with the usual gates (tests/parity.py),
    on every scoring path: K2 exact (d = 64), K2 int8, K3 fused CNF (the c3
    instantiation J = 24), K3 match-all, the bf16 prefilter (child process),
    the exhaustive k > 4096 path and row shards.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import hyre_oracle as O
from tests.helpers import hits, run_batch, to_cnf
from tests.parity import check_topk

pytestmark = [pytest.mark.gpu]


@pytest.fixture(scope="module")
def hy():
    import paper_2402_13435_b200 as hy
    return hy


def _cnf_index(hy, n, dim, C, V, max_ids, seed, dtype="f32"):
    from paper_2402_13435_b200 import workloads as W
    w = W.Workload("t", n, dim, C, V, 7, max_ids, 10, 16, "cnf", seed=seed, qseed=seed + 1)
    so, ids, emb = W.cnf_docs(w)
    b = hy.IndexBuilder(hy.IndexConfig(C, C * max_ids, dim))
    b.add_documents(so, ids, emb)
    prod = b.freeze(hy.make_codec(dim, 64, seed))
    ref = O.Frozen(n, C, C * max_ids, dim, 64, seed, np.array(prod.attributes), np.array(prod.offsets),
                   np.array(prod.embeddings), np.array(prod.signatures), np.array(prod.zero_flags))
    return prod, ref


def _queries(hy, dim, C, V, B, k, qseed, match_all_every=0, draws=7):
    from paper_2402_13435_b200 import workloads as W
    raws, qemb = W.queries(W.Workload("q", 0, dim, C, V, draws, 3, 10, B, "cnf", qseed=qseed), B)
    out = []
    for i, raw in enumerate(raws):
        cl = [] if (match_all_every and i % match_all_every == 0) else O.normalize_query(raw, C)
        kk = k[i % len(k)] if isinstance(k, (list, tuple)) else k
        out.append(hy.HybridQuery(to_cnf(cl), qemb[i], kk, hy.ExecOptions(quant_enabled=False)))
    return out


def _weights(n, seed):
    rs = np.random.default_rng(seed)
    w = rs.random(n).astype(np.float32)
    w[rs.integers(0, n, n // 50)] = 0.0  # some zero-weight rows
    w[rs.integers(0, n, n // 50)] = 1.0
    return w


def _check(ref, queries, got, w, emb=None):
    emb = ref.embeddings if emb is None else emb
    for i, (q, (st, gr, gs)) in enumerate(zip(queries, got)):
        assert st == 0, (i, st)
        cl = [(c.slot, c.attribute_ids) for c in q.terms.clauses]
        rows = O.full_scan_tbr(ref, cl)
        qq, _ = O.unit_embedding(q.embedding)
        er, es = O.top_k(rows, O.weighted_scores(emb, qq, rows, w), q.k)
        check_topk(gr, gs, er, es, O.weighted_scores(emb, qq, gr, w))


def test_identity_weights_reproduce_the_unweighted_results_exactly(hy):
    prod, ref = _cnf_index(hy, 120_000, 128, 8, 20, 3, 5)
    dev = prod.device(0, "f32")
    qs = _queries(hy, 128, 8, 20, 64, [100, 10, 1000], 7)
    base64, _, _ = run_batch(hy.Executor(dev, 64), qs)
    one = hy.Executor(dev, 1)
    base1 = [run_batch(one, [q])[0][0] for q in qs[:3]]
    dev.set_row_weights(np.ones(120_000, np.float32))
    try:
        w64, _, var = run_batch(hy.Executor(dev, 64), qs)
        one = hy.Executor(dev, 1)
        w1 = [run_batch(one, [q])[0][0] for q in qs[:3]]
    finally:
        dev.set_row_weights(None)
    assert list(var[:3]) == [24, 1, 2]
    for a, b in zip(base64 + base1, w64 + w1):
        assert a[0] == b[0] and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


@pytest.mark.parametrize("B", [1, 4, 64])
def test_weighted_cnf_batches_match_the_weighted_oracle(hy, B):
    # B = 1 / 4: K1 mask + K2 int8 prefilter + K4p; B = 64: fused CNF K3
    # (c3 instantiation J = 24, u8 ids, 2 chunks) with the IMAD admission
    prod, ref = _cnf_index(hy, 150_000, 128, 8, 20, 3, 11)
    dev = prod.device(0, "f32")
    w = _weights(150_000, 3)
    dev.set_row_weights(w)
    try:
        qs = _queries(hy, 128, 8, 20, B, [100, 10, 1000, 1], 13)
        got, path, var = run_batch(hy.Executor(dev, B), qs)
        if B == 64:
            assert path & 1 and path & 2 and list(var[:3]) == [24, 1, 2], (path, var)
        _check(ref, qs, got, w)
        if B == 64:  # batch transparency holds with weights: singles bit-exact
            one = hy.Executor(dev, 1)
            for i in (0, 31):
                g1, _, _ = run_batch(one, [qs[i]])
                assert np.array_equal(g1[0][1], got[i][1]) and np.array_equal(g1[0][2], got[i][2])
    finally:
        dev.set_row_weights(None)


@pytest.mark.parametrize("B,dtype", [(1, "f32"), (32, "f32"), (64, "bf16")])
def test_weighted_match_all_batches(hy, B, dtype):
    prod, ref = _cnf_index(hy, 90_001, 128, 4, 6, 3, 21)
    dev = prod.device(0, dtype)
    w = _weights(90_001, 8)
    dev.set_row_weights(w)
    emb = ref.embeddings
    if dtype == "bf16":
        import torch
        emb = torch.from_numpy(ref.embeddings).to(torch.bfloat16).float().numpy()
    try:
        qs = _queries(hy, 128, 4, 6, B, [100, 7, 500], 23, match_all_every=1)
        got, _, _ = run_batch(hy.Executor(dev, B), qs)
        _check(ref, qs, got, w, emb)
    finally:
        dev.set_row_weights(None)


@pytest.mark.parametrize("match_all", [False, True])
def test_weighted_single_query_on_a_larger_index(hy, match_all):
    # 400K rows, d = 128, B = 1: K1 mask (or none for match-all) + K2 int8 prefilter + K4p
    prod, ref = _cnf_index(hy, 400_000, 128, 8, 20, 3, 71)
    dev = prod.device(0, "f32")
    w = _weights(400_000, 14)
    dev.set_row_weights(w)
    try:
        qs = _queries(hy, 128, 8, 20, 3, [100, 10, 1], 73, match_all_every=1 if match_all else 0, draws=13)
        one = hy.Executor(dev, 1)
        got = [run_batch(one, [q])[0][0] for q in qs]
        _check(ref, qs, got, w)
    finally:
        dev.set_row_weights(None)


def test_weighted_exact_k2_path_d64(hy):
    # d = 64: no int8 plane, K2 scores exactly and compares w x clamp(dot)
    prod, ref = _cnf_index(hy, 100_000, 64, 4, 12, 3, 31)
    dev = prod.device(0, "f32")
    w = _weights(100_000, 9)
    dev.set_row_weights(w)
    try:
        for B in (1, 3):
            qs = _queries(hy, 64, 4, 12, B, [100, 5], 33 + B)
            got, _, _ = run_batch(hy.Executor(dev, B), qs)
            _check(ref, qs, got, w)
    finally:
        dev.set_row_weights(None)


def test_weighted_exhaustive_large_k(hy):
    # k > 4096 takes the exhaustive exact path (rescore every eligible row)
    prod, ref = _cnf_index(hy, 30_000, 64, 2, 4, 2, 41)
    dev = prod.device(0, "f32")
    w = _weights(30_000, 10)
    dev.set_row_weights(w)
    try:
        qs = _queries(hy, 64, 2, 4, 2, [6000, 20000], 43, match_all_every=2)
        got, _, _ = run_batch(hy.Executor(dev, 2), qs)
        _check(ref, qs, got, w)
    finally:
        dev.set_row_weights(None)


def test_weighted_row_shards_equal_the_single_index(hy):
    prod, ref = _cnf_index(hy, 80_000, 128, 8, 20, 3, 51)
    w = _weights(80_000, 12)
    qs = _queries(hy, 128, 8, 20, 16, [100, 10], 53)
    sh = hy.ShardedIndex(prod, 2, devices=[0, 0])
    sh.set_row_weights(w)
    out = hy.ShardedExecutor(sh, max_batch=16).execute_batch(hy.BatchRequest(qs))
    got = [(0 if o.ok else 1, *hits(o.result)) for o in out]
    _check(ref, qs, got, w)


def test_weight_validation(hy):
    prod, _ = _cnf_index(hy, 1_000, 64, 2, 4, 2, 61)
    dev = prod.device(0, "f32")
    with pytest.raises(hy.ValidationError, match="expected 1000 weights, got 999"):
        dev.set_row_weights(np.ones(999, np.float32))
    bad = np.ones(1000, np.float32)
    bad[7] = 1.5
    with pytest.raises(hy.ValidationError, match="row weight 7 = 1.5"):
        dev.set_row_weights(bad)
    bad[7] = np.nan
    with pytest.raises(hy.ValidationError, match="row weight 7"):
        dev.set_row_weights(bad)
    dev.set_row_weights(np.zeros(1000, np.float32))  # all-zero weights: every score 0, rows ascending
    q = hy.HybridQuery(hy.CnfQuery(), np.ones(64, np.float32), 5, hy.ExecOptions(quant_enabled=False))
    r = hy.Executor(dev, 1).execute(q)
    assert [h.row_id for h in r.hits] == [0, 1, 2, 3, 4] and all(h.score == 0.0 for h in r.hits)
    dev.set_row_weights(None)


def test_weighted_bf16_prefilter_in_a_fresh_process():
    # the K3 bf16 prefilter (weighted FFMA admission) is selected per process
    import subprocess
    import sys
    env = dict(os.environ, HYRE_PREFILTER="bf16")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        os.path.join(root, "tests", "test_gpu_weights.py"), "-k",
                        "weighted_cnf_batches or weighted_match_all"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
