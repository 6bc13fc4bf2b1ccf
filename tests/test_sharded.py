"""Row-sharded executor (hyre_sharded_*) on one GPU: G
shards of the same device run the same code as G GPUs (peer-memory reads
are plain loads on one device).  Sharded results must equal the unsharded
executor's bit for bit -- per-row eligibility and scores do not depend on
the shard, the merge is exact, and the quant pre-selection is global -- and
match the compiled reference."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import ref as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hy():
    import paper_2402_13435_b200 as hy
    return hy


def _index(hy, n, dim=128, C=8, V=20, draws=13, max_ids=3, seed=3, qseed=4):
    from paper_2402_13435_b200 import workloads as W
    w = W.Workload("s", n, dim, C, V, draws, max_ids, 100, 64, "cnf", seed=seed, qseed=qseed)
    so, ids, emb = W.docs(w)
    b = hy.IndexBuilder(hy.IndexConfig(C, C * max_ids, dim))
    b.add_documents(so, ids, emb, doc_id_prefix="d")
    return w, (so, ids, emb), b.freeze(hy.make_codec(dim, w.num_bits, seed))


def _queries(hy, w, b, ks, quant=False, qk=0, term_only_every=0, match_all_every=0):
    from paper_2402_13435_b200 import workloads as W
    raws, qemb = W.queries(w, b)
    out = []
    for i, raw in enumerate(raws):
        cq = hy.CnfQuery() if (match_all_every and i % match_all_every == 0) else hy.normalize_query(raw, w.num_clauses)
        emb = None if (term_only_every and i % term_only_every == 1) else qemb[i]
        out.append(hy.HybridQuery(cq, emb, ks[i % len(ks)], hy.ExecOptions(quant_enabled=quant, quant_k=qk)))
    return out


def _same(a, b):
    assert len(a) == len(b)
    for i, (x, y) in enumerate(zip(a, b)):
        assert x.ok == y.ok, i
        gx = [(h.row_id, h.score) for h in x.result.hits]
        gy = [(h.row_id, h.score) for h in y.result.hits]
        assert gx == gy, (i, gx[:5], gy[:5], len(gx), len(gy))


@pytest.mark.parametrize("G", [2, 3, 4])
def test_sharded_batch_equals_unsharded(hy, G):
    w, _, prod = _index(hy, 300_000)
    qs = _queries(hy, w, 64, [100, 10, 1, 700], term_only_every=9, match_all_every=13)
    one = hy.Executor(prod, max_batch=64).execute_batch(hy.BatchRequest(qs))
    sh = hy.ShardedExecutor(prod, G, devices=[0] * G, max_batch=64)
    assert sh.info() == (G, [0] * G)
    _same(sh.execute_batch(hy.BatchRequest(qs)), one)
    # the same executor again (scratch reuse across batches) and single queries (K2 path)
    _same(sh.execute_batch(hy.BatchRequest(qs[:5])), one[:5])
    for q, o in zip(qs[:3], one[:3]):
        assert [(h.row_id, h.score) for h in sh.execute(q).hits] == [(h.row_id, h.score) for h in o.result.hits]


@pytest.mark.parametrize("B", [4, 9, 64])
def test_sharded_quant_is_global(hy, B):
    # quant_k below the matches: per-shard preselection would keep G x quant_k
    # rows; the global one keeps exactly quant_k (pipeline.cpp:126-130)
    w, (so, ids, emb), prod = _index(hy, 200_000)
    qs = _queries(hy, w, B, [10, 100], quant=True, qk=1500)
    one = hy.Executor(prod, max_batch=B).execute_batch(hy.BatchRequest(qs))
    sh = hy.ShardedExecutor(prod, 3, devices=[0, 0, 0], max_batch=B)
    _same(sh.execute_batch(hy.BatchRequest(qs)), one)
    if R.available():
        ref = R.RefIndex.build(so.astype(np.uint32), ids, emb, w.num_clauses, w.max_num_attr, w.num_bits, w.seed, "d")
        for q, o in zip(qs[:8], one[:8]):
            cl = [(c.slot, list(c.attribute_ids)) for c in q.terms.clauses]
            rr, _ = ref.execute(cl, q.embedding, q.k, True, 1500)
            got = np.asarray([h.row_id for h in o.result.hits])
            # survivor sets are bit-exact, so ties aside the hits agree
            assert len(np.intersect1d(got, rr)) >= len(rr) - 2


def test_sharded_large_k_and_term_only_beyond_select(hy):
    w, _, prod = _index(hy, 120_000, dim=64, C=4, draws=13)
    qs = _queries(hy, w, 6, [5000, 20000, 100], term_only_every=2)
    one = hy.Executor(prod, max_batch=8).execute_batch(hy.BatchRequest(qs))
    sh = hy.ShardedExecutor(prod, 4, devices=[0] * 4, max_batch=8)
    _same(sh.execute_batch(hy.BatchRequest(qs)), one)
    assert max(len(o.result.hits) for o in one) > 4096


def test_k_above_a_shard_rows_returns_min_k_all_rows(hy):
    # k larger than one shard's rows must still return min(k, all rows)
    w, _, prod = _index(hy, 1000, dim=32, C=2, V=4, draws=4)
    qs = [hy.HybridQuery(hy.CnfQuery(), np.ones(32, np.float32), 600, hy.ExecOptions(False)),
          hy.HybridQuery(hy.CnfQuery(), None, 900, hy.ExecOptions(False))]
    one = hy.Executor(prod, max_batch=2).execute_batch(hy.BatchRequest(qs))
    sh = hy.ShardedExecutor(prod, 4, devices=[0] * 4, max_batch=2)
    out = sh.execute_batch(hy.BatchRequest(qs))
    _same(out, one)
    assert len(out[0].result.hits) == 600 and len(out[1].result.hits) == 900


def test_sharded_validation_errors_fail_their_slot(hy):
    w, _, prod = _index(hy, 5000, dim=16, C=2, V=4, draws=2)
    sh = hy.ShardedExecutor(prod, 2, devices=[0, 0], max_batch=4)
    good = hy.HybridQuery(hy.CnfQuery(), np.ones(16, np.float32), 5, hy.ExecOptions(False))
    bad = hy.HybridQuery(hy.CnfQuery(), np.ones(7, np.float32), 5, hy.ExecOptions(False))
    out = sh.execute_batch(hy.BatchRequest([good, bad]))
    assert out[0].ok and not out[1].ok
    assert out[1].error == "embedding: expected dim 16, got 7"
    with pytest.raises(hy.ValidationError):
        hy.ShardedExecutor(prod, 17, max_batch=4)
