"""Row-sharded multi-GPU path.

Rows are split into contiguous shards, each shard returns its local top-K
with *global* row ids, one all-gather moves the B x K (row, score) lists and
an exact merge on (score desc, row asc) reproduces the unsharded answer
(the global top-K is a subset of the union of shard top-Ks).

* CPU: world_size-2 gloo run of the shard -> all_gather -> merge logic with
  the oracle scoring each shard (hy.merge_topk is the product's host merge).
* GPU: G shards emulated sequentially on one device through the same device
  merge bench.py uses under torchrun (hyre_batch_merge_gathered).
"""

from __future__ import annotations

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import hyre_oracle as O


def _corpus():
    spec = O.CorpusSpec(num_docs=3000, dim=16, num_clauses=2, attr_universe=6, num_bits=64, seed=9)
    return O.make_corpus(spec)


def _queries(fr, b=6):
    rng = O.MT19937_64(5)
    spec = O.CorpusSpec(num_docs=3000, dim=16, num_clauses=2, attr_universe=6)
    return [(O.random_query(spec, rng), O.random_unit_vector(16, rng), 1 + (i * 7) % 40) for i in range(b)]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2402_13435_b200 as hy
    docs, fr = _corpus()
    n = fr.num_docs
    rb, re_ = rank * n // world, (rank + 1) * n // world
    dt = np.dtype([("row", np.uint32), ("score", np.float32)])
    ok = True
    for clauses, emb, k in _queries(fr):
        # shard-local work: eligibility + scores over [rb, re_) only, global row ids
        rows = O.full_scan_tbr(fr, clauses)
        rows = rows[(rows >= rb) & (rows < re_)]
        q, _ = O.unit_embedding(emb)
        r, s = O.top_k(rows, O.scores_rows(fr.embeddings, q, rows), k)
        local = np.zeros(k, dt)
        local["row"][: len(r)] = r
        local["score"][: len(r)] = s
        t = torch.from_numpy(local.view(np.uint32).astype(np.int64))
        cnt = torch.tensor([len(r)])
        gathered = [torch.zeros_like(t) for _ in range(world)]
        counts = [torch.zeros_like(cnt) for _ in range(world)]
        dist.all_gather(gathered, t)
        dist.all_gather(counts, cnt)
        lists = [g.numpy().astype(np.uint32).view(dt)[: int(c)] for g, c in zip(gathered, counts)]
        merged = hy.merge_topk(lists, k)
        er, es = O.execute(fr, clauses, emb, k, quant_enabled=False)
        ok &= merged["row"].tolist() == er.tolist()
        ok &= np.array_equal(merged["score"], es)
    out[rank] = ok
    dist.destroy_process_group()


def test_sharded_merge_gloo_world2():
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert out[0] and out[1]


@pytest.mark.gpu
@pytest.mark.parametrize("G,B,packed", [(3, 4, False), (4, 16, False), (3, 4, True), (4, 16, True)])
def test_device_shard_merge_emulated_on_one_gpu(G, B, packed):
    """G row shards on one GPU, each with its own executor; their device
    results are stacked like an NCCL all-gather (three arrays, or one packed
    record per shard as bench.py gathers them) and merged on device."""
    import ctypes as C

    import paper_2402_13435_b200 as hy
    from paper_2402_13435_b200 import _lib as L
    from tests.helpers import hits, to_cnf
    from tests.parity import assert_topk_match

    spec = O.CorpusSpec(num_docs=20_000, dim=64, num_clauses=2, attr_universe=6, num_bits=64, seed=3)
    docs, fr = O.make_corpus(spec)
    b = hy.IndexBuilder(hy.IndexConfig(2, fr.max_num_attr, 64))
    for d in docs:
        b.add_document(hy.DocumentInput(d.doc_id, d.clauses, d.embedding))
    frozen = b.freeze(hy.make_codec(64, 64, spec.seed + 1000))
    rng = O.MT19937_64(17)
    batch = hy.BatchRequest()
    for i in range(B):
        cl = O.random_query(spec, rng)
        emb = O.random_unit_vector(64, rng) if i % 3 else None  # mix term-only queries
        batch.queries.append(hy.HybridQuery(to_cnf(cl), emb, 5 + 11 * i, hy.ExecOptions(quant_enabled=False)))
    pack = hy.QueryPack(batch.queries)
    n = spec.num_docs
    shards = []
    for g in range(G):
        dev = hy.DeviceIndex(frozen, 0, "f32", True, g * n // G, (g + 1) * n // G)
        ex = hy.Executor(dev, max_batch=B)
        assert L.lib().hyre_batch_prepare(ex._h, pack.arr, B) == 0
        assert L.lib().hyre_batch_run(ex._h) == 0
        assert L.lib().hyre_batch_settle(ex._h) == 0  # final device results before the gather
        shards.append((dev, ex))
    # gather: [G][stride] hits, [G][B] offsets, [G][B] counts (device buffers)
    res = []
    for dev, ex in shards:
        hp, nh, op, cp = C.c_void_p(), C.c_uint64(), C.c_void_p(), C.c_void_p()
        assert L.lib().hyre_batch_device_results(ex._h, C.byref(hp), C.byref(nh), C.byref(op), C.byref(cp)) == 0
        torch.cuda.synchronize()
        res.append((hp.value, nh.value, op.value, cp.value))
    stride = max(r[1] for r in res)
    g_hits = torch.zeros(G, stride * 2, dtype=torch.int32, device="cuda")
    g_off = torch.zeros(G, B, dtype=torch.int64, device="cuda")
    g_cnt = torch.zeros(G, B, dtype=torch.int32, device="cuda")
    class Dev:  # wraps a library device pointer for torch (as bench.py does)
        def __init__(self, ptr, n, typestr):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}

    for g, (hp, nh, op, cp) in enumerate(res):
        g_hits[g, : nh * 2].copy_(torch.as_tensor(Dev(hp, nh * 2, "<i4"), device="cuda"))
        g_off[g].copy_(torch.as_tensor(Dev(op, B, "<i8"), device="cuda"))
        g_cnt[g].copy_(torch.as_tensor(Dev(cp, B, "<i4"), device="cuda"))
    torch.cuda.synchronize()
    ex0 = shards[0][1]
    if packed:
        hw = stride * 2
        rw = hw + 3 * B + (3 * B) % 2
        g_rec = torch.zeros(G, rw, dtype=torch.int32, device="cuda")
        g_rec[:, :hw] = g_hits
        g_rec[:, hw:hw + 2 * B] = g_off.view(torch.int32)
        g_rec[:, hw + 2 * B:hw + 3 * B] = g_cnt
        torch.cuda.synchronize()
        assert L.lib().hyre_batch_merge_packed(ex0._h, g_rec.data_ptr(), G, rw, hw) == 0
    else:
        assert L.lib().hyre_batch_merge_gathered(ex0._h, g_hits.data_ptr(), g_off.data_ptr(), g_cnt.data_ptr(), G,
                                                 stride) == 0
    caps = [q.k for q in batch.queries]
    offs = np.concatenate([[0], np.cumsum(caps)[:-1]]).astype(np.uint64)
    out = (L.hyre_hit * sum(caps))()
    counts = np.zeros(B, np.uint32)
    sts = np.zeros(B, np.int32)
    assert L.lib().hyre_batch_fetch(ex0._h, out, offs.ctypes.data_as(L.u64p), counts.ctypes.data_as(L.u32p),
                                    sts.ctypes.data_as(L.i32p), None) == 0
    for i, q in enumerate(batch.queries):
        got = [out[int(offs[i]) + j] for j in range(counts[i])]
        gr = np.asarray([h.row for h in got], np.int64)
        gs = np.asarray([h.score for h in got], np.float32)
        clauses = [(c.slot, c.attribute_ids) for c in q.terms.clauses]
        er, es = O.execute(fr, clauses, q.embedding, q.k, quant_enabled=False)
        if q.embedding is None:
            assert gr.tolist() == er.tolist()
        else:
            assert_topk_match(fr, q.embedding, gr, gs, er, es)
