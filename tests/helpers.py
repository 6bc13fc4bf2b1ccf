"""Builds the same corpus into the product (libhyre_b200) and the oracle."""

from __future__ import annotations

import numpy as np

from oracle import hyre_oracle as O


def product_index(docs, num_clauses, max_num_attr, dim, num_bits, seed, clause_names=None):
    import paper_2402_13435_b200 as hy
    b = hy.IndexBuilder(hy.IndexConfig(num_clauses, max_num_attr, dim, list(clause_names or [])))
    for d in docs:
        b.add_document(hy.DocumentInput(d.doc_id, d.clauses, d.embedding))
    return b.freeze(hy.make_codec(dim, num_bits, seed))


def corpus_pair(spec: O.CorpusSpec):
    docs, ref = O.make_corpus(spec)
    prod = product_index(docs, spec.num_clauses, ref.max_num_attr, spec.dim, spec.num_bits, spec.seed + 1000)
    return docs, ref, prod


def to_cnf(clauses):
    import paper_2402_13435_b200 as hy
    return hy.CnfQuery([hy.CnfClause(int(s), [int(i) for i in ids]) for s, ids in clauses])


def hits(result):
    return (np.asarray([h.row_id for h in result.hits], np.int64),
            np.asarray([h.score for h in result.hits], np.float32))


def cnf_workload(n, dim, num_clauses, vocab, draws, b, seed=11, qseed=7):
    """SURVEY §8(d) c1/c3 workload via the native generator if available, else Python."""
    offs, ids, emb = O.cnf_workload_docs(n, dim, num_clauses, vocab, seed)
    qs, qemb = O.cnf_workload_queries(b, dim, num_clauses, vocab, draws, qseed)
    return offs, ids, emb, qs, qemb


def run_batch(ex, queries):
    """execute_batch through the C-ABI split form (prepare / run / fetch)
    without per-hit Python objects -> (list of (status, rows, scores), path
    flags, K3 variant {J, id bytes, query chunks, Np})."""
    import ctypes as C

    import paper_2402_13435_b200 as hy
    from paper_2402_13435_b200 import _lib as L
    lib = L.lib()
    pack = hy.QueryPack(queries)
    b = len(queries)
    n = ex.index().num_docs()
    caps = [max(0, min(q.k, n)) for q in queries]
    offs = np.zeros(b, np.uint64)
    offs[1:] = np.cumsum(caps)[:-1]
    hits = np.zeros(max(1, sum(caps)) * 2, np.uint32)
    counts = np.zeros(b, np.uint32)
    st = np.zeros(b, np.int32)
    hy.hyre._check(lib.hyre_batch_prepare(ex._h, pack.arr, b))
    path = int(lib.hyre_batch_path(ex._h))
    var = np.zeros(4, np.uint32)
    lib.hyre_batch_tc_variant(ex._h, var.ctypes.data_as(L.u32p))
    hy.hyre._check(lib.hyre_batch_run(ex._h))
    hy.hyre._check(lib.hyre_batch_fetch(ex._h, hits.ctypes.data_as(C.POINTER(L.hyre_hit)),
                                        offs.ctypes.data_as(L.u64p), counts.ctypes.data_as(L.u32p),
                                        st.ctypes.data_as(L.i32p), None))
    out = []
    for i in range(b):
        o, c = int(offs[i]), int(counts[i])
        h = hits[2 * o: 2 * (o + c)].reshape(-1, 2)
        out.append((int(st[i]), h[:, 0].astype(np.int64), h[:, 1].view(np.float32).copy()))
    return out, path, tuple(int(x) for x in var)
