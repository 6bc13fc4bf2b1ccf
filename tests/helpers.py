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
