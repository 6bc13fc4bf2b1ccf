"""Synthetic workloads of SURVEY.md §8(d) (measurement infrastructure,
the analogue of the reference's make_bench_index / run_bench,
proj/src/bench.cpp:42-131).

Generation runs in libhyre_synth.so (std::mt19937_64, the reference's RNG
conventions); indexes are built through the product IndexBuilder / freeze.

Configs (BASELINE.json):
  c1  100K x d64 fp32, 4-clause CNF (V=20/slot, 7 draws), B=1, K=100
  c2  1M x d128, match-all, B=1/256, K=100
  c3  10M x d128 fp32, 8-clause CNF (V=20/slot, 13 draws, ~5% selectivity), B=64, K=100
  c4  50M x d128 bf16, match-all, B=1/1024, K=100
  c5  50M, 1 slot of Zipf(1.1) link ids over a 100K vocab, term-only, K=1000
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SYNTH_PATH = os.path.join(HERE, "libhyre_synth.so")

_synth = None


def synth():
    global _synth
    if _synth is None:
        if not os.path.exists(SYNTH_PATH):
            raise ImportError(f"{SYNTH_PATH} missing: run make -C paper_2402_13435_b200/csrc")
        L = C.CDLL(SYNTH_PATH)
        L.synth_cnf_docs.restype = C.c_uint64
        L.synth_cnf_docs.argtypes = [C.c_uint32] * 6 + [C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.synth_cnf_queries.restype = None
        L.synth_cnf_queries.argtypes = [C.c_uint32] * 5 + [C.c_uint64, C.c_void_p, C.c_void_p]
        L.synth_unit_vectors.restype = None
        L.synth_unit_vectors.argtypes = [C.c_uint32] * 3 + [C.c_uint64, C.c_void_p]
        L.synth_zipf_docs.restype = C.c_uint64
        L.synth_zipf_docs.argtypes = [C.c_uint32] * 4 + [C.c_double, C.c_uint32, C.c_uint64, C.c_void_p,
                                                         C.c_void_p, C.c_void_p]
        _synth = L
    return _synth


@dataclass
class Workload:
    name: str
    n: int
    dim: int
    num_clauses: int
    vocab: int          # ids per slot (cnf) or vocabulary (zipf)
    draws: int          # query ids drawn per slot (cnf)
    max_ids: int        # max ids per doc per slot
    k: int
    batch: int
    kind: str           # "cnf" | "match_all" | "zipf"
    dtype: str = "f32"
    num_bits: int = 512
    seed: int = 42
    qseed: int = 4242

    @property
    def max_num_attr(self) -> int:
        return self.num_clauses * self.max_ids


WORKLOADS = {
    "c1": Workload("c1", 100_000, 64, 4, 20, 7, 3, 100, 1, "cnf"),
    "c2": Workload("c2", 1_000_000, 128, 1, 1, 0, 1, 100, 256, "match_all"),
    "c3": Workload("c3", 10_000_000, 128, 8, 20, 13, 3, 100, 64, "cnf"),
    "c4": Workload("c4", 50_000_000, 128, 1, 1, 0, 1, 100, 1024, "match_all", dtype="bf16"),
    "c5": Workload("c5", 50_000_000, 16, 1, 100_000, 0, 8, 1000, 1, "zipf"),
}


def cnf_docs(w: Workload, row_begin: int = 0, row_end: Optional[int] = None):
    row_end = w.n if row_end is None else row_end
    rows = row_end - row_begin
    so = np.zeros(rows * w.num_clauses + 1, np.uint64)
    ids = np.zeros(max(1, rows * w.num_clauses * w.max_ids), np.uint32)
    emb = np.zeros((rows, w.dim), np.float32)
    n_ids = synth().synth_cnf_docs(row_begin, row_end, w.dim, w.num_clauses, w.vocab, w.max_ids, w.seed,
                                   so.ctypes.data, ids.ctypes.data, emb.ctypes.data)
    return so, ids[:n_ids], emb


def match_all_docs(w: Workload, row_begin: int = 0, row_end: Optional[int] = None):
    row_end = w.n if row_end is None else row_end
    rows = row_end - row_begin
    emb = np.zeros((rows, w.dim), np.float32)
    synth().synth_unit_vectors(row_begin, row_end, w.dim, w.seed, emb.ctypes.data)
    # one slot holding a single constant id per doc (the index needs >= 1 clause)
    so = np.arange(rows + 1, dtype=np.uint64)
    ids = np.ones(rows, np.uint32)
    return so, ids, emb


def zipf_docs(w: Workload, row_begin: int = 0, row_end: Optional[int] = None):
    row_end = w.n if row_end is None else row_end
    rows = row_end - row_begin
    so = np.zeros(rows + 1, np.uint64)
    ids = np.zeros(rows * w.max_ids, np.uint32)
    emb = np.zeros((rows, w.dim), np.float32)
    n_ids = synth().synth_zipf_docs(row_begin, row_end, w.dim, w.vocab, 1.1, w.max_ids, w.seed, so.ctypes.data,
                                    ids.ctypes.data, emb.ctypes.data)
    return so, ids[:n_ids], emb


def docs(w: Workload, row_begin: int = 0, row_end: Optional[int] = None):
    return {"cnf": cnf_docs, "match_all": match_all_docs, "zipf": zipf_docs}[w.kind](w, row_begin, row_end)


def queries(w: Workload, b: Optional[int] = None, high_pass: bool = True):
    """-> (list of raw {slot: ids} maps, f32 [b, dim] embeddings or None)."""
    b = w.batch if b is None else b
    if w.kind == "cnf":
        ids = np.zeros(b * w.num_clauses * w.draws, np.uint32)
        emb = np.zeros((b, w.dim), np.float32)
        synth().synth_cnf_queries(b, w.dim, w.num_clauses, w.vocab, w.draws, w.qseed, ids.ctypes.data,
                                  emb.ctypes.data)
        ids = ids.reshape(b, w.num_clauses, w.draws)
        raws = [{c: ids[q, c].tolist() for c in range(w.num_clauses)} for q in range(b)]
        return raws, emb
    if w.kind == "match_all":
        emb = np.zeros((b, w.dim), np.float32)
        synth().synth_unit_vectors(0, b, w.dim, w.qseed, emb.ctypes.data)
        return [{} for _ in range(b)], emb
    # zipf term-only: high pass = 32 head ids, low pass = 8 tail ids
    rs = np.random.default_rng(w.qseed)
    if high_pass:
        raws = [{0: list(range(1, 33))} for _ in range(b)]
    else:
        raws = [{0: rs.integers(50_001, 100_001, size=8).tolist()} for _ in range(b)]
    return raws, None


def build_frozen(w: Workload, row_begin: int = 0, row_end: Optional[int] = None):
    """Generates the corpus rows [row_begin, row_end) and freezes them with the
    product IndexBuilder (doc ids "d<global row>")."""
    so, ids, emb = docs(w, row_begin, row_end)
    return freeze_docs(w, so, ids, emb, row_begin)


def freeze_docs(w: Workload, so, ids, emb, row_begin: int = 0):
    """Freezes generated rows with the product IndexBuilder."""
    import paper_2402_13435_b200 as hy
    b = hy.IndexBuilder(hy.IndexConfig(w.num_clauses, w.max_num_attr, w.dim))
    if row_begin:
        # keep global doc ids: pad the running row counter with a distinct prefix per shard
        b.add_documents(so, ids, emb, doc_id_prefix=f"d{row_begin}+")
    else:
        b.add_documents(so, ids, emb, doc_id_prefix="d")
    return b.freeze(hy.make_codec(w.dim, w.num_bits, w.seed))
