"""ORACLE / TEST INFRASTRUCTURE ONLY -- ctypes binding of oracle/_ref/libhyre_ref.so.

``libhyre_ref.so`` is the *unmodified* reference engine
(/root/reference/proj/src/{corpus,term_match,quantizer,knn,pipeline,bench}.cpp)
compiled by ``oracle/Makefile`` together with ``oracle/ref_shim.cpp``.  It is
the checker for the CUDA path and the timed CPU baseline; nothing in the
product package may import this module.
"""

from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libhyre_ref.so")

u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)


class RefQuery(C.Structure):
    _fields_ = [
        ("n_clauses", C.c_uint32),
        ("slots", u32p),
        ("id_offsets", u32p),
        ("ids", u32p),
        ("embedding", f32p),
        ("embedding_dim", C.c_uint32),
        ("k", C.c_uint32),
        ("quant_enabled", C.c_uint32),
        ("quant_k", C.c_uint32),
        ("granularity", C.c_uint32),
    ]


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle` (needs /root/reference)")
        L = C.CDLL(LIB_PATH)
        L.ref_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def _p(a, t):
    return a.ctypes.data_as(t)


class QueryPack:
    """Holds numpy buffers alive for a RefQuery array."""

    def __init__(self, queries: Sequence[tuple]):
        # queries: (clauses [(slot, ids)], embedding | None, k, quant_enabled, quant_k, granularity)
        self.keep = []
        self.arr = (RefQuery * max(1, len(queries)))()
        for i, (clauses, emb, k, qe, qk, g) in enumerate(queries):
            slots = np.asarray([s for s, _ in clauses], np.uint32)
            offs = np.zeros(len(clauses) + 1, np.uint32)
            flat = []
            for j, (_, ids) in enumerate(clauses):
                flat.extend(ids)
                offs[j + 1] = len(flat)
            ids = np.asarray(flat, np.uint32)
            e = None if emb is None else np.ascontiguousarray(emb, np.float32)
            self.keep += [slots, offs, ids, e]
            q = self.arr[i]
            q.n_clauses = len(clauses)
            q.slots = _p(slots, u32p)
            q.id_offsets = _p(offs, u32p)
            q.ids = _p(ids, u32p)
            q.embedding = _p(e, f32p) if e is not None else None
            q.embedding_dim = 0 if e is None else len(e)
            q.k, q.quant_enabled, q.quant_k, q.granularity = k, int(bool(qe)), qk, g


class RefIndex:
    """The reference FrozenIndex (built by IndexBuilder::freeze or FrozenIndex::load)."""

    def __init__(self, handle):
        self.h = handle
        shape = np.zeros(6, np.uint32)
        lib().ref_shape(self.h, _p(shape, u32p))
        self.num_docs, self.num_clauses, self.max_num_attr, self.dim, self.num_bits, self.num_words = map(int, shape)

    def __del__(self):
        try:
            if self.h:
                lib().ref_free(self.h)
        except Exception:
            pass

    @classmethod
    def build(cls, slot_offsets, ids, embeddings, num_clauses, max_num_attr, num_bits, seed,
              doc_prefix: str = "doc") -> "RefIndex":
        so = np.ascontiguousarray(slot_offsets, np.uint32)
        ids = np.ascontiguousarray(ids, np.uint32)
        emb = np.ascontiguousarray(embeddings, np.float32)
        n, dim = emb.shape
        h = C.c_void_p()
        _check(lib().ref_build(C.c_uint32(n), C.c_uint32(num_clauses), C.c_uint32(max_num_attr),
                               C.c_uint32(dim), _p(so, u32p), _p(ids, u32p), _p(emb, f32p),
                               C.c_uint32(num_bits), C.c_uint64(seed), doc_prefix.encode(), C.byref(h)))
        return cls(h)

    @classmethod
    def load(cls, path: str) -> "RefIndex":
        h = C.c_void_p()
        _check(lib().ref_load(path.encode(), C.byref(h)))
        return cls(h)

    def save(self, path: str) -> None:
        _check(lib().ref_save(self.h, path.encode()))

    def export(self):
        n = self.num_docs
        att = np.zeros((n, self.max_num_attr), np.uint32)
        off = np.zeros((n, self.num_clauses + 1), np.uint32)
        emb = np.zeros((n, self.dim), np.float32)
        sig = np.zeros((n, self.num_words), np.uint64)
        zf = np.zeros(n, np.uint8)
        lib().ref_export(self.h, _p(att, u32p), _p(off, u32p), _p(emb, f32p), _p(sig, u64p),
                         zf.ctypes.data_as(C.POINTER(C.c_uint8)))
        return att, off, emb, sig, zf

    def doc_id(self, row: int) -> str:
        buf = C.create_string_buffer(256)
        lib().ref_doc_id(self.h, C.c_uint32(row), buf, C.c_uint32(256))
        return buf.value.decode()

    def full_scan_tbr(self, clauses) -> np.ndarray:
        qp = QueryPack([(clauses, None, 1, False, 0, 100)])
        out = np.zeros(self.num_docs, np.uint32)
        n = C.c_uint64()
        _check(lib().ref_full_scan_tbr(self.h, C.byref(qp.arr[0]), _p(out, u32p), C.c_uint64(len(out)),
                                       C.byref(n)))
        return out[: n.value].astype(np.int64)

    def batch_scan_tbr(self, queries, batch_ids) -> list:
        """pipeline.cpp:75-93 -> [(row, batch_id)] in (row, query position) order."""
        qp = QueryPack([(c, None, 1, False, 0, 100) for c in queries])
        bid = np.ascontiguousarray(batch_ids, np.uint32)
        n = C.c_uint64()
        _check(lib().ref_batch_scan_tbr(self.h, qp.arr, C.c_uint32(len(queries)), _p(bid, u32p), None,
                                        C.c_uint64(0), C.byref(n)))
        out = np.zeros(2 * max(1, n.value), np.uint32)
        _check(lib().ref_batch_scan_tbr(self.h, qp.arr, C.c_uint32(len(queries)), _p(bid, u32p), _p(out, u32p),
                                        C.c_uint64(n.value), C.byref(n)))
        return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(n.value)]

    def validate(self, clauses, emb, k, granularity=100) -> None:
        qp = QueryPack([(clauses, emb, k, False, 0, granularity)])
        _check(lib().ref_validate_query(self.h, C.byref(qp.arr[0])))

    def execute(self, clauses, emb, k, quant_enabled=True, quant_k=0, granularity=100, timings=None):
        qp = QueryPack([(clauses, emb, k, quant_enabled, quant_k, granularity)])
        rows = np.zeros(k, np.uint32)
        sc = np.zeros(k, np.float32)
        n = C.c_uint32()
        t = np.zeros(5, np.float64)
        _check(lib().ref_execute(self.h, C.byref(qp.arr[0]), _p(rows, u32p), _p(sc, f32p), C.c_uint32(k),
                                 C.byref(n), t.ctypes.data_as(C.POINTER(C.c_double))))
        if timings is not None:
            timings[:] = t
        m = min(n.value, k)
        return rows[:m].astype(np.int64), sc[:m]

    def execute_batch(self, queries, max_batch: Optional[int] = None):
        """queries: [(clauses, emb, k, quant_enabled, quant_k, granularity)] ->
        [(ok, rows, scores)]"""
        b = len(queries)
        cap = max(q[2] for q in queries)
        qp = QueryPack(queries)
        rows = np.zeros((b, cap), np.uint32)
        sc = np.zeros((b, cap), np.float32)
        cnt = np.zeros(b, np.uint32)
        st = np.zeros(b, np.int32)
        _check(lib().ref_execute_batch(self.h, qp.arr, C.c_uint32(b), C.c_uint32(max_batch or b),
                                       _p(rows, u32p), _p(sc, f32p), C.c_uint32(cap), _p(cnt, u32p),
                                       st.ctypes.data_as(C.POINTER(C.c_int32))))
        out = []
        for i in range(b):
            m = min(int(cnt[i]), cap)
            out.append((st[i] == 0, rows[i, :m].astype(np.int64), sc[i, :m].copy()))
        return out

    def execute_parallel(self, queries, threads: int, want_hits: bool = True):
        """ExecutorPool-style throughput run -> (seconds, [(rows, scores)])."""
        b = len(queries)
        cap = max(q[2] for q in queries)
        qp = QueryPack(queries)
        rows = np.zeros((b, cap), np.uint32)
        sc = np.zeros((b, cap), np.float32)
        cnt = np.zeros(b, np.uint32)
        secs = C.c_double()
        _check(lib().ref_execute_parallel(self.h, qp.arr, C.c_uint32(b), C.c_uint32(threads),
                                          _p(rows, u32p) if want_hits else None,
                                          _p(sc, f32p) if want_hits else None, C.c_uint32(cap),
                                          _p(cnt, u32p), C.byref(secs)))
        hits = [(rows[i, : min(int(cnt[i]), cap)].astype(np.int64), sc[i, : min(int(cnt[i]), cap)].copy())
                for i in range(b)]
        return secs.value, hits

    def exact_scores(self, q, rows):
        q = np.ascontiguousarray(q, np.float32)
        rows = np.ascontiguousarray(rows, np.uint32)
        out = np.zeros(len(rows), np.float32)
        ren = C.c_int32()
        _check(lib().ref_exact_scores(self.h, _p(q, f32p), C.c_uint32(len(q)), _p(rows, u32p),
                                      C.c_uint64(len(rows)), _p(out, f32p), C.byref(ren)))
        return out, bool(ren.value)

    def bucket_top_k(self, rows, scores, k, granularity=100):
        rows = np.ascontiguousarray(rows, np.uint32)
        scores = np.ascontiguousarray(scores, np.float32)
        ro = np.zeros(max(k, 1), np.uint32)
        so = np.zeros(max(k, 1), np.float32)
        n = C.c_uint32()
        _check(lib().ref_bucket_top_k(self.h, _p(rows, u32p), _p(scores, f32p), C.c_uint64(len(rows)),
                                      C.c_uint32(k), C.c_uint32(granularity), _p(ro, u32p), _p(so, f32p),
                                      C.byref(n)))
        m = min(n.value, k)
        return ro[:m].astype(np.int64), so[:m]

    def preselect(self, qwords, rows, quant_k):
        qw = np.ascontiguousarray(qwords, np.uint64)
        rows = np.ascontiguousarray(rows, np.uint32)
        out = np.zeros(len(rows), np.uint32)
        n = C.c_uint64()
        _check(lib().ref_preselect(self.h, _p(qw, u64p), _p(rows, u32p), C.c_uint64(len(rows)),
                                   C.c_uint32(quant_k), _p(out, u32p), C.byref(n)))
        return out[: n.value].astype(np.int64)


def normalize_query(raw: dict, num_clauses: int) -> List[tuple]:
    slots = np.asarray(list(raw.keys()), np.uint32)
    offs = np.zeros(len(raw) + 1, np.uint32)
    flat = []
    for i, s in enumerate(raw):
        flat.extend(raw[s])
        offs[i + 1] = len(flat)
    ids = np.asarray(flat if flat else [0], np.uint32)
    n = C.c_uint32()
    os_ = np.zeros(len(raw) + 1, np.uint32)
    oo = np.zeros(len(raw) + 2, np.uint32)
    oi = np.zeros(max(1, len(flat)), np.uint32)
    _check(lib().ref_normalize_query(C.c_uint32(len(raw)), _p(slots, u32p), _p(offs, u32p), _p(ids, u32p),
                                     C.c_uint32(num_clauses), C.byref(n), _p(os_, u32p), _p(oo, u32p),
                                     _p(oi, u32p)))
    return [(int(os_[c]), [int(x) for x in oi[oo[c]:oo[c + 1]]]) for c in range(n.value)]


def encode(dim: int, num_bits: int, seed: int, x) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    w = np.zeros((num_bits + 63) // 64, np.uint64)
    _check(lib().ref_encode(C.c_uint32(dim), C.c_uint32(num_bits), C.c_uint64(seed), _p(x, f32p), _p(w, u64p)))
    return w


def codec(dim: int, num_bits: int, seed: int):
    max_rounds = num_bits  # upper bound (>= 1 bin per round)
    n_rounds = C.c_uint32()
    perm = np.zeros(max_rounds * dim, np.uint32)
    signs = np.zeros(max_rounds * dim, np.float32)
    bounds = np.zeros(max_rounds * (dim + 1), np.uint32)
    nb = np.zeros(max_rounds, np.uint32)
    _check(lib().ref_codec(C.c_uint32(dim), C.c_uint32(num_bits), C.c_uint64(seed), C.byref(n_rounds),
                           _p(perm, u32p), _p(signs, f32p), _p(bounds, u32p), _p(nb, u32p)))
    out, pos = [], 0
    for r in range(n_rounds.value):
        out.append((perm[r * dim:(r + 1) * dim].copy(), signs[r * dim:(r + 1) * dim].copy(),
                    bounds[pos:pos + nb[r]].copy()))
        pos += int(nb[r])
    return out


class ShardedRef:
    """The reference over G FrozenIndex shards of one corpus (SURVEY.md §8(d)
    sharded oracle; oracle/ref_shim.cpp ref_build_shards /
    ref_execute_sharded).  Hybrid results are merged by (score desc, global
    row asc) and term-only ones concatenated in shard order, which equals the
    unsharded reference exactly with quant off."""

    def __init__(self, slot_offsets, ids, embeddings, num_clauses, max_num_attr, num_bits, seed,
                 shards: Optional[int] = None, threads: Optional[int] = None, doc_prefix: str = "d"):
        so = np.ascontiguousarray(slot_offsets, np.uint64)
        ids = np.ascontiguousarray(ids if len(ids) else np.zeros(1, np.uint32), np.uint32)
        emb = np.ascontiguousarray(embeddings, np.float32)
        n, dim = emb.shape
        self.num_docs, self.dim = n, dim
        threads = threads or os.cpu_count() or 1
        g = shards or max(1, min(64, -(-n // 1_000_000)))
        g = max(g, min(threads, max(1, n // 100_000)))  # use the cores even for small corpora
        self.g = g
        hs = (C.c_void_p * g)()
        self.bases = np.zeros(g, np.uint64)
        L = lib()
        L.ref_build_shards.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.c_uint32, C.c_uint64, C.c_char_p, C.c_uint32, C.c_uint32,
                                       C.c_void_p, C.c_void_p]
        _check(L.ref_build_shards(n, num_clauses, max_num_attr, dim, so.ctypes.data, ids.ctypes.data,
                                  emb.ctypes.data, num_bits, seed, doc_prefix.encode(), g, threads,
                                  C.cast(hs, C.c_void_p), self.bases.ctypes.data))
        self.hs = hs
        self.shards = [RefIndex(C.c_void_p(hs[s])) for s in range(g)]  # owns (frees) the handles

    def execute(self, queries, threads: Optional[int] = None):
        """queries: [(clauses, emb, k, quant_enabled, quant_k, granularity)] ->
        (seconds, [(status, rows, scores)]) with GLOBAL rows."""
        b = len(queries)
        cap = max(q[2] for q in queries)
        qp = QueryPack(queries)
        rows = np.zeros((b, cap), np.uint32)
        sc = np.zeros((b, cap), np.float32)
        cnt = np.zeros(b, np.uint32)
        st = np.zeros(b, np.int32)
        secs = C.c_double()
        L = lib()
        L.ref_execute_sharded.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint32, C.c_uint32,
                                          C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p]
        _check(L.ref_execute_sharded(C.cast(self.hs, C.c_void_p), self.bases.ctypes.data, self.g,
                                     C.cast(qp.arr, C.c_void_p), b, threads or os.cpu_count() or 1,
                                     rows.ctypes.data, sc.ctypes.data, cap, cnt.ctypes.data, st.ctypes.data,
                                     C.byref(secs)))
        return secs.value, [(int(st[i]), rows[i, :cnt[i]].astype(np.int64), sc[i, :cnt[i]].copy())
                            for i in range(b)]

    def exact_scores(self, q, global_rows):
        """The reference's exact_scores (knn.cpp:8-40) of arbitrary global rows."""
        rows = np.asarray(global_rows, np.int64)
        out = np.zeros(len(rows), np.float32)
        shard = np.searchsorted(self.bases.astype(np.int64), rows, side="right") - 1
        for s in np.unique(shard):
            sel = shard == s
            out[sel], _ = self.shards[s].exact_scores(q, rows[sel] - int(self.bases[s]))
        return out
