"""Python mirror of the reference's hot-path API (proj/include/hyre/*.hpp).

Same names, argument meaning and error behaviour as the reference so that
parity tests read like the reference's own doctest suites:

* ``IndexBuilder(IndexConfig)``, ``add_document``, ``freeze(make_codec(...))``
  -- corpus.hpp:36-52
* ``FrozenIndex`` accessors, ``save``/``load`` -- corpus.hpp:57-124
* ``normalize_query`` / ``full_scan_tbr`` -- term_match.hpp:31-45
* ``encode`` / ``quant_score`` / ``preselect`` -- quantizer.hpp:48-74
* ``exact_scores`` / ``bucket_top_k`` -- knn.hpp:24-35
* ``Executor.execute`` / ``execute_batch``, ``validate_query`` -- pipeline.hpp:57-100

Every call goes through the C-ABI of ``libhyre_b200.so``; all query-path
compute runs in hand-written sm_100a kernels.  There is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _lib as L
from ._lib import hyre_hit, hyre_query

# ---------------------------------------------------------------------------
# Errors (common.hpp:15-33, knn.cpp:59-61)
# ---------------------------------------------------------------------------


class ValidationError(ValueError):
    """hyre::ValidationError (std::invalid_argument); the message names the field."""


class LoadError(RuntimeError):
    """hyre::LoadError with a distinguishable cause."""

    class Cause(IntEnum):
        kBadMagic = 0
        kVersionMismatch = 1
        kTruncated = 2
        kChecksum = 3

    def __init__(self, cause: "LoadError.Cause", msg: str):
        super().__init__(msg)
        self._cause = cause

    def cause(self) -> "LoadError.Cause":
        return self._cause


class ScoreDomainError(ArithmeticError):
    """std::domain_error raised by bucket_top_k for a score outside [-1, 1]."""


class DeviceError(RuntimeError):
    """CUDA / allocation failure inside the library (std::runtime_error)."""


def _check(rc: int) -> None:
    if rc == L.HYRE_OK:
        return
    msg = (L.lib().hyre_last_error() or b"").decode()
    if rc == L.HYRE_INVALID_ARGUMENT:
        raise ValidationError(msg)
    if rc == L.HYRE_OUT_OF_RANGE:
        raise ScoreDomainError(msg)
    if rc == L.HYRE_LOAD_ERROR:
        raise LoadError(LoadError.Cause(L.lib().hyre_last_load_cause()), msg)
    raise DeviceError(f"[status {rc}] {msg}")


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


# ---------------------------------------------------------------------------
# Codec (quantizer.hpp:17-76)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class QuantCodec:
    """Deterministic in (dim, num_bits, seed) (quantizer.hpp:46-52); the
    rounds are re-derived inside the library exactly as FrozenIndex::load does."""

    dim: int
    num_bits: int
    seed: int

    def num_words(self) -> int:
        return (self.num_bits + 63) // 64


def make_codec(dim: int, num_bits: int, seed: int) -> QuantCodec:
    if dim == 0:
        raise ValidationError("codec dim must be >= 1")
    if num_bits == 0:
        raise ValidationError("codec numBits must be >= 1")
    return QuantCodec(dim, num_bits, seed)


@dataclass
class Signature:
    num_bits: int
    words: np.ndarray  # u64

    def bit(self, b: int) -> bool:
        return bool((int(self.words[b // 64]) >> (b % 64)) & 1)

    def __eq__(self, other) -> bool:
        return self.num_bits == other.num_bits and np.array_equal(self.words, other.words)


def encode(codec: QuantCodec, embedding) -> Signature:
    x = np.ascontiguousarray(embedding, np.float32)
    if len(x) != codec.dim:
        raise ValidationError(f"embedding length {len(x)} != codec dim {codec.dim}")
    w = np.zeros(codec.num_words(), np.uint64)
    _check(L.lib().hyre_encode(codec.dim, codec.num_bits, codec.seed, _p(x, L.f32p), _p(w, L.u64p)))
    return Signature(codec.num_bits, w)


def quant_score_words(a, b, num_bits: int) -> int:
    a = np.ascontiguousarray(a, np.uint64)
    b = np.ascontiguousarray(b, np.uint64)
    return int(L.lib().hyre_quant_score_words(_p(a, L.u64p), _p(b, L.u64p), len(a), num_bits))


def quant_score(a: Signature, b: Signature) -> int:
    if a.num_bits != b.num_bits:
        raise ValidationError("signature width mismatch")
    return quant_score_words(a.words, b.words, a.num_bits)


# ---------------------------------------------------------------------------
# Index build (corpus.hpp)
# ---------------------------------------------------------------------------
@dataclass
class IndexConfig:
    num_clauses: int = 0
    max_num_attr: int = 0
    dim: int = 0
    clause_names: List[str] = field(default_factory=list)


@dataclass
class DocumentInput:
    doc_id: str = ""
    clauses: List[List[int]] = field(default_factory=list)
    embedding: Sequence[float] = field(default_factory=list)


class IndexBuilder:
    """Single-writer staging area (corpus.hpp:36-52)."""

    def __init__(self, config: IndexConfig):
        names = [n.encode() for n in config.clause_names]
        arr = (C.c_char_p * max(1, len(names)))(*names) if names else None
        h = C.c_void_p()
        _check(L.lib().hyre_builder_create(config.num_clauses, config.max_num_attr, config.dim, arr, len(names),
                                           C.byref(h)))
        self._h = h
        self._dim = config.dim

    def __del__(self):
        if getattr(self, "_h", None):
            L.lib().hyre_builder_destroy(self._h)
            self._h = None

    def add_document(self, doc: DocumentInput) -> int:
        offs = np.zeros(len(doc.clauses) + 1, np.uint32)
        flat: List[int] = []
        for i, cl in enumerate(doc.clauses):
            flat.extend(int(x) for x in cl)
            offs[i + 1] = len(flat)
        ids = np.asarray(flat if flat else [0], np.uint32)
        emb = np.ascontiguousarray(doc.embedding, np.float32)
        if emb.size == 0:
            emb = np.zeros(1, np.float32)
            elen = 0
        else:
            elen = len(emb)
        row = C.c_uint32()
        _check(L.lib().hyre_builder_add_document(self._h, doc.doc_id.encode(), len(doc.clauses), _p(offs, L.u32p),
                                                 _p(ids, L.u32p), _p(emb, L.f32p), elen, C.byref(row)))
        return row.value

    def add_documents(self, slot_offsets, ids, embeddings, doc_id_prefix: str = "d") -> None:
        """Bulk add of n documents with ids ``prefix + row`` (flat CSR clause ids)."""
        so = np.ascontiguousarray(slot_offsets, np.uint64)
        ids = np.ascontiguousarray(ids if len(ids) else np.zeros(1), np.uint32)
        emb = np.ascontiguousarray(embeddings, np.float32)
        _check(L.lib().hyre_builder_add_documents(self._h, emb.shape[0], doc_id_prefix.encode(), _p(so, L.u64p),
                                                  _p(ids, L.u32p), _p(emb, L.f32p)))

    def size(self) -> int:
        return int(L.lib().hyre_builder_size(self._h))

    def freeze(self, codec: QuantCodec, device: Optional[int] = None) -> "FrozenIndex":
        """corpus.cpp:54-129; device=<ordinal> computes it on that GPU
        (bit-identical arrays, same errors) -- for large builds."""
        if codec.dim != self._dim:
            raise ValidationError("codec dim != index dim")
        h = C.c_void_p()
        if device is None:
            _check(L.lib().hyre_builder_freeze(self._h, codec.num_bits, codec.seed, C.byref(h)))
        else:
            _check(L.lib().hyre_builder_freeze_device(self._h, codec.num_bits, codec.seed, int(device), C.byref(h)))
        return FrozenIndex(h)


class FrozenIndex:
    """Immutable searchable corpus (corpus.hpp:57-124).  Host arrays are
    zero-copy numpy views; the device column store is created on first use."""

    def __init__(self, handle):
        self._h = handle
        s = L.hyre_shape()
        L.lib().hyre_frozen_shape(self._h, C.byref(s))
        self._shape = s
        n, a, c, d, w = s.num_docs, s.max_num_attr, s.num_clauses, s.dim, s.num_words

        def view(fn, ctype, shape, dtype):
            ptr = fn(self._h)
            if not ptr or int(np.prod(shape)) == 0:
                return np.zeros(shape, dtype)
            arr = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), shape=shape)
            arr.flags.writeable = False
            return arr

        lib = L.lib()
        self.attributes = view(lib.hyre_frozen_attributes, C.c_uint32, (n, a), np.uint32)
        self.offsets = view(lib.hyre_frozen_offsets, C.c_uint32, (n, c + 1), np.uint32)
        self.embeddings = view(lib.hyre_frozen_embeddings, C.c_float, (n, d), np.float32)
        self.signatures = view(lib.hyre_frozen_signatures, C.c_uint64, (n, w), np.uint64)
        self.zero_flags = view(lib.hyre_frozen_zero_flags, C.c_uint8, (n,), np.uint8)
        self._devices: Dict[tuple, "DeviceIndex"] = {}

    def __del__(self):
        if getattr(self, "_h", None):
            self._devices.clear()
            L.lib().hyre_frozen_destroy(self._h)
            self._h = None

    @classmethod
    def from_arrays(cls, attributes, offsets, embeddings, num_bits: int, seed: int, signatures=None,
                    zero_flags=None, doc_id_prefix: str = "d") -> "FrozenIndex":
        att = np.ascontiguousarray(attributes, np.uint32)
        off = np.ascontiguousarray(offsets, np.uint32)
        emb = np.ascontiguousarray(embeddings, np.float32)
        n, a = att.shape
        sig = None if signatures is None else np.ascontiguousarray(signatures, np.uint64)
        zf = None if zero_flags is None else np.ascontiguousarray(zero_flags, np.uint8)
        h = C.c_void_p()
        _check(L.lib().hyre_frozen_from_arrays(
            n, off.shape[1] - 1, a, emb.shape[1], num_bits, seed, _p(att, L.u32p), _p(off, L.u32p),
            _p(emb, L.f32p), None if sig is None else _p(sig, L.u64p), None if zf is None else _p(zf, L.u8p),
            None, doc_id_prefix.encode(), C.byref(h)))
        return cls(h)

    # -- shape ---------------------------------------------------------------
    def num_docs(self) -> int:
        return self._shape.num_docs

    def num_clauses(self) -> int:
        return self._shape.num_clauses

    def max_num_attr(self) -> int:
        return self._shape.max_num_attr

    def dim(self) -> int:
        return self._shape.dim

    def codec(self) -> QuantCodec:
        return QuantCodec(self._shape.dim, self._shape.num_bits, self._shape.seed)

    def clause_names(self) -> List[str]:
        return [L.lib().hyre_frozen_clause_name(self._h, c).decode() for c in range(self.num_clauses())]

    # -- accessors (corpus.hpp:68-103) --------------------------------------
    def attribute_row(self, row: int) -> np.ndarray:
        return self.attributes[row]

    def offsets_row(self, row: int) -> np.ndarray:
        return self.offsets[row]

    def clause_slice(self, row: int, clause: int) -> np.ndarray:
        o = self.offsets[row]
        return self.attributes[row, o[clause]:o[clause + 1]]

    def embedding_row(self, row: int) -> np.ndarray:
        return self.embeddings[row]

    def signature_words(self, row: int) -> np.ndarray:
        return self.signatures[row]

    def signature_row(self, row: int) -> Signature:
        return Signature(self._shape.num_bits, self.signatures[row].copy())

    def embedding_is_zero(self, row: int) -> bool:
        return bool(self.zero_flags[row])

    def doc_id(self, row: int) -> str:
        s = L.lib().hyre_frozen_doc_id(self._h, row)
        if s is None:
            raise IndexError(row)
        return s.decode()

    def row_of(self, doc_id: str) -> Optional[int]:
        r = L.lib().hyre_frozen_row_of(self._h, doc_id.encode())
        return None if r < 0 else int(r)

    def resolve_clause_slot(self, name: str) -> int:
        return int(L.lib().hyre_frozen_resolve_clause_slot(self._h, name.encode()))

    def save(self, path: str) -> None:
        _check(L.lib().hyre_frozen_save(self._h, str(path).encode()))

    @staticmethod
    def load(path: str) -> "FrozenIndex":
        h = C.c_void_p()
        _check(L.lib().hyre_frozen_load(str(path).encode(), C.byref(h)))
        return FrozenIndex(h)

    def __eq__(self, other: "FrozenIndex") -> bool:
        return (self.num_docs() == other.num_docs() and self.num_clauses() == other.num_clauses()
                and self.max_num_attr() == other.max_num_attr() and self.dim() == other.dim()
                and self.clause_names() == other.clause_names()
                and np.array_equal(self.attributes, other.attributes)
                and np.array_equal(self.offsets, other.offsets)
                and np.array_equal(self.embeddings.view(np.uint32), other.embeddings.view(np.uint32))
                and np.array_equal(self.signatures, other.signatures)
                and np.array_equal(self.zero_flags, other.zero_flags)
                and all(self.doc_id(r) == other.doc_id(r) for r in range(self.num_docs()))
                and self.codec() == other.codec())

    # -- device column store -------------------------------------------------
    def device(self, device: int = 0, dtype: str = "f32", tensor_path: bool = True, row_begin: int = 0,
               row_end: int = 0) -> "DeviceIndex":
        key = (device, dtype, tensor_path, row_begin, row_end)
        if key not in self._devices:
            self._devices[key] = DeviceIndex(self, device, dtype, tensor_path, row_begin, row_end)
        return self._devices[key]


class DeviceIndex:
    """The FrozenIndex (or a row shard of it) resident in one GPU's HBM."""

    def __init__(self, frozen: FrozenIndex, device: int = 0, dtype: str = "f32", tensor_path: bool = True,
                 row_begin: int = 0, row_end: int = 0, row_offset: int = 0):
        o = L.hyre_index_options(device, L.HYRE_EMB_BF16 if dtype == "bf16" else L.HYRE_EMB_F32, row_begin,
                                 row_end, int(tensor_path), row_offset)
        h = C.c_void_p()
        _check(L.lib().hyre_index_create(frozen._h, C.byref(o), C.byref(h)))
        self._h = h
        self.frozen = frozen
        self.dtype = dtype

    def __del__(self):
        if getattr(self, "_h", None):
            L.lib().hyre_index_destroy(self._h)
            self._h = None

    def set_row_weights(self, weights) -> None:
        """Learned per-row weights (north star; no reference counterpart):
        hybrid scores become w[row] x clamp(cosine), w in [0, 1], one weight
        per row of this index; None restores the pure cosine."""
        if weights is None:
            _check(L.lib().hyre_index_set_row_weights(self._h, None, 0))
            return
        w = np.ascontiguousarray(weights, np.float32)
        _check(L.lib().hyre_index_set_row_weights(self._h, _p(w, L.f32p), w.size))

    def stats(self) -> dict:
        s = L.hyre_index_stats()
        _check(L.lib().hyre_index_stats_get(self._h, C.byref(s)))
        return {n: int(getattr(s, n)) for n, _ in L.hyre_index_stats._fields_}


# ---------------------------------------------------------------------------
# Queries (term_match.hpp, pipeline.hpp)
# ---------------------------------------------------------------------------
@dataclass
class CnfClause:
    slot: int = 0
    attribute_ids: List[int] = field(default_factory=list)


@dataclass
class CnfQuery:
    clauses: List[CnfClause] = field(default_factory=list)

    def match_all(self) -> bool:
        return not self.clauses


def normalize_query(raw: Dict[int, Sequence[int]], num_clauses: int) -> CnfQuery:
    slots = np.asarray(list(raw.keys()) or [0], np.uint32)
    offs = np.zeros(len(raw) + 1, np.uint32)
    flat: List[int] = []
    for i, s in enumerate(raw):
        flat.extend(int(x) for x in raw[s])
        offs[i + 1] = len(flat)
    ids = np.asarray(flat or [0], np.uint32)
    n = C.c_uint32()
    os_ = np.zeros(len(raw) + 1, np.uint32)
    oo = np.zeros(len(raw) + 2, np.uint32)
    oi = np.zeros(max(1, len(flat)), np.uint32)
    _check(L.lib().hyre_normalize_query(len(raw), _p(slots, L.u32p), _p(offs, L.u32p), _p(ids, L.u32p),
                                        num_clauses, C.byref(n), _p(os_, L.u32p), _p(oo, L.u32p),
                                        _p(oi, L.u32p)))
    return CnfQuery([CnfClause(int(os_[c]), [int(x) for x in oi[oo[c]:oo[c + 1]]]) for c in range(n.value)])


@dataclass
class ExecOptions:
    quant_enabled: bool = True
    quant_k: int = 0
    granularity: int = 100

    def effective_quant_k(self, k: int) -> int:
        return self.quant_k if self.quant_k != 0 else 200 * k


@dataclass
class HybridQuery:
    terms: CnfQuery = field(default_factory=CnfQuery)
    embedding: Optional[Sequence[float]] = None
    k: int = 10
    options: ExecOptions = field(default_factory=ExecOptions)


@dataclass
class BatchRequest:
    queries: List[HybridQuery] = field(default_factory=list)


@dataclass
class StageTimings:
    tbr_ms: float = 0.0
    quant_ms: float = 0.0
    ebr_ms: float = 0.0
    topk_ms: float = 0.0
    total_ms: float = 0.0


@dataclass
class Messenger:
    row_id: int = 0
    batch_id: int = 0
    score: float = 0.0


@dataclass
class ScoredDoc:
    doc_id: str = ""
    row_id: int = 0
    score: float = 0.0


@dataclass
class TopKResult:
    hits: List[ScoredDoc] = field(default_factory=list)


@dataclass
class QueryOutcome:
    ok: bool = False
    result: TopKResult = field(default_factory=TopKResult)
    error: str = ""


@dataclass
class ScoredMessengers:
    items: List[Messenger] = field(default_factory=list)
    query_was_renormalized: bool = False


class QueryPack:
    """Packs HybridQuery objects into a contiguous hyre_query array whose
    pointers stay valid as long as the pack lives."""

    def __init__(self, queries: Sequence[HybridQuery]):
        self.keep = []
        self.arr = (hyre_query * max(1, len(queries)))()
        for i, q in enumerate(queries):
            cl = q.terms.clauses
            slots = np.asarray([c.slot for c in cl] or [0], np.uint32)
            offs = np.zeros(len(cl) + 1, np.uint32)
            flat: List[int] = []
            for j, c in enumerate(cl):
                flat.extend(int(x) for x in c.attribute_ids)
                offs[j + 1] = len(flat)
            ids = np.asarray(flat or [0], np.uint32)
            emb = None if q.embedding is None else np.ascontiguousarray(q.embedding, np.float32)
            if emb is not None and emb.size == 0:
                emb = np.zeros(1, np.float32)
                edim = 0
            else:
                edim = 0 if emb is None else len(emb)
            self.keep += [slots, offs, ids, emb]
            s = self.arr[i]
            s.n_clauses = len(cl)
            s.slots = _p(slots, L.u32p)
            s.id_offsets = _p(offs, L.u32p)
            s.ids = _p(ids, L.u32p)
            s.embedding = None if emb is None else _p(emb, L.f32p)
            s.embedding_dim = edim
            s.k = max(0, int(q.k))
            s.quant_enabled = int(bool(q.options.quant_enabled))
            s.quant_k = int(q.options.quant_k)
            s.granularity = max(0, int(q.options.granularity))


def validate_query(index: FrozenIndex, query: HybridQuery) -> None:
    pack = QueryPack([query])
    _check(L.lib().hyre_validate_query(index._h, C.byref(pack.arr[0])))


def _timings(t: L.hyre_timings) -> StageTimings:
    return StageTimings(t.tbr_ms, t.quant_ms, t.ebr_ms, t.topk_ms, t.total_ms)


class Executor:
    """One in-flight batch per executor (pipeline.hpp:66-96); scratch is sized
    from (rows, max_batch) at construction on the executor's device."""

    def __init__(self, index, max_batch: int = 16, device: int = 0, dtype: str = "f32",
                 tensor_path: bool = True):
        if max_batch < 1:
            raise ValidationError("maxBatch must be >= 1")
        self._dev = index if isinstance(index, DeviceIndex) else index.device(device, dtype, tensor_path)
        self._index = self._dev.frozen
        h = C.c_void_p()
        _check(L.lib().hyre_executor_create(self._dev._h, max_batch, C.byref(h)))
        self._h = h
        self._max_batch = max_batch

    def __del__(self):
        if getattr(self, "_h", None):
            L.lib().hyre_executor_destroy(self._h)
            self._h = None

    def index(self) -> FrozenIndex:
        return self._index

    def max_batch(self) -> int:
        return self._max_batch

    def _result(self, hits, n: int) -> TopKResult:
        return TopKResult([ScoredDoc(self._index.doc_id(h.row), int(h.row), float(np.float32(h.score)))
                           for h in hits[:n]])

    def execute(self, query: HybridQuery, timings: Optional[StageTimings] = None) -> TopKResult:
        pack = QueryPack([query])
        cap = max(1, min(max(query.k, 1), self._index.num_docs()))
        hits = (hyre_hit * cap)()
        n = C.c_uint32()
        t = L.hyre_timings()
        _check(L.lib().hyre_execute(self._h, C.byref(pack.arr[0]), hits, C.byref(n), C.byref(t)))
        if timings is not None:
            timings.__dict__.update(_timings(t).__dict__)
        return self._result(hits, n.value)

    def execute_batch(self, batch: BatchRequest, timings: Optional[StageTimings] = None) -> List[QueryOutcome]:
        qs = batch.queries
        b = len(qs)
        pack = QueryPack(qs)
        caps = [max(0, min(max(q.k, 0), self._index.num_docs())) for q in qs]
        offs = np.zeros(max(b, 1), np.uint64)
        if b:
            offs[:b] = np.concatenate([[0], np.cumsum(caps)[:-1]])
        hits = (hyre_hit * max(1, sum(caps)))()
        counts = np.zeros(max(b, 1), np.uint32)
        st = np.zeros(max(b, 1), np.int32)
        t = L.hyre_timings()
        _check(L.lib().hyre_execute_batch(self._h, pack.arr, b, hits, _p(offs, L.u64p), _p(counts, L.u32p),
                                          _p(st, L.i32p), C.byref(t)))
        if timings is not None:
            timings.__dict__.update(_timings(t).__dict__)
        out = []
        for i in range(b):
            if st[i] != L.HYRE_OK:
                out.append(QueryOutcome(False, TopKResult(), L.lib().hyre_executor_slot_error(self._h, i).decode()))
            else:
                base = int(offs[i])
                out.append(QueryOutcome(True, self._result(hits[base:base + int(counts[i])], int(counts[i])), ""))
        return out

    # -- stage entry points ---------------------------------------------------
    def full_scan_tbr(self, query: CnfQuery, batch_id: int = 0) -> List[Messenger]:
        rows = self.full_scan_rows(query)
        return [Messenger(int(r), batch_id, 0.0) for r in rows]

    def full_scan_rows(self, query: CnfQuery) -> np.ndarray:
        pack = QueryPack([HybridQuery(terms=query, k=1)])
        out = np.zeros(max(1, self._index.num_docs()), np.uint32)
        n = C.c_uint64()
        _check(L.lib().hyre_full_scan_tbr(self._h, C.byref(pack.arr[0]), _p(out, L.u32p), len(out), C.byref(n)))
        return out[: n.value].astype(np.int64)

    def batch_scan_tbr(self, queries: Sequence[CnfQuery], batch_ids: Sequence[int]) -> List[Messenger]:
        """pipeline.cpp:75-93: one pass over the rows for every query; the
        matches ordered by (rowId, query position), stamped with batch_ids."""
        if len(batch_ids) != len(queries):
            raise ValidationError("batch_ids must have one id per query")
        if not queries:
            return []
        pack = QueryPack([HybridQuery(terms=q, k=1) for q in queries])
        bid = np.ascontiguousarray(batch_ids, np.uint32)
        n = C.c_uint64()
        _check(L.lib().hyre_batch_scan_tbr(self._h, pack.arr, len(queries), _p(bid, L.u32p), None, 0, C.byref(n)))
        out = (L.hyre_messenger * max(1, n.value))()
        _check(L.lib().hyre_batch_scan_tbr(self._h, pack.arr, len(queries), _p(bid, L.u32p), out, n.value,
                                           C.byref(n)))
        return [Messenger(int(m.row_id), int(m.batch_id), 0.0) for m in out[: n.value]]

    def exact_scores(self, query_embedding, candidates: Sequence[Messenger]) -> ScoredMessengers:
        q = np.ascontiguousarray(query_embedding, np.float32)
        rows = np.asarray([m.row_id for m in candidates] or [0], np.uint32)
        n = len(candidates)
        out = np.zeros(max(1, n), np.float32)
        ren = C.c_int32()
        qq = q if q.size else np.zeros(1, np.float32)
        _check(L.lib().hyre_exact_scores(self._h, _p(qq, L.f32p), len(q), _p(rows, L.u32p), n, _p(out, L.f32p),
                                         C.byref(ren)))
        items = [Messenger(m.row_id, m.batch_id, float(out[i])) for i, m in enumerate(candidates)]
        return ScoredMessengers(items, bool(ren.value))

    def bucket_top_k(self, scored: ScoredMessengers, k: int, granularity: int = 100) -> TopKResult:
        rows = np.asarray([m.row_id for m in scored.items] or [0], np.uint32)
        sc = np.asarray([m.score for m in scored.items] or [0], np.float32)
        n = len(scored.items)
        cap = max(1, min(max(k, 1), n))
        hits = (hyre_hit * cap)()
        cnt = C.c_uint32()
        _check(L.lib().hyre_bucket_top_k(self._h, _p(rows, L.u32p), _p(sc, L.f32p), n, k, granularity, hits,
                                         C.byref(cnt)))
        return self._result(hits, cnt.value)

    def preselect(self, query_signature: Signature, candidates: Sequence[Messenger], quant_k: int) -> List[Messenger]:
        rows = np.asarray([m.row_id for m in candidates] or [0], np.uint32)
        n = len(candidates)
        out = np.zeros(max(1, n), np.uint32)
        cnt = C.c_uint64()
        qw = np.ascontiguousarray(query_signature.words, np.uint64)
        _check(L.lib().hyre_preselect(self._h, _p(qw, L.u64p), _p(rows, L.u32p), n, quant_k, _p(out, L.u32p),
                                      C.byref(cnt)))
        by_row = {m.row_id: m for m in candidates}
        return [by_row[int(r)] for r in out[: cnt.value]]


class ShardedIndex:
    """A FrozenIndex row-sharded over devices (hyre_sharded_index_*,
    SURVEY §8(e)): shard g = rows [g N / G, (g + 1) N / G) on devices[g]
    (default g % device count; shards may share a device)."""

    def __init__(self, frozen: FrozenIndex, n_shards: int, devices: Optional[Sequence[int]] = None,
                 dtype: str = "f32", tensor_path: bool = True):
        self.frozen = frozen
        devs = None if devices is None else np.ascontiguousarray(devices, np.int32)
        o = L.hyre_sharded_index_options(n_shards, None if devs is None else _p(devs, L.i32p),
                                         L.HYRE_EMB_BF16 if dtype == "bf16" else L.HYRE_EMB_F32, int(tensor_path))
        h = C.c_void_p()
        _check(L.lib().hyre_sharded_index_create(frozen._h, C.byref(o), C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            L.lib().hyre_sharded_index_destroy(self._h)
            self._h = None

    def set_row_weights(self, weights) -> None:
        """DeviceIndex.set_row_weights over every shard (weights in global row order)."""
        if weights is None:
            _check(L.lib().hyre_sharded_index_set_row_weights(self._h, None, 0))
            return
        w = np.ascontiguousarray(weights, np.float32)
        _check(L.lib().hyre_sharded_index_set_row_weights(self._h, _p(w, L.f32p), w.size))

    def info(self):
        """-> (n_shards, [device of each shard])."""
        n = C.c_uint32()
        devs = np.zeros(16, np.int32)
        _check(L.lib().hyre_sharded_index_info(self._h, C.byref(n), _p(devs, L.i32p)))
        return int(n.value), devs[: n.value].tolist()


class ShardedExecutor:
    """Executor over a ShardedIndex (hyre_sharded_* in include/hyre_b200.h):
    one Executor + stream per shard, per-shard top-K merged exactly on shard
    0's device through peer memory, global quant pre-selection.  Same
    execute / execute_batch contract and results as Executor.  `index` is a
    ShardedIndex, or a FrozenIndex sharded here into `n_shards`."""

    def __init__(self, index, n_shards: int = 1, devices: Optional[Sequence[int]] = None, dtype: str = "f32",
                 tensor_path: bool = True, max_batch: int = 16):
        if max_batch < 1:
            raise ValidationError("maxBatch must be >= 1")
        self._sx = index if isinstance(index, ShardedIndex) else ShardedIndex(index, n_shards, devices, dtype,
                                                                              tensor_path)
        self._index = self._sx.frozen
        h = C.c_void_p()
        _check(L.lib().hyre_sharded_create(self._sx._h, max_batch, C.byref(h)))
        self._h = h
        self._max_batch = max_batch

    def __del__(self):
        if getattr(self, "_h", None):
            L.lib().hyre_sharded_destroy(self._h)
            self._h = None

    def index(self) -> FrozenIndex:
        return self._index

    def max_batch(self) -> int:
        return self._max_batch

    def info(self):
        return self._sx.info()

    def execute(self, query: HybridQuery, timings: Optional[StageTimings] = None) -> TopKResult:
        out = self.execute_batch(BatchRequest([query]), timings)[0]
        if not out.ok:
            raise ValidationError(out.error)
        return out.result

    def execute_batch(self, batch: BatchRequest, timings: Optional[StageTimings] = None) -> List[QueryOutcome]:
        qs = batch.queries
        b = len(qs)
        pack = QueryPack(qs)
        caps = [max(0, min(max(q.k, 0), self._index.num_docs())) for q in qs]
        offs = np.zeros(max(b, 1), np.uint64)
        if b:
            offs[:b] = np.concatenate([[0], np.cumsum(caps)[:-1]])
        hits = (hyre_hit * max(1, sum(caps)))()
        counts = np.zeros(max(b, 1), np.uint32)
        st = np.zeros(max(b, 1), np.int32)
        t = L.hyre_timings()
        _check(L.lib().hyre_sharded_execute_batch(self._h, pack.arr, b, hits, _p(offs, L.u64p), _p(counts, L.u32p),
                                                  _p(st, L.i32p), C.byref(t)))
        if timings is not None:
            timings.__dict__.update(_timings(t).__dict__)
        out = []
        for i in range(b):
            if st[i] != L.HYRE_OK:
                out.append(QueryOutcome(False, TopKResult(), L.lib().hyre_sharded_slot_error(self._h, i).decode()))
            else:
                base = int(offs[i])
                n = int(counts[i])
                out.append(QueryOutcome(True, TopKResult([ScoredDoc(self._index.doc_id(h.row), int(h.row),
                                                                    float(np.float32(h.score)))
                                                          for h in hits[base:base + n]]), ""))
        return out


class ExecutorPool:
    """The B200 ExecutorPool (service.cpp:99-141, ServiceConfig workers /
    max_batch, service.hpp:19-26) with dynamic request batching: `workers`
    executors, each with its own CUDA stream; concurrent search() calls are
    grouped into execute_batch calls of up to max_batch queries, waiting at
    most max_wait_us for a batch to fill.  search() is thread-safe (the ctypes
    call releases the GIL) and returns what Executor.execute would."""

    def __init__(self, index, workers: int = 2, max_batch: int = 16, max_wait_us: int = 200, device: int = 0,
                 dtype: str = "f32", tensor_path: bool = True):
        self._dev = index if isinstance(index, DeviceIndex) else index.device(device, dtype, tensor_path)
        self._index = self._dev.frozen
        h = C.c_void_p()
        _check(L.lib().hyre_pool_create(self._dev._h, workers, max_batch, max_wait_us, C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            L.lib().hyre_pool_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def search(self, query: HybridQuery) -> TopKResult:
        pack = QueryPack([query])
        cap = max(1, min(max(query.k, 1), self._index.num_docs()))
        hits = (hyre_hit * cap)()
        n = C.c_uint32()
        _check(L.lib().hyre_pool_search(self._h, C.byref(pack.arr[0]), hits, C.byref(n)))
        return TopKResult([ScoredDoc(self._index.doc_id(h.row), int(h.row), float(np.float32(h.score)))
                           for h in hits[: n.value]])

    def stats(self) -> tuple:
        """(batches run, queries served)."""
        b, q = C.c_uint64(), C.c_uint64()
        _check(L.lib().hyre_pool_stats(self._h, C.byref(b), C.byref(q)))
        return int(b.value), int(q.value)


# Free functions over a per-index default executor (pipeline.hpp:98-100 and
# the public stage functions the reference's tests call directly).
def _default_executor(index: FrozenIndex, max_batch: int = 1) -> Executor:
    ex = getattr(index, "_default_exec", None)
    if ex is None or ex.max_batch() < max_batch:
        ex = Executor(index, max(max_batch, 16))
        index._default_exec = ex
    return ex


def full_scan_tbr(index: FrozenIndex, query: CnfQuery, batch_id: int = 0) -> List[Messenger]:
    return _default_executor(index).full_scan_tbr(query, batch_id)


def batch_scan_tbr(index: FrozenIndex, queries: Sequence[CnfQuery], batch_ids: Sequence[int]) -> List[Messenger]:
    return _default_executor(index, max(1, len(queries))).batch_scan_tbr(queries, batch_ids)


def clause_matches(index: FrozenIndex, row_id: int, clause: CnfClause) -> bool:
    """Host two-pointer intersection of one row (term_match.cpp:34-54); the
    device path never calls this -- it is the per-row predicate of the API."""
    a = index.clause_slice(row_id, clause.slot)
    return bool(np.intersect1d(a, np.asarray(clause.attribute_ids, np.uint32)).size)


def exact_scores(index: FrozenIndex, query_embedding, candidates: Sequence[Messenger]) -> ScoredMessengers:
    return _default_executor(index).exact_scores(query_embedding, candidates)


def bucket_top_k(index: FrozenIndex, scored: ScoredMessengers, k: int, granularity: int = 100) -> TopKResult:
    return _default_executor(index).bucket_top_k(scored, k, granularity)


def preselect(index: FrozenIndex, query_signature: Signature, candidates: Sequence[Messenger],
              quant_k: int) -> List[Messenger]:
    return _default_executor(index).preselect(query_signature, candidates, quant_k)


def execute(index: FrozenIndex, query: HybridQuery) -> TopKResult:
    return _default_executor(index).execute(query)


def execute_batch(index: FrozenIndex, batch: BatchRequest) -> List[QueryOutcome]:
    return _default_executor(index, max(1, len(batch.queries))).execute_batch(batch)


def merge_topk(lists: Sequence[np.ndarray], k: int) -> np.ndarray:
    """Exact merge of per-shard (row u32, score f32) hit lists."""
    arrs = [np.ascontiguousarray(l, dtype=np.dtype([("row", np.uint32), ("score", np.float32)])) for l in lists]
    ptrs = (C.POINTER(hyre_hit) * max(1, len(arrs)))(*[a.ctypes.data_as(C.POINTER(hyre_hit)) for a in arrs])
    counts = np.asarray([len(a) for a in arrs] or [0], np.uint32)
    out = np.zeros(max(1, k), dtype=arrs[0].dtype if arrs else np.dtype([("row", np.uint32), ("score", np.float32)]))
    n = C.c_uint32()
    _check(L.lib().hyre_merge_topk(ptrs, _p(counts, L.u32p), len(arrs), k,
                                   out.ctypes.data_as(C.POINTER(hyre_hit)), C.byref(n)))
    return out[: n.value]
