"""ORACLE / TEST INFRASTRUCTURE ONLY -- never imported by the product path.

A numpy restatement of the reference's hybrid-retrieval hot path
(/root/reference/proj, "hyre"): F-TBR CNF term scan, sign-quant
pre-selection, exact cosine scoring and bucket top-K, plus the reference's
deterministic test-corpus generators.  Only ``tests/``, ``bench.py``'s
``cpu_baseline`` leg and ``__graft_entry__.smoke()`` may import it, and only
as the checker.

Parity status: PINNED.  ``tests/test_oracle.py`` checks every function here
against golden vectors produced by the *compiled reference itself*
(``oracle/_ref/libhyre_ref.so``, built from /root/reference sources by
``oracle/Makefile``; fixtures written by ``tests/golden/make_golden.py``) and
against the reference's own hand-written known-answer tests.

Arithmetic notes
----------------
* ``exact_scores`` accumulates in float32, in dimension order, with separate
  multiply and add (the reference's ``dot += q[d] * row[d]``, knn.cpp:36, is
  compiled without FMA contraction).  numpy float32 elementwise ops are IEEE
  single mul/add, so vectorising across rows while looping over d is
  bit-identical to the reference's scalar loop.
* Row normalisation (corpus.cpp:109-119), query renormalisation
  (pipeline.cpp:19-28, knn.cpp:17-29) and signature aggregation
  (quantizer.cpp:57-66) are done in double exactly as the reference does.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

MASK64 = (1 << 64) - 1


class ValidationError(ValueError):
    """Mirror of hyre::ValidationError (common.hpp:15-18)."""


class DomainError(ArithmeticError):
    """Mirror of std::domain_error thrown by bucket_top_k (knn.cpp:59-61)."""


# ---------------------------------------------------------------------------
# std::mt19937_64 (the reference's only RNG; common.hpp:166, test_util.hpp:29)
# ---------------------------------------------------------------------------
class MT19937_64:
    """Bit-exact std::mt19937_64 (Matsumoto & Nishimura 64-bit MT)."""

    _N, _M = 312, 156
    _MATRIX_A = 0xB5026F5AA96619E9
    _UPPER, _LOWER = 0xFFFFFFFF80000000, 0x7FFFFFFF

    def __init__(self, seed: int = 5489):
        mt = [0] * self._N
        mt[0] = seed & MASK64
        for i in range(1, self._N):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & MASK64
        self._mt = mt
        self._idx = self._N

    def _twist(self) -> None:
        mt, n, m = self._mt, self._N, self._M
        a, up, lo = self._MATRIX_A, self._UPPER, self._LOWER
        for i in range(n):
            x = (mt[i] & up) | (mt[(i + 1) % n] & lo)
            xa = x >> 1
            if x & 1:
                xa ^= a
            mt[i] = mt[(i + m) % n] ^ xa
        self._idx = 0

    def __call__(self) -> int:
        if self._idx >= self._N:
            self._twist()
        x = self._mt[self._idx]
        self._idx += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & MASK64


def unit_uniform(rng: MT19937_64) -> float:
    """test_util.hpp:29-31 / bench.cpp:21: (rng() >> 11) * 2^-53."""
    return float(rng() >> 11) * (2.0 ** -53)


def random_unit_vector(dim: int, rng: MT19937_64) -> np.ndarray:
    """test_util.hpp:33-48 (== bench.cpp:16-32 random_unit)."""
    v = np.empty(dim, dtype=np.float32)
    norm_sq = 0.0
    for i in range(dim):
        x = np.float32(2.0 * unit_uniform(rng) - 1.0)
        v[i] = x
        norm_sq += float(x) * float(x)
    if norm_sq == 0.0:
        v[0] = 1.0
        return v
    inv = 1.0 / math.sqrt(norm_sq)
    return (v.astype(np.float64) * inv).astype(np.float32)


# ---------------------------------------------------------------------------
# Index build (corpus.cpp:15-129)
# ---------------------------------------------------------------------------
@dataclass
class Doc:
    doc_id: str
    clauses: List[List[int]]
    embedding: np.ndarray


@dataclass
class Frozen:
    num_docs: int
    num_clauses: int
    max_num_attr: int
    dim: int
    num_bits: int
    seed: int
    attributes: np.ndarray  # u32 [N, A]
    offsets: np.ndarray  # u32 [N, C+1]
    embeddings: np.ndarray  # f32 [N, d]
    signatures: np.ndarray  # u64 [N, W]
    zero: np.ndarray  # u8 [N]
    doc_ids: List[str] = field(default_factory=list)

    def clause_slice(self, row: int, c: int) -> np.ndarray:
        o = self.offsets[row]
        return self.attributes[row, o[c]:o[c + 1]]


def freeze(docs: Sequence[Doc], num_clauses: int, max_num_attr: int, dim: int,
           num_bits: int, seed: int) -> Frozen:
    """IndexBuilder::add_document checks (corpus.cpp:29-52) + freeze (:54-129)."""
    if num_clauses == 0:
        raise ValidationError("numClauses must be >= 1")
    if dim == 0:
        raise ValidationError("dim must be >= 1")
    if max_num_attr == 0:
        raise ValidationError("maxNumAttr must be >= 1")
    seen = set()
    for d in docs:
        if d.doc_id in seen:
            raise ValidationError("duplicate docId: " + d.doc_id)
        seen.add(d.doc_id)
        if len(d.clauses) != num_clauses:
            raise ValidationError(f"clauses: expected {num_clauses} clause slots, got {len(d.clauses)}")
        if len(d.embedding) != dim:
            raise ValidationError(f"embedding: expected dim {dim}, got {len(d.embedding)}")
        for cl in d.clauses:
            if any(i == 0 for i in cl):
                raise ValidationError(f"attribute id 0 is reserved for padding (docId {d.doc_id})")
    if not docs:
        raise ValidationError("no documents staged")
    canon = [[sorted(set(cl)) for cl in d.clauses] for d in docs]
    too_wide = [d.doc_id for d, cn in zip(docs, canon) if sum(len(x) for x in cn) > max_num_attr]
    if too_wide:
        raise ValidationError(f"documents wider than maxNumAttr={max_num_attr}:" + "".join(" " + i for i in too_wide))
    n = len(docs)
    attributes = np.zeros((n, max_num_attr), dtype=np.uint32)
    offsets = np.zeros((n, num_clauses + 1), dtype=np.uint32)
    for r, cn in enumerate(canon):
        pos = 0
        for c in range(num_clauses):
            offsets[r, c] = pos
            attributes[r, pos:pos + len(cn[c])] = cn[c]
            pos += len(cn[c])
        offsets[r, num_clauses] = pos
    raw = np.stack([np.asarray(d.embedding, dtype=np.float32) for d in docs]).astype(np.float64)
    norm_sq = np.zeros(n, dtype=np.float64)
    for j in range(dim):  # sequential double accumulation, corpus.cpp:110-111
        norm_sq += raw[:, j] * raw[:, j]
    zero = (norm_sq == 0.0).astype(np.uint8)
    inv = np.where(norm_sq == 0.0, 0.0, 1.0 / np.sqrt(np.where(norm_sq == 0.0, 1.0, norm_sq)))
    emb = (raw * inv[:, None]).astype(np.float32)
    emb[zero.astype(bool)] = 0.0
    codec = make_codec(dim, num_bits, seed)
    sigs = encode_rows(codec, emb)
    return Frozen(n, num_clauses, max_num_attr, dim, num_bits, seed, attributes, offsets,
                  emb, sigs, zero, [d.doc_id for d in docs])


# ---------------------------------------------------------------------------
# Sign-quant codec (quantizer.cpp:12-84)
# ---------------------------------------------------------------------------
@dataclass
class Codec:
    dim: int
    num_bits: int
    seed: int
    rounds: List[tuple]  # (perm u32[dim], signs f32[dim], bounds u32[bins+1])

    @property
    def num_words(self) -> int:
        return (self.num_bits + 63) // 64


def make_codec(dim: int, num_bits: int, seed: int) -> Codec:
    if dim == 0:
        raise ValidationError("codec dim must be >= 1")
    if num_bits == 0:
        raise ValidationError("codec numBits must be >= 1")
    rng = MT19937_64(seed)
    rounds = []
    emitted = 0
    while emitted < num_bits:
        perm = list(range(dim))
        for i in range(dim, 1, -1):  # deterministic_shuffle, common.hpp:166-172
            j = rng() % i
            perm[i - 1], perm[j] = perm[j], perm[i - 1]
        signs = [1.0 if (rng() & 1) else -1.0 for _ in range(dim)]
        bins = min(num_bits - emitted, dim)
        base, extra = dim // bins, dim % bins
        bounds = [0]
        for b in range(bins):
            bounds.append(bounds[-1] + base + (1 if b < extra else 0))
        rounds.append((np.array(perm, dtype=np.int64), np.array(signs, dtype=np.float64),
                       np.array(bounds, dtype=np.int64)))
        emitted += bins
    return Codec(dim, num_bits, seed, rounds)


def encode_rows(codec: Codec, x: np.ndarray) -> np.ndarray:
    """encode() for each row of x (f32 [n, dim]) -> u64 [n, words]."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float32)).astype(np.float64)
    n = x.shape[0]
    words = np.zeros((n, codec.num_words), dtype=np.uint64)
    bit = 0
    for perm, signs, bounds in codec.rounds:
        for b in range(len(bounds) - 1):
            if bit >= codec.num_bits:
                break
            agg = np.zeros(n, dtype=np.float64)
            for i in range(bounds[b], bounds[b + 1]):  # sequential double sum
                agg += signs[i] * x[:, perm[i]]
            on = agg >= 0.0  # sign(0) = +1
            words[on, bit // 64] |= np.uint64(1) << np.uint64(bit % 64)
            bit += 1
    return words


def quant_score_words(a: np.ndarray, b: np.ndarray, num_bits: int) -> np.ndarray:
    """popcount(~(a^b)) with the tail of the last word masked (quantizer.cpp:72-84).

    a: u64 [W] (query), b: u64 [n, W] -> u32 [n].
    """
    same = ~(np.asarray(b, dtype=np.uint64) ^ np.asarray(a, dtype=np.uint64)[None, :])
    if num_bits % 64:
        same[:, -1] &= np.uint64((1 << (num_bits % 64)) - 1)
    bytes_ = same.view(np.uint8).reshape(same.shape[0], -1)
    return np.unpackbits(bytes_, axis=1).sum(axis=1).astype(np.uint32)


def preselect(index: Frozen, qsig: np.ndarray, rows: np.ndarray, quant_k: int) -> np.ndarray:
    """quantizer.cpp:100-138: keep quant_k best (agreement desc, row asc), row-ordered."""
    if quant_k < 1:
        raise ValidationError("quantK must be >= 1")
    rows = np.asarray(rows, dtype=np.int64)
    if len(rows) <= quant_k:
        return rows.copy()
    s = quant_score_words(qsig, index.signatures[rows], index.num_bits).astype(np.int64)
    order = np.lexsort((rows, -s))[:quant_k]
    return np.sort(rows[order])


# ---------------------------------------------------------------------------
# Term matching (term_match.cpp)
# ---------------------------------------------------------------------------
def normalize_query(raw: Dict[int, Sequence[int]], num_clauses: int) -> List[tuple]:
    """term_match.cpp:7-30 -> [(slot, sorted unique ids)], ascending slot."""
    out = []
    for slot in sorted(raw):
        if slot >= num_clauses:
            raise ValidationError(f"unknown clause slot {slot} (index has {num_clauses})")
        ids = list(raw[slot])
        if any(i == 0 for i in ids):
            raise ValidationError("attribute id 0 is reserved for padding")
        ids = sorted(set(ids))
        if not ids:
            continue
        out.append((slot, ids))
    return out


def full_scan_tbr(index: Frozen, clauses: Sequence[tuple]) -> np.ndarray:
    """term_match.cpp:56-78: rows where every clause intersects the doc slice."""
    n = index.num_docs
    ok = np.ones(n, dtype=bool)
    if not clauses:
        return np.arange(n, dtype=np.int64)
    pos = np.arange(index.max_num_attr)[None, :]
    for slot, ids in clauses:
        lo = index.offsets[:, slot].astype(np.int64)[:, None]
        hi = index.offsets[:, slot + 1].astype(np.int64)[:, None]
        in_slice = (pos >= lo) & (pos < hi)
        hit = np.isin(index.attributes, np.asarray(ids, dtype=np.uint32)) & in_slice
        ok &= hit.any(axis=1)
    return np.nonzero(ok)[0].astype(np.int64)


def batch_scan_tbr(index: Frozen, queries: Sequence, batch_ids: Sequence[int]) -> list:
    """pipeline.cpp:75-93: one pass over the rows; for each row, every query
    (in batch position order) whose clauses all match emits (row, batch_id)."""
    rows = [set(full_scan_tbr(index, q).tolist()) for q in queries]
    out = []
    for r in sorted(set().union(*rows)) if rows else []:
        for qi, s in enumerate(rows):
            if r in s:
                out.append((r, int(batch_ids[qi])))
    return out


# ---------------------------------------------------------------------------
# Scoring and selection (knn.cpp, pipeline.cpp)
# ---------------------------------------------------------------------------
def unit_embedding(raw: np.ndarray) -> tuple:
    """pipeline.cpp:19-28 / knn.cpp:17-29 -> (unit f32, renormalized?)."""
    raw = np.asarray(raw, dtype=np.float32)
    norm_sq = 0.0
    for v in raw:
        norm_sq += float(v) * float(v)
    if norm_sq != 0.0 and abs(norm_sq - 1.0) > 1e-6:
        inv = 1.0 / math.sqrt(norm_sq)
        return (raw.astype(np.float64) * inv).astype(np.float32), True
    return raw.copy(), False


def scores_rows(emb: np.ndarray, q: np.ndarray, rows: np.ndarray) -> np.ndarray:
    """Sequential fp32 mul/add dot + clamp (knn.cpp:33-38), vectorised over rows."""
    sub = emb[np.asarray(rows, dtype=np.int64)]
    dot = np.zeros(sub.shape[0], dtype=np.float32)
    q = np.asarray(q, dtype=np.float32)
    for d in range(sub.shape[1]):
        dot = dot + q[d] * sub[:, d]
    return np.clip(dot, np.float32(-1.0), np.float32(1.0))


def exact_scores(index: Frozen, query: np.ndarray, rows: np.ndarray) -> tuple:
    if len(query) != index.dim:
        raise ValidationError(f"query embedding dim {len(query)} != index dim {index.dim}")
    q, renorm = unit_embedding(query)
    return scores_rows(index.embeddings, q, rows), renorm


def top_k(rows: np.ndarray, scores: np.ndarray, k: int, granularity: int = 100) -> tuple:
    """bucket_top_k (knn.cpp:42-95); result == full sort (score desc, row asc)."""
    if k < 1:
        raise ValidationError("k must be >= 1")
    if granularity < 1:
        raise ValidationError("granularity must be >= 1")
    rows = np.asarray(rows, dtype=np.int64)
    scores = np.asarray(scores, dtype=np.float32)
    bad = (scores < -1.0) | (scores > 1.0)
    if bad.any():
        raise DomainError(f"score {float(scores[bad][0]):f} outside the documented [-1, 1] bounds")
    order = np.lexsort((rows, -scores.astype(np.float64)))[:k]
    return rows[order], scores[order]


def validate_query(index: Frozen, clauses: Sequence[tuple], embedding, k: int,
                   granularity: int = 100) -> None:
    """pipeline.cpp:44-73 (messages verbatim)."""
    if k < 1:
        raise ValidationError("k must be >= 1")
    if granularity < 1:
        raise ValidationError("granularity must be >= 1")
    if embedding is not None and len(embedding) != index.dim:
        raise ValidationError(f"embedding: expected dim {index.dim}, got {len(embedding)}")
    last = None
    for slot, ids in clauses:
        if slot >= index.num_clauses:
            raise ValidationError(f"unknown clause slot {slot}")
        if last is not None and slot <= last:
            raise ValidationError("clause slots must be ascending and unique")
        last = slot
        if len(ids) == 0:
            raise ValidationError(f"clause {slot} has no attribute ids")
        for i, a in enumerate(ids):
            if a == 0:
                raise ValidationError("attribute id 0 is reserved for padding")
            if i > 0 and a <= ids[i - 1]:
                raise ValidationError("clause attribute ids must be strictly increasing (use normalize_query)")


def weighted_scores(emb: np.ndarray, q: np.ndarray, rows: np.ndarray, row_weights) -> np.ndarray:
    """The north star's learned-weight epilogue (no reference counterpart; the
    reference score is the pure cosine, knn.cpp:36-37): w[row] x clamp(dot),
    one fp32 multiply of the reference's exact score."""
    s = scores_rows(emb, q, rows)
    if row_weights is None:
        return s
    return (np.asarray(row_weights, np.float32)[np.asarray(rows, np.int64)] * s).astype(np.float32)


def execute(index: Frozen, clauses: Sequence[tuple], embedding: Optional[np.ndarray], k: int,
            quant_enabled: bool = True, quant_k: int = 0, granularity: int = 100, row_weights=None) -> tuple:
    """Executor::execute (pipeline.cpp:108-145) -> (rows i64[], scores f32[]);
    row_weights: the learned per-row weights (weighted_scores)."""
    validate_query(index, clauses, embedding, k, granularity)
    matches = full_scan_tbr(index, clauses)
    if len(matches) == 0:
        return np.zeros(0, np.int64), np.zeros(0, np.float32)
    if embedding is None:
        take = matches[:k]
        return take, np.zeros(len(take), np.float32)
    q, _ = unit_embedding(embedding)
    qk = quant_k if quant_k != 0 else 200 * k
    if quant_enabled and len(matches) > qk:
        qsig = encode_rows(make_codec(index.dim, index.num_bits, index.seed), q)[0]
        matches = preselect(index, qsig, matches, qk)
    s = weighted_scores(index.embeddings, q, matches, row_weights)
    return top_k(matches, s, k, granularity)


# ---------------------------------------------------------------------------
# Deterministic corpora (test_util.hpp:54-117) and the §8(d) synthetic workloads
# ---------------------------------------------------------------------------
@dataclass
class CorpusSpec:
    num_docs: int = 100
    dim: int = 16
    num_clauses: int = 2
    max_attrs_per_clause: int = 4
    attr_universe: int = 50
    num_bits: int = 64
    seed: int = 1


def make_corpus_docs(spec: CorpusSpec) -> tuple:
    """test_util.hpp:69-101 -> (docs, widest)."""
    rng = MT19937_64(spec.seed)
    docs, widest = [], 1
    for i in range(spec.num_docs):
        clauses, width = [], 0
        for _ in range(spec.num_clauses):
            count = rng() % (spec.max_attrs_per_clause + 1)
            cl = [1 + (rng() % spec.attr_universe) for _ in range(count)]
            width += len(set(cl))
            clauses.append(cl)
        widest = max(widest, width)
        docs.append(Doc(f"doc{i}", clauses, random_unit_vector(spec.dim, rng)))
    return docs, widest


def make_corpus(spec: CorpusSpec) -> tuple:
    docs, widest = make_corpus_docs(spec)
    return docs, freeze(docs, spec.num_clauses, widest, spec.dim, spec.num_bits, spec.seed + 1000)


def random_query(spec: CorpusSpec, rng: MT19937_64) -> List[tuple]:
    """test_util.hpp:105-117."""
    raw = {}
    for c in range(spec.num_clauses):
        if rng() % 2 == 0:
            continue
        count = 1 + rng() % 4
        raw[c] = [1 + (rng() % spec.attr_universe) for _ in range(count)]
    return normalize_query(raw, spec.num_clauses)


def reference_tbr(docs: Sequence[Doc], clauses: Sequence[tuple]) -> np.ndarray:
    """test_util.hpp:126-147 hash-set oracle over the staged docs."""
    out = []
    for r, d in enumerate(docs):
        if all(set(d.clauses[slot]) & set(ids) for slot, ids in clauses):
            out.append(r)
    return np.asarray(out, dtype=np.int64)


def cnf_workload_docs(n: int, dim: int, num_clauses: int, vocab_per_slot: int, seed: int,
                      max_ids_per_slot: int = 3) -> tuple:
    """SURVEY §8(d) c1/c3 generator (pure Python; small n only).

    Doc-major RNG order: per slot a = 1 + rng()%3 ids, each
    1 + c*V + rng()%V, then random_unit_vector(dim).  Returns raw
    (slot_offsets u32 [n*C+1], ids u32[], embeddings f32 [n, dim]).
    """
    rng = MT19937_64(seed)
    offs, ids, embs = [0], [], []
    for _ in range(n):
        for c in range(num_clauses):
            a = 1 + rng() % max_ids_per_slot
            for _ in range(a):
                ids.append(1 + c * vocab_per_slot + rng() % vocab_per_slot)
            offs.append(len(ids))
        embs.append(random_unit_vector(dim, rng))
    return (np.asarray(offs, np.uint64), np.asarray(ids, np.uint32),
            np.stack(embs).astype(np.float32))


def cnf_workload_queries(b: int, dim: int, num_clauses: int, vocab_per_slot: int, draws: int,
                         seed: int) -> tuple:
    """SURVEY §8(d) query generator: per slot `draws` ids with replacement, then
    random_unit_vector(dim). Returns ([clauses], f32 [b, dim])."""
    rng = MT19937_64(seed)
    qs, embs = [], []
    for _ in range(b):
        raw = {}
        for c in range(num_clauses):
            raw[c] = [1 + c * vocab_per_slot + rng() % vocab_per_slot for _ in range(draws)]
        qs.append(normalize_query(raw, num_clauses))
        embs.append(random_unit_vector(dim, rng))
    return qs, np.stack(embs).astype(np.float32)
