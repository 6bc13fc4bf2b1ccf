"""Tie-aware top-K comparator (correctness gates 2-3).

Exact score equality is impossible between the oracle's sequential
no-FMA fp32 dot and the GPU's FMA/tree reduction, so hybrid results are
compared with:
  * score tolerance eps(s) = max(REL_TOL * |s|, ABS_TOL) per hit
    (north star: 1e-3 relative for fp32; 2e-5 absolute floor for near-zero
    cosines -- the worst-case rounding of two d=128 unit-vector dots is
    ~1.5e-5);
  * identical hit sets except for rows tied with the K-th score (within eps);
  * the GPU list ordered by (GPU score desc, row asc) exactly.
Term-only results (integer rows) must be identical.
"""

from __future__ import annotations

import numpy as np

REL_TOL = 1e-3
ABS_TOL = 2e-5
BF16_ABS_TOL = 2.5e-3  # single-pass bf16 query rounding


def eps(s, rel=REL_TOL, abs_=ABS_TOL):
    return np.maximum(rel * np.abs(np.asarray(s, np.float64)), abs_)


def assert_topk_match(ref_index, query_embedding, got_rows, got_scores, ref_rows, ref_scores,
                      rel=REL_TOL, abs_=ABS_TOL, emb_override=None):
    """ref_index: oracle Frozen (numpy) used to score GPU rows exactly as the
    reference would; emb_override: embedding matrix actually scored (bf16 upcast)."""
    from oracle import hyre_oracle as O

    got_rows = np.asarray(got_rows, np.int64)
    got_scores = np.asarray(got_scores, np.float32)
    ref_rows = np.asarray(ref_rows, np.int64)
    ref_scores = np.asarray(ref_scores, np.float32)
    assert len(got_rows) == len(ref_rows), f"hit count {len(got_rows)} != oracle {len(ref_rows)}"
    if len(ref_rows) == 0:
        return
    q, _ = O.unit_embedding(query_embedding)
    emb = ref_index.embeddings if emb_override is None else emb_override
    check_topk(got_rows, got_scores, ref_rows, ref_scores, O.scores_rows(emb, q, got_rows), rel, abs_)


def check_topk(got_rows, got_scores, ref_rows, ref_scores, oracle_of_got, rel=REL_TOL, abs_=ABS_TOL):
    """Gates 2-3 given the oracle's own score of every returned row
    (`oracle_of_got`, e.g. the compiled reference's exact_scores)."""
    got_rows = np.asarray(got_rows, np.int64)
    got_scores = np.asarray(got_scores, np.float32)
    ref_rows = np.asarray(ref_rows, np.int64)
    ref_scores = np.asarray(ref_scores, np.float32)
    oracle_of_got = np.asarray(oracle_of_got, np.float64)
    assert len(got_rows) == len(ref_rows), f"hit count {len(got_rows)} != oracle {len(ref_rows)}"
    if len(ref_rows) == 0:
        return
    assert len(set(got_rows.tolist())) == len(got_rows), "duplicate rows in GPU result"
    e_got = eps(oracle_of_got, rel, abs_)
    # (b) every GPU score within tolerance of the oracle's score for that row
    bad = np.abs(got_scores.astype(np.float64) - oracle_of_got) > e_got
    assert not bad.any(), (f"score mismatch rows {got_rows[bad][:5]} gpu {got_scores[bad][:5]} "
                           f"oracle {oracle_of_got[bad][:5]}")
    tau = float(ref_scores[-1])
    e_tau = float(eps(tau, rel, abs_))
    # (a) all oracle hits clearly above the boundary are present
    must = set(ref_rows[ref_scores > tau + e_tau].tolist())
    missing = must - set(got_rows.tolist())
    assert not missing, f"oracle hits missing from GPU result: {sorted(missing)[:10]}"
    # (c) GPU hits outside the oracle set are boundary ties
    extra = ~np.isin(got_rows, ref_rows)
    if extra.any():
        assert (oracle_of_got[extra] >= tau - 2 * e_tau).all(), (
            f"non-tied extra rows {got_rows[extra]} scores {oracle_of_got[extra]} tau {tau}")
    # (d) ordered by (score desc, row asc) on the GPU's own scores
    key = np.lexsort((got_rows, -got_scores.astype(np.float64)))
    assert np.array_equal(key, np.arange(len(got_rows))), "GPU hits not in (score desc, row asc) order"
    # (e) positionally, only near-ties may swap
    assert (np.abs(oracle_of_got - ref_scores.astype(np.float64)) <= 2 * eps(ref_scores, rel, abs_) + 1e-12).all()
