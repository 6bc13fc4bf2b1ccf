"""Generates tests/golden/*.json from the *compiled reference* (oracle/_ref,
built by `make -C oracle` from /root/reference sources).  Run here, where
/root/reference exists; the fixtures are committed so the GPU box (which has
no /root/reference) and the CPU tests can pin the oracle and the product.

    python tests/golden/make_golden.py

Scores are stored as float32 bit patterns (hex) so comparisons are exact.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import hyre_oracle as O  # noqa: E402
from oracle import ref as R  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def f32hex(a):
    return [f"{int(x):08x}" for x in np.asarray(a, np.float32).view(np.uint32)]


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def ref_from_docs(docs, num_clauses, widest, dim, num_bits, seed):
    offs, ids = [0], []
    for d in docs:
        for cl in d.clauses:
            ids += list(cl)
            offs.append(len(ids))
    emb = np.stack([np.asarray(d.embedding, np.float32) for d in docs])
    return R.RefIndex.build(np.asarray(offs, np.uint32), np.asarray(ids or [0], np.uint32), emb, num_clauses,
                            widest, num_bits, seed)


def corpus(spec):
    docs, widest = O.make_corpus_docs(spec)
    return docs, widest, ref_from_docs(docs, spec.num_clauses, widest, spec.dim, spec.num_bits, spec.seed + 1000)


def main():
    fixtures = {}

    # --- freeze layout digests (test_corpus.cpp:50-215 style corpora) -------
    fz = []
    for spec in [O.CorpusSpec(num_docs=20, dim=8, seed=5), O.CorpusSpec(num_docs=37, dim=6, num_bits=96),
                 O.CorpusSpec(num_docs=300, dim=12, num_clauses=2, attr_universe=10, seed=501)]:
        docs, widest, ri = corpus(spec)
        att, off, emb, sig, zf = ri.export()
        fz.append({"spec": spec.__dict__, "widest": widest,
                   "sha256": digest(att, off, emb.view(np.uint32), sig, zf),
                   "doc_ids": [ri.doc_id(0), ri.doc_id(spec.num_docs - 1)]})
    fixtures["freeze"] = fz

    # --- TBR on random corpora (test_term_match.cpp:119-132) ----------------
    tbr = []
    spec = O.CorpusSpec(num_docs=60, num_clauses=3, attr_universe=12)
    rng = O.MT19937_64(99)
    for trial in range(25):
        spec.seed = 1000 + trial
        docs, widest, ri = corpus(spec)
        q = O.random_query(spec, rng)
        tbr.append({"seed": spec.seed, "query": q, "rows": ri.full_scan_tbr(q).tolist()})
    fixtures["tbr"] = tbr

    # --- batch scan stream (pipeline.cpp:75-93, test_pipeline.cpp:221-235) ---
    bs = []
    rng = O.MT19937_64(123)
    for trial in range(6):
        spec.seed = 2000 + trial
        docs, widest, ri = corpus(spec)
        qs = [O.random_query(spec, rng) for _ in range(1 + trial)]
        if trial == 3:
            qs.append([])  # match-all
        ids = [7 * i + trial for i in range(len(qs))]
        bs.append({"seed": spec.seed, "queries": qs, "batch_ids": ids,
                   "stream": [list(p) for p in ri.batch_scan_tbr(qs, ids)]})
    fixtures["batch_scan"] = bs

    # --- hybrid search, quant off and on (test_pipeline.cpp:124-197) --------
    hyb = []
    spec = O.CorpusSpec(num_docs=300, dim=12, num_clauses=2, attr_universe=10)
    rng = O.MT19937_64(41)
    for trial in range(12):
        spec.seed = 500 + trial
        docs, widest, ri = corpus(spec)
        terms = O.random_query(spec, rng)
        raw = np.asarray([np.float32(4.0 * O.unit_uniform(rng) - 2.0) for _ in range(spec.dim)], np.float32)
        for qe, qk in [(False, 0), (True, 30)]:
            rows, sc = ri.execute(terms, raw, 10, quant_enabled=qe, quant_k=qk)
            hyb.append({"seed": spec.seed, "terms": terms, "raw": f32hex(raw), "k": 10, "quant": qe, "quant_k": qk,
                        "rows": rows.tolist(), "scores": f32hex(sc)})
    fixtures["hybrid"] = hyb

    # --- quant pre-selection at scale (acceptance.cpp:125-202 flavour) ------
    qt = []
    spec = O.CorpusSpec(num_docs=4000, dim=16, num_bits=256, num_clauses=1, max_attrs_per_clause=1,
                        attr_universe=2, seed=7)
    docs, widest, ri = corpus(spec)
    rng = O.MT19937_64(13)
    for t in range(8):
        raw = O.random_unit_vector(spec.dim, rng)
        terms = [(0, [1])] if t % 2 else []
        qk = [60, 200, 1000, 0][t % 4]
        rows, sc = ri.execute(terms, raw, 1 + t, quant_enabled=True, quant_k=qk)
        qt.append({"terms": terms, "raw": f32hex(raw), "k": 1 + t, "quant_k": qk, "rows": rows.tolist(),
                   "scores": f32hex(sc)})
    fixtures["quant"] = {"spec": spec.__dict__, "cases": qt}

    # --- codec + encode (test_quantizer.cpp:71-187) --------------------------
    cd = {}
    for (d, b, s) in [(4, 512, 3), (8, 12, 3), (10, 13, 3), (16, 96, 11)]:
        rounds = R.codec(d, b, s)
        cd[f"{d}_{b}_{s}"] = {"n_rounds": len(rounds), "first_perm": rounds[0][0].tolist(),
                              "first_signs": rounds[0][1].tolist(),
                              "bounds": [r[2].tolist() for r in rounds[-2:]]}
    rng = O.MT19937_64(4)
    enc = []
    for d, b, s in [(16, 64, 9), (24, 128, 31), (128, 512, 42)]:
        x = O.random_unit_vector(d, rng)
        enc.append({"dim": d, "bits": b, "seed": s, "x": f32hex(x),
                    "words": [f"{int(w):016x}" for w in R.encode(d, b, s, x)]})
    fixtures["codec"] = cd
    fixtures["encode"] = enc

    # --- bucket top-K over planted ties (test_knn.cpp:145-171) --------------
    spec = O.CorpusSpec(num_docs=500, dim=8, num_clauses=1, seed=77)
    docs, widest, ri = corpus(spec)
    rng = O.MT19937_64(123)
    tk = []
    for g in (1, 2, 100):
        for k in (1, 7, 100, 499, 500):
            s = np.asarray([np.float32(2.0 * O.unit_uniform(rng) - 1.0) for _ in range(500)], np.float32)
            s[17] = s[401] = s[88]
            rows, sc = ri.bucket_top_k(np.arange(500), s, k, g)
            tk.append({"g": g, "k": k, "scores": f32hex(s), "rows": rows.tolist()})
    fixtures["topk"] = tk

    # --- c1 workload slice: 20K docs x d64, 4-clause CNF -----
    n, dim, C, V = 20_000, 64, 4, 20
    offs, ids, emb = O.cnf_workload_docs(n, dim, C, V, 11)
    ri = R.RefIndex.build(offs.astype(np.uint32), ids, emb, C, 3 * C, 512, 42, "d")
    qs, qemb = O.cnf_workload_queries(6, dim, C, V, 7, 7)
    c1 = []
    for i, q in enumerate(qs):
        rows, sc = ri.execute(q, qemb[i], 100, quant_enabled=False)
        c1.append({"query": q, "emb": f32hex(qemb[i]), "rows": rows.tolist(), "scores": f32hex(sc),
                   "n_tbr": len(ri.full_scan_tbr(q))})
    att, off, e, sig, zf = ri.export()
    fixtures["c1_slice"] = {"n": n, "dim": dim, "clauses": C, "vocab": V, "seed": 11, "qseed": 7, "draws": 7,
                            "sha256": digest(att, off, e.view(np.uint32), sig, zf), "queries": c1}

    # --- normalize_query / validate_query messages ---------------------------
    msgs = {}
    for name, raw, nc in [("unknown_slot", {2: [1]}, 2), ("zero_id", {0: [0]}, 2)]:
        try:
            R.normalize_query(raw, nc)
        except R.RefError as e:
            msgs[name] = str(e)
    fixtures["messages"] = msgs

    with open(os.path.join(OUT, "reference_fixtures.json"), "w") as f:
        json.dump(fixtures, f, separators=(",", ":"))
    print("wrote", os.path.join(OUT, "reference_fixtures.json"))


if __name__ == "__main__":
    main()
