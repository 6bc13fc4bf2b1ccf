"""B200-native hybrid retrieval hot path (arXiv 2402.13435, "hyre").

Drop-in for the reference's query path (proj/include/hyre): CNF term
eligibility, exact cosine scoring and top-K, executed by hand-written sm_100a
kernels behind the C-ABI in include/hyre_b200.h.

The product API (IndexBuilder, Executor, ...) is loaded on first use:
accessing any of it maps libhyre_b200.so and fails loudly if it has not been
built.  Importing only the synthetic-workload generators
(``paper_2402_13435_b200.workloads``, libhyre_synth.so) does not map the
product library, so the reference arm of bench.py runs without it.
"""

_EXPORTS = (
    "BatchRequest", "CnfClause", "CnfQuery", "DeviceError", "DeviceIndex", "DocumentInput", "ExecOptions", "Executor",
    "ExecutorPool", "FrozenIndex", "HybridQuery", "IndexBuilder", "IndexConfig", "LoadError", "Messenger",
    "QuantCodec", "QueryOutcome", "QueryPack", "ScoreDomainError", "ScoredDoc", "ScoredMessengers", "ShardedExecutor", "ShardedIndex",
    "Signature", "StageTimings", "TopKResult", "ValidationError", "bucket_top_k", "clause_matches", "encode",
    "batch_scan_tbr", "exact_scores", "execute", "execute_batch", "full_scan_tbr", "make_codec", "merge_topk", "normalize_query",
    "preselect", "quant_score", "quant_score_words", "validate_query", "hyre")


def load():
    """Maps libhyre_b200.so (raises ImportError if it is missing) and returns
    the API module."""
    import importlib
    importlib.import_module(__name__ + "._lib").lib()
    return importlib.import_module(__name__ + ".hyre")


def __getattr__(name):
    if name in _EXPORTS:
        mod = load()
        return mod if name == "hyre" else getattr(mod, name)  # ("hyre": the API module itself)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")


def __dir__():
    return sorted(list(globals()) + list(_EXPORTS))
