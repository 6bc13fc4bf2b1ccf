"""B200-native hybrid retrieval hot path (arXiv 2402.13435, "hyre").

Drop-in for the reference's query path (proj/include/hyre): CNF term
eligibility, exact cosine scoring and top-K, executed by hand-written sm_100a
kernels behind the C-ABI in include/hyre_b200.h.  Importing the package loads
libhyre_b200.so and fails loudly if it has not been built.
"""

from ._lib import lib as _load_lib

_load_lib()

from .hyre import *  # noqa: E402,F401,F403
from .hyre import (  # noqa: E402,F401
    BatchRequest, CnfClause, CnfQuery, DeviceError, DeviceIndex, DocumentInput, ExecOptions, Executor, ExecutorPool,
    FrozenIndex, HybridQuery, IndexBuilder, IndexConfig, LoadError, Messenger, QuantCodec, QueryOutcome,
    ScoreDomainError, ScoredDoc, ScoredMessengers, Signature, StageTimings, TopKResult, ValidationError,
    bucket_top_k, clause_matches, encode, exact_scores, execute, execute_batch, full_scan_tbr, make_codec,
    merge_topk, normalize_query, preselect, quant_score, quant_score_words, validate_query)
