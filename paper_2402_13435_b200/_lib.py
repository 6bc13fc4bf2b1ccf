"""ctypes binding of libhyre_b200.so (the C-ABI in include/hyre_b200.h).

The shared library is built in-tree by ``paper_2402_13435_b200/csrc/Makefile``
(``__graft_entry__.build()``).  There is no fallback: if the library is
missing, importing the package raises immediately.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhyre_b200.so")

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
i32p = C.POINTER(C.c_int32)
f32p = C.POINTER(C.c_float)
vp = C.c_void_p

HYRE_OK, HYRE_INVALID_ARGUMENT, HYRE_OUT_OF_RANGE, HYRE_LOAD_ERROR = 0, 1, 2, 3
HYRE_CUDA_ERROR, HYRE_OUT_OF_MEMORY, HYRE_INTERNAL = 4, 5, 6
HYRE_EMB_F32, HYRE_EMB_BF16 = 0, 1


class hyre_query(C.Structure):
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


class hyre_hit(C.Structure):
    _fields_ = [("row", C.c_uint32), ("score", C.c_float)]


class hyre_messenger(C.Structure):
    _fields_ = [("row_id", C.c_uint32), ("batch_id", C.c_uint32), ("score", C.c_float)]


class hyre_timings(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("tbr_ms", "quant_ms", "ebr_ms", "topk_ms", "total_ms")]


class hyre_shape(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in ("num_docs", "num_clauses", "max_num_attr", "dim", "num_bits",
                                          "num_words")] + [("seed", C.c_uint64)]


class hyre_index_options(C.Structure):
    _fields_ = [("device", C.c_int32), ("emb_dtype", C.c_uint32), ("row_begin", C.c_uint32),
                ("row_end", C.c_uint32), ("tensor_path", C.c_uint32), ("row_offset", C.c_uint32)]


class hyre_sharded_index_options(C.Structure):
    _fields_ = [("n_shards", C.c_uint32), ("devices", i32p), ("emb_dtype", C.c_uint32), ("tensor_path", C.c_uint32)]


class hyre_index_stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "num_rows", "row_base", "dim", "row_stride", "num_terms", "bitmap_terms", "csr_terms", "postings",
        "embedding_bytes", "tensor_bytes", "bitmap_bytes", "csr_bytes", "signature_bytes", "forward_bytes")]


# name -> (restype, argtypes); every symbol declared in include/hyre_b200.h.
SIGNATURES = {
    "hyre_last_error": (C.c_char_p, []),
    "hyre_last_load_cause": (C.c_int, []),
    "hyre_abi_version": (C.c_int, []),
    "hyre_builder_create": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_char_p), C.c_uint32,
                                      C.POINTER(vp)]),
    "hyre_builder_destroy": (None, [vp]),
    "hyre_builder_add_document": (C.c_int, [vp, C.c_char_p, C.c_uint32, u32p, u32p, f32p, C.c_uint32, u32p]),
    "hyre_builder_add_documents": (C.c_int, [vp, C.c_uint32, C.c_char_p, u64p, u32p, f32p]),
    "hyre_builder_size": (C.c_uint32, [vp]),
    "hyre_schema_read_json": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
    "hyre_schema_create": (C.c_int, [C.c_uint32, C.POINTER(C.c_char_p), C.c_uint32, C.POINTER(vp)]),
    "hyre_schema_destroy": (None, [vp]),
    "hyre_schema_num_clauses": (C.c_uint32, [vp]),
    "hyre_schema_clause_name": (C.c_char_p, [vp, C.c_uint32]),
    "hyre_schema_dim": (C.c_uint32, [vp]),
    "hyre_documents_read_jsonl": (C.c_int, [C.c_char_p, vp, C.POINTER(vp)]),
    "hyre_documents_destroy": (None, [vp]),
    "hyre_documents_count": (C.c_uint32, [vp]),
    "hyre_documents_widest": (C.c_uint32, [vp]),
    "hyre_documents_id": (C.c_char_p, [vp, C.c_uint32]),
    "hyre_documents_slot_offsets": (u64p, [vp]),
    "hyre_documents_ids": (u32p, [vp]),
    "hyre_documents_embeddings": (f32p, [vp]),
    "hyre_builder_add_document_set": (C.c_int, [vp, vp, u32p]),
    "hyre_links_read_json": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
    "hyre_links_destroy": (None, [vp]),
    "hyre_links_num_nodes": (C.c_uint32, [vp]),
    "hyre_links_count": (C.c_uint32, [vp, C.c_int32]),
    "hyre_links_name": (C.c_char_p, [vp, C.c_int32, C.c_uint32]),
    "hyre_links_ids": (u32p, [vp, C.c_int32, C.c_uint32, u32p]),
    "hyre_builder_freeze": (C.c_int, [vp, C.c_uint32, C.c_uint64, C.POINTER(vp)]),
    "hyre_builder_freeze_device": (C.c_int, [vp, C.c_uint32, C.c_uint64, C.c_int32, C.POINTER(vp)]),
    "hyre_frozen_from_arrays": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                          u32p, u32p, f32p, u64p, u8p, C.POINTER(C.c_char_p), C.c_char_p,
                                          C.POINTER(vp)]),
    "hyre_frozen_save": (C.c_int, [vp, C.c_char_p]),
    "hyre_frozen_load": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
    "hyre_frozen_destroy": (None, [vp]),
    "hyre_frozen_shape": (None, [vp, C.POINTER(hyre_shape)]),
    "hyre_frozen_attributes": (vp, [vp]),
    "hyre_frozen_offsets": (vp, [vp]),
    "hyre_frozen_embeddings": (vp, [vp]),
    "hyre_frozen_signatures": (vp, [vp]),
    "hyre_frozen_zero_flags": (vp, [vp]),
    "hyre_frozen_doc_id": (C.c_char_p, [vp, C.c_uint32]),
    "hyre_frozen_row_of": (C.c_int64, [vp, C.c_char_p]),
    "hyre_frozen_resolve_clause_slot": (C.c_int32, [vp, C.c_char_p]),
    "hyre_frozen_clause_name": (C.c_char_p, [vp, C.c_uint32]),
    "hyre_encode": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint64, f32p, u64p]),
    "hyre_quant_score_words": (C.c_uint32, [u64p, u64p, C.c_uint32, C.c_uint32]),
    "hyre_normalize_query": (C.c_int, [C.c_uint32, u32p, u32p, u32p, C.c_uint32, u32p, u32p, u32p, u32p]),
    "hyre_validate_query": (C.c_int, [vp, C.POINTER(hyre_query)]),
    "hyre_index_create": (C.c_int, [vp, C.POINTER(hyre_index_options), C.POINTER(vp)]),
    "hyre_index_destroy": (None, [vp]),
    "hyre_index_set_row_weights": (C.c_int, [vp, f32p, C.c_uint64]),
    "hyre_sharded_index_set_row_weights": (C.c_int, [vp, f32p, C.c_uint64]),
    "hyre_index_stats_get": (C.c_int, [vp, C.POINTER(hyre_index_stats)]),
    "hyre_executor_create": (C.c_int, [vp, C.c_uint32, C.POINTER(vp)]),
    "hyre_executor_destroy": (None, [vp]),
    "hyre_executor_stream": (vp, [vp]),
    "hyre_execute": (C.c_int, [vp, C.POINTER(hyre_query), C.POINTER(hyre_hit), u32p, C.POINTER(hyre_timings)]),
    "hyre_execute_batch": (C.c_int, [vp, C.POINTER(hyre_query), C.c_uint32, C.POINTER(hyre_hit), u64p, u32p,
                                     i32p, C.POINTER(hyre_timings)]),
    "hyre_executor_slot_error": (C.c_char_p, [vp, C.c_uint32]),
    "hyre_batch_prepare": (C.c_int, [vp, C.POINTER(hyre_query), C.c_uint32]),
    "hyre_batch_run": (C.c_int, [vp]),
    "hyre_batch_fetch": (C.c_int, [vp, C.POINTER(hyre_hit), u64p, u32p, i32p, C.POINTER(hyre_timings)]),
    "hyre_batch_kernel_count": (C.c_uint32, [vp]),
    "hyre_batch_path": (C.c_uint32, [vp]),
    "hyre_batch_cnf_group": (C.c_uint32, [vp]),
    "hyre_batch_tc_variant": (None, [vp, u32p]),
    "hyre_batch_recovery": (C.c_int, [vp, u32p]),
    "hyre_sharded_index_create": (C.c_int, [vp, C.POINTER(hyre_sharded_index_options), C.POINTER(vp)]),
    "hyre_sharded_index_destroy": (None, [vp]),
    "hyre_sharded_index_info": (C.c_int, [vp, u32p, i32p]),
    "hyre_sharded_create": (C.c_int, [vp, C.c_uint32, C.POINTER(vp)]),
    "hyre_sharded_destroy": (None, [vp]),
    "hyre_sharded_execute_batch": (C.c_int, [vp, C.POINTER(hyre_query), C.c_uint32, C.POINTER(hyre_hit), u64p, u32p,
                                             i32p, C.POINTER(hyre_timings)]),
    "hyre_sharded_slot_error": (C.c_char_p, [vp, C.c_uint32]),
    "hyre_sharded_prepare": (C.c_int, [vp, C.POINTER(hyre_query), C.c_uint32]),
    "hyre_sharded_run": (C.c_int, [vp]),
    "hyre_sharded_settle": (C.c_int, [vp]),
    "hyre_sharded_fetch": (C.c_int, [vp, C.POINTER(hyre_hit), u64p, u32p, i32p, C.POINTER(hyre_timings)]),
    "hyre_sharded_stream": (vp, [vp]),
    "hyre_sharded_kernel_count": (C.c_uint32, [vp]),
    "hyre_sharded_recovery": (C.c_int, [vp, u32p]),
    "hyre_batch_eligible": (C.c_int, [vp, u32p]),
    "hyre_batch_term_bytes": (C.c_uint64, [vp]),
    "hyre_batch_scan_bytes": (C.c_uint64, [vp]),
    "hyre_batch_settle": (C.c_int32, [vp]),
    "hyre_pool_create": (C.c_int, [vp, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(vp)]),
    "hyre_pool_destroy": (None, [vp]),
    "hyre_pool_search": (C.c_int, [vp, vp, vp, u32p]),
    "hyre_pool_stats": (C.c_int, [vp, u64p, u64p]),
    "hyre_batch_stage_ms": (C.c_int, [vp, f32p]),
    "hyre_batch_stage_ms_hist": (C.c_int, [vp, C.c_uint32, f32p]),
    "hyre_batch_set_stage_events": (C.c_int, [vp, C.c_int]),
    "hyre_batch_io_bytes": (C.c_int, [vp, u64p, u64p]),
    "hyre_batch_merge_packed": (C.c_int, [vp, vp, C.c_uint32, C.c_uint64, C.c_uint64]),
    "hyre_batch_merge_gathered": (C.c_int, [vp, vp, vp, vp, C.c_uint32, C.c_uint64]),
    "hyre_batch_device_results": (C.c_int, [vp, C.POINTER(vp), u64p, C.POINTER(vp), C.POINTER(vp)]),
    "hyre_full_scan_tbr": (C.c_int, [vp, C.POINTER(hyre_query), u32p, C.c_uint64, u64p]),
    "hyre_batch_scan_tbr": (C.c_int, [vp, C.POINTER(hyre_query), C.c_uint32, u32p, C.POINTER(hyre_messenger),
                                      C.c_uint64, u64p]),
    "hyre_exact_scores": (C.c_int, [vp, f32p, C.c_uint32, u32p, C.c_uint64, f32p, i32p]),
    "hyre_bucket_top_k": (C.c_int, [vp, u32p, f32p, C.c_uint64, C.c_uint32, C.c_uint32, C.POINTER(hyre_hit),
                                    u32p]),
    "hyre_preselect": (C.c_int, [vp, u64p, u32p, C.c_uint64, C.c_uint32, u32p, u64p]),
    "hyre_merge_topk": (C.c_int, [C.POINTER(C.POINTER(hyre_hit)), u32p, C.c_uint32, C.c_uint32,
                                  C.POINTER(hyre_hit), u32p]),
}

_lib = None


def lib():
    """Loads libhyre_b200.so; raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "or `make -C paper_2402_13435_b200/csrc` (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib
