"""ctypes mirror of include/gdlog_b200.h (the C-ABI of libgdlog_b200.so).

Struct layouts here must match the header byte for byte; tests/test_abi.py
checks the sizes against the C compiler's view.  Loading the library is
explicit and loud: there is no CPU fallback for the product path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

GD_MAX_ARITY = 8
GD_MAX_FILTERS = 8
GD_MAX_STEPS = 6
GD_MAX_VARIANTS = 8

GD_OK = 0
GD_ERR_LOGIC = 1
GD_ERR_CONFIG = 2
GD_ERR_USAGE = 3
GD_ERR_LOAD = 4
GD_ERR_PLAN = 5
GD_ERR_BUDGET = 6
GD_ERR_CUDA = 7
GD_ERR_UNSUPPORTED = 8
GD_ERR_INVALID_ARG = 9
GD_ERR_NCCL = 10

GD_OUTER_COL = 0
GD_INNER_COL = 1
GD_CONSTANT = 2
GD_FULL = 0
GD_DELTA = 1

PHASES = ("index", "join", "dedup", "difference", "merge", "other")  # stats.hpp:15-16
KCLASSES = ("sort_pass", "sort_hist", "diff_merge", "join_probe", "join_materialize", "index_build",
            "select", "other", "difference", "join_insert", "loop_ctl")  # gdlog_b200.h GD_KCLASS_COUNT

u32 = C.c_uint32
u64 = C.c_uint64


GD_LOOP_GRAPH = 0
GD_EXCHANGE_PEER, GD_EXCHANGE_NCCL = 0, 1
GD_LOOP_EAGER = 1
GD_LOOP_BATCH = 2


class gd_device_config(C.Structure):
    """gd_device_config (gdlog_b200.h): device-only knobs of a context."""
    _fields_ = [
        ("size", u32),
        ("resident_loop", C.c_int32),
        ("loop_mode", C.c_int32),
        ("loop_batch", u32),
        ("min_capacities", C.c_int32),
        ("split_insert", C.c_int32),
        ("dense_inner", C.c_int32),
        ("index_growth", u32),
        ("insert_waves", u32),
        ("rehash_cas_only", C.c_int32),
        ("zone_slots", u32),
        ("partition_loop", C.c_int32),
        ("hash_dedup", C.c_int32),
        ("hash_dedup_min_rows", u64),
        ("dedup_part_slots", u64),
        ("dedup_split", C.c_int32),
        ("host_unpack", C.c_int32),
        ("download_direct_frac", C.c_double),
        ("download_chunk_rows", u64),
        ("sort_items", u32),
        ("trace", u32),
        ("warp_expand", C.c_int32),
        ("sort_digit_bits", u32),
        ("heavy_rows", u64),
        ("sort_pipeline", C.c_int32),
        ("partition_exchange", u32),
        ("sort_pipeline_min_keys", u64),
        ("temp_limit_rows", u64),
        ("peer_timeout_ms", u32),
        ("insert_slots", u32),
        ("insert_pipeline", u32),
        ("insert_per_thread", u32),
        ("sort_ballot", u32),
        ("l2_fetch_bytes", u32),
        ("sort_min_ctas", u32),
        ("expand_keys_per_lane", u32),
        ("warp_append", u32),
        ("precount", u32),
        ("count_ctas_per_sm", u32),
        ("download_delta", u32),
        ("index_load_pct", u32),
        ("download_pipeline", u32),
        ("download_pipeline_min_rows", u64),
        ("gate_in_insert", u32),
        ("pdl", u32),
        ("count_ahead", u32),
        ("chain_chunk_rows", u64),
        ("log_growth", u32),
        ("download_overlap_pack", u32),
    ]


class gd_operand(C.Structure):
    _fields_ = [("kind", u32), ("column", u32), ("value", u64)]


class gd_filter(C.Structure):
    _fields_ = [("lhs", gd_operand), ("rhs", gd_operand), ("require_equal", u32), ("reserved", u32)]


class gd_join_step(C.Structure):
    _fields_ = [
        ("inner_rel", u32),
        ("join_column_count", u32),
        ("inner_perm", u32 * GD_MAX_ARITY),
        ("proj_arity", u32),
        ("nfilters", u32),
        ("proj", gd_operand * GD_MAX_ARITY),
        ("filters", gd_filter * GD_MAX_FILTERS),
    ]


class gd_variant(C.Structure):
    _fields_ = [
        ("src_rel", u32),
        ("src_version", u32),
        ("src_perm", u32 * GD_MAX_ARITY),
        ("nsteps", u32),
        ("sel_arity", u32),
        ("nsel_filters", u32),
        ("reserved", u32),
        ("steps", gd_join_step * GD_MAX_STEPS),
        ("sel_proj", gd_operand * GD_MAX_ARITY),
        ("sel_filters", gd_filter * GD_MAX_FILTERS),
    ]


class gd_rule_plan(C.Structure):
    _fields_ = [
        ("rule_index", u32),
        ("head_rel", u32),
        ("head_arity", u32),
        ("recursive", u32),
        ("nvariants", u32),
        ("reserved", u32),
        ("variants", gd_variant * GD_MAX_VARIANTS),
    ]


class gd_container_view(C.Structure):
    _fields_ = [
        ("rows", C.c_void_p),
        ("n", u64),
        ("arity", u32),
        ("canonical", u32),
        ("index_prefix_len", u32),
        ("reserved", u32),
        ("load_factor", C.c_double),
    ]


class gd_join_spec(C.Structure):
    _fields_ = [
        ("join_column_count", u32),
        ("proj_arity", u32),
        ("nfilters", u32),
        ("reserved", u32),
        ("proj", gd_operand * GD_MAX_ARITY),
        ("filters", gd_filter * GD_MAX_FILTERS),
    ]


class gd_engine_config(C.Structure):
    _fields_ = [
        ("memory_budget_bytes", u64),
        ("ebm_enabled", u32),
        ("alpha", u32),
        ("load_factor", C.c_double),
        ("workers", u32),
        ("reserved", u32),
        ("stride_rows", u64),
    ]


class gd_run_stats(C.Structure):
    _fields_ = [
        ("phase_seconds", C.c_double * 6),
        ("total_seconds", C.c_double),
        ("iterations", u64),
        ("buffer_allocations", u64),
        ("charge_events", u64),
        ("peak_tracked_bytes", u64),
        ("peak_temp_bytes", u64),
        ("join_tuples", u64),
        ("device_bytes_peak", u64),
        ("kernel_seconds", C.c_double * 6),
        ("algo_bytes", u64 * 6),
    ]


class gd_iter_record(C.Structure):
    _fields_ = [
        ("delta_in", u64),
        ("join", u64),
        ("new_unique", u64),
        ("delta_out", u64),
        ("full_after", u64),
    ]


P = C.c_void_p
PU64 = C.POINTER(u64)
PU32 = C.POINTER(u32)

# name -> (restype, argtypes); the full exported surface of gdlog_b200.h.
SIGNATURES = {
    "gd_abi_version": (C.c_int, []),
    "gd_ctx_create": (C.c_int, [C.c_int, P, C.POINTER(P)]),
    "gd_ctx_destroy": (C.c_int, [P]),
    "gd_last_error": (C.c_char_p, [P]),
    "gd_last_error_phase": (C.c_char_p, [P]),
    "gd_ctx_kernel_launches": (u64, [P]),
    "gd_ctx_synchronize": (C.c_int, [P]),
    "gd_ctx_trim": (C.c_int, [P]),
    "gd_ctx_set_profiling": (C.c_int, [P, C.c_int]),
    "gd_ctx_profile_read": (C.c_int, [P, P, P, P]),
    "gd_ctx_profile_reset": (C.c_int, [P]),
    "gd_ctx_host_counters": (C.c_int, [P, P, P, P, P]),
    "gd_ctx_transfer_bytes": (C.c_int, [P, P, P]),
    "gd_device_config_default": (None, [C.POINTER(gd_device_config)]),
    "gd_ctx_set_device_config": (C.c_int, [P, C.POINTER(gd_device_config)]),
    "gd_ctx_get_device_config": (C.c_int, [P, C.POINTER(gd_device_config)]),
    "gd_prefix_hash": (C.c_int, [P, P, u64, u32, u32, P]),
    "gd_canonicalize": (C.c_int, [P, P, u64, u32, P, PU64]),
    "gd_sort_keys_device": (C.c_int, [P, P, P, u64, u32, C.POINTER(C.c_int)]),
    "gd_permute_columns": (C.c_int, [P, P, u64, u32, C.c_int, P, u32, P, PU64]),
    "gd_group_starts": (C.c_int, [P, P, u64, u32, C.c_int, u32, P, PU64]),
    "gd_index_lookup": (C.c_int, [P, P, u64, u32, C.c_int, u32, C.c_double, P, u64, u32, P, P, PU64, PU64]),
    "gd_join_count": (C.c_int, [P, C.POINTER(gd_container_view), C.POINTER(gd_container_view),
                                C.POINTER(gd_join_spec), PU64]),
    "gd_join_materialize": (C.c_int, [P, C.POINTER(gd_container_view), C.POINTER(gd_container_view),
                                      C.POINTER(gd_join_spec), P, u64]),
    "gd_select_project": (C.c_int, [P, P, u64, u32, C.POINTER(gd_operand), u32, C.POINTER(gd_filter), u32,
                                    P, PU64]),
    "gd_merge_sorted": (C.c_int, [P, P, u64, C.c_int, P, u64, C.c_int, u32, u64, P]),
    "gd_difference": (C.c_int, [P, P, u64, C.c_int, P, u64, C.c_int, u32, P, PU64]),
    "gd_engine_create": (C.c_int, [P, C.POINTER(gd_engine_config), u32, PU32, PU32, C.POINTER(C.c_char_p),
                                   C.POINTER(P)]),
    "gd_engine_destroy": (C.c_int, [P]),
    "gd_engine_set_plans": (C.c_int, [P, C.POINTER(gd_rule_plan), u32]),
    "gd_engine_load_edb": (C.c_int, [P, u32, P, u64, C.c_int]),
    "gd_engine_load_edb_tsv": (C.c_int, [P, u32, C.c_char_p, P, u64]),
    "gd_engine_relation_tsv": (C.c_int, [P, u32, P, u64, P]),
    "gd_parse_facts": (C.c_int, [P, C.c_char_p, P, u64, u32, P, u64, P]),
    "gd_facts_all_integers": (C.c_int, [P, P, u64, P]),
    "gd_rows_to_tsv": (C.c_int, [P, P, u64, u32, P, u64, P]),
    "gd_engine_load_edb_device": (C.c_int, [P, u32, P, u64, C.c_int]),
    "gd_engine_seed": (C.c_int, [P]),
    "gd_engine_iterate": (C.c_int, [P]),
    "gd_engine_run": (C.c_int, [P]),
    "gd_engine_relation_count": (C.c_int, [P, u32, PU64]),
    "gd_engine_relation_download": (C.c_int, [P, u32, P, u64]),
    "gd_engine_relation_download_device": (C.c_int, [P, u32, P, u64]),
    "gd_engine_relation_digest": (C.c_int, [P, u32, PU64]),
    "gd_engine_stats": (C.c_int, [P, C.POINTER(gd_run_stats)]),
    "gd_engine_accountant": (C.c_int, [P, P, PU64, PU64, PU64, PU64]),
    "gd_engine_delta_history": (C.c_int, [P, u32, P, u64, PU64]),
    "gd_engine_iter_log": (C.c_int, [P, u32, C.POINTER(gd_iter_record), u64, PU64]),
    "gd_engine_encoding": (C.c_int, [P, PU32, PU32, PU32]),
    "gd_engine_set_partition": (C.c_int, [P, u32, u32]),
    "gd_engine_exchange_words": (C.c_int, [P, PU32]),
    "gd_engine_partition_begin": (C.c_int, [P, P, C.POINTER(P)]),
    "gd_engine_partition_end": (C.c_int, [P, P, u64, PU64]),
    "gd_engine_partition_finish": (C.c_int, [P]),
    "gd_nccl_unique_id": (C.c_int, [P]),
    "gd_nccl_comm_create": (C.c_int, [P, P, u32, u32, C.POINTER(P)]),
    "gd_nccl_comm_destroy": (C.c_int, [P]),
    "gd_engine_run_partitioned": (C.c_int, [P, P, u64, PU64]),
    "gd_loopback_hub_create": (C.c_int, [u32, C.POINTER(P)]),
    "gd_loopback_hub_destroy": (C.c_int, [P]),
    "gd_loopback_comm_create": (C.c_int, [P, u32, C.POINTER(P)]),
}

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("GDLOG_B200_LIB", PKG_DIR / "lib" / "libgdlog_b200.so"))

_lib = None


def load_library(path: Path | str | None = None) -> C.CDLL:
    """Loads libgdlog_b200.so (built in-tree by __graft_entry__.build()).

    Raises RuntimeError when the library is missing: the product path has
    no CPU fallback.
    """
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise RuntimeError(
            f"libgdlog_b200.so not found at {p}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    lib = C.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib
