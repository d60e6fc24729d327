"""ctypes binding of libhopgnn.so (include/hopgnn.h).

The product path has no fallback: if the shared library is missing or does
not load, every entry point raises ``RuntimeError`` (the CUDA extension is
the only implementation).
"""
from __future__ import annotations

import ctypes as C
import os

from .errors import ConfigError, InvariantViolation

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhopgnn.so")
MAX_LAYERS = 6
MAX_GROUP = 16  # HG_MAX_GROUP

_lib = None


class MgLayout(C.Structure):
    _fields_ = [("n_layers", C.c_int32),
                ("fanout", C.c_int32 * MAX_LAYERS),
                ("cap_lay", C.c_int32 * (MAX_LAYERS + 1)),
                ("cap_need", C.c_int32 * (MAX_LAYERS + 1)),
                ("cand_cap", C.c_int32),
                ("sort_cap", C.c_int32),
                ("smem_bytes", C.c_int32),
                ("ws_root_ints", C.c_int32)]


_P7 = C.c_void_p * (MAX_LAYERS + 1)


class MgBatch(C.Structure):
    _fields_ = [("need_ids", _P7), ("need_off", _P7), ("in_layer", _P7), ("self_pos", _P7),
                ("nbr_off", _P7), ("nbr_idx", _P7), ("pair_off", _P7), ("totals", C.c_void_p),
                ("nbr_vid1", C.c_void_p), ("self_vid1", C.c_void_p)]


MAX_SHARDS = 16  # HG_MAX_SHARDS


class CsrShards(C.Structure):
    """hg_csr_shards (include/hopgnn.h section 4)."""

    _fields_ = [("n_shards", C.c_int32), ("offsets", C.c_void_p * MAX_SHARDS),
                ("targets", C.c_void_p * MAX_SHARDS), ("vstart", C.c_int64 * (MAX_SHARDS + 1)),
                ("home_of", C.c_void_p), ("row_of", C.c_void_p)]


class GraphTables(C.Structure):
    _fields_ = [("n", C.c_int64), ("n_blocks", C.c_int32), ("n_levels", C.c_int32),
                ("key", C.c_uint64), ("deg_key", C.c_uint64), ("thr_in", C.c_uint32), ("in_always", C.c_int32),
                ("block_start", C.c_int64 * 65), ("a", C.c_uint64 * 64),
                ("c", C.c_uint64 * 64), ("a_inv", C.c_uint64 * 64), ("cum", C.c_uint64 * 64),
                ("lvl_size", C.c_int64 * 64), ("deg_lo", C.c_int64 * 64),
                ("deg_span", C.c_int64 * 64)]


_P7V = C.c_void_p * 7


class StepDesc(C.Structure):
    """hg_step_desc (include/hopgnn.h section 5)."""

    _fields_ = [("n_layers", C.c_int32), ("arch", C.c_int32), ("act_dtype", C.c_int32),
                ("feat_dim", C.c_int32), ("feat_ld", C.c_int32), ("hidden", C.c_int32),
                ("n_classes", C.c_int32), ("max_roots", C.c_int32),
                ("max_rows", C.c_int32 * 7), ("in_dim", C.c_int32 * 7),
                ("split_k", C.c_int32), ("use_tc", C.c_int32),
                ("features", C.c_void_p), ("feat_row", C.c_void_p), ("roots", C.c_void_p),
                ("label_state", C.c_uint64), ("mg", MgBatch),
                ("W", _P7V), ("b", _P7V), ("Wc", C.c_void_p), ("Wlp", _P7V), ("Wclp", C.c_void_p),
                ("gW", _P7V), ("gb", _P7V), ("gWc", C.c_void_p),
                ("agg", _P7V), ("h", _P7V), ("dh", _P7V), ("dagg", C.c_void_p),
                ("logits", C.c_void_p), ("loss", C.c_void_p), ("lowp_scratch", C.c_void_p),
                ("Wb", _P7V), ("feat_peers", C.c_void_p), ("feat_home", C.c_void_p),
                ("stage_base", C.c_void_p), ("stage_row", C.c_void_p), ("rank", C.c_int32),
                ("agg1_ready", C.c_int32), ("WcT", C.c_void_p), ("Wcp", C.c_void_p),
                ("dl_lowp", C.c_void_p), ("root_rows", C.c_int32 * 7),
                ("lowp_fresh", C.c_int32), ("max_deg", C.c_int32 * 7),
                ("lowp_layered", C.c_int32), ("row_handle", C.c_void_p),
                ("labels", C.c_void_p)]


V, I32, I64, U64, SZ = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_size_t
PSZ = C.POINTER(C.c_size_t)
PI64 = C.POINTER(C.c_int64)

# name -> argtypes (every function returns int status)
SIGNATURES = {
    "hg_version": [],
    "hg_device_sync": [V],
    "hg_launch_count": [C.POINTER(C.c_longlong), C.c_int],
    "hg_prof_enable": [C.c_int],
    "hg_prof_read": [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int)],
    "hg_stamp": [C.c_void_p, C.c_void_p],
    "hg_sample_frontier": [V, V, I64, V, I64, I32, U64, V, V, I64, PI64, V],
    "hg_feature_rows": [V, I64, I32, U64, V, V],
    "hg_feature_table": [V, I64, I64, I32, I32, U64, I32, V, V],
    "hg_epoch_permutation": [I64, U64, V, V, PSZ, V],
    "hg_glorot": [I32, I32, U64, I32, V, V],
    "hg_iter_stage": [V, V, I64, V, I32, I32, I32, V, V, V],
    "hg_iter_stage_group": [V, V, I64, V, I32, I32, I32, I32, V, V, V],
    "hg_bench_mix64": [I32, I64, V, V],
    "hg_iter_stage_ranged": [V, V, V, I64, V, I32, I32, I32, V, V, V, V],
    "hg_graph_raw_degrees": [C.POINTER(GraphTables), V, V],
    "hg_graph_fill": [C.POINTER(GraphTables), I64, I64, V, V, V],
    "hg_graph_canonicalize": [I64, I64, V, V, V, V, PSZ, V],
    "hg_graph_compact": [I64, I64, V, V, V, V, V],
    "hg_exclusive_scan_i64": [V, V, I64, V, PSZ, V],
    "hg_pick_k_smallest": [V, I64, I64, U64, V, V],
    "hg_sbm_edges": [V, I64, I32, U64, I32, U64, U64, V, V, I64, PI64, V],
    "hg_partition_greedy": [V, V, I64, I32, I64, V, V, V, V],
    "hg_partition_leftovers": [V, I64, I32, V, V],
    "hg_mg_plan_layout": [I32, C.POINTER(I32), C.POINTER(MgLayout)],
    "hg_mg_build": [V, V, I64, V, I32, V, I32, C.POINTER(MgLayout), V, C.POINTER(MgBatch),
                    V, V],
    "hg_mg_build_n": [V, V, I64, V, I32, V, V, I32, C.POINTER(MgLayout), V, C.POINTER(MgBatch),
                      V, V],
    "hg_mg_build_mode": [I32],
    "hg_mg_build_group": [V, V, I64, V, I32, I32, V, V, I32, C.POINTER(MgLayout), V,
                          C.POINTER(MgBatch), V, I32, V],
    "hg_mg_build_group_sharded": [C.POINTER(CsrShards), I64, V, I32, I32, V, V, I32,
                                  C.POINTER(MgLayout), V, C.POINTER(MgBatch), V, I32, V],
    "hg_set_fused_head": [I32],
    "hg_set_side_budget": [I32, I32],
    "hg_set_fused_top": [I32],
    "hg_top_trace": [C.c_void_p],
    "hg_train_step": [C.POINTER(StepDesc), I32, V],
    "hg_train_step_sgd": [C.POINTER(StepDesc), I32, V, V, I64, C.c_float, C.c_float, I32, V],
    "hg_set_persist": [I32, I32, I32],
    "hg_persist_trace": [C.c_void_p],
    "hg_forward": [C.POINTER(StepDesc), I32, V],
    "hg_sgd_update": [V, V, V, I64, C.c_float, C.c_float, V],
    "hg_sgd_refresh": [C.POINTER(StepDesc), V, V, I64, C.c_float, C.c_float, I32, V],
    "hg_allreduce_sgd_refresh": [V, C.POINTER(StepDesc), V, V, I64, C.c_float, C.c_float, V],
    "hg_gemm_bf16": [V, I64, C.c_int, V, I64, C.c_int, V, I64, I32, I32, I32, I32, V, I32, V],
    "hg_alloc": [C.c_size_t, C.POINTER(C.c_void_p)],
    "hg_memcpy_d2d": [V, V, C.c_size_t, V],
    "hg_flag_if_differ": [V, V, I64, V, V],
    "hg_remote_account_group": [V, V, I32, V, I32, V, I64, V, V, I32, V, V],
    "hg_resolve_rows_group": [V, V, I32, V, I32, V, V, V, V],
    "hg_p2p_region_bytes": [I32, I64, PI64],
    "hg_p2p_allreduce": [V, I64, V, I32, I32, V, V, V, V],
    "hg_free": [V],
    "hg_ipc_handle": [V, V],
    "hg_ipc_open": [V, C.POINTER(C.c_void_p)],
    "hg_ipc_close": [V],
    "hg_remote_account": [V, V, I32, V, I32, V, V, V, V],
    "hg_remote_clear": [V, V, I32, V, V],
    "hg_nccl_unique_id": [V],
    "hg_nccl_init": [V, C.c_int, C.c_int, C.POINTER(C.c_void_p)],
    "hg_nccl_destroy": [V],
    "hg_allreduce_sgd": [V, V, V, I64, C.c_float, C.c_float, V],
    "hg_shift": [V, C.c_int, C.c_int, C.c_int, V, V, V, V, I64, V],
    "hg_pregather_peer": [V, V, V, I32, V, V, I32, V, V, V, V, I32, V, V, V, V, V],
    "hg_pregather_peer_at": [V, V, V, I32, V, V, I32, V, V, V, V, I32, V, V, V, I32, V, V, V],
    "hg_pregather_push": [V, V, V, I32, I32, V, V, I32, V, V, I32, V, V, I64, I64, I64, I64, I64,
                          V, V, I32, V, V, V, V],
    "hg_step_prologue": [C.POINTER(StepDesc), I32, I32, V],
    "hg_resolve_rows": [V, V, V, I32, V, V, V, V],
    "hg_pregather_push_multi": [V, V, I32, V, I32, I32, V, V, I32, V, V, I32, V, V, I64, I64,
                                I64, I64, I64, V, V, V],
    "hg_remote_account_at": [V, V, V, I32, V, V, V, I32, I32, V, V],
    "hg_step_prologue_group": [C.POINTER(C.POINTER(StepDesc)), I32, I32, V],
    "hg_debug_build_phases": [C.POINTER(C.c_longlong), C.c_int],
}


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"libhopgnn.so not built ({LIB_PATH}); run `python -m paper_2409_00657_b200.build`"
                " — there is no CPU fallback")
        h = C.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            fn = getattr(h, name)
            fn.argtypes = args
            fn.restype = C.c_int
        h.hg_last_error.argtypes = []
        h.hg_last_error.restype = C.c_char_p
        _lib = h
    return _lib


def check(status: int, what: str = "") -> None:
    """Map hg_status to the reference's exception types (errors.py:4-12)."""
    if status == 0:
        return
    msg = lib().hg_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if status == 1:
        raise ValueError(msg)
    if status == 2:
        raise ConfigError(msg)
    if status == 3:
        raise InvariantViolation(msg)
    raise RuntimeError(f"hopgnn status {status}: {msg}")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)


def flag_status(code: int, what: str) -> None:
    """Raise for a device-side error flag read back by the caller."""
    if code == 0:
        return
    if code == 1:
        raise ValueError(f"{what}: index out of range (device flag)")
    if code == 3:
        raise InvariantViolation(f"{what}: device invariant violated")
    raise RuntimeError(f"{what}: device error flag {code}")


def launch_count(reset: bool = False) -> int:
    v = C.c_longlong(0)
    call("hg_launch_count", C.byref(v), int(reset))
    return int(v.value)


def prof_enable(on: bool) -> None:
    call("hg_prof_enable", int(on))


def prof_read(site: int):
    """(total ms, launches) recorded at a profiling site since prof_enable."""
    t, n = C.c_double(0), C.c_int(0)
    call("hg_prof_read", site, C.byref(t), C.byref(n))
    return t.value, n.value


(PROF_BUILD, PROF_AGG1, PROF_GEMM1, PROF_DW1, PROF_STEP, PROF_AGG2, PROF_SGD, PROF_PG_MARK,
 PROF_PG_COPY, PROF_PG_CLEAR) = range(10)
