"""ctypes mirror of include/pqtg.h (the C-ABI boundary) and the loader of libpqtg.so.

The product path has no CPU fallback: if the CUDA library is missing, `lib()` raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "_build" / "libpqtg.so"

PQTG_OK = 0
STATUS = {
    -1: "BAD_DIM",
    -2: "CONFIG",
    -3: "FORMAT",
    -4: "UNSUPPORTED",
    -5: "OOM",
    -6: "CUDA",
    -7: "ARG",
    -8: "NCCL",
}


class PqtgConfig(C.Structure):
    """pqtg_config — field-for-field pqt::PqtConfig (include/pqt/codebook.hpp:12-36)."""

    _fields_ = [
        ("dim", C.c_uint32),
        ("p_tree", C.c_uint32),
        ("k1", C.c_uint32),
        ("k2", C.c_uint32),
        ("w", C.c_uint32),
        ("p_line", C.c_uint32),
        ("hash_size", C.c_uint64),
        ("candidate_budget", C.c_uint32),
        ("rerank_exact", C.c_uint32),
        ("resort_bins", C.c_uint32),
        ("train_iters", C.c_uint32),
        ("seed", C.c_uint64),
    ]


class PqtgIndexView(C.Structure):
    _fields_ = [
        ("config", PqtgConfig),
        ("n", C.c_uint64),
        ("level1", C.c_void_p),
        ("level2", C.c_void_p),
        ("d2", C.c_void_p),
        ("table_count", C.c_uint32),
        ("table_len", C.c_uint32),
        ("table_slopes", C.c_void_p),
        ("table_entries", C.c_void_p),
        ("offsets", C.c_void_p),
        ("ids", C.c_void_p),
        ("lambda_q", C.c_void_p),
        ("pair_id", C.c_void_p),
        ("shard_lo", C.c_uint64),
        ("shard_hi", C.c_uint64),
    ]


class PqtgQueryStats(C.Structure):
    _fields_ = [
        ("bins_visited", C.c_uint64),
        ("candidates", C.c_uint64),
        ("exact_evals", C.c_uint64),
    ]


class PqtgIndexInfo(C.Structure):
    _fields_ = [
        ("config", PqtgConfig),
        ("n", C.c_uint64),
        ("shard_lo", C.c_uint64),
        ("shard_hi", C.c_uint64),
        ("list_len", C.c_uint32),
        ("pair_count", C.c_uint32),
        ("pair_width", C.c_uint32),
        ("code_row_bytes", C.c_uint32),
        ("device_bytes", C.c_uint64),
        ("device", C.c_int),
    ]


# Every symbol include/pqtg.h declares, with its ctypes signature (restype, argtypes).
_vp = C.c_void_p
_u32 = C.c_uint32
_u64 = C.c_uint64
SIGNATURES = {
    "pqtg_abi_version": (C.c_int, []),
    "pqtg_last_error": (C.c_char_p, []),
    "pqtg_device_ok": (C.c_int, [C.c_int]),
    "pqtg_set_kernel_variant": (C.c_int, [C.c_int]),
    "pqtg_index_create": (C.c_int, [C.POINTER(PqtgIndexView), C.c_int, C.POINTER(_vp)]),
    "pqtg_index_load": (C.c_int, [C.c_char_p, C.c_int, _u64, _u64, C.POINTER(_vp)]),
    "pqtg_index_create_shard": (C.c_int, [C.POINTER(PqtgIndexView), _vp, _vp, C.c_int, C.POINTER(_vp)]),
    "pqtg_index_info_get": (C.c_int, [_vp, C.POINTER(PqtgIndexInfo)]),
    "pqtg_index_destroy": (None, [_vp]),
    "pqtg_index_attach_database": (C.c_int, [_vp, _vp, _u64, _u32]),
    "pqtg_workspace_create": (C.c_int, [_vp, _u64, C.POINTER(_vp)]),
    "pqtg_workspace_destroy": (None, [_vp]),
    "pqtg_workspace_set_chunks": (C.c_int, [_vp, _u32]),
    "pqtg_workspace_stage_ms": (C.c_int, [_vp, C.POINTER(C.c_float)]),
    "pqtg_workspace_status": (C.c_int, [_vp]),
    "pqtg_workspace_query_times": (C.c_int, [_vp, C.c_int]),
    "pqtg_debug_rerank_phases": (C.c_int, [_vp]),
    "pqtg_debug_query_clocks": (C.c_int, [_vp, C.c_uint64, _vp]),
    "pqtg_workspace_read_query_times": (C.c_int, [_vp, _u64, _vp]),
    "pqtg_workspace_read": (C.c_int, [_vp, _u64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pqtg_search": (C.c_int, [_vp, _vp, _vp, _u64, _u32, _u32, _vp, _vp, _vp, _vp]),
    "pqtg_search_device": (C.c_int, [_vp, _vp, _vp, _u64, _u32, _vp, _vp, _vp, _vp, _vp]),
    "pqtg_build_codes": (C.c_int, [C.POINTER(PqtgConfig), _vp, _vp, _vp, _vp, _vp, _vp, _u64, _vp, _vp, _vp, _vp, _vp]),
    "pqtg_bin_stream_host": (C.c_int64, [C.POINTER(PqtgIndexView), _vp, _u64, _vp]),
    "pqtg_merge_topk_host": (C.c_int, [_u32, _u64, _u32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pqtg_merge_topk_device": (C.c_int, [_u32, _u64, _u32, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pqtg_shard_range": (C.c_int, [_u64, _u32, _u32, C.POINTER(_u64), C.POINTER(_u64)]),
    "pqtg_brute_force_knn": (C.c_int, [_vp, _u64, _u32, _vp, _u64, _u32, C.c_int, _vp, _vp, _vp, _vp]),
    "pqtg_brute_force_knn_device": (C.c_int, [_vp, _u64, _u32, _vp, _u64, _u32, _vp, _vp, _vp, _vp]),
    "pqtg_nccl_unique_id": (C.c_int, [_vp]),
    "pqtg_sharded_create_nccl": (C.c_int, [_vp, _vp, _u32, _u32, _u64, C.POINTER(_vp)]),
    "pqtg_sharded_create_local": (C.c_int, [C.POINTER(_vp), _u32, _u64, C.POINTER(_vp)]),
    "pqtg_sharded_local_ranks": (C.c_int, [_vp]),
    "pqtg_sharded_create_sim": (C.c_int, [_vp, _u32, _u32, _u64, C.POINTER(_vp)]),
    "pqtg_sharded_workspace": (_vp, [_vp, _u32]),
    "pqtg_sharded_search_device": (C.c_int, [_vp, C.POINTER(_vp), _u64, _u32, C.c_int, C.POINTER(_vp),
                                             C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp)]),
    "pqtg_sharded_search": (C.c_int, [_vp, _vp, _u64, _u32, _u32, _vp, _vp, _vp, _vp]),
    "pqtg_sharded_stage_ms": (C.c_int, [_vp, C.POINTER(C.c_float)]),
    "pqtg_sharded_destroy": (None, [_vp]),
}

_LIB = None


class PqtgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"pqtg {STATUS.get(status, status)}: {msg}")
        self.status = status


def lib():
    """Load libpqtg.so (built in-tree by build.py). Raises if it is missing: no fallback."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the GPU query path has no CPU fallback)"
            )
        so = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(so, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = so
    return _LIB


def check(status: int) -> None:
    if status != PQTG_OK:
        msg = lib().pqtg_last_error()
        raise PqtgError(status, msg.decode() if msg else "")
