"""ctypes binding of the C ABI in ``include/pat.h`` (libpatb200.so, built in-tree).

There is no fallback: if the shared library is missing or fails to load, every
entry point raises.  PyTorch only provides device memory and streams."""

from __future__ import annotations

import ctypes as C
import os

from . import errors

LIB_PATH = os.environ.get("PAT_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpatb200.so")

PAT_DTYPE_F16 = 0
PAT_DTYPE_BF16 = 1
SPLIT_MODES = {"none": 0, "reference": 1, "native": 2}
PAT_PLAN_HOST_ONLY = 1
PAT_PLAN_FORWARD_ONLY = 2
PAT_PLAN_PAIR_ITEMS = 4
PAT_PLAN_ALL_PARTIALS = 8
PAT_DECODE_SAME_TABLE = 1

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
u8p = C.POINTER(C.c_uint8)


class PlanOptions(C.Structure):
    _fields_ = [("num_heads", C.c_int32), ("num_kv_heads", C.c_int32), ("head_dim", C.c_int32),
                ("split_mode", C.c_int32), ("num_sms", C.c_int32), ("flags", C.c_int32),
                ("tc_min_rows", C.c_int32)]


class PlanInfo(C.Structure):
    _fields_ = [("num_queries", C.c_int32), ("block_size", C.c_int32), ("n_packs", C.c_int32),
                ("n_pack_q", C.c_int32), ("n_pack_blk", C.c_int32), ("n_units", C.c_int32),
                ("n_items", C.c_int32), ("n_slots", C.c_int32), ("n_merge_q", C.c_int32),
                ("on_device", C.c_int32), ("unique_tokens", C.c_int64),
                ("n_fwd_kernels", C.c_int32), ("n_launches", C.c_int32)]


class CostModel(C.Structure):
    _fields_ = [("tc_item_ns", C.c_double), ("tc_item_row_ns", C.c_double), ("tc_step_ns", C.c_double),
                ("stream_item_ns", C.c_double), ("hbm_bytes_per_ns", C.c_double)]


# (name, restype, argtypes) -- the complete exported surface of include/pat.h
SIGNATURES = [
    ("pat_set_cost_model", C.c_int, [C.POINTER(CostModel)]),
    ("pat_get_cost_model", C.c_int, [C.POINTER(CostModel)]),
    ("pat_plan_create_host", C.c_int, [C.c_int32, i64p, i32p, i32p, C.c_int32, C.POINTER(PlanOptions),
                                       C.POINTER(C.c_void_p)]),
    ("pat_table_hash_device", C.c_int, [C.c_int32, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_void_p,
                                        C.c_void_p]),
    ("pat_plan_create_device", C.c_int, [C.c_int32, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_int32,
                                         C.POINTER(PlanOptions), C.c_void_p, C.POINTER(C.c_void_p)]),
    ("pat_plan_create_units", C.c_int, [C.c_int32, i64p, i32p, i32p, C.c_int32, C.c_int32, i64p, i32p, i64p,
                                        i32p, i32p, C.POINTER(PlanOptions), C.POINTER(C.c_void_p)]),
    ("pat_plan_info_get", C.c_int, [C.c_void_p, C.POINTER(PlanInfo)]),
    ("pat_plan_export_packs", C.c_int, [C.c_void_p, i32p, i32p, i32p, i32p, i32p, u8p]),
    ("pat_plan_export_units", C.c_int, [C.c_void_p, i32p, i32p, i32p, i32p, i32p, i32p]),
    ("pat_workspace_bytes", C.c_size_t, [C.c_void_p]),
    ("pat_forward", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                              C.c_size_t, C.c_int32, C.c_float, C.c_void_p]),
    ("pat_plan_destroy", None, [C.c_void_p]),
    ("pat_decoder_create", C.c_int, [C.POINTER(PlanOptions), C.c_int32, C.c_int32, C.c_int32,
                                     C.POINTER(C.c_void_p)]),
    ("pat_decoder_workspace_bytes", C.c_size_t, [C.c_void_p]),
    ("pat_decoder_forward", C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_int32,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                      C.c_size_t, C.c_int32, C.c_float, C.c_int32, C.c_void_p]),
    ("pat_decoder_status", C.c_int, [C.c_void_p, C.c_void_p, i32p]),
    ("pat_decoder_destroy", None, [C.c_void_p]),
    ("pat_last_error", C.c_char_p, []),
    ("pat_version", C.c_char_p, []),
]

_lib = None


def lib():
    """Load libpatb200.so (once).  Raises if it is missing: there is no CPU path."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise errors.NativeError(
                f"{LIB_PATH} is missing -- build it with `python -m paper_2511_22333_b200.build` "
                "(or __graft_entry__.build())")
        h = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def check(status: int, what: str = "") -> None:
    if status != 0:
        msg = lib().pat_last_error().decode(errors="replace")
        cls = errors.STATUS.get(status, errors.NativeError)
        raise cls(f"{what}: {msg}" if what else msg)


def ptr(arr, ctype):
    """Pointer to a contiguous numpy array's data."""
    return arr.ctypes.data_as(C.POINTER(ctype))
