"""ctypes binding of libgsmat_b200.so (the C ABI in include/gsmat_b200.h).

There is no CPU fallback: importing the executor without the built library,
or calling it on a machine without a CUDA device, raises.
"""

from __future__ import annotations

import ctypes as C
import re
import os
import threading
from pathlib import Path

from . import errors

LIB_PATH = Path(os.environ.get("GSM_LIB") or Path(__file__).resolve().parent / "_lib" / "libgsmat_b200.so")

GSM_OK = 0
GSM_ERR_VALUE = 1
GSM_ERR_STORE_FORMAT = 2
GSM_ERR_UNKNOWN_PREDICATE = 3
GSM_ERR_RESOURCE = 4
GSM_ERR_CUDA = 5
GSM_ERR_UNSORTED = 6
GSM_ERR_UNKNOWN_ID = 7
GSM_ERR_PARSE = 8
GSM_ERR_DEVICE_MEMORY = 9

GSM_BUDGET_SEQUENTIAL = 0
GSM_BUDGET_PARALLEL = 1

STEP_KINDS = ("scan", "empty", "expand", "filter", "cross", "gate")  # GSM_STEP_*

#: Every symbol include/gsmat_b200.h declares (checked by tests/test_capi.py).
EXPORTS = (
    "gsm_device_count",
    "gsm_store_create",
    "gsm_store_put_predicate",
    "gsm_store_put_predicate_shard",
    "gsm_store_load_files",
    "gsm_store_finalize",
    "gsm_store_device_bytes",
    "gsm_store_free",
    "gsm_context_create",
    "gsm_context_free",
    "gsm_context_stream",
    "gsm_execute",
    "gsm_execute_batch",
    "gsm_execute_seeded",
    "gsm_partition_rows",
    "gsm_cross_rows",
    "gsm_table_join",
    "gsm_result_shape",
    "gsm_result_copy",
    "gsm_result_device_ptr",
    "gsm_result_free",
    "gsm_results_shape",
    "gsm_results_copy",
    "gsm_last_error",
    "gsm_kernel_launches",
    "gsm_store_put_dictionary",
    "gsm_decode_rows",
    "gsm_text_data",
    "gsm_text_free",
    "gsm_ntriples_parse",
    "gsm_build_store",
    "gsm_sort_triples",
    "gsm_context_capacity",
    "gsm_execute_batch_into",
    "gsm_execute_into",
    "gsm_result_fingerprint",
)


class Pattern(C.Structure):
    """gsm_pattern"""

    _fields_ = [
        ("s_var", C.c_int32),
        ("o_var", C.c_int32),
        ("s_const", C.c_uint32),
        ("o_const", C.c_uint32),
        ("pid", C.c_int32),
        ("empty", C.c_int32),
    ]


class Report(C.Structure):
    """gsm_report"""

    _fields_ = [
        ("rows", C.POINTER(C.c_int64)),
        ("prealloc_total", C.POINTER(C.c_int64)),
        ("device_ms", C.POINTER(C.c_float)),
        ("kind", C.POINTER(C.c_int32)),
        ("arity", C.POINTER(C.c_int32)),
        ("total_device_ms", C.c_float),
        ("h2d_bytes", C.c_int64),
        ("d2h_bytes", C.c_int64),
        ("kernels", C.c_int64),
        ("fused", C.POINTER(C.c_int32)),
    ]


class Query(C.Structure):
    """gsm_query"""

    _fields_ = [
        ("steps", C.POINTER(Pattern)),
        ("n_steps", C.c_int32),
        ("proj", C.POINTER(C.c_int32)),
        ("n_proj", C.c_int32),
        ("distinct", C.c_int32),
        ("row_budget", C.c_int64),
        ("budget_mode", C.c_int32),
        ("part_index", C.c_int64),
        ("part_count", C.c_int64),
        ("report", C.POINTER(Report)),
    ]


_lock = threading.Lock()
_lib: C.CDLL | None = None


def lib() -> C.CDLL:
    """Load the CUDA library (once).  Raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()' or "
                "make -C paper_1807_07691_b200/csrc)"
            )
        L = C.CDLL(os.fspath(LIB_PATH))
        vp = C.c_void_p
        i32, i64 = C.c_int32, C.c_int64
        P = C.POINTER
        sig = {
            "gsm_device_count": (i32, [P(i32)]),
            "gsm_store_create": (i32, [i32, i64, i32, P(vp)]),
            "gsm_store_put_predicate": (i32, [vp, i32, vp, vp, i64]),
            "gsm_store_put_predicate_shard": (i32, [vp, i32, vp, i64, vp, i64]),
            "gsm_store_load_files": (i32, [vp, i32, P(i32), P(C.c_char_p), P(C.c_char_p), P(i64)]),
            "gsm_store_finalize": (i32, [vp]),
            "gsm_store_put_dictionary": (i32, [vp, C.c_char_p, i64, vp, vp, i64]),
            "gsm_decode_rows": (i32, [vp, vp, i64, i32, P(vp)]),
            "gsm_text_data": (i32, [vp, P(C.c_void_p), P(i64)]),
            "gsm_text_free": (i32, [vp]),
            "gsm_ntriples_parse": (i32, [C.c_char_p, i64, i32, P(vp)]),
            "gsm_build_store": (i32, [C.c_char_p, C.c_char_p, i32, i32, P(i64)]),
            "gsm_sort_triples": (i32, [i32, vp, vp, vp, i64, i32, P(vp), P(vp), P(i64)]),
            "gsm_store_device_bytes": (i32, [vp, P(i64)]),
            "gsm_store_free": (i32, [vp]),
            "gsm_context_create": (i32, [vp, i64, P(vp)]),
            "gsm_context_free": (i32, [vp]),
            "gsm_context_stream": (i32, [vp, P(C.c_uint64)]),
            "gsm_context_capacity": (i32, [vp, P(i64)]),
            "gsm_execute": (
                i32,
                [vp, P(Pattern), i32, P(i32), i32, i32, i64, i32, i64, i64, P(Report), P(vp)],
            ),
            "gsm_execute_batch": (i32, [P(vp), i32, P(Query), P(i32), P(vp), P(C.c_float)]),
            "gsm_execute_into": (
                i32,
                [vp, P(Pattern), i32, P(i32), i32, i32, i64, i32, i64, i64, P(Report), vp, i64,
                 P(i64), P(i32), P(vp)],
            ),
            "gsm_execute_batch_into": (
                i32, [P(vp), i32, P(Query), P(i32), P(vp), P(i64), P(i64), P(i32), P(vp),
                      P(C.c_float)]),
            "gsm_execute_seeded": (
                i32,
                [vp, vp, i64, P(i32), i32, P(Pattern), i32, P(i32), i32, i32, i64, i32,
                 P(Report), P(vp)],
            ),
            "gsm_partition_rows": (i32, [vp, vp, i64, i32, i32, i64, i32, vp, P(i64)]),
            "gsm_cross_rows": (i32, [vp, vp, i64, i32, vp, i64, i32, vp]),
            "gsm_table_join": (
                i32,
                [vp, vp, i64, i32, vp, i64, i32, P(i32), P(i32), i32, i64, i32, P(i64), vp, P(vp)],
            ),
            "gsm_result_shape": (i32, [vp, P(i64), P(i32)]),
            "gsm_result_copy": (i32, [vp, vp]),
            "gsm_result_device_ptr": (i32, [vp, P(C.c_uint64)]),
            "gsm_result_free": (i32, [vp]),
            "gsm_result_fingerprint": (i32, [vp, P(C.c_uint64)]),
            "gsm_results_shape": (i32, [P(vp), i32, P(i64), P(i32)]),
            "gsm_results_copy": (i32, [P(vp), i32, P(vp), i32]),
            "gsm_last_error": (C.c_char_p, []),
            "gsm_kernel_launches": (i64, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
        return L


def last_error() -> str:
    msg = lib().gsm_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(status: int) -> None:
    """Map a gsm_status to the reference's exception classes."""
    if status == GSM_OK:
        return
    raise_status(status, last_error())


def raise_status(status: int, msg: str) -> None:
    if status == GSM_ERR_DEVICE_MEMORY:
        raise errors.DeviceMemoryError(msg)
    if status == GSM_ERR_RESOURCE:
        raise errors.ResourceLimitError(msg)
    if status == GSM_ERR_STORE_FORMAT:
        raise errors.StoreFormatError(msg)
    if status == GSM_ERR_UNKNOWN_PREDICATE:
        pid = int(msg.rsplit(" ", 1)[-1]) if msg and msg.rsplit(" ", 1)[-1].isdigit() else -1
        raise errors.UnknownPredicateError(pid)
    if status in (GSM_ERR_VALUE, GSM_ERR_UNSORTED):
        raise ValueError(msg)
    if status == GSM_ERR_PARSE:
        m = re.match(r"line (\d+): (.*)$", msg, re.S)
        if m:
            raise errors.ParseError(m.group(2), int(m.group(1)))
        raise errors.ParseError(msg)
    if status == GSM_ERR_UNKNOWN_ID:
        tail = msg.rsplit(" ", 1)[-1] if msg else ""
        raise errors.UnknownIdError("node", int(tail) if tail.isdigit() else -1)
    raise errors.DeviceError(msg or f"gsm status {status}")


def device_count() -> int:
    n = C.c_int32(0)
    st = lib().gsm_device_count(C.byref(n))
    if st != GSM_OK:
        return 0
    return int(n.value)


def kernel_launches() -> int:
    return int(lib().gsm_kernel_launches())
