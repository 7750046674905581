"""TEST INFRASTRUCTURE ONLY: ctypes wrapper of oracle/gsm_oracle.c.

``run(matrices, plan_patterns, projection, distinct, budget, mode)`` evaluates
a plan exactly like the reference's ``execute`` (executor.py:296-368) and
returns the projected rows in the reference's order plus the per-step
(rows, prealloc_total) report.  Patterns are any objects with the reference's
EncodedPattern attributes (s, p, o, empty); ``matrices`` maps pid -> an object
with (n, 2) uint64 arrays ``so`` and ``os`` (or lists ``so_pairs``/``os_pairs``).
"""

from __future__ import annotations

import ctypes as C
import subprocess
import threading
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "liborc.so"
GSMGEN = HERE / "_build" / "gsmgen"

ORC_OK, ORC_ERR_VALUE, ORC_ERR_RESOURCE, ORC_ERR_NOMEM = 0, 1, 4, 6


class OrcPred(C.Structure):
    _fields_ = [("nnz", C.c_int64), ("so", C.c_void_p), ("os", C.c_void_p)]


class OrcPattern(C.Structure):
    _fields_ = [
        ("s_var", C.c_int32),
        ("o_var", C.c_int32),
        ("s_const", C.c_int64),
        ("o_const", C.c_int64),
        ("pid", C.c_int32),
        ("empty", C.c_int32),
    ]


class OracleResourceError(Exception):
    """The reference would raise ResourceLimitError with this message."""


_lock = threading.Lock()
_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not LIB.exists() or not GSMGEN.exists():
                build()
            L = C.CDLL(str(LIB))
            L.orc_execute.restype = C.c_int
            L.orc_execute.argtypes = [
                C.POINTER(OrcPred), C.c_int32, C.POINTER(OrcPattern), C.c_int32,
                C.POINTER(C.c_int32), C.c_int32, C.c_int32, C.c_int64, C.c_int32,
                C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                C.POINTER(C.POINTER(C.c_int64)), C.POINTER(C.c_int64),
            ]
            L.orc_execute_part.restype = C.c_int
            L.orc_execute_part.argtypes = [
                C.POINTER(OrcPred), C.c_int32, C.POINTER(OrcPattern), C.c_int32,
                C.POINTER(C.c_int32), C.c_int32, C.c_int32, C.c_int64, C.c_int32,
                C.c_int64, C.c_int64,
                C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                C.POINTER(C.POINTER(C.c_int64)), C.POINTER(C.c_int64),
            ]
            L.orc_last_error.restype = C.c_char_p
            L.orc_free.argtypes = [C.c_void_p]
            _lib = L
    return _lib


def _arrays(m) -> tuple[np.ndarray, np.ndarray]:
    so = getattr(m, "so", None)
    os_ = getattr(m, "os", None)
    if so is None:
        so = np.asarray(m.so_pairs, dtype=np.uint64).reshape(-1, 2)
        os_ = np.asarray(m.os_pairs, dtype=np.uint64).reshape(-1, 2)
    return np.ascontiguousarray(so, dtype=np.uint64), np.ascontiguousarray(os_, dtype=np.uint64)


class PreparedStore:
    """Pair arrays of every predicate, kept alive for repeated oracle runs."""

    def __init__(self, matrices):
        self.max_pid = max(matrices) if matrices else 0
        self.keep = []
        self.preds = (OrcPred * (self.max_pid + 1))()
        for pid, m in matrices.items():
            so, os_ = _arrays(m)
            self.keep += [so, os_]
            self.preds[pid] = OrcPred(so.shape[0], so.ctypes.data, os_.ctypes.data)


def run(store, patterns, projection, distinct=False, budget=(1 << 62), mode="sequential",
        partition=(0, 1), as_array=False):
    """Returns (rows: list[tuple], step_rows: list[int], step_prealloc: list[int]).

    ``partition=(i, k)`` keeps only the i-th of k contiguous slices of the
    first step's rows (the executor's multi-GPU row partitioning).  With
    ``as_array`` the rows come back as an (n, k) int64 array (no tuples)."""
    if not isinstance(store, PreparedStore):
        store = PreparedStore(store)
    n = len(patterns)
    var_of: dict[str, int] = {}
    arr = (OrcPattern * max(1, n))()
    for i, p in enumerate(patterns):
        r = arr[i]
        for end in ("s", "o"):
            t = getattr(p, end)
            if isinstance(t, str):
                setattr(r, end + "_var", var_of.setdefault(t, len(var_of)))
                setattr(r, end + "_const", 0)
            else:
                setattr(r, end + "_var", -1)
                setattr(r, end + "_const", int(t))
        r.pid = int(p.p)
        r.empty = 1 if getattr(p, "empty", False) else 0
    proj = [var_of[v] for v in projection]
    proj_arr = (C.c_int32 * max(1, len(proj)))(*proj)
    srows = (C.c_int64 * max(1, n))()
    spre = (C.c_int64 * max(1, n))()
    out = C.POINTER(C.c_int64)()
    nout = C.c_int64(0)
    L = lib()
    rc = L.orc_execute_part(store.preds, store.max_pid, arr, n, proj_arr, len(proj),
                            1 if distinct else 0, int(budget), 1 if mode == "parallel" else 0,
                            int(partition[0]), int(partition[1]), srows, spre, C.byref(out),
                            C.byref(nout))
    if rc == ORC_ERR_RESOURCE:
        raise OracleResourceError(L.orc_last_error().decode())
    if rc != ORC_OK:
        raise ValueError(L.orc_last_error().decode() or f"oracle error {rc}")
    try:
        k = len(proj)
        cnt = int(nout.value)
        if as_array:
            rows = (np.ctypeslib.as_array(out, shape=(cnt * k,)).reshape(cnt, k).copy()
                    if cnt and k else np.zeros((cnt, k), dtype=np.int64))
        elif cnt and k:
            flat = np.ctypeslib.as_array(out, shape=(cnt * k,)).copy()
            rows = [tuple(r) for r in flat.reshape(cnt, k).tolist()]
        else:
            rows = [()] * cnt
    finally:
        L.orc_free(out)
    return rows, list(srows[:n]), list(spre[:n])


def gsmgen(*args: str) -> None:
    """Run the synthetic store generator (datagen/gsmgen.c)."""
    if not GSMGEN.exists():
        build()
    subprocess.run([str(GSMGEN), *args], check=True, stdout=subprocess.DEVNULL)


def fingerprint(rows) -> tuple[int, int, int]:
    """Order-independent multiset fingerprint (count, sum, xor) of id tuples
    (SURVEY.md §8(c)): splitmix64 chained over the tuple's ids."""
    M = (1 << 64) - 1
    s = x = 0
    for r in rows:
        h = 0x9E3779B97F4A7C15
        for v in r:
            z = (h ^ int(v)) & M
            z = (z + 0x9E3779B97F4A7C15) & M
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
            h = z ^ (z >> 31)
        s = (s + h) & M
        x ^= h
    return len(rows), s, x


def fingerprint_array(a: np.ndarray) -> tuple[int, int, int]:
    """Vectorised :func:`fingerprint` over an (n, k) integer array."""
    a = np.asarray(a, dtype=np.uint64)
    n = a.shape[0]
    if n == 0:
        return 0, 0, 0
    with np.errstate(over="ignore"):
        h = np.full(n, 0x9E3779B97F4A7C15, dtype=np.uint64)
        for c in range(a.shape[1]):
            z = h ^ a[:, c]
            z = z + np.uint64(0x9E3779B97F4A7C15)
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            h = z ^ (z >> np.uint64(31))
        s = int(h.sum(dtype=np.uint64))
        x = int(np.bitwise_xor.reduce(h))
    return n, s, x
