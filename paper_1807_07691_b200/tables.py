"""Table-level join functions on the GPU, mirroring the reference executor's
unit API (/root/reference/pkg/src/gsmat/executor.py:130-293):

  sm_join(left, right, join_vars, row_budget)            executor.py:168-194
  parallel_sm_join(left, right, join_vars, worker_count,
                   prealloc, row_budget)                  executor.py:218-280
  cross_product(left, right, row_budget)                  executor.py:155-165
  preallocate(left, right, first_var) -> PreallocPlan     executor.py:197-215
  match_counts(left, right, join_vars) -> Counter         executor.py:283-293
  regroup(table, var)                                     executor.py:130-137

``left``/``right`` are any binding tables with ``schema`` and ``rows`` (the
reference's BindingTable or ours).  The joins run through ``gsm_table_join``
(the right table is indexed on the device: stable radix sort by the first
join variable + a run hash, then the same count/scan/scatter kernels as
execute()).  ``sm_join`` returns rows in the reference's order (left rows in
order, candidates in right-table order); the budget rules and messages are the
reference's (sequential: emitted rows; parallel: the pre-allocated total E).
``regroup`` is a host-side reordering (it only changes row order).
"""

from __future__ import annotations

import ctypes as C
import atexit
import threading
from collections import Counter
from dataclasses import dataclass

import numpy as np

from . import _lib
from .executor import DEFAULT_ROW_BUDGET, BindingTable, _fetch


@dataclass
class PreallocPlan:
    """executor.PreallocPlan (executor.py:52-64)."""

    keys: list[int]
    counts: list[int]
    offsets: list[int]
    total: int


_ctx_lock = threading.Lock()
_ctx: dict[int, tuple] = {}


def _context(device: int = 0):
    """A context over an empty device store: table joins need no store."""
    with _ctx_lock:
        hit = _ctx.get(device)
        if hit is None:
            L = _lib.lib()
            store = C.c_void_p()
            _lib.check(L.gsm_store_create(device, 0, 0, C.byref(store)))
            _lib.check(L.gsm_store_finalize(store))
            ctx = C.c_void_p()
            _lib.check(L.gsm_context_create(store, 1 << 20, C.byref(ctx)))
            hit = _ctx[device] = (store, ctx)
            if len(_ctx) == 1:
                atexit.register(_free_contexts)
        return hit[1]


def _free_contexts() -> None:
    L = _lib.lib()
    with _ctx_lock:
        for store, ctx in _ctx.values():
            L.gsm_context_free(ctx)
            L.gsm_store_free(store)
        _ctx.clear()


def _rows_array(table) -> np.ndarray:
    arr = getattr(table, "_array", None)
    k = len(table.schema)
    if arr is not None and getattr(table, "_rows", None) is None:
        a = np.ascontiguousarray(arr, dtype=np.uint32)
    else:
        rows = table.rows
        a = np.asarray(rows, dtype=np.uint64).reshape(len(rows), k) if rows else np.zeros((0, k), np.uint64)
        if a.size and int(a.max()) >= 2**32:
            raise ValueError("table ids must be < 2^32")
        a = np.ascontiguousarray(a, dtype=np.uint32)
    return a.reshape(-1, k) if k else np.zeros((len(table), 0), np.uint32)


def _layout(left, right, join_vars):
    """_join_layout (executor.py:140-152): positions and output schema."""
    jl = [list(left.schema).index(v) for v in join_vars]
    jr = [list(right.schema).index(v) for v in join_vars]
    left_set = set(left.schema)
    rcols = [v for v in right.schema if v not in left_set]
    return jl, jr, tuple(left.schema) + tuple(rcols)


def _join(left, right, join_vars, row_budget, budget_mode, want_counts=False, counts_only=False):
    L = _lib.lib()
    la, ra = _rows_array(left), _rows_array(right)
    if join_vars:
        jl, jr, schema = _layout(left, right, join_vars)
    else:
        jl, jr, schema = [], [], tuple(left.schema) + tuple(right.schema)
    nj = len(jl)
    jl_a = (C.c_int32 * max(1, nj))(*jl)
    jr_a = (C.c_int32 * max(1, nj))(*jr)
    E = C.c_int64(0)
    counts = np.zeros(la.shape[0], dtype=np.int64) if want_counts else None
    res = C.c_void_p()
    st = L.gsm_table_join(
        _context(), la.ctypes.data if la.size else None, la.shape[0], la.shape[1],
        ra.ctypes.data if ra.size else None, ra.shape[0], ra.shape[1], jl_a, jr_a, nj,
        min(int(row_budget), (1 << 63) - 1), budget_mode, C.byref(E),
        counts.ctypes.data if (counts is not None and counts.size) else None,
        None if counts_only else C.byref(res))
    _lib.check(st)
    if counts_only:
        return None, int(E.value), counts
    out = _fetch(L, res)
    return BindingTable(schema, array=out), int(E.value), counts


def sm_join(left, right, join_vars: list[str], row_budget: int = DEFAULT_ROW_BUDGET) -> BindingTable:
    """executor.sm_join (executor.py:168-194) on the GPU, same row order."""
    if not join_vars:
        return cross_product(left, right, row_budget)
    return _join(left, right, join_vars, row_budget, _lib.GSM_BUDGET_SEQUENTIAL)[0]


def parallel_sm_join(left, right, join_vars: list[str], worker_count: int = 1,
                     prealloc: PreallocPlan | None = None,
                     row_budget: int = DEFAULT_ROW_BUDGET) -> BindingTable:
    """executor.parallel_sm_join (executor.py:218-280): the pre-allocation
    budget rule (E > budget raises); ``worker_count`` is accepted for
    signature compatibility."""
    if not join_vars:
        return cross_product(left, right, row_budget)
    if prealloc is not None and prealloc.total > row_budget:
        from .errors import ResourceLimitError

        raise ResourceLimitError(
            f"pre-allocated join region of {prealloc.total} rows exceeds budget {row_budget}")
    return _join(left, right, join_vars, row_budget, _lib.GSM_BUDGET_PARALLEL)[0]


def cross_product(left, right, row_budget: int = DEFAULT_ROW_BUDGET) -> BindingTable:
    """executor.cross_product (executor.py:155-165)."""
    return _join(left, right, [], row_budget, _lib.GSM_BUDGET_SEQUENTIAL)[0]


def preallocate(left, right, first_var: str) -> PreallocPlan:
    """executor.preallocate (executor.py:197-215): the device computes every
    left row's first-variable match count N_r (a counts-only table join: no
    candidate is materialised, O(|L| + |R|) device memory); rows are grouped
    by key in first-occurrence order (N[g] = sum of N_r over the group)."""
    _, E, counts = _join(left, right, [first_var], (1 << 62), _lib.GSM_BUDGET_PARALLEL,
                         want_counts=True, counts_only=True)
    la = _rows_array(left)
    if la.shape[0] == 0:
        return PreallocPlan([], [], [], 0)
    keys = la[:, list(left.schema).index(first_var)].astype(np.int64)
    uniq, first, inv = np.unique(keys, return_index=True, return_inverse=True)
    sums = np.zeros(len(uniq), dtype=np.int64)  # exact int64 group sums
    np.add.at(sums, inv.reshape(-1), counts)
    order = np.argsort(first, kind="stable")
    gk = uniq[order].tolist()
    gc = sums[order].tolist()
    offs = np.concatenate(([0], np.cumsum(sums[order])[:-1])).astype(np.int64).tolist()
    return PreallocPlan(gk, gc, offs, int(E))


def match_counts(left, right, join_vars: list[str]) -> Counter:
    """executor.match_counts (executor.py:283-293): the boolean sparse-matrix
    product's value cells."""
    joined = sm_join(left, right, join_vars)
    keep = [i for i, v in enumerate(joined.schema) if v not in join_vars]
    return Counter(tuple(row[i] for i in keep) for row in joined.rows)


def regroup(table, var: str) -> BindingTable:
    """executor.regroup (executor.py:130-137): stable group-by on ``var`` in
    first-occurrence key order (a reordering; no join work)."""
    a = _rows_array(table)
    if a.shape[0] == 0:
        return BindingTable(table.schema, array=a, sorted_by=var)
    col = a[:, list(table.schema).index(var)]
    _, first, inv = np.unique(col, return_index=True, return_inverse=True)
    rank = np.argsort(np.argsort(first, kind="stable"), kind="stable")[inv]
    order = np.argsort(rank, kind="stable")
    return BindingTable(table.schema, array=a[order], sorted_by=var)
