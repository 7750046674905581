"""The drop-in executor: ``execute(query, plan, store, mode="gpu", ...)``.

Same signature, argument meaning, result type and error behaviour as the
reference's ``gsmat.executor.execute``
(/root/reference/pkg/src/gsmat/executor.py:296-368), but the whole plan runs
as a chain of hand-written sm_100a kernels (csrc/gsm_exec.cu) over the
HBM-resident store, through the C ABI in include/gsmat_b200.h.

* ``query``/``plan`` may come from the reference (``gsmat.qparser`` /
  ``gsmat.planner``) or from :mod:`.frontend`; only the attributes the
  reference's execute reads are used (patterns' s/p/o/empty/source,
  ``plan.steps[i].pattern``, ``projection``, ``distinct``).
* ``store`` is a :class:`.storage.DeviceStore` (``storage.load``) or a
  reference ``Store`` (uploaded once and cached).
* ``mode``: "gpu" (default) evaluates with the reference's DEFAULT mode's
  budget rule, the sequential one: a join raises ResourceLimitError when its
  EMITTED rows exceed ``row_budget`` (executor.py:192-193), so a query whose
  pre-filter candidate total E is large but whose output is small (the
  device filters while expanding) is answered, as ``gsmat query`` answers it.
  "sequential" is the same rule; "parallel" selects the parallel mode's
  pre-allocation rule (E > budget, executor.py:237-241). Every mode runs on
  the GPU; there is no CPU path.
* The result is a :class:`BindingTable` whose ``rows`` are the projected id
  tuples (bag; row order is not contractual); ``array`` holds
  the same rows as an (n, k) uint32 numpy array without building tuples.
"""

from __future__ import annotations

import ctypes as C
import operator
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import DeviceMemoryError, ResourceLimitError
from .storage import DeviceStore, from_store

DEFAULT_ROW_BUDGET = 10**8
_MODES = ("gpu", "sequential", "parallel")


class BindingTable:
    """An n-ary relation over variables, bag semantics (executor.py:40-49)."""

    def __init__(self, schema, rows=None, sorted_by=None, array=None, view=None):
        self.schema = tuple(schema)
        self.sorted_by = sorted_by
        self._rows = list(rows) if rows is not None else None
        self._array = array
        # (buffer, offset, rows, columns): the rows already sit in a host
        # buffer shared by a batch's results; the (n, k) view of them is made
        # when first asked for
        self._view = view

    @property
    def rows(self) -> list[tuple[int, ...]]:
        if self._rows is None:
            a = self._array if self._view is None else self.array
            if a is None:
                self._rows = []
            elif a.shape[1] == 0:
                self._rows = [()] * a.shape[0]
            else:
                self._rows = list(map(tuple, a.tolist()))
        return self._rows

    @rows.setter
    def rows(self, value) -> None:
        self._rows = list(value)
        self._array = None
        self._view = None

    @property
    def array(self) -> np.ndarray:
        if self._array is None:
            if self._view is not None:
                buf, off, r, k = self._view
                self._array = buf[off:off + r * k].reshape(r, k)
                self._view = None
            else:
                rows = self._rows or []
                self._array = np.asarray(rows, dtype=np.uint64).reshape(len(rows), len(self.schema))
        return self._array

    def __len__(self) -> int:
        if self._rows is not None:
            return len(self._rows)
        if self._view is not None:
            return self._view[2]
        return 0 if self._array is None else int(self._array.shape[0])

    def __eq__(self, other) -> bool:
        if not hasattr(other, "schema") or not hasattr(other, "rows"):
            return NotImplemented
        return tuple(self.schema) == tuple(other.schema) and self.rows == list(other.rows)

    def __repr__(self) -> str:
        return f"BindingTable(schema={self.schema!r}, rows={len(self)} rows)"


@dataclass
class StepReport:
    pattern_text: str
    rows: int
    prealloc_total: int
    seconds: float


@dataclass
class ExecutionReport:
    """executor.ExecutionReport (executor.py:74-91); seconds are device time.

    Extra device-side fields (not in the reference): per-step ``kinds``,
    ``arities`` and ``fused`` (1 = the step ran inside the previous step's
    kernel, so its input table was never materialised), the whole-query ``device_seconds``, the bytes copied each way
    (``h2d_bytes``, ``d2h_bytes``, result rows included) and ``kernels``.
    """

    steps: list[StepReport] = field(default_factory=list)
    preparations: int = 0
    uses: int = 0
    kinds: list[str] = field(default_factory=list)
    arities: list[int] = field(default_factory=list)
    fused: list[int] = field(default_factory=list)
    device_seconds: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    kernels: int = 0
    chunks: int = 0  # left-row chunks the plan ran in (0 = one pass)
    exchanged_bytes: int = 0  # multi-GPU: bytes this rank sent to its peers
    collectives: int = 0
    host_syncs: int = 0

    @property
    def intermediate_total(self) -> int:
        return sum(s.rows for s in self.steps)

    def lines(self) -> list[str]:
        out = [
            f"{i}\t{s.pattern_text}\t{s.rows}\t{s.prealloc_total}\t{s.seconds:.6f}"
            for i, s in enumerate(self.steps, start=1)
        ]
        out.append(f"preparations\t{self.preparations}\tuses\t{self.uses}")
        return out


def _pattern_text(pattern) -> str:
    src = getattr(pattern, "source", None)
    return src.text() if src is not None and hasattr(src, "text") else repr(pattern)


_PATTERN = operator.attrgetter("pattern")


def compile_plan(query, plan):
    """Plan -> (steps, gsm_pattern array, projection index array, n_proj).

    Variables get small integer ids in order of first appearance in the plan.
    The encoding is cached on the plan object (keyed by its patterns and the
    projection) so repeated executions skip it.
    """
    # List equality short-circuits on identity, so an unchanged plan costs a
    # C-level pass; equal-but-new pattern objects encode identically.
    pats = list(map(_PATTERN, plan.steps))
    cached = getattr(plan, "__dict__", {}).get("_gsm_compiled")
    if cached is not None and cached[0] == pats and cached[1] == query.projection:
        return cached[2]
    compiled = _compile(query, plan)
    try:
        plan.__dict__["_gsm_compiled"] = (pats, list(query.projection), compiled)
    except (AttributeError, TypeError):
        pass
    return compiled


def _compile(query, plan):
    steps = [st.pattern for st in plan.steps]
    var_id: dict[str, int] = {}
    arr = (_lib.Pattern * len(steps))()
    for i, pat in enumerate(steps):
        rec = arr[i]
        for end in ("s", "o"):
            term = getattr(pat, end)
            if isinstance(term, str):
                vid = var_id.setdefault(term, len(var_id))
                setattr(rec, f"{end}_var", vid)
                setattr(rec, f"{end}_const", 0)
            else:
                setattr(rec, f"{end}_var", -1)
                tid = int(term)
                setattr(rec, f"{end}_const", tid if 0 <= tid < 2**32 else 0)
        rec.pid = int(pat.p) if 0 <= int(pat.p) < 2**31 else 0
        rec.empty = 1 if getattr(pat, "empty", False) else 0
    proj = []
    for v in query.projection:
        if v not in var_id:
            raise ValueError(f"projected variable {v} is not bound by the plan")
        proj.append(var_id[v])
    proj_arr = (C.c_int32 * max(1, len(proj)))(*proj)
    return steps, arr, proj_arr, len(proj)


def _budget_mode(mode: str) -> int:
    """"gpu" and "sequential" -> emitted-rows rule; "parallel" -> E rule."""
    return _lib.GSM_BUDGET_PARALLEL if mode == "parallel" else _lib.GSM_BUDGET_SEQUENTIAL


def execute(
    query,
    plan,
    store,
    mode: str = "gpu",
    worker_count: int = 1,
    row_budget: int = DEFAULT_ROW_BUDGET,
    report: ExecutionReport | None = None,
    *,
    partition: tuple[int, int] = (0, 1),
    chunks: int | None = None,
) -> BindingTable:
    """Evaluate a plan on the GPU and project onto the query's projection.

    ``worker_count`` is accepted for signature compatibility (the grid is
    sized from the device).  ``partition=(i, k)`` evaluates only the i-th of
    k contiguous slices of the first step's rows (multi-GPU row partitioning,
    see :mod:`.distributed`).  A plan whose intermediate tables exceed device
    memory is evaluated in left-row chunks (:func:`_execute_chunked`);
    ``chunks=k`` forces at least k of them.
    """
    if mode not in _MODES:
        raise ValueError(f"unknown mode {mode!r}")
    if not plan.steps:
        raise ValueError("cannot execute an empty plan")
    if chunks is not None and tuple(partition) != (0, 1):
        raise ValueError("chunks and partition cannot be combined")
    dstore = store if isinstance(store, DeviceStore) else from_store(store)
    if getattr(dstore, "shard", None) is not None and dstore.shard[1] > 1:
        raise ValueError(
            f"store holds shard {dstore.shard} only; evaluate it with sharded.execute_sharded")
    steps, arr, proj_arr, nproj = compile_plan(query, plan)
    n = len(steps)
    budget_mode = _budget_mode(mode)
    budget = min(int(row_budget), (1 << 63) - 1)

    rep_struct = None
    bufs = None
    if report is not None:
        rep_struct, bufs = _new_report(n)

    L = _lib.lib()
    part, parts = partition
    if chunks is not None:
        return _execute_chunked(dstore, query, steps, arr, proj_arr, nproj, budget, budget_mode,
                                report, "rows", _pow2(chunks))
    # the rows land in a host buffer sized by this plan's previous result
    # (gsm_execute_into); a larger result comes back as a handle
    pd = getattr(plan, "__dict__", None)
    hint = pd.get("_gsm_ids", 0) if pd is not None else 0
    cap = hint + hint // 8
    buf = np.empty(max(cap, 1), dtype=np.uint32)
    res, nrows, ncols = C.c_void_p(), C.c_int64(0), C.c_int32(0)
    st = L.gsm_execute_into(
        dstore.context(), arr, n, proj_arr, nproj, 1 if query.distinct else 0, budget,
        budget_mode, int(part), int(parts), C.byref(rep_struct) if rep_struct is not None else None,
        buf.ctypes.data, cap, C.byref(nrows), C.byref(ncols), C.byref(res),
    )
    if st == _lib.GSM_ERR_DEVICE_MEMORY and (part, parts) == (0, 1):
        return _execute_chunked(dstore, query, steps, arr, proj_arr, nproj, budget, budget_mode,
                                report, "rows", _first_parts(dstore, _lib.last_error()))
    _lib.check(st)
    r, k = int(nrows.value), int(ncols.value)
    out = _fetch(L, res) if res.value else buf[:r * k].reshape(r, k)
    if pd is not None:
        pd["_gsm_ids"] = r * max(k, 1)
    if report is not None:
        _fill_report(report, steps, rep_struct, *bufs)
    return BindingTable(tuple(query.projection), array=out)


@dataclass(frozen=True)
class ResultSummary:
    """What :func:`execute_summary` returns instead of the rows: the row
    count and an order-independent multiset fingerprint (wrapping sum and
    xor of a per-row splitmix64 chain over the row's ids; the same value for
    the same bag of rows whatever their order)."""

    schema: tuple
    rows: int
    sum: int
    xor: int

    @property
    def fingerprint(self) -> tuple[int, int, int]:
        return self.rows, self.sum, self.xor


_M64 = (1 << 64) - 1
# GSM_BATCH_INTO=0: execute_batch copies every result after the whole batch
# (A/B of the in-flight copy; tools/e2e_ab.py)
_BATCH_INTO = os.environ.get("GSM_BATCH_INTO", "1") != "0"


def fingerprint_rows(a: np.ndarray) -> tuple[int, int, int]:
    """Host-side twin of ``gsm_result_fingerprint`` for an (n, k) id array."""
    a = np.asarray(a, dtype=np.uint64)
    n = int(a.shape[0])
    if n == 0:
        return 0, 0, 0
    with np.errstate(over="ignore"):
        h = np.full(n, 0x9E3779B97F4A7C15, dtype=np.uint64)
        for c in range(a.shape[1]):
            z = (h ^ a[:, c]) + np.uint64(0x9E3779B97F4A7C15)
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            h = z ^ (z >> np.uint64(31))
        return n, int(h.sum(dtype=np.uint64)), int(np.bitwise_xor.reduce(h))


def execute_summary(query, plan, store, mode: str = "gpu", row_budget: int = DEFAULT_ROW_BUDGET,
                    report: ExecutionReport | None = None, *, chunks: int | None = None
                    ) -> ResultSummary:
    """Evaluate a plan like :func:`execute` but return only the result's row
    count and multiset fingerprint, computed on the device: the rows never
    reach the host, so results larger than host memory (a 19G-row star on a
    power-law store) can still be answered and checked.  Plans whose
    intermediates exceed device memory run in left-row chunks, each chunk's
    result reduced on the device.  Budget rules and errors as in
    :func:`execute` (on the whole plan's counters)."""
    if mode not in _MODES:
        raise ValueError(f"unknown mode {mode!r}")
    if not plan.steps:
        raise ValueError("cannot execute an empty plan")
    dstore = store if isinstance(store, DeviceStore) else from_store(store)
    if getattr(dstore, "shard", None) is not None and dstore.shard[1] > 1:
        raise ValueError(
            f"store holds shard {dstore.shard} only; evaluate it with sharded.execute_sharded")
    steps, arr, proj_arr, nproj = compile_plan(query, plan)
    budget_mode = _budget_mode(mode)
    budget = min(int(row_budget), (1 << 63) - 1)
    parts0 = _pow2(chunks) if chunks is not None else 1
    return _execute_chunked(dstore, query, steps, arr, proj_arr, nproj, budget, budget_mode,
                            report, "summary", parts0)


# slices are row-granular (k_slice_pick), so splitting stops only when one
# first-table row's own chain outgrows the device
_MAX_PARTS = 1 << 30
_NO_BUDGET = (1 << 63) - 1


def _pow2(k: int) -> int:
    k = int(k)
    if k < 1:
        raise ValueError("chunks must be >= 1")
    p = 1
    while p < k:
        p <<= 1
    return min(p, _MAX_PARTS)


def _first_parts(dstore, msg: str) -> int:
    """Chunk count for a plan that failed with "intermediate result of R rows
    x k columns exceeds device memory": enough chunks for 8*R*k bytes (two
    arena halves) to fit the context's capacity, with 25% headroom (equal-E
    chunks balance the first join only, so later steps may split further)."""
    import re

    m = re.search(r"of (\d+) rows x (\d+) columns", msg)
    cap = C.c_int64(0)
    _lib.check(_lib.lib().gsm_context_capacity(dstore.context(), C.byref(cap)))
    if not m or cap.value <= 0:
        return 2
    need = 8 * int(m.group(1)) * max(1, int(m.group(2)))
    return _pow2(max(2, -(-need * 5 // (4 * cap.value))))


def _host_budget_bytes() -> int:
    try:
        return int(os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE") * 0.5)
    except (ValueError, OSError, AttributeError):
        return 1 << 40


def _check_budget_totals(kinds, rows, pre, budget: int, budget_mode: int) -> None:
    """The three budget rules of complete_query (executor.py:158-163,
    192-193, 237-241) applied, in plan order, to counters summed over the
    left-row chunks: the same error the one-pass evaluation raises."""
    for s in range(1, len(kinds)):
        k = kinds[s]
        if k in ("cross", "gate"):
            nl = rows[s - 1]
            nr = (rows[s] // nl) if nl else 0
            if nl * nr > budget:
                raise ResourceLimitError(f"cross product of {nl} x {nr} rows exceeds budget {budget}")
        elif k in ("expand", "filter"):
            if budget_mode == _lib.GSM_BUDGET_PARALLEL and pre[s] > budget:
                raise ResourceLimitError(
                    f"pre-allocated join region of {pre[s]} rows exceeds budget {budget}")
            if budget_mode == _lib.GSM_BUDGET_SEQUENTIAL and rows[s] > budget:
                raise ResourceLimitError(f"join output exceeds row budget {budget}")


def _dedupe_first(a: np.ndarray) -> np.ndarray:
    """DISTINCT across chunks: first occurrence of every row, in order."""
    if a.shape[0] <= 1 or a.shape[1] == 0:
        return a[:1] if a.shape[1] == 0 else a
    v = np.ascontiguousarray(a).view(np.dtype((np.void, a.dtype.itemsize * a.shape[1])))
    _, first = np.unique(v.reshape(-1), return_index=True)
    return a[np.sort(first)]


def _execute_chunked(dstore, query, steps, arr, proj_arr, nproj, budget, budget_mode, report,
                     sink: str, parts0: int):
    """Left-row chunking (SURVEY.md §5, §7 hard part 2; the sizing it
    replaces is executor.py:197-215): the plan runs once per slice of its
    first table (``gsm_execute`` part/parts: equal-E slices, so the union
    of the slices of ``parts`` is the slice of ``parts/2`` they refine), each
    slice's intermediates sized to the device.  A slice that still overflows
    is split in two in place, so the slices stay in first-table order and
    the concatenated rows are the one-pass result.  Budgets are checked on
    the summed counters; each slice's rows are copied out (``sink="rows"``)
    or reduced to a fingerprint on the device (``sink="summary"``) before
    the next slice runs."""
    from collections import deque

    L = _lib.lib()
    ctx = dstore.context()
    n = len(steps)
    distinct = 1 if query.distinct else 0
    keep_rows = sink == "rows" or distinct
    rows_t, pre_t, ms_t = [0] * n, [0] * n, [0.0] * n
    meta = None
    pieces: list[np.ndarray] = []
    held = 0
    host_cap = _host_budget_bytes() if keep_rows else 0
    cnt = fsum = fxor = 0
    done = 0
    dev_s = 0.0
    h2d = d2h = kern = 0
    queue = deque((i, parts0) for i in range(parts0))
    while queue:
        part, parts = queue.popleft()
        rep_struct, bufs = _new_report(n)
        res = C.c_void_p()
        st = L.gsm_execute(ctx, arr, n, proj_arr, nproj, distinct, _NO_BUDGET, budget_mode,
                           part, parts, C.byref(rep_struct), C.byref(res))
        if st == _lib.GSM_ERR_DEVICE_MEMORY:
            msg = _lib.last_error()
            if parts >= _MAX_PARTS:
                raise DeviceMemoryError(f"{msg} (in one of {parts} left-row chunks)")
            queue.appendleft((2 * part + 1, 2 * parts))
            queue.appendleft((2 * part, 2 * parts))
            continue
        _lib.check(st)
        done += 1
        rows_buf, pre_buf, ms_buf, kind_buf, ar_buf, fused_buf = bufs
        for i in range(n):
            rows_t[i] += int(rows_buf[i])
            pre_t[i] += int(pre_buf[i])
            ms_t[i] += float(ms_buf[i])
        if meta is None:
            meta = ([_lib.STEP_KINDS[kind_buf[i]] for i in range(n)],
                    [int(ar_buf[i]) for i in range(n)], [int(fused_buf[i]) for i in range(n)])
        dev_s += rep_struct.total_device_ms / 1e3
        h2d += int(rep_struct.h2d_bytes)
        d2h += int(rep_struct.d2h_bytes)
        kern += int(rep_struct.kernels)
        if keep_rows:
            nrows = C.c_int64(0)
            ncols = C.c_int32(0)
            L.gsm_result_shape(res, C.byref(nrows), C.byref(ncols))
            held += 4 * int(nrows.value) * int(ncols.value)
            if held > host_cap:
                L.gsm_result_free(res)
                raise ResourceLimitError(
                    f"result of more than {held // max(4 * nproj, 1)} rows exceeds host memory "
                    "(execute_summary returns its count and fingerprint)")
            pieces.append(_fetch(L, res))
        else:
            fp = (C.c_uint64 * 3)()
            try:
                _lib.check(L.gsm_result_fingerprint(res, fp))
            finally:
                L.gsm_result_free(res)
            cnt += int(fp[0])
            fsum = (fsum + int(fp[1])) & _M64
            fxor ^= int(fp[2])
    kinds, arities, fused = meta
    _check_budget_totals(kinds, rows_t, pre_t, budget, budget_mode)
    if keep_rows:
        out = np.concatenate(pieces) if pieces else np.empty((0, nproj), dtype=np.uint32)
        if distinct:
            out = _dedupe_first(out)
    if report is not None:
        seen: set[int] = set()
        for pat in steps:
            if pat.p not in seen:
                seen.add(pat.p)
                report.preparations += 1
            report.uses += 1
        for i, pat in enumerate(steps):
            report.steps.append(StepReport(_pattern_text(pat), rows_t[i], pre_t[i], ms_t[i] / 1e3))
        if isinstance(report, ExecutionReport):
            report.kinds.extend(kinds)
            report.arities.extend(arities)
            report.fused.extend(fused)
            report.device_seconds += dev_s
            report.h2d_bytes += h2d
            report.d2h_bytes += d2h
            report.kernels += kern
            report.chunks = done
    schema = tuple(query.projection)
    if sink == "rows":
        return BindingTable(schema, array=out)
    if keep_rows:
        return ResultSummary(schema, *fingerprint_rows(out))
    return ResultSummary(schema, cnt, fsum, fxor)


def _fetch(L, res) -> np.ndarray:
    """Copy a gsm_result's rows into a new (n, k) uint32 array and free it."""
    try:
        nrows = C.c_int64(0)
        ncols = C.c_int32(0)
        _lib.check(L.gsm_result_shape(res, C.byref(nrows), C.byref(ncols)))
        out = np.empty((int(nrows.value), int(ncols.value)), dtype=np.uint32)
        if out.size:
            _lib.check(L.gsm_result_copy(res, out.ctypes.data))
    finally:
        L.gsm_result_free(res)
    return out


def _new_report(n: int):
    bufs = ((C.c_int64 * n)(), (C.c_int64 * n)(), (C.c_float * n)(), (C.c_int32 * n)(),
            (C.c_int32 * n)(), (C.c_int32 * n)())
    rep = _lib.Report(*bufs[:5])
    rep.fused = bufs[5]
    return rep, bufs


def _fill_report(report, steps, rep_struct, rows_buf, pre_buf, ms_buf, kind_buf, ar_buf,
                 fused_buf) -> None:
    # matrix_of(): one preparation per distinct pid, one use per step (executor.py:315-325)
    seen: set[int] = set()
    for pat in steps:
        if pat.p not in seen:
            seen.add(pat.p)
            report.preparations += 1
        report.uses += 1
    for i, pat in enumerate(steps):
        report.steps.append(
            StepReport(_pattern_text(pat), int(rows_buf[i]), int(pre_buf[i]), float(ms_buf[i]) / 1e3)
        )
    if not isinstance(report, ExecutionReport):
        return  # the reference's own ExecutionReport: its fields only
    for i in range(len(steps)):
        report.kinds.append(_lib.STEP_KINDS[kind_buf[i]])
        report.arities.append(int(ar_buf[i]))
        report.fused.append(int(fused_buf[i]))
    report.device_seconds += rep_struct.total_device_ms / 1e3
    report.h2d_bytes += int(rep_struct.h2d_bytes)
    report.d2h_bytes += int(rep_struct.d2h_bytes)
    report.kernels += int(rep_struct.kernels)



class _PreparedBatch:
    """ctypes records of one batch of (query, plan) items, reused while the
    plans keep their compiled encoding (see :func:`compile_plan`)."""

    __slots__ = ("items", "compiled", "ctx_arr", "qarr", "outs", "statuses", "nrows", "ncols",
                 "nrows_np", "ncols_np", "dsts", "caps", "offsets", "total_cap", "ms", "steps",
                 "schemas", "sig")


def _size_slices(prep, sizes) -> None:
    """Per-query slices of the batch's host buffer: the last result sizes
    (ids) plus 1/8 headroom, so a result that varies a little still lands in
    place."""
    off = 0
    offsets = []
    for i, sz in enumerate(sizes):
        cap = sz + sz // 8
        prep.caps[i] = cap
        offsets.append(off)
        off += cap
    prep.offsets = offsets
    prep.total_cap = off


def _batch_sig(items):
    """Everything a batch's encoding depends on, flattened: every plan
    step's pattern (EncodedPattern is frozen, so equal patterns encode
    equally), every projection and DISTINCT flag.  One comprehension over
    the batch instead of a compile_plan validation per query."""
    return ([s.pattern for _, p in items for s in p.steps],
            [(len(p.steps), q.projection, q.distinct) for q, p in items])


def _prepared_batch(dstore, items, budget_mode: int, budget: int) -> _PreparedBatch:
    cache = dstore.__dict__.setdefault("_batch_prep", {})
    # ids only pick the cache slot (a reused id is caught by the signature)
    key = (tuple(map(id, items)), budget_mode, budget)
    sig = _batch_sig(items)
    prep = cache.get(key)
    if prep is not None and prep.sig == sig:
        return prep
    compiled = [compile_plan(q, p) for q, p in items]
    n = len(items)
    prep = _PreparedBatch()
    prep.items = items  # keeps the queries and plans (and so their ids) alive
    prep.compiled = compiled
    prep.sig = sig
    ctxs = dstore.context_pool(n)
    prep.ctx_arr = (C.c_void_p * n)(*[c.value for c in ctxs])
    prep.qarr = (_lib.Query * n)()
    for i, ((query, plan), (steps, arr, proj_arr, nproj)) in enumerate(zip(items, compiled)):
        if not steps:
            raise ValueError("cannot execute an empty plan")
        q = prep.qarr[i]
        q.steps = arr
        q.n_steps = len(steps)
        q.proj = proj_arr
        q.n_proj = nproj
        q.distinct = 1 if query.distinct else 0
        q.part_index, q.part_count = 0, 1
        q.row_budget = budget
        q.budget_mode = budget_mode
        q.report = None
    prep.outs = (C.c_void_p * n)()
    prep.statuses = (C.c_int32 * n)()
    prep.nrows = (C.c_int64 * n)()
    prep.ncols = (C.c_int32 * n)()
    prep.nrows_np = np.frombuffer(prep.nrows, dtype=np.int64)  # views of the ctypes arrays
    prep.ncols_np = np.frombuffer(prep.ncols, dtype=np.int32)
    prep.dsts = (C.c_void_p * n)()
    prep.caps = (C.c_int64 * n)()
    _size_slices(prep, [0] * n)
    prep.ms = C.c_float(0.0)
    prep.steps = [c[0] for c in compiled]
    prep.schemas = [tuple(q.projection) for q, _ in items]
    if len(cache) >= 64:
        cache.clear()
    cache[key] = prep
    return prep


def execute_batch(items, store, mode: str = "gpu", row_budget: int = DEFAULT_ROW_BUDGET,
                  reports: list | None = None, batch_timing: list | None = None) -> list[BindingTable]:
    """Evaluate independent queries concurrently (``gsm_execute_batch``).

    ``items`` is a sequence of ``(query, plan)``; query i runs on its own
    context/stream, and all launch sequences are enqueued before any is
    awaited.  Same results and errors as calling :func:`execute` on each in
    order (the first failing query's exception is raised).  When
    ``batch_timing`` is a list, the batch's device time in seconds is appended.
    """
    if mode not in _MODES:
        raise ValueError(f"unknown mode {mode!r}")
    items = list(items)
    if not items:
        return []
    dstore = store if isinstance(store, DeviceStore) else from_store(store)
    if getattr(dstore, "shard", None) is not None and dstore.shard[1] > 1:
        raise ValueError(
            f"store holds shard {dstore.shard} only; evaluate it with sharded.execute_sharded")
    n = len(items)
    budget_mode = _budget_mode(mode)
    budget = min(int(row_budget), (1 << 63) - 1)
    prep = _prepared_batch(dstore, items, budget_mode, budget)
    qarr = prep.qarr
    rep_bufs = None
    if reports is not None:
        rep_bufs = []
        for i, (_, plan) in enumerate(items):
            rep_struct, bufs = _new_report(len(plan.steps))
            qarr[i].report = C.pointer(rep_struct)
            rep_bufs.append((rep_struct, bufs))
    L = _lib.lib()
    ms = prep.ms
    # One host buffer for all results, sized by this batch's previous
    # results: each query's rows are copied into their slice as soon as the
    # query finishes (gsm_execute_batch_into), overlapping the rest of the
    # batch; a result that outgrew its slice is copied afterwards.
    caps = prep.caps if _BATCH_INTO else None
    buf = np.empty(prep.total_cap, dtype=np.uint32)
    base = buf.ctypes.data
    dsts = prep.dsts
    dsts[:] = [base + 4 * off for off in prep.offsets]
    try:
        st = L.gsm_execute_batch_into(prep.ctx_arr, n, qarr, prep.statuses, dsts, caps,
                                      prep.nrows, prep.ncols, prep.outs,
                                      C.byref(ms) if batch_timing is not None else None)
    finally:
        if reports is not None:
            for i in range(n):
                qarr[i].report = None
    outs = prep.outs
    if st != _lib.GSM_OK:
        msg = _lib.last_error()
        L.gsm_results_copy(outs, n, None, 1)
        if st == _lib.GSM_ERR_DEVICE_MEMORY:
            # a query's intermediates exceed device memory: evaluate the
            # batch one query at a time, the oversize ones in left-row chunks
            return [execute(q, p, dstore, mode=mode, row_budget=row_budget,
                            report=None if reports is None else reports[i])
                    for i, (q, p) in enumerate(items)]
        _lib.raise_status(st, msg)
    nr = prep.nrows_np.tolist()
    nc = prep.ncols_np.tolist()
    results = []
    grown = False
    for i, (sch, r, k, off) in enumerate(zip(prep.schemas, nr, nc, prep.offsets)):
        if outs[i]:  # did not fit its slice: copy it now, give the slice room next time
            a = np.empty((r, k), dtype=np.uint32)
            st = L.gsm_result_copy(outs[i], a.ctypes.data) if a.size else _lib.GSM_OK
            L.gsm_result_free(outs[i])
            outs[i] = None
            _lib.check(st)
            results.append(BindingTable(sch, array=a))
            grown = True
        else:  # already in its slice of buf: the (n, k) view is made on first use
            results.append(BindingTable(sch, view=(buf, off, r, k)))
    if grown:
        _size_slices(prep, [r * max(k, 1) for r, k in zip(nr, nc)])
    if reports is not None:
        for i in range(n):
            rep_struct, bufs = rep_bufs[i]
            _fill_report(reports[i], prep.steps[i], rep_struct, *bufs)
    if batch_timing is not None:
        batch_timing.append(ms.value / 1e3)
    return results
