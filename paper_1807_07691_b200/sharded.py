"""Sharded execution over torch.distributed (SURVEY.md §8(e) "sharded mode").

For stores that do not fit one GPU: shard i of n holds the CSR rows of the
subjects and the CSC rows of the objects whose ids fall in id range i
(``storage.load(dir, shard=(i, n))``, owner(id) = (id-1)*n // node_count).
Every join step of the reference's chain (executor.py:340-356) looks up the
row value of its first join variable J[0] in one orientation, so a binding row
must sit on the shard owning that value: before a step whose key differs from
the current partitioning, rows are regrouped by owner on the device
(``gsm_partition_rows``) and exchanged with one all-to-all; the step itself
runs locally on the device (``gsm_execute_seeded``).  Consecutive steps keyed
on the same variable (stars) need no exchange.  Cross products (J0)
all-gather the right table.  Per-step counters are all-reduced, so the
reference's budget rules (executor.py:158-163, 192-193, 237-241) apply to the
global counts with the reference's messages on every rank.  DISTINCT
(executor.py:360-367) exchanges projected rows by a hash of the tuple, then
deduplicates locally.  With NCCL the exchanged tensors stay on the device
(NVLink); with gloo they go through host memory.
"""

from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import _lib
from .errors import ResourceLimitError
from .executor import (
    DEFAULT_ROW_BUDGET,
    BindingTable,
    ExecutionReport,
    StepReport,
    _pattern_text,
    compile_plan,
)

_HUGE = 1 << 62


def _torch():
    import torch
    import torch.distributed as dist

    return torch, dist


class _CAI:
    """__cuda_array_interface__ view of library-owned device rows."""

    def __init__(self, ptr: int, n: int, k: int):
        self.__cuda_array_interface__ = {"shape": (n, k), "typestr": "<i4", "data": (ptr, False),
                                         "version": 3, "strides": None}


def pattern_vars(rec) -> list[int]:
    """Schema of a scanned pattern (executor.py:101-110) as variable ids."""
    out: list[int] = []
    for v in (rec.s_var, rec.o_var):
        if v >= 0 and v not in out:
            out.append(v)
    return out


def exchange_plan(recs) -> list[dict]:
    """Per join step: kind ("cross" / "join"), the key variable, the output
    schema, and whether the rows must be exchanged first (SURVEY.md §8(e):
    consecutive steps keyed on the same variable need no exchange).

    The first scan of R1 / R4 patterns is partitioned by its subject (local
    CSR rows); R2 / R3 / R5 scans live on the owner of the constant."""
    first = recs[0]
    schema = pattern_vars(first)
    part_var = first.s_var if (first.s_var >= 0 and first.o_var >= 0) else None
    out = []
    for rec in recs[1:]:
        rs = pattern_vars(rec)
        jv = [v for v in schema if v in rs]
        new = schema + [v for v in rs if v not in schema]
        if not jv:
            out.append({"kind": "cross", "key": None, "schema": new, "exchange": False})
        else:
            key = jv[0]
            out.append({"kind": "join", "key": key, "schema": new, "exchange": part_var != key})
            part_var = key
        schema = new
    return out


class _Shard:
    """One rank's view: its shard store, the library context, and the
    collectives.  Library launches, torch ops and NCCL collectives are all
    enqueued on the context's own stream (``gsm_context_stream`` wrapped as a
    torch ExternalStream), so nothing synchronises the host between them; the
    host waits only where it needs a size: once inside each library call
    (its result size) and once per exchange (the all-to-all's split sizes)."""

    def __init__(self, store, group):
        torch, dist = _torch()
        self.torch, self.dist, self.group = torch, dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if store.shard is not None and tuple(store.shard) != (self.rank, self.world):
            raise ValueError(f"store shard {store.shard} != (rank, world) {(self.rank, self.world)}")
        self.store = store
        self.L = _lib.lib()
        self.ctx = store.context()
        self.nccl = dist.get_backend(group) == "nccl"
        self.cdev = torch.device("cuda", store.device)
        self.xdev = self.cdev if self.nccl else torch.device("cpu")
        sp = C.c_uint64(0)
        _lib.check(self.L.gsm_context_stream(self.ctx, C.byref(sp)))
        self.stream = torch.cuda.ExternalStream(int(sp.value), device=self.cdev)
        self.sent_bytes = 0      # rows this rank sent to other ranks (exchanges, all-gathers)
        self.collectives = 0
        self.host_syncs = 0

    # -- device tables -------------------------------------------------------
    def take(self, res, k: int):
        """gsm_result -> owned (n, k) int32 CUDA tensor (frees the result)."""
        torch, L = self.torch, self.L
        try:
            n = C.c_int64(0)
            kk = C.c_int32(0)
            _lib.check(L.gsm_result_shape(res, C.byref(n), C.byref(kk)))
            n = int(n.value)
            if n == 0 or k == 0:
                return torch.zeros((n, k), dtype=torch.int32, device=self.cdev)
            ptr = C.c_uint64(0)
            _lib.check(L.gsm_result_device_ptr(res, C.byref(ptr)))
            return torch.as_tensor(_CAI(int(ptr.value), n, k), device=self.cdev).clone()
        finally:
            L.gsm_result_free(res)

    def run(self, seed, seed_vars, recs, proj, distinct=False):
        """gsm_execute_seeded (seed is None: recs[0] is a scan).  Returns the
        rows and this rank's per-step (rows, E, kind) counters."""
        L = self.L
        n = len(recs)
        nrep = n + (1 if seed is not None else 0)
        bufs = ((C.c_int64 * max(1, nrep))(), (C.c_int64 * max(1, nrep))(), None,
                (C.c_int32 * max(1, nrep))(), (C.c_int32 * max(1, nrep))())
        rep = _lib.Report(bufs[0], bufs[1], None, bufs[3], bufs[4])
        arr = (_lib.Pattern * max(1, n))(*recs)
        parr = (C.c_int32 * max(1, len(proj)))(*proj)
        res = C.c_void_p()
        if seed is None:
            st = L.gsm_execute(self.ctx, arr, n, parr, len(proj), int(distinct), _HUGE,
                               _lib.GSM_BUDGET_PARALLEL, 0, 1, C.byref(rep), C.byref(res))
        else:
            # the seed was written by torch ops on the context's stream
            seed = seed.contiguous()
            sv = (C.c_int32 * max(1, len(seed_vars)))(*seed_vars)
            st = L.gsm_execute_seeded(self.ctx, seed.data_ptr() if seed.numel() else None,
                                      int(seed.shape[0]), sv, len(seed_vars), arr, n, parr,
                                      len(proj), int(distinct), _HUGE, _lib.GSM_BUDGET_PARALLEL,
                                      C.byref(rep), C.byref(res))
        _lib.check(st)
        self.host_syncs += 1
        rows = self.take(res, len(proj))
        return rows, [int(bufs[0][i]) for i in range(nrep)], [int(bufs[1][i]) for i in range(nrep)], \
            [_lib.STEP_KINDS[bufs[3][i]] for i in range(nrep)]

    # -- collectives -----------------------------------------------------------
    def gather_counts(self, vals: list[int]) -> list[list[int]]:
        """All-gather one int64 vector per rank (ONE collective, one host read)."""
        torch = self.torch
        t = torch.tensor(vals, dtype=torch.int64, device=self.xdev)
        out = torch.empty((self.world * len(vals),), dtype=torch.int64, device=self.xdev)
        self.dist.all_gather_into_tensor(out, t, group=self.group)  # rank-major concatenation
        out = out.view(self.world, len(vals))
        self.collectives += 1
        self.host_syncs += 1
        return out.cpu().tolist()

    def partition(self, rows, key_col: int):
        """Group rows by owner shard on the device -> (grouped rows, send counts)."""
        rows = rows.contiguous()
        n, k = int(rows.shape[0]), int(rows.shape[1])
        counts = (C.c_int64 * self.world)()
        grouped = self.torch.empty_like(rows)
        _lib.check(self.L.gsm_partition_rows(
            self.ctx, rows.data_ptr() if rows.numel() else None, n, k, key_col,
            self.store.node_count, self.world, grouped.data_ptr() if grouped.numel() else None,
            counts))
        self.host_syncs += 1
        return grouped, [int(counts[i]) for i in range(self.world)]

    def all_to_all(self, grouped, send: list[int], recv: list[int]):
        torch, dist = self.torch, self.dist
        k = int(grouped.shape[1])
        self.sent_bytes += 4 * k * (sum(send) - send[self.rank])
        if k == 0:
            return torch.zeros((sum(recv), 0), dtype=torch.int32, device=self.cdev)
        out = torch.empty((sum(recv), k), dtype=torch.int32, device=self.xdev)
        dist.all_to_all_single(out, grouped.to(self.xdev), output_split_sizes=recv,
                               input_split_sizes=send, group=self.group)
        self.collectives += 1
        return out.to(self.cdev)

    def cross(self, left, right):
        """Local left rows x the whole right table (gsm_cross_rows)."""
        torch = self.torch
        nl, a = int(left.shape[0]), int(left.shape[1])
        nr, b = int(right.shape[0]), int(right.shape[1])
        out = torch.empty((nl * nr, a + b), dtype=torch.int32, device=self.cdev)
        if out.numel():
            left = left.contiguous()
            right = right.to(self.cdev).contiguous()
            _lib.check(self.L.gsm_cross_rows(self.ctx, left.data_ptr() if left.numel() else None,
                                             nl, a, right.data_ptr() if right.numel() else None,
                                             nr, b, out.data_ptr()))
        return out

    def allgather_rows(self, rows, sizes: list[int] | None = None):
        """All-gather variable-size row blocks; ``sizes`` (every rank's row
        count) may come from an earlier counts collective."""
        torch, dist = self.torch, self.dist
        n, k = int(rows.shape[0]), int(rows.shape[1])
        if sizes is None:
            sizes = [r[0] for r in self.gather_counts([n])]
        mx = max(sizes) if sizes else 0
        buf = torch.zeros((mx, max(k, 1)), dtype=torch.int32, device=self.xdev)
        if n and k:
            buf[:n, :k] = rows.to(self.xdev)
        parts = torch.empty((self.world * mx, max(k, 1)), dtype=torch.int32, device=self.xdev)
        dist.all_gather_into_tensor(parts, buf, group=self.group)
        parts = parts.view(self.world, mx, max(k, 1))
        self.collectives += 1
        self.sent_bytes += 4 * k * n * (self.world - 1)
        return torch.cat([parts[r, :m, :k] for r, m in enumerate(sizes)], dim=0), sizes


def _check_budget(i: int, kind: str, rows: int, e: int, prev_rows: int, budget: int, seq: bool):
    """The reference's budget rule of step i on GLOBAL counters
    (executor.py:158-163 cross, 192-193 sequential, 237-241 parallel)."""
    if kind in ("cross", "gate"):
        if prev_rows and rows > budget:
            raise ResourceLimitError(
                f"cross product of {prev_rows} x {rows // prev_rows} rows exceeds budget {budget}")
    elif not seq and e > budget:
        raise ResourceLimitError(f"pre-allocated join region of {e} rows exceeds budget {budget}")
    elif seq and rows > budget:
        raise ResourceLimitError(f"join output exceeds row budget {budget}")


def execute_sharded(query, plan, store, mode: str = "gpu", row_budget: int = DEFAULT_ROW_BUDGET,
                    report: ExecutionReport | None = None, gather: bool = True,
                    group=None) -> BindingTable:
    """executor.execute (executor.py:296-368) over the shards of ``group``.

    ``store`` is this rank's shard (``load(dir, shard=(rank, world))``; a full
    store also works: every rank then holds everything and the exchanges
    still partition the work).  Returns the whole result on rank 0 when
    ``gather`` (else this rank's part).  ``report`` receives the global
    per-step counters, and (ExecutionReport of this package) the bytes this
    rank sent, the collectives and the host synchronisations.

    Every rank runs the same sequence of collectives.  The per-step counters
    ride on the next collective the plan needs anyway (an exchange's split
    sizes, the cross product's gather, the final gather), so the budget rules
    are checked on global counts in plan order with the reference's messages
    -- raised on every rank, possibly a few local steps after the violating
    one."""
    if mode not in ("gpu", "sequential", "parallel"):
        raise ValueError(f"unknown mode {mode!r}")
    if not plan.steps:
        raise ValueError("cannot execute an empty plan")
    sh = _Shard(store, group)
    with sh.torch.cuda.stream(sh.stream):
        return _execute_sharded(sh, query, plan, mode, int(row_budget), report, gather)


def _execute_sharded(sh, query, plan, mode, budget, report, gather):
    torch = sh.torch
    steps, arr, proj_arr, nproj = compile_plan(query, plan)
    recs = [arr[i] for i in range(len(steps))]
    proj = [int(proj_arr[i]) for i in range(nproj)]
    sched = exchange_plan(recs)
    seq = mode != "parallel"  # "gpu" applies the sequential rule, as execute() does
    n_steps = len(steps)
    loc_rows = [0] * n_steps   # this rank's counters
    loc_e = [0] * n_steps
    glob_rows: list[int | None] = [None] * n_steps  # global, once a collective carried them
    glob_e: list[int | None] = [None] * n_steps
    kinds: list[str] = [""] * n_steps
    secs: list[float] = [0.0] * n_steps
    checked = 0  # steps [0, checked) passed the budget rules

    def absorb(gathered):
        """Sum the counter block of an all-gather, then check every step
        whose global counters are now known, in plan order."""
        nonlocal checked
        for i in range(n_steps):
            glob_rows[i] = sum(r[i] for r in gathered)
            glob_e[i] = sum(r[n_steps + i] for r in gathered)
        while checked < n_steps and checked <= known:
            i = checked
            if i > 0:
                _check_budget(i, kinds[i], glob_rows[i], glob_e[i], glob_rows[i - 1], budget, seq)
            checked += 1

    t0 = time.perf_counter()
    schema = pattern_vars(recs[0])
    cur, r0, _, k0 = sh.run(None, None, recs[:1], schema)
    loc_rows[0], kinds[0] = r0[0], k0[0]
    secs[0] = time.perf_counter() - t0
    known = 0

    for j, st in enumerate(sched, start=1):
        t0 = time.perf_counter()
        rec = recs[j]
        if st["kind"] == "cross":
            right, _, _, _ = sh.run(None, None, [rec], pattern_vars(rec))
            # the right table's gather carries every counter so far + |L|
            g = sh.gather_counts(loc_rows + loc_e + [int(right.shape[0]), int(cur.shape[0])])
            known = j - 1
            absorb(g)
            nl = sum(r[-1] for r in g)
            full_right, _ = sh.allgather_rows(right, [r[-2] for r in g])
            nr = int(full_right.shape[0])
            if nl * nr > budget:
                raise ResourceLimitError(
                    f"cross product of {nl} x {nr} rows exceeds budget {budget}")
            cur = sh.cross(cur, full_right)
            loc_rows[j], loc_e[j], kinds[j] = int(cur.shape[0]), 0, "cross"
        else:
            if st["exchange"] and sh.world > 1:
                grouped, send = sh.partition(cur, schema.index(st["key"]))
                g = sh.gather_counts(loc_rows + loc_e + send)
                known = j - 1
                absorb(g)
                recv = [r[2 * n_steps + sh.rank] for r in g]
                cur = sh.all_to_all(grouped, send, recv)
            cur, r, e, k = sh.run(cur, schema, [rec], st["schema"])
            loc_rows[j], loc_e[j], kinds[j] = r[1], e[1], k[1]
        schema = st["schema"]
        secs[j] = time.perf_counter() - t0

    # projection (executor.py:358-359) and DISTINCT on the union (:360-367):
    # rows are exchanged by a hash of the projected tuple, then deduplicated
    # locally (the projected columns get fresh variable ids: a projection may
    # repeat a variable)
    cur, _, _, _ = sh.run(cur, schema, [], proj)
    if query.distinct and proj and sh.world > 1:
        grouped, send = sh.partition(cur, -1)
        g = sh.gather_counts(loc_rows + loc_e + send)
        known = n_steps - 1
        absorb(g)
        cur = sh.all_to_all(grouped, send, [r[2 * n_steps + sh.rank] for r in g])
    if query.distinct and proj:
        ids = list(range(len(proj)))
        cur, _, _, _ = sh.run(cur, ids, [], ids, distinct=True)

    # the final counters (and the result sizes for the gather): one collective
    g = sh.gather_counts(loc_rows + loc_e + [int(cur.shape[0])])
    known = n_steps - 1
    absorb(g)
    sizes = [r[-1] for r in g]

    if report is not None:
        seen: set[int] = set()
        for pat in steps:
            if pat.p not in seen:
                seen.add(pat.p)
                report.preparations += 1
            report.uses += 1
        for i, pat in enumerate(steps):
            report.steps.append(StepReport(_pattern_text(pat), int(glob_rows[i]), int(glob_e[i]),
                                           secs[i]))
        report.kinds = kinds
        if isinstance(report, ExecutionReport):
            report.exchanged_bytes += sh.sent_bytes
            report.collectives += sh.collectives
            report.host_syncs += sh.host_syncs

    if not gather:
        return BindingTable(tuple(query.projection), array=cur.cpu().numpy().astype(np.uint32))
    full, _ = sh.allgather_rows(cur, sizes)
    if report is not None and isinstance(report, ExecutionReport):
        report.exchanged_bytes += 4 * int(cur.shape[1]) * int(cur.shape[0]) * (sh.world - 1)
        report.collectives += 1
    if sh.rank != 0:
        return BindingTable(tuple(query.projection), array=cur.cpu().numpy().astype(np.uint32))
    out = full.cpu().numpy().astype(np.uint32)
    if query.distinct and not proj:
        out = out[:1]  # zero-arity rows: DISTINCT keeps at most one ()
    return BindingTable(tuple(query.projection), array=out)
