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
            with torch.cuda.device(self.cdev):
                return torch.as_tensor(_CAI(int(ptr.value), n, k), device=self.cdev).clone()
        finally:
            L.gsm_result_free(res)

    def run(self, seed, seed_vars, recs, proj, distinct=False):
        """gsm_execute_seeded (seed is None: recs[0] is a scan)."""
        torch, L = self.torch, self.L
        n = len(recs)
        nrep = n + (1 if seed is not None else 0)
        bufs = ((C.c_int64 * max(1, nrep))(), (C.c_int64 * max(1, nrep))(), None,
                (C.c_int32 * max(1, nrep))(), (C.c_int32 * max(1, nrep))())
        rep = _lib.Report(bufs[0], bufs[1], None, bufs[3], bufs[4])
        arr = (_lib.Pattern * max(1, n))(*recs)
        parr = (C.c_int32 * max(1, len(proj)))(*proj)
        res = C.c_void_p()
        torch.cuda.synchronize(self.cdev)
        if seed is None:
            st = L.gsm_execute(self.ctx, arr, n, parr, len(proj), int(distinct), _HUGE,
                               _lib.GSM_BUDGET_PARALLEL, 0, 1, C.byref(rep), C.byref(res))
        else:
            seed = seed.contiguous()
            sv = (C.c_int32 * max(1, len(seed_vars)))(*seed_vars)
            st = L.gsm_execute_seeded(self.ctx, seed.data_ptr() if seed.numel() else None,
                                      int(seed.shape[0]), sv, len(seed_vars), arr, n, parr,
                                      len(proj), int(distinct), _HUGE, _lib.GSM_BUDGET_PARALLEL,
                                      C.byref(rep), C.byref(res))
        _lib.check(st)
        rows = self.take(res, len(proj))
        return rows, [int(bufs[0][i]) for i in range(nrep)], [int(bufs[1][i]) for i in range(nrep)], \
            [_lib.STEP_KINDS[bufs[3][i]] for i in range(nrep)]

    # -- collectives -----------------------------------------------------------
    def allreduce(self, vals: list[int]) -> list[int]:
        t = self.torch.tensor(vals, dtype=self.torch.int64, device=self.xdev)
        self.dist.all_reduce(t, group=self.group)
        return [int(x) for x in t.cpu().tolist()]

    def exchange(self, rows, key_col: int):
        """Regroup rows by owner shard (device) and all-to-all them."""
        torch, dist = self.torch, self.dist
        rows = rows.contiguous()
        n, k = int(rows.shape[0]), int(rows.shape[1])
        counts = (C.c_int64 * self.world)()
        grouped = torch.empty_like(rows)
        _lib.check(self.L.gsm_partition_rows(
            self.ctx, rows.data_ptr() if rows.numel() else None, n, k, key_col,
            self.store.node_count, self.world, grouped.data_ptr() if grouped.numel() else None,
            counts))
        send = [int(counts[i]) for i in range(self.world)]
        sc = torch.tensor(send, dtype=torch.int64, device=self.xdev)
        rc = torch.empty_like(sc)
        dist.all_to_all_single(rc, sc, group=self.group)
        recv_n = [int(x) for x in rc.cpu().tolist()]
        if k == 0:
            return torch.zeros((sum(recv_n), 0), dtype=torch.int32, device=self.cdev)
        out = torch.empty((sum(recv_n), k), dtype=torch.int32, device=self.xdev)
        dist.all_to_all_single(out, grouped.to(self.xdev), output_split_sizes=recv_n,
                               input_split_sizes=send, group=self.group)
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
            torch.cuda.synchronize(self.cdev)
            _lib.check(self.L.gsm_cross_rows(self.ctx, left.data_ptr() if left.numel() else None,
                                             nl, a, right.data_ptr() if right.numel() else None,
                                             nr, b, out.data_ptr()))
        return out

    def allgather_rows(self, rows):
        torch, dist = self.torch, self.dist
        n, k = int(rows.shape[0]), int(rows.shape[1])
        sizes = torch.tensor([n], dtype=torch.int64, device=self.xdev)
        alls = [torch.zeros_like(sizes) for _ in range(self.world)]
        dist.all_gather(alls, sizes, group=self.group)
        alls = [int(t.item()) for t in alls]
        mx = max(alls) if alls else 0
        buf = torch.zeros((mx, max(k, 1)), dtype=torch.int32, device=self.xdev)
        if n and k:
            buf[:n, :k] = rows.to(self.xdev)
        parts = [torch.zeros_like(buf) for _ in range(self.world)]
        dist.all_gather(parts, buf, group=self.group)
        return torch.cat([p[:m, :k] for p, m in zip(parts, alls)], dim=0), alls


def execute_sharded(query, plan, store, mode: str = "gpu", row_budget: int = DEFAULT_ROW_BUDGET,
                    report: ExecutionReport | None = None, gather: bool = True,
                    group=None) -> BindingTable:
    """executor.execute (executor.py:296-368) over the shards of ``group``.

    ``store`` is this rank's shard (``load(dir, shard=(rank, world))``; a full
    store also works: every rank then holds everything and the exchanges
    still partition the work).  Returns the whole result on rank 0 when
    ``gather`` (else this rank's part)."""
    if mode not in ("gpu", "sequential", "parallel"):
        raise ValueError(f"unknown mode {mode!r}")
    if not plan.steps:
        raise ValueError("cannot execute an empty plan")
    sh = _Shard(store, group)
    torch = sh.torch
    steps, arr, proj_arr, nproj = compile_plan(query, plan)
    recs = [arr[i] for i in range(len(steps))]
    proj = [int(proj_arr[i]) for i in range(nproj)]
    sched = exchange_plan(recs)
    budget = int(row_budget)
    seq = mode == "sequential"

    step_rows: list[int] = []
    step_e: list[int] = []
    kinds: list[str] = []
    secs: list[float] = []

    t0 = time.perf_counter()
    schema = pattern_vars(recs[0])
    cur, r0, _, k0 = sh.run(None, None, recs[:1], schema)
    g = sh.allreduce([r0[0]])
    step_rows.append(g[0])
    step_e.append(0)
    kinds.append(k0[0])
    secs.append(time.perf_counter() - t0)

    for j, st in enumerate(sched, start=1):
        t0 = time.perf_counter()
        rec = recs[j]
        if st["kind"] == "cross":
            right, _, _, _ = sh.run(None, None, [rec], pattern_vars(rec))
            full_right, _ = sh.allgather_rows(right)
            nl, nr = sh.allreduce([int(cur.shape[0])])[0], int(full_right.shape[0])
            if nl * nr > budget:
                raise ResourceLimitError(
                    f"cross product of {nl} x {nr} rows exceeds budget {budget}")
            cur = sh.cross(cur, full_right)
            rows_g, e_g, kind = nl * nr, 0, "cross"
        else:
            if st["exchange"] and sh.world > 1:
                cur = sh.exchange(cur, schema.index(st["key"]))
            cur, r, e, k = sh.run(cur, schema, [rec], st["schema"])
            rows_g, e_g = sh.allreduce([r[1], e[1]])
            kind = k[1]
            if not seq and e_g > budget:
                raise ResourceLimitError(
                    f"pre-allocated join region of {e_g} rows exceeds budget {budget}")
            if seq and rows_g > budget:
                raise ResourceLimitError(f"join output exceeds row budget {budget}")
        schema = st["schema"]
        step_rows.append(rows_g)
        step_e.append(e_g)
        kinds.append(kind)
        secs.append(time.perf_counter() - t0)

    # projection (executor.py:358-359) and DISTINCT on the union (:360-367):
    # rows are exchanged by a hash of the projected tuple, then deduplicated
    # locally (the projected columns get fresh variable ids: a projection may
    # repeat a variable)
    cur, _, _, _ = sh.run(cur, schema, [], proj)
    if query.distinct and proj:
        if sh.world > 1:
            cur = sh.exchange(cur, -1)
        ids = list(range(len(proj)))
        cur, _, _, _ = sh.run(cur, ids, [], ids, distinct=True)

    if report is not None:
        seen: set[int] = set()
        for pat in steps:
            if pat.p not in seen:
                seen.add(pat.p)
                report.preparations += 1
            report.uses += 1
        for i, pat in enumerate(steps):
            report.steps.append(StepReport(_pattern_text(pat), step_rows[i], step_e[i], secs[i]))
        report.kinds = kinds

    if not gather:
        return BindingTable(tuple(query.projection), array=cur.cpu().numpy().astype(np.uint32))
    full, _ = sh.allgather_rows(cur)
    if sh.rank != 0:
        return BindingTable(tuple(query.projection), array=cur.cpu().numpy().astype(np.uint32))
    out = full.cpu().numpy().astype(np.uint32)
    if query.distinct and not proj:
        out = out[:1]  # zero-arity rows: DISTINCT keeps at most one ()
    return BindingTable(tuple(query.projection), array=out)
