"""Multi-GPU execution: one process per GPU over torch.distributed.

The store is read-only and every join step is independent per left row (the
reference already splits left-key groups over workers, executor.py:267-276),
so with the store replicated on every GPU a query shards with NO exchange
between plan steps: rank r of W evaluates rows [n*r/W, n*(r+1)/W) of the
first step's table through the whole chain (``gsm_execute`` part_index /
part_count).  The only collectives are on the per-step counters (one
all-reduce, so the row-budget rules -- emitted rows for "gpu"/"sequential"
(executor.py:192-193), E for "parallel" (executor.py:237-241), |L|x|R| for
cross products (executor.py:158-163) -- are applied to the GLOBAL counts and
every rank raises the same ResourceLimitError) and, optionally, the
gather of the result rows to rank 0.  DISTINCT is applied to the union.

``runner`` defaults to the CUDA executor; the CPU tests inject the C oracle's
row-partitioned evaluation to check this plumbing under ``gloo``.
"""

from __future__ import annotations

from typing import Callable

import numpy as np

from .errors import ResourceLimitError
from .executor import DEFAULT_ROW_BUDGET, BindingTable, ExecutionReport, StepReport

# runner(query, plan, store, partition, report) -> (n, k) integer array of projected rows
Runner = Callable[..., np.ndarray]


def _device_runner(query, plan, store, partition, report, mode):
    from .executor import execute

    res = execute(query, plan, store, mode=mode, row_budget=(1 << 62), report=report,
                  partition=partition)
    return res.array


def _torch():
    import torch
    import torch.distributed as dist

    return torch, dist


def _tensor_device(dist):
    import torch

    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def execute_distributed(query, plan, store, mode: str = "gpu", row_budget: int = DEFAULT_ROW_BUDGET,
                        report: ExecutionReport | None = None, gather: bool = True,
                        runner: Runner | None = None, group=None) -> BindingTable:
    """Row-partitioned evaluation of one query over all ranks of ``group``.

    Returns the full result on rank 0 when ``gather`` (else every rank's own
    slice).  ``report`` receives the global per-step counters.
    """
    torch, dist = _torch()
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    dev = _tensor_device(dist)
    local_rep = ExecutionReport()
    distinct = bool(query.distinct)
    run = runner or (lambda q, p, s, part, rep: _device_runner(q, p, s, part, rep, mode))

    class _NoDistinct:  # rank-local rows stay a bag; DISTINCT runs on the union
        def __init__(self, q):
            self.patterns = getattr(q, "patterns", None)
            self.projection = q.projection
            self.distinct = False
            self.variables = getattr(q, "variables", None)

    rows = np.asarray(run(_NoDistinct(query) if distinct else query, plan, store, (rank, world),
                          local_rep))
    k = len(query.projection)
    if rows.ndim != 2:
        rows = rows.reshape(-1, k) if k else np.zeros((rows.shape[0], 0), dtype=np.uint32)

    # global step counters: rows and E summed over the partitions
    n_steps = len(plan.steps)
    cnt = torch.zeros(2 * n_steps + 1, dtype=torch.int64, device=dev)
    for i, s in enumerate(local_rep.steps[:n_steps]):
        cnt[i] = s.rows
        cnt[n_steps + i] = s.prealloc_total
    cnt[2 * n_steps] = rows.shape[0]
    dist.all_reduce(cnt, group=group)
    cnt = cnt.cpu().tolist()
    step_rows, step_e = cnt[:n_steps], cnt[n_steps:2 * n_steps]
    kinds = local_rep.kinds or [""] * n_steps
    for i in range(1, n_steps):
        if kinds[i] in ("cross", "gate"):
            # cross_product's rule (executor.py:158-163) on the GLOBAL tables:
            # every rank crossed its slice of L with the whole right table R,
            # so the summed step rows are |L| * |R|
            n_left = step_rows[i - 1]
            if n_left and step_rows[i] > row_budget:
                raise ResourceLimitError(
                    f"cross product of {n_left} x {step_rows[i] // n_left} rows exceeds "
                    f"budget {row_budget}")
            continue
        if mode == "parallel" and step_e[i] > row_budget:
            raise ResourceLimitError(
                f"pre-allocated join region of {step_e[i]} rows exceeds budget {row_budget}")
        if mode != "parallel" and step_rows[i] > row_budget:
            raise ResourceLimitError(f"join output exceeds row budget {row_budget}")
    if report is not None:
        for i, pat in enumerate(plan.steps):
            src = getattr(pat.pattern, "source", None)
            text = src.text() if src is not None else repr(pat.pattern)
            secs = local_rep.steps[i].seconds if i < len(local_rep.steps) else 0.0
            report.steps.append(StepReport(text, int(step_rows[i]), int(step_e[i]), secs))
        report.kinds = list(kinds)
        if isinstance(report, ExecutionReport):
            report.fused = list(local_rep.fused)
            report.arities = list(local_rep.arities)

    if not gather:
        return BindingTable(tuple(query.projection), array=rows)

    # variable-size gather to rank 0: all-gather counts, pad, all-gather rows
    sizes = torch.tensor([rows.shape[0]], dtype=torch.int64, device=dev)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    all_sizes = [int(t.item()) for t in all_sizes]
    mx = max(all_sizes) if all_sizes else 0
    buf = torch.zeros((mx, max(k, 1)), dtype=torch.int64, device=dev)
    if rows.shape[0] and k:
        buf[: rows.shape[0], :k] = torch.from_numpy(rows.astype(np.int64)).to(dev)
    parts = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    if rank != 0:
        return BindingTable(tuple(query.projection), array=rows)
    full = np.concatenate([p[:n, :k].cpu().numpy() for p, n in zip(parts, all_sizes)], axis=0)
    if distinct and full.shape[0]:
        if k == 0:
            full = full[:1]
        else:
            _, first = np.unique(full, axis=0, return_index=True)
            full = full[np.sort(first)]
    return BindingTable(tuple(query.projection), array=full.astype(np.uint32))
