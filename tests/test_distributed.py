"""Multi-process (gloo, world_size 2) checks of the row-partitioned multi-GPU
plumbing (paper_1807_07691_b200/distributed.py).  The per-rank evaluator is
the C oracle's row-partitioned run (same split rule as gsm_execute), so the
partition / global budget / gather / DISTINCT logic is exercised on CPU."""

from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import REPO, lubm_queries

QUERIES = dict(lubm_queries())
UB = "PREFIX ub: <http://swat.cse.lehigh.edu/onto/univ-bench.owl#> "
RDF = "PREFIX rdf: <http://www.w3.org/1999/02/22-rdf-syntax-ns#> "
CROSS = (RDF + UB + "SELECT * WHERE { ?x rdf:type ub:FullProfessor . "
         "?y rdf:type ub:Course . }")
# (name, query, row budget or None, mode)
CASES = [
    ("q09", QUERIES["q09"], None, "gpu"),
    ("q08", QUERIES["q08"], None, "gpu"),
    ("q02", QUERIES["q02"], None, "gpu"),
    ("distinct", UB + "SELECT DISTINCT ?d WHERE { ?x ub:memberOf ?d . ?x ub:takesCourse ?c . }",
     None, "gpu"),
    ("cross", CROSS, None, "gpu"),
    ("budget_par", QUERIES["q09"], 10, "parallel"),
    ("budget_seq", QUERIES["q09"], 10, "gpu"),
    ("budget_cross", CROSS, 50, "gpu"),
]


def _kinds(plan) -> list[str]:
    """Step kinds as the executor reports them: a step sharing no variable
    with the steps before it is a cross product (a gate when it has none)."""
    bound: set = set()
    kinds = []
    for i, st in enumerate(plan.steps):
        vs = {t for t in (st.pattern.s, st.pattern.o) if isinstance(t, str)}
        kinds.append("scan" if i == 0 else "join" if vs & bound else "cross" if vs else "gate")
        bound |= vs
    return kinds


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, store_dir, out_dir):
    sys.path.insert(0, str(REPO))
    sys.path.insert(0, str(REPO / "tests"))
    import torch.distributed as dist

    from hoststore import HostStore, plan_for
    from oracle import oracle as orc
    from paper_1807_07691_b200.distributed import execute_distributed
    from paper_1807_07691_b200.errors import ResourceLimitError
    from paper_1807_07691_b200.executor import ExecutionReport, StepReport

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    store = HostStore(store_dir)
    prep = orc.PreparedStore(store.matrices)

    def runner(q, plan, st, part, rep):
        rows, srows, spre = orc.run(prep, [s.pattern for s in plan.steps], q.projection,
                                    q.distinct, partition=part)
        for i, s in enumerate(plan.steps):
            rep.steps.append(StepReport(s.pattern.source.text(), srows[i], spre[i], 0.0))
        rep.kinds = _kinds(plan)
        return np.asarray(rows, dtype=np.uint32).reshape(len(rows), len(q.projection))

    results = {}
    for name, text, budget, mode in CASES:
        q, plan = plan_for(store, text)
        try:
            rep = ExecutionReport()
            res = execute_distributed(q, plan, store, runner=runner, report=rep, mode=mode,
                                      row_budget=budget if budget is not None else 10**8)
            results[name] = ("ok", orc.fingerprint_array(res.array), [s.rows for s in rep.steps],
                             [s.prealloc_total for s in rep.steps])
        except ResourceLimitError as exc:
            results[name] = ("ResourceLimitError", str(exc))
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), np.array([results], dtype=object))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_row_partitioned_two_ranks(tmp_path, store_factory):
    from hoststore import HostStore, plan_for
    from oracle import oracle as orc

    store_dir = store_factory("lubm", univ=1, seed=0)
    mp.start_processes(_worker, args=(2, _free_port(), str(store_dir), str(tmp_path)), nprocs=2,
                       join=True, start_method="spawn")
    r0 = np.load(tmp_path / "rank0.npy", allow_pickle=True)[0]
    r1 = np.load(tmp_path / "rank1.npy", allow_pickle=True)[0]
    store = HostStore(store_dir)
    prep = orc.PreparedStore(store.matrices)
    for name, text, budget, mode in CASES:
        q, plan = plan_for(store, text)
        if budget is not None:
            # the same error, raised on every rank, as the whole-store oracle
            # (the reference's rule for the mode: "gpu" = the sequential one)
            with pytest.raises(orc.OracleResourceError) as exc:
                orc.run(prep, [s.pattern for s in plan.steps], q.projection, q.distinct,
                        budget=budget, mode="parallel" if mode == "parallel" else "sequential")
            assert r0[name] == ("ResourceLimitError", str(exc.value)) == r1[name], name
            continue
        rows, srows, spre = orc.run(prep, [s.pattern for s in plan.steps], q.projection,
                                    q.distinct)
        exp = np.asarray(rows, dtype=np.uint32).reshape(len(rows), len(q.projection))
        assert r0[name][0] == "ok"
        assert tuple(r0[name][1]) == orc.fingerprint_array(exp), name
        assert r0[name][2] == srows and r1[name][2] == srows, name
        assert r0[name][3] == spre, name
