"""Sharded mode (paper_1807_07691_b200/sharded.py): every rank
holds one id-range shard of the store; rows are exchanged by owner between
steps.  Ranks are separate processes sharing the one GPU and exchanging over
gloo (NCCL needs one GPU per rank); the result union, the per-step global
counters and the budget errors must equal the oracle's on the whole store."""

from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import GOLDEN, REPO, lubm_queries

pytestmark = pytest.mark.gpu

UB = "PREFIX ub: <http://swat.cse.lehigh.edu/onto/univ-bench.owl#> "


def _cases():
    cases = [(n, t, None, "gpu") for n, t in lubm_queries()]
    cdir = GOLDEN.parents[1] / "datagen" / "queries" / "lubm_complex"
    cases += [(f.stem, f.read_text(), None, "gpu") for f in sorted(cdir.glob("*.rq"))]
    cases += [
        ("distinct", UB + "SELECT DISTINCT ?d WHERE { ?x ub:memberOf ?d . ?x ub:takesCourse ?c . }",
         None, "gpu"),
        ("distinct2", UB + "SELECT DISTINCT ?c ?d WHERE { ?x ub:memberOf ?d . ?x ub:takesCourse ?c . }",
         None, "gpu"),
        ("cross", UB + "SELECT * WHERE { ?x ub:headOf ?d . ?y ub:subOrganizationOf ?u . }", None, "gpu"),
        ("star", UB + "SELECT * WHERE { ?x ub:memberOf ?d . ?x ub:emailAddress ?e . "
         "?x ub:telephone ?t . }", None, "gpu"),
        ("budget_par", dict(lubm_queries())["q09"], 10, "parallel"),
        ("budget_seq", dict(lubm_queries())["q09"], 10, "sequential"),
        ("budget_cross", UB + "SELECT * WHERE { ?x ub:headOf ?d . ?y ub:subOrganizationOf ?u . }",
         100, "gpu"),
    ]
    return cases


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, store_dir, out_dir):
    sys.path.insert(0, str(REPO))
    sys.path.insert(0, str(REPO / "tests"))
    import torch
    import torch.distributed as dist

    import paper_1807_07691_b200 as g
    from oracle import oracle as orc
    from paper_1807_07691_b200.errors import ResourceLimitError
    from paper_1807_07691_b200.sharded import execute_sharded

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    store = g.load(store_dir, shard=(rank, world))
    results = {}
    for name, text, budget, mode in _cases():
        q = g.bind_constants(g.parse_query(text), store.dictionary)
        plan = g.make_plan(q, store.stats)
        try:
            rep = g.ExecutionReport()
            res = execute_sharded(q, plan, store, mode=mode, report=rep,
                                  row_budget=budget if budget is not None else 1 << 62)
            results[name] = ("ok", [str(x) for x in orc.fingerprint_array(res.array)],
                             [s.rows for s in rep.steps], [s.prealloc_total for s in rep.steps],
                             res.array.shape[0])
        except ResourceLimitError as exc:
            results[name] = ("ResourceLimitError", str(exc))
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), np.array([results], dtype=object))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_union_matches_oracle(tmp_path, store_factory, world):
    from hoststore import HostStore, plan_for
    from oracle import oracle as orc

    store_dir = store_factory("lubm", univ=1, seed=6)
    mp.start_processes(_worker, args=(world, _free_port(), str(store_dir), str(tmp_path)),
                       nprocs=world, join=True, start_method="spawn")
    res = [np.load(tmp_path / f"rank{r}.npy", allow_pickle=True)[0] for r in range(world)]
    store = HostStore(store_dir)
    prep = orc.PreparedStore(store.matrices)
    for name, text, budget, mode in _cases():
        q, plan = plan_for(store, text)
        pats = [s.pattern for s in plan.steps]
        omode = "sequential" if mode == "sequential" else "parallel"
        try:
            rows, srows, spre = orc.run(prep, pats, q.projection, q.distinct,
                                        budget=budget if budget is not None else 1 << 62,
                                        mode=omode)
        except orc.OracleResourceError as exc:
            for r in range(world):
                assert res[r][name][0] == "ResourceLimitError", (name, r, res[r][name])
                assert res[r][name][1] == str(exc), (name, r)
            continue
        exp = np.asarray(rows, dtype=np.uint32).reshape(len(rows), len(q.projection))
        for r in range(world):
            assert res[r][name][0] == "ok", (name, r, res[r][name])
            assert res[r][name][2] == srows, (name, r)
            assert res[r][name][3] == spre, (name, r)
        assert [int(x) for x in res[0][name][1]] == list(orc.fingerprint_array(exp)), name
        assert res[0][name][4] == exp.shape[0], name
