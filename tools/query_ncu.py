#!/usr/bin/env python
"""Run one LUBM query repeatedly (target for ncu captures of its kernels).
    python tools/query_ncu.py q09 [--univ 10] [--reps 4]"""
import argparse
import sys
import tempfile
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

import bench  # noqa: E402
import paper_1807_07691_b200 as g  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("query")
    ap.add_argument("--univ", type=int, default=10)
    ap.add_argument("--reps", type=int, default=4)
    args = ap.parse_args()
    with tempfile.TemporaryDirectory() as tmp:
        store = g.load(bench._gen_store(Path(tmp), args.univ, 0), device=0)
        text = dict(bench._queries())[args.query]
        q = g.bind_constants(g.parse_query(text), store.dictionary)
        plan = g.make_plan(q, store.stats)
        for _ in range(args.reps):
            res = g.execute(q, plan, store)
        rep = g.ExecutionReport()
        g.execute(q, plan, store, report=rep)
        print(args.query, len(res), rep.kinds, [s.rows for s in rep.steps], rep.kernels)


if __name__ == "__main__":
    main()
