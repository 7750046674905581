#!/usr/bin/env python
"""Device time of power-law queries (median of 5 after warm-up) on a
generated store: python tools/pl_time.py --triples 100000000"""
import argparse
import statistics
import subprocess
import sys
import tempfile
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
import paper_1807_07691_b200 as g  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--triples", type=int, default=100_000_000)
ap.add_argument("--store", default=None)
ap.add_argument("--only", default=None, help="comma-separated query names")
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
with tempfile.TemporaryDirectory() as tmp:
    sd = args.store
    if not sd:
        sd = f"{tmp}/pl"
        subprocess.run([str(REPO / "oracle/_build/gsmgen"), "powerlaw", "--triples", str(args.triples),
                        "--predicates", "40", "--seed", "0", "--out", sd], check=True, stdout=subprocess.DEVNULL)
    st = g.load(sd)
    for f in sorted((REPO / "datagen/queries/powerlaw").glob("*.rq")):
        if args.only and f.stem not in args.only.split(","):
            continue
        q = g.bind_constants(g.parse_query(f.read_text()), st.dictionary)
        plan = g.make_plan(q, st.stats)
        try:
            g.execute(q, plan, st, row_budget=1 << 62)
        except g.ResourceLimitError:
            print(f.stem, "infeasible")
            continue
        ts = []
        for _ in range(args.reps):
            rep = g.ExecutionReport()
            g.execute(q, plan, st, row_budget=1 << 62, report=rep)
            ts.append(rep.device_seconds)
        print(f.stem, "rows", [s.rows for s in rep.steps], "ms", round(1e3 * statistics.median(ts), 3))
