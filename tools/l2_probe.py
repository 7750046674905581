#!/usr/bin/env python
"""How much of the small-query latency is cold DRAM (diagnostic, not the bench).

LUBM-U Q1-Q14: device time of every query (a one-query execute_batch) and of
the 14-query batch, (cold) right after a 256 MB L2 flush and (warm) right
after the same call ran, medians over --reps.  With GSM_L2_PREFETCH toggled
by the caller this A/Bs the plan-level L2 prefetch branch.
Usage: python tools/l2_probe.py [--univ 10] [--reps 30]
"""
from __future__ import annotations

import argparse
import json
import statistics
import subprocess
import sys
import tempfile
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--univ", type=int, default=10)
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--label", default="")
    args = ap.parse_args()
    import torch

    import paper_1807_07691_b200 as g

    with tempfile.TemporaryDirectory() as tmp:
        subprocess.run([str(REPO / "oracle/_build/gsmgen"), "lubm", "--univ", str(args.univ),
                        "--out", f"{tmp}/s"], check=True, stdout=subprocess.DEVNULL)
        store = g.load(f"{tmp}/s")
    items = []
    for f in sorted((REPO / "datagen/queries/lubm").glob("*.rq")):
        q = g.bind_constants(g.parse_query(f.read_text()), store.dictionary)
        items.append((f.stem, q, g.make_plan(q, store.stats)))
    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda:0")

    def timed(batch, cold):
        if cold:
            flush.add_(1)
            torch.cuda.synchronize()
        bt = []
        g.execute_batch(batch, store, batch_timing=bt)
        return 1e3 * bt[0]

    out = {"label": args.label, "univ": args.univ, "cold": {}, "warm": {}}
    for name, q, plan in items + [("batch", None, None)]:
        batch = [(q, plan)] if q is not None else [(q, p) for _, q, p in items]
        for _ in range(3):
            timed(batch, True)
        cold = [timed(batch, True) for _ in range(args.reps)]
        warm = []
        for _ in range(args.reps):
            warm.append(timed(batch, False))
        out["cold"][name] = round(statistics.median(cold), 4)
        out["warm"][name] = round(statistics.median(warm), 4)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
