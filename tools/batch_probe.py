#!/usr/bin/env python
"""Where the batched LUBM step's device time goes (diagnostic; GPU box).

Runs execute_batch over subsets of Q1-Q14 on the bench store (LUBM U=10),
L2 flushed before every batch, and prints the median device time of each
subset next to the single-query latencies: the gap between the batch and
its slowest member is the cost of running the members concurrently.
Usage: python tools/batch_probe.py [--reps 30]
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
import tempfile
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--univ", type=int, default=10)
    args = ap.parse_args()
    import torch

    import paper_1807_07691_b200 as g

    with tempfile.TemporaryDirectory() as tmp:
        store = g.load(bench._gen_store(Path(tmp), args.univ, 0), device=0)
        qs = {}
        for name, text in bench._queries():
            q = g.bind_constants(g.parse_query(text), store.dictionary)
            qs[name] = (q, g.make_plan(q, store.stats))
        flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda:0")

        def timed(names):
            items = [qs[n] for n in names]
            out = []
            for i in range(args.reps + 3):
                flush.add_(1)
                torch.cuda.synchronize()
                bt = []
                g.execute_batch(items, store, batch_timing=bt)
                if i >= 3:
                    out.append(bt[0] * 1e6)
            return round(statistics.median(out), 1)

        names = sorted(qs)
        single = {n: timed([n]) for n in names}
        heavy = sorted(names, key=lambda n: -single[n])[:3]
        light = [n for n in names if n not in heavy]
        res = {"single_us": single, "all": timed(names), "heavy": heavy,
               "heavy_only": timed(heavy), "light_only": timed(light),
               "all_minus_slowest": timed([n for n in names if n != heavy[0]])}
        for h in heavy:
            res[f"{h}+light"] = timed([h] + light)
        # store-sized kernels only: the two slowest alone, twice each
        res["slowest_x2"] = timed([heavy[0], heavy[0]])
        res["slowest_x4"] = timed([heavy[0]] * 4)
        res["light_x2"] = timed(light + light)
        print(json.dumps(res))


if __name__ == "__main__":
    main()
