#!/usr/bin/env python
"""Diagnostic: kernels per replay and device time of one query run repeatedly
on one context (capture -> hinted re-capture -> warm replays without k_init),
with and without an L2 flush before each run."""
import statistics
import sys
import tempfile
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
import bench  # noqa: E402


def main():
    import torch

    import paper_1807_07691_b200 as g

    with tempfile.TemporaryDirectory() as tmp:
        store = g.load(bench._gen_store(Path(tmp), 10, 0), device=0)
        flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda:0")
        for name, text in bench._queries():
            if name not in ("q01", "q06", "q08", "q09"):
                continue
            q = g.bind_constants(g.parse_query(text), store.dictionary)
            plan = g.make_plan(q, store.stats)
            ks, ts = [], []
            for i in range(40):
                flush.add_(1)
                torch.cuda.synchronize()
                bt = []
                rep = g.ExecutionReport()
                g.execute_batch([(q, plan)], store, reports=[rep], batch_timing=bt)
                ks.append(rep.kernels)
                ts.append(bt[0] * 1e6)
            print(name, "kernels", ks[:5], "...", ks[-1], "us first", [round(t, 1) for t in ts[:4]],
                  "median later", round(statistics.median(ts[5:]), 1))


if __name__ == "__main__":
    main()
