#!/usr/bin/env python
"""End-to-end execute_batch time of the bench step (LUBM-10 Q1-Q14, L2
flushed before every call), median over --reps: run under different
GSM_* settings back to back on one box to A/B a host-path change."""
import argparse
import json
import os
import statistics
import sys
import tempfile
import time
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=300)
    ap.add_argument("--store", default=None)
    args = ap.parse_args()
    import torch

    import paper_1807_07691_b200 as g

    with tempfile.TemporaryDirectory() as tmp:
        sd = args.store or bench._gen_store(Path(tmp), 10, 0)
        store = g.load(sd, device=0)
        items = []
        for _, text in bench._queries():
            q = g.bind_constants(g.parse_query(text), store.dictionary)
            items.append((q, g.make_plan(q, store.stats)))
        flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda:0")
        wall, dev = [], []
        for i in range(args.reps + 10):
            flush.add_(1)
            torch.cuda.synchronize()
            bt = []
            t0 = time.perf_counter()
            g.execute_batch(items, store, batch_timing=bt)
            t = time.perf_counter() - t0
            if i >= 10:
                wall.append(t * 1e6)
                dev.append(bt[0] * 1e6)
        env = {k: v for k, v in os.environ.items() if k.startswith(("GSM_", "CUDA_DEVICE_MAX"))}
        print(json.dumps({"env": env, "e2e_us": round(statistics.median(wall), 1),
                          "device_us": round(statistics.median(dev), 1)}))


if __name__ == "__main__":
    main()
