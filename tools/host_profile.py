#!/usr/bin/env python
"""Host-side cost of the public batch API on the bench workload (LUBM-10
Q1-Q14): cProfile of repeated execute_batch() calls (no L2 flush, so the
device part is as short as it gets) and the split between the C call
(gsm_execute_batch) and the Python around it.  GPU box only."""
import cProfile
import pstats
import sys
import tempfile
import time
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

import bench  # noqa: E402
import paper_1807_07691_b200 as g  # noqa: E402


def main():
    with tempfile.TemporaryDirectory() as tmp:
        store = g.load(bench._gen_store(Path(tmp), 10, 0), device=0)
        items = []
        for _, text in bench._queries():
            q = g.bind_constants(g.parse_query(text), store.dictionary)
            items.append((q, g.make_plan(q, store.stats)))
        for _ in range(20):
            g.execute_batch(items, store)
        n = 500
        t0 = time.perf_counter()
        for _ in range(n):
            g.execute_batch(items, store)
        wall = (time.perf_counter() - t0) / n
        bt = []
        for _ in range(n):
            g.execute_batch(items, store, batch_timing=bt)
        print(f"execute_batch wall {wall * 1e6:.1f} us, device {1e6 * sum(bt) / len(bt):.1f} us")
        pr = cProfile.Profile()
        pr.enable()
        for _ in range(n):
            g.execute_batch(items, store)
        pr.disable()
        pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
