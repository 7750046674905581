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
        # split: the C call vs the Python around it
        from paper_1807_07691_b200 import _lib
        L = _lib.lib()
        acc = {}
        for name in ("gsm_execute_batch_into", "gsm_result_copy", "gsm_result_free"):
            f = getattr(L, name)

            def wrap(*a, _f=f, _n=name):
                t = time.perf_counter()
                r = _f(*a)
                acc[_n] = acc.get(_n, 0.0) + time.perf_counter() - t
                return r
            setattr(L, name, wrap)
        t0 = time.perf_counter()
        for _ in range(n):
            g.execute_batch(items, store)
        wall = (time.perf_counter() - t0) / n
        print(f"wrapped: wall {wall * 1e6:.1f} us; " +
              ", ".join(f"{k} {v / n * 1e6:.1f} us" for k, v in acc.items()))
        for name in list(acc):
            delattr(L, name) if name in L.__dict__ else None
        # per-query step breakdown (device events inside the library)
        for (q, plan), (qn, _) in zip(items, bench._queries()):
            ms = []
            for _ in range(20):
                rep = g.ExecutionReport()
                g.execute(q, plan, store, report=rep)
                ms.append(rep)
            rep = ms[-1]
            print(qn, f"{rep.device_seconds * 1e6:.1f} us",
                  [(k, s.rows, round(s.seconds * 1e6, 1)) for k, s in zip(rep.kinds, rep.steps)],
                  "kernels", rep.kernels)
        pr = cProfile.Profile()
        pr.enable()
        for _ in range(n):
            g.execute_batch(items, store)
        pr.disable()
        pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
