#!/usr/bin/env python
"""Per-query latency breakdown on the GPU (diagnostic, not the bench).

For every LUBM query: median wall time of the public execute() (with and
without a report), of the bare C call (gsm_execute + copy, plan already
encoded), and the device time the library measured (CUDA events), plus the
per-step device times.  Usage: python tools/latency_probe.py [--univ 10] [--reps 50]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--univ", type=int, default=10)
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    import numpy as np

    import paper_1807_07691_b200 as g
    from paper_1807_07691_b200 import _lib
    from paper_1807_07691_b200.executor import compile_plan

    with tempfile.TemporaryDirectory() as tmp:
        subprocess.run([str(REPO / "oracle/_build/gsmgen"), "lubm", "--univ", str(args.univ),
                        "--out", f"{tmp}/s"], check=True, stdout=subprocess.DEVNULL)
        store = g.load(f"{tmp}/s")
        L = _lib.lib()
        out = {}
        for f in sorted((REPO / "datagen/queries/lubm").glob("*.rq")):
            q = g.bind_constants(g.parse_query(f.read_text()), store.dictionary)
            plan = g.make_plan(q, store.stats)
            for _ in range(5):
                g.execute(q, plan, store)
            t_full, t_rep, t_c, dev, steps = [], [], [], [], []
            for _ in range(args.reps):
                t0 = time.perf_counter()
                g.execute(q, plan, store)
                t_full.append(time.perf_counter() - t0)
                rep = g.ExecutionReport()
                t0 = time.perf_counter()
                g.execute(q, plan, store, report=rep)
                t_rep.append(time.perf_counter() - t0)
                dev.append(rep.device_seconds)
                steps.append([s.seconds for s in rep.steps])
            _, arr, proj, k = compile_plan(q, plan)
            ctx = store.context()
            for _ in range(args.reps):
                res = C.c_void_p()
                t0 = time.perf_counter()
                _lib.check(L.gsm_execute(ctx, arr, len(plan.steps), proj, k, int(q.distinct),
                                         10**8, 1, 0, 1, None, C.byref(res)))
                n = C.c_int64()
                kk = C.c_int32()
                L.gsm_result_shape(res, C.byref(n), C.byref(kk))
                buf = np.empty((n.value, kk.value), np.uint32)
                if buf.size:
                    L.gsm_result_copy(res, buf.ctypes.data)
                L.gsm_result_free(res)
                t_c.append(time.perf_counter() - t0)
            med = lambda x: round(1e6 * statistics.median(x), 1)  # noqa: E731
            out[f.stem] = {"execute_us": med(t_full), "execute_report_us": med(t_rep),
                           "c_call_us": med(t_c), "device_us": med(dev),
                           "steps_device_us": [round(1e6 * statistics.median(c), 1) for c in zip(*steps)],
                           "kinds": rep.kinds, "rows": [s.rows for s in rep.steps]}
            print(f.stem, json.dumps(out[f.stem]), flush=True)
        print(json.dumps(out))


if __name__ == "__main__":
    main()
