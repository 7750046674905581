#!/usr/bin/env python
"""Per-block phase timeline of a join kernel (diagnostic; GPU box only).

Loads the trace build of the library (make -C paper_1807_07691_b200/csrc
trace -> libgsmat_b200_trace.so), runs one query on the LUBM store and reads
the %globaltimer stamps thread 0 of every block wrote at the phase
boundaries of its first tiles (gsm_common.cuh trace_at):
  0 prologue done, 1 tile grabbed, 2 count done, 3 scan + publish done,
  4 look-back done (non-window path), 5 tile done, 6 window look-back done
  (round 0's loads in flight), 7 window round 0 stored; (3,7) = block end.
Usage: python tools/trace_probe.py [--query takesCourse_classmates|qNN] [--univ 10]
"""
from __future__ import annotations

import argparse
import ctypes as C
import os
import statistics
import sys
import tempfile
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
os.environ.setdefault("GSM_LIB", str(REPO / "paper_1807_07691_b200/_lib/libgsmat_b200_trace.so"))
sys.path.insert(0, str(REPO))

import bench  # noqa: E402
import paper_1807_07691_b200 as g  # noqa: E402
from paper_1807_07691_b200 import _lib  # noqa: E402

SLOTS = 32


def pct(v, q):
    v = sorted(v)
    return v[min(len(v) - 1, int(q * len(v)))] if v else 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--query", default="takesCourse_classmates")
    ap.add_argument("--univ", type=int, default=10)
    ap.add_argument("--powerlaw", type=int, default=0, help="power-law store of this many triples")
    ap.add_argument("--text", default=None, help="query text (overrides --query)")
    args = ap.parse_args()
    L = _lib.lib()
    L.gsm_trace_dump.argtypes = [C.c_void_p, C.c_int64]
    L.gsm_trace_reset.argtypes = []
    with tempfile.TemporaryDirectory() as tmp:
        if args.powerlaw:
            import subprocess
            sd = Path(tmp) / "pl"
            subprocess.run([str(REPO / "oracle/_build/gsmgen"), "powerlaw", "--triples", str(args.powerlaw),
                            "--predicates", "40", "--seed", "0", "--out", str(sd)], check=True,
                           stdout=subprocess.DEVNULL)
            store = g.load(sd, device=0)
        else:
            store = g.load(bench._gen_store(Path(tmp), args.univ, 0), device=0)
        text = args.text or dict(bench.PROBES).get(args.query) or dict(bench._queries())[args.query]
        q = g.bind_constants(g.parse_query(text), store.dictionary)
        plan = g.make_plan(q, store.stats)
        for _ in range(3):
            g.execute(q, plan, store, row_budget=1 << 62)
        L.gsm_trace_reset()
        rep = g.ExecutionReport()
        g.execute(q, plan, store, row_budget=1 << 62, report=rep)
        n = 8192 * SLOTS * 2
        buf = (C.c_uint64 * n)()
        L.gsm_trace_dump(buf, n)
    print(args.query, "steps", rep.kinds, [s.rows for s in rep.steps],
          "device us", round(rep.device_seconds * 1e6, 1))
    blocks = []
    for b in range(8192):
        base = b * SLOTS * 2
        st = {}
        for s in range(SLOTS):
            gt = buf[base + 2 * s]
            if gt:
                st[s] = gt
        if st:
            blocks.append(st)
    if not blocks:
        print("no stamps")
        return
    t0 = min(min(st.values()) for st in blocks)
    end = max(max(st.values()) for st in blocks)
    print(f"blocks with stamps: {len(blocks)}, span {(end - t0) / 1e3:.2f} us")
    starts = [st.get(0, 0) - t0 for st in blocks if 0 in st]
    ends = [st.get(31, 0) - t0 for st in blocks if 31 in st]
    print(f"block start  us: p10 {pct(starts, .1)/1e3:.2f} p50 {pct(starts, .5)/1e3:.2f} "
          f"p90 {pct(starts, .9)/1e3:.2f} max {max(starts)/1e3:.2f}")
    print(f"block end    us: p10 {pct(ends, .1)/1e3:.2f} p50 {pct(ends, .5)/1e3:.2f} "
          f"p90 {pct(ends, .9)/1e3:.2f} max {max(ends)/1e3:.2f}")
    tiles = [sum(1 for it in range(4) if it * 8 + 1 in st) for st in blocks]
    print("tiles per block:", {k: tiles.count(k) for k in sorted(set(tiles))})
    names = {(1, 2): "count", (2, 3): "scan+publish", (3, 4): "look-back",
             (4, 5): "scatter", (3, 6): "window look-back", (6, 7): "window round 0",
             (7, 5): "window rounds 1+", (3, 5): "look-back+scatter", (1, 5): "tile"}
    for it in range(3):
        rows = []
        for (a, b), nm in names.items():
            d = [st[it * 8 + b] - st[it * 8 + a] for st in blocks
                 if it * 8 + a in st and it * 8 + b in st]
            if d:
                rows.append(f"{nm} p50 {statistics.median(d)/1e3:.2f} p90 {pct(d, .9)/1e3:.2f} "
                            f"max {max(d)/1e3:.2f}")
        gs = [st[it * 8 + 1] - t0 for st in blocks if it * 8 + 1 in st]
        if gs:
            print(f"tile #{it}: grabbed at p50 {statistics.median(gs)/1e3:.2f} us, "
                  f"{len(gs)} blocks | " + " | ".join(rows))
    # active blocks over time (10 buckets)
    nb = 12
    hist = [0] * nb
    for st in blocks:
        a, b = st.get(0), st.get(31)
        if a is None or b is None:
            continue
        for k in range(nb):
            lo = t0 + (end - t0) * k / nb
            hi = t0 + (end - t0) * (k + 1) / nb
            if a < hi and b > lo:
                hist[k] += 1
    print("blocks alive per 1/12 of the span:", hist)


if __name__ == "__main__":
    main()
