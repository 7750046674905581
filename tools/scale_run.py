#!/usr/bin/env python
"""Scale runs with parity and a CPU baseline: BASELINE.json configs[2]
(LUBM-style U=1000, ~130M triples, complex cyclic / snowflake queries on
1 B200) and the configs[4] power-law model (generate.py, hub-heavy chain
joins) at single-GPU scale (--kind powerlaw --triples N).

For every query of datagen/queries/lubm and datagen/queries/lubm_complex:
  * GPU: warm-up, then median device latency (CUDA events) over --reps runs,
    result rows, join rows, per-step report;
  * parity: the C oracle (oracle/gsm_oracle.c, the reference executor
    restated, 1 core) on the same store — multiset fingerprint (count, sum,
    xor of splitmix64 row hashes) and, when the result has at most
    --exact-rows rows, an exact lexicographic comparison;
  * the oracle's wall time is the CPU baseline at this scale (the Python
    reference needs ~550 MB RAM and ~13 s per million triples to build, so
    it is not run here; SURVEY.md §7 "Oracle at scale").
Row budget is 2^62 in both engines.  One JSON line per query,
then a summary line.  Usage:
    python tools/scale_run.py --univ 1000 [--reps 5] [--skip-oracle-above 400000000]
    python tools/scale_run.py --kind powerlaw --triples 200000000 --predicates 40
    python tools/scale_run.py --kind watdiv --scale 1000      (configs[3], ~104M triples)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))


def summary_run(g, q, plan, store, budget, name, why):
    """execute_summary twice: with the chunk count the executor picks, then
    with twice as many chunks (different slice boundaries, so a dropped or
    doubled row would change the fingerprint)."""
    rep = g.ExecutionReport()
    t0 = time.perf_counter()
    s1 = g.execute_summary(q, plan, store, row_budget=budget, report=rep)
    wall = time.perf_counter() - t0
    rep2 = g.ExecutionReport()
    s2 = g.execute_summary(q, plan, store, row_budget=budget, report=rep2,
                           chunks=max(2, 2 * rep.chunks))
    join = sum(s.rows for s in rep.steps[1:])
    return {"query": name, "mode": "execute_summary (rows not materialised on the host)",
            "why": why, "rows": s1.rows, "fingerprint": [s1.rows, s1.sum, s1.xor],
            "chunks": rep.chunks, "step_rows": [s.rows for s in rep.steps],
            "step_prealloc": [s.prealloc_total for s in rep.steps], "kinds": rep.kinds,
            "gpu_ms": round(1e3 * rep.device_seconds, 3), "wall_s": round(wall, 3),
            "join_rows": join, "join_rows_per_s": round(join / max(rep.device_seconds, 1e-9), 1),
            "rechunked": {"chunks": rep2.chunks, "same_fingerprint": s2.fingerprint == s1.fingerprint,
                          "same_step_rows": [s.rows for s in rep2.steps] == [s.rows for s in rep.steps]},
            "parity": "oracle not run (intermediate beyond host RAM); see the reduced-store "
                      "chunked parity in tests/test_gpu_chunked.py"}


def degree_stats(store_dir, np, top=4):
    """Largest out/in degree of the biggest predicates (the hub sizes the
    skew produces; SURVEY.md §8(d) T4 asks for hubs of 1e5-1e6)."""
    d = Path(store_dir)
    sizes = sorted(((f.stat().st_size, f) for f in d.glob("p*.so")), reverse=True)[:top]
    out = {}
    for _, f in sizes:
        pid = f.stem
        for ext, what in (("so", "max_out"), ("os", "max_in")):
            keys = np.fromfile(d / f"{pid}.{ext}", dtype="<u8")[0::2]
            if keys.size:
                b = np.flatnonzero(np.diff(keys)) + 1
                runs = np.diff(np.concatenate(([0], b, [keys.size])))
                out.setdefault(pid, {"pairs": int(keys.size)})[what] = int(runs.max())
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", choices=["lubm", "powerlaw", "watdiv"], default="lubm")
    ap.add_argument("--scale", type=int, default=1000, help="watdiv scale (1000 ~ 100M triples)")
    ap.add_argument("--univ", type=int, default=1000)
    ap.add_argument("--triples", type=int, default=100_000_000)
    ap.add_argument("--predicates", type=int, default=40)
    ap.add_argument("--node-skew", type=float, default=0.5,
                    help="powerlaw endpoint exponent (generate.py NODE_SKEW; T4 uses 0.9)")
    ap.add_argument("--qdir", default=None,
                    help="query directory under datagen/queries (default: the kind's own)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--exact-rows", type=int, default=20_000_000)
    ap.add_argument("--skip-oracle-above", type=int, default=400_000_000,
                    help="skip the oracle when a step materialises more rows (host RAM guard)")
    ap.add_argument("--store", default=None, help="reuse an existing store directory")
    ap.add_argument("--only", default=None, help="comma-separated query names to run")
    ap.add_argument("--summary", default="",
                    help="comma-separated query names evaluated by execute_summary only (results "
                         "larger than host memory)")
    args = ap.parse_args()

    import numpy as np

    import paper_1807_07691_b200 as g
    from oracle import oracle as orc

    import bench

    peak = bench._peaks()[0].get("hbm_gbs", 6650.0)

    subprocess.run(["make", "-s", "-C", str(REPO / "oracle")], check=True)
    tmp = tempfile.mkdtemp(prefix="gsm_scale_")
    store_dir = args.store or f"{tmp}/{args.kind}"
    t0 = time.perf_counter()
    if not args.store or not Path(args.store, "meta").exists():  # --store DIR: generated once
        gen = [str(REPO / "oracle/_build/gsmgen"), args.kind, "--seed", str(args.seed),
               "--out", store_dir]
        if args.kind == "lubm":
            gen += ["--univ", str(args.univ)]
        elif args.kind == "watdiv":
            gen += ["--scale", str(args.scale)]
        else:  # generate.py's model (Zipf predicates, i^-0.5 endpoints, nodes = triples/4)
            gen += ["--triples", str(args.triples), "--predicates", str(args.predicates),
                    "--node-skew", str(args.node_skew)]
        subprocess.run(gen, check=True, stdout=subprocess.DEVNULL)
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    store = g.load(store_dir)
    t_load = time.perf_counter() - t0
    print(json.dumps({"store": store_dir, "triples": store.triple_count,
                      "nodes": store.node_count, "gen_s": round(t_gen, 1),
                      "load_s": round(t_load, 2), "device_bytes": store.device_bytes()}),
          flush=True)
    prep = orc.PreparedStore(store.matrices)
    if args.kind == "powerlaw":
        print(json.dumps({"degrees": degree_stats(store_dir, np)}), flush=True)
    if args.qdir:
        qfiles = sorted((REPO / "datagen/queries" / args.qdir).glob("*.rq"))
    elif args.kind == "lubm":
        qfiles = sorted((REPO / "datagen/queries/lubm").glob("*.rq")) + \
            sorted((REPO / "datagen/queries/lubm_complex").glob("*.rq"))
    else:
        qfiles = sorted((REPO / f"datagen/queries/{args.kind}").glob("*.rq"))
    summary = {"gpu_ms": 0.0, "cpu_s": 0.0, "join_rows": 0, "parity_ok": 0, "parity_checked": 0}
    if args.only:
        keep = set(args.only.split(","))
        qfiles = [f for f in qfiles if f.stem in keep]
    for qf in qfiles:
        q = g.bind_constants(g.parse_query(qf.read_text()), store.dictionary)
        plan = g.make_plan(q, store.stats)
        budget = 1 << 62
        if qf.stem in set(args.summary.split(",")):
            print(json.dumps(summary_run(g, q, plan, store, budget, qf.stem, "--summary")), flush=True)
            summary["summary_only"] = summary.get("summary_only", 0) + 1
            continue
        try:
            res = g.execute(q, plan, store, row_budget=budget)
        except g.ResourceLimitError as e:
            # the rows do not fit host memory: count + fingerprint on the
            # device, the plan in left-row chunks where its intermediates
            # exceed device memory
            print(json.dumps(summary_run(g, q, plan, store, budget, qf.stem, str(e))), flush=True)
            summary["summary_only"] = summary.get("summary_only", 0) + 1
            continue
        dev = []
        rep = None
        for _ in range(args.reps):
            rep = g.ExecutionReport()
            g.execute(q, plan, store, row_budget=budget, report=rep)
            dev.append(rep.device_seconds)
        rec = {"query": qf.stem, "rows": len(res), "step_rows": [s.rows for s in rep.steps],
               "step_prealloc": [s.prealloc_total for s in rep.steps], "kinds": rep.kinds,
               "gpu_ms": round(1e3 * statistics.median(dev), 3),
               "join_rows": sum(s.rows for s in rep.steps[1:])}
        if rep.chunks:
            rec["chunks"] = rep.chunks
        rec["join_rows_per_s"] = round(rec["join_rows"] / statistics.median(dev), 1)
        # HBM roofline of the whole query: algorithmic bytes of its join steps
        # (bench._step_bytes) / device time
        # (fused intermediates are not billed: bench.query_bytes)
        qbytes = bench.query_bytes(rep, len(q.projection))
        gbps = qbytes / statistics.median(dev) / 1e9
        rec["bytes"] = int(qbytes)
        rec["achieved_GBps"] = round(gbps, 1)
        rec["hbm_frac"] = round(gbps / peak, 4)
        if max(rec["step_rows"]) <= args.skip_oracle_above:
            t0 = time.perf_counter()
            rows, srows, spre = orc.run(prep, [s.pattern for s in plan.steps], q.projection,
                                        q.distinct, budget=budget)
            rec["cpu_oracle_s"] = round(time.perf_counter() - t0, 3)
            exp = np.asarray(rows, dtype=np.uint32).reshape(len(rows), len(q.projection))
            del rows
            ok = orc.fingerprint_array(exp) == orc.fingerprint_array(res.array)
            ok = ok and srows == rec["step_rows"] and spre == rec["step_prealloc"]
            if ok and len(res) <= args.exact_rows and exp.shape[1]:
                a = res.array[np.lexsort(res.array.T[::-1])]
                b = exp[np.lexsort(exp.T[::-1])]
                ok = bool(np.array_equal(a, b))
                rec["exact_compare"] = True
            rec["parity"] = bool(ok)
            summary["parity_checked"] += 1
            summary["parity_ok"] += int(ok)
            summary["cpu_s"] += rec["cpu_oracle_s"]
        else:
            rec["parity"] = "skipped (host RAM guard)"
        summary["gpu_ms"] += rec["gpu_ms"]
        summary["join_rows"] += rec["join_rows"]
        print(json.dumps(rec), flush=True)
    print(json.dumps({"summary": summary}), flush=True)
    if not args.store:
        subprocess.run(["rm", "-rf", tmp])


if __name__ == "__main__":
    main()
