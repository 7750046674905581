#!/usr/bin/env python
"""Benchmark: LUBM-style query latency and join output rows/s on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--univ U] [--seed S]

Workload (BASELINE.json configs[1]): LUBM-style synthetic store at scale U
(default 10, ~1.38M triples, datagen/gsmgen) and queries Q1-Q14
(datagen/queries/lubm, plain BGPs).  One "step" = the 14 queries executed
once, each through the public drop-in API
(``paper_1807_07691_b200.execute``), with L2 flushed before every step (the
store is smaller than the 126 MB L2).

* value          join output rows / s (sum over join steps of StepReport.rows,
                 SURVEY.md §8(d)), device time (CUDA events around each query
                 inside the library), whole job over all ranks
* e2e            the same through execute() as a user calls it: host-side plan
                 encoding, H2D of the query block from pinned memory, kernels,
                 D2H of the result rows into host numpy arrays (wall clock)
* roofline       dominant kernel class (join kernel), algorithmic bytes per
                 SURVEY.md §8(d) / its measured event time vs MEASURED_PEAKS.json
* cpu_baseline   the C oracle port (oracle/gsm_oracle.c, 1 core) on the same
                 queries, bounded sample
* --impl reference  the unmodified reference package (oracle/_ref) on the host
                 cores, mode="parallel", worker_count=os.cpu_count()

Multi-GPU (torchrun): every rank holds a replica of the store and serves its
own copy of the query stream (weak scaling, no data-path collective); timing
is the max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))

QDIR = REPO / "datagen" / "queries" / "lubm"
W_ID = 4  # bytes per id


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--univ", type=int, default=10)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-probe", action="store_true")
    ap.add_argument("--only-probe", action="store_true", help="run only the kernel probe (ncu)")
    ap.add_argument("--probe", default=None, help="with --only-probe: run just this probe")
    return ap.parse_args()


# Kernel-at-scale probe on the same store: self-joins whose expand step writes
# tens of millions of rows, so the join kernel's HBM roofline is measured
# where bandwidth (not launch latency) decides.  Not part of `value`.
# SELECT * keeps the written bytes equal to the expand's full output (a+1
# columns) whether or not the projection is fused into the kernel.
PROBES = [
    ("memberOf_coworkers", "PREFIX ub: <http://swat.cse.lehigh.edu/onto/univ-bench.owl#> "
     "SELECT * WHERE { ?x ub:memberOf ?d . ?y ub:memberOf ?d . }"),
    ("takesCourse_classmates", "PREFIX ub: <http://swat.cse.lehigh.edu/onto/univ-bench.owl#> "
     "SELECT * WHERE { ?x ub:takesCourse ?c . ?y ub:takesCourse ?c . }"),
]


def run_probe(g, store, peaks, reps=5, only=None):
    out = {}
    for name, text in PROBES:
        if only and name != only:
            continue
        q = g.bind_constants(g.parse_query(text), store.dictionary)
        plan = g.make_plan(q, store.stats)
        best = None
        # one untimed run first: it sizes the arena / result buffer, so the
        # timed runs are the steady state (with the projection fused when it is)
        g.execute(q, plan, store, report=g.ExecutionReport(), row_budget=1 << 62)
        for _ in range(reps):
            rep = g.ExecutionReport()
            g.execute(q, plan, store, report=rep, row_budget=1 << 62)
            st = rep.steps[1]
            L, a = rep.steps[0].rows, rep.arities[0]
            b = _step_bytes(rep.kinds[1], L, a, st.prealloc_total, st.rows, rep.arities[1])
            if best is None or st.seconds < best[1]:
                best = (b, st.seconds, st.rows, rep.kinds[1])
        gbs = best[0] / best[1] / 1e9
        out[name] = {"kernel": f"k_tilescan<{best[3]}>", "rows_out": best[2],
                     "bytes": best[0], "us": round(1e6 * best[1], 1), "achieved_GBps": round(gbs, 1),
                     "frac": round(gbs / peaks["hbm_gbs"], 4)}
    return out


def _dist():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _ensure_built():
    lib = REPO / "paper_1807_07691_b200" / "_lib" / "libgsmat_b200.so"
    if not lib.exists():
        subprocess.run(["make", "-s", "-C", str(REPO / "paper_1807_07691_b200" / "csrc")], check=True)
    subprocess.run(["make", "-s", "-C", str(REPO / "oracle")], check=True)


def _gen_store(tmp: Path, univ: int, seed: int) -> Path:
    out = tmp / f"lubm{univ}"
    subprocess.run([str(REPO / "oracle" / "_build" / "gsmgen"), "lubm", "--univ", str(univ),
                    "--seed", str(seed), "--out", str(out)], check=True, stdout=subprocess.DEVNULL)
    return out


def _queries():
    return [(f.stem, f.read_text()) for f in sorted(QDIR.glob("*.rq"))]


def _peaks():
    try:
        return json.loads((REPO / "MEASURED_PEAKS.json").read_text()), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples: list[list[str]] = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(s[0]) for s in self.samples if len(s) >= 6 and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) >= 6 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples if len(s) >= 6
                          for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def _join_rows(rep_steps) -> int:
    return sum(s.rows for s in rep_steps[1:])


def _step_bytes(kind: str, L: int, a: int, E: int, O: int, out_a: int) -> int:
    """Algorithmic HBM bytes of one join step."""
    if kind == "expand":
        return W_ID * L * a + 16 * L + W_ID * E + W_ID * O * out_a
    if kind == "filter":
        return W_ID * L * a + 16 * L + W_ID * L + W_ID * O * out_a
    if kind == "cross":
        return W_ID * O * out_a  # reads are O(|L|+|R|), dominated by the write
    return 0


def run_ours(args):
    import numpy as np
    import torch

    rank, world, local = _dist()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    import paper_1807_07691_b200 as g
    from paper_1807_07691_b200 import _lib

    with tempfile.TemporaryDirectory() as tmp:
        store_dir = _gen_store(Path(tmp), args.univ, args.seed)
        store = g.load(store_dir, device=local)
        queries = []
        for name, text in _queries():
            q = g.bind_constants(g.parse_query(text), store.dictionary)
            queries.append((name, q, g.make_plan(q, store.stats)))
        triples = store.triple_count
        flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=f"cuda:{local}")  # 256 MB > L2
        if args.only_probe:
            print(json.dumps(run_probe(g, store, _peaks()[0], reps=5, only=args.probe)))
            return

        items = [(q, plan) for _, q, plan in queries]

        def one_step(collect):
            """One step = the 14 queries, three passes, each after an L2 flush:
            (A) one by one with a report: per-query device latency (CUDA
                events inside the library), step counters, per-kernel times;
            (B) one by one exactly as a user calls execute() (no report), wall
                clock incl. H2D of the query block and D2H of the result rows;
            (C) the same 14 queries as one execute_batch() call (concurrent
                streams): device time (events) and wall clock;
            (D) one by one again, each as a one-query execute_batch() whose
                device time is taken around the whole launch sequence only
                (no per-step events): the per-query latency."""
            flush.add_(1)
            torch.cuda.synchronize()
            per_q = []
            for name, q, plan in queries:
                rep = g.ExecutionReport()
                res = g.execute(q, plan, store, report=rep)
                per_q.append((name, rep, len(res)))
            flush.add_(1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for name, q, plan in queries:
                g.execute(q, plan, store)
            wall_seq = time.perf_counter() - t0
            flush.add_(1)
            torch.cuda.synchronize()
            bt = []
            t0 = time.perf_counter()
            g.execute_batch(items, store, batch_timing=bt)
            wall_batch = time.perf_counter() - t0
            flush.add_(1)
            torch.cuda.synchronize()
            lat_q = {}
            for name, q, plan in queries:
                one = []
                g.execute_batch([(q, plan)], store, batch_timing=one)
                lat_q[name] = one[0]
            return {"per_q": per_q, "wall_seq": wall_seq, "wall_batch": wall_batch,
                    "dev_batch": bt[0], "lat": lat_q}

        clk = ClockSampler(local).__enter__()  # sampling starts before warm-up (nvidia-smi start-up)
        time.sleep(0.5)
        for _ in range(max(3, args.warmup)):
            one_step(False)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        launches0 = _lib.kernel_launches()
        steps = []
        n_before = len(clk.samples)
        for _ in range(args.steps):
            steps.append(one_step(True))
        torch.cuda.synchronize()
        time.sleep(0.25)
        clk.__exit__(None, None, None)
        if len(clk.samples) - n_before >= 3:
            clk.samples = clk.samples[n_before:]
        if world > 1:
            torch.distributed.barrier()
        launches = _lib.kernel_launches() - launches0

        all_q = [x for st_ in steps for x in st_["per_q"]]
        dev_seq = sum(sum(st_["lat"].values()) for st_ in steps)
        dev_s = sum(st_["dev_batch"] for st_ in steps)
        wall_seq = sum(st_["wall_seq"] for st_ in steps)
        wall_s = sum(st_["wall_batch"] for st_ in steps)
        rows = sum(_join_rows(rep.steps) for _, rep, _ in all_q)
        delta = sum(rep.intermediate_total for _, rep, _ in all_q)
        h2d = sum(rep.h2d_bytes for _, rep, _ in all_q) / args.steps
        d2h = sum(rep.d2h_bytes for _, rep, _ in all_q) / args.steps

        # roofline per kernel class from the per-step device events
        cls: dict[str, list[float]] = {}
        for _, rep, _ in all_q:
            for i in range(1, len(rep.steps)):
                k = rep.kinds[i]
                if k not in ("expand", "filter", "cross"):
                    continue
                L = rep.steps[i - 1].rows
                a = rep.arities[i - 1]
                b = _step_bytes(k, L, a, rep.steps[i].prealloc_total, rep.steps[i].rows,
                                rep.arities[i])
                c = cls.setdefault(k, [0.0, 0.0, 0])
                c[0] += b
                c[1] += rep.steps[i].seconds
                c[2] += 1

        lat = {}
        for name, *_ in queries:
            lat[name] = round(1e3 * statistics.median(st_["lat"][name] for st_ in steps), 4)

        if world > 1:
            t = torch.tensor([dev_s, wall_s, dev_seq, wall_seq], dtype=torch.float64,
                             device=f"cuda:{local}")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            r = torch.tensor([rows], dtype=torch.float64, device=f"cuda:{local}")
            torch.distributed.all_reduce(r)
            dev_s, wall_s, dev_seq, wall_seq = (float(x) for x in t)
            rows_all = float(r[0])
        else:
            rows_all = float(rows)

        if rank != 0:
            torch.distributed.destroy_process_group()
            return
        peaks, peak_kind = _peaks()
        # The join kernels (k_tilescan for single steps, k_group for fused
        # [filter][expand][filter] groups) are one tile-scan machine; fused
        # steps report their group's time on the group's first step, so the
        # roofline is taken over all join steps together.
        roof = None
        if cls:
            tb = sum(v[0] for v in cls.values())
            tt = sum(v[1] for v in cls.values())
            nl = sum(v[2] for v in cls.values())
            achieved = tb / tt / 1e9 if tt > 0 else 0.0
            traffic = None
            tp = REPO / "profiles" / "ncu_traffic.json"
            if tp.exists():
                try:
                    tj = json.loads(tp.read_text())
                    traffic = tj.get("join", tj.get("filter"))
                except Exception:
                    traffic = None
            roof = {"bound": "hbm", "kernel": "join kernels (k_tilescan / k_group)",
                    "achieved": round(achieved, 2), "peak": peaks["hbm_gbs"],
                    "peak_source": peak_kind, "unit": "GB/s",
                    "frac": round(achieved / peaks["hbm_gbs"], 5), "traffic": traffic,
                    "steps": nl, "bytes_per_step": int(tb / max(1, nl)),
                    "us_per_step": round(1e6 * tt / max(1, nl), 3),
                    "classes": {k: {"bytes": int(v[0]), "steps": v[2], "ms": round(1e3 * v[1], 3)}
                                for k, v in cls.items()}}

        probe = None
        if not args.no_probe:
            # (a) as a user runs it: the projection is fused into the expand,
            #     which writes the row-major result directly;
            # (b) the expand kernel alone writing columnar binding tables (as
            #     for every non-final step): a subprocess with projection
            #     fusion off, timing only the expand step.
            probe = {"fused_projection": run_probe(g, store, peaks)}
            env = dict(os.environ, GSM_NO_PROJ_FUSION="1")
            out = subprocess.run([sys.executable, str(REPO / "bench.py"), "--only-probe",
                                  "--univ", str(args.univ), "--seed", str(args.seed)],
                                 env=env, capture_output=True, text=True)
            try:
                probe["expand_kernel_columnar"] = json.loads(out.stdout.strip().splitlines()[-1])
            except Exception:
                probe["expand_kernel_columnar"] = {"error": out.stderr[-400:]}
        cpu = None
        if not args.no_cpu_baseline and world == 1:  # the CPU baseline is an N=1 measurement
            cpu = cpu_baseline_port(store, queries, args.cpu_seconds)

        value = rows_all / dev_s if dev_s > 0 else 0.0
        line = {
            "metric": "LUBM-style join output rows/sec (per-query latency in latency_ms)",
            "value": round(value, 1),
            "unit": "rows/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": max(3, args.warmup),
            "ms_per_step": round(1e3 * dev_s / args.steps, 4),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "u32",
            "data": "synthetic (datagen/gsmgen lubm, seeded)",
            "config": {"workload": f"LUBM-style U={args.univ} ({triples} triples), Q1-Q14 "
                                   "(datagen/queries/lubm), one step = 14 queries "
                                   "(executed concurrently via execute_batch)",
                       "univ": args.univ, "seed": args.seed, "triples": triples,
                       "l2": "flushed before every step (256 MB write)",
                       "parallelism": f"replica x{world}"},
            "e2e": {"value": round(rows_all / wall_s, 1) if wall_s > 0 else 0.0, "unit": "rows/s",
                    "ms_per_step": round(1e3 * wall_s / args.steps, 4),
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
            "sequential": {"value": round(rows_all / dev_seq, 1) if dev_seq > 0 else 0.0,
                           "ms_per_step": round(1e3 * dev_seq / args.steps, 4),
                           "e2e": round(rows_all / wall_seq, 1) if wall_seq > 0 else 0.0,
                           "e2e_ms_per_step": round(1e3 * wall_seq / args.steps, 4),
                           "note": "queries one at a time (value/e2e above: the step's 14 "
                                   "queries as one execute_batch call on 14 streams)"},
            "latency_ms": lat,
            "join_rows_per_step": rows // args.steps,
            "intermediate_rows_per_step": delta // args.steps,
            "roofline": roof,
            "roofline_probe": probe,
            "cpu_baseline": cpu,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
        if world > 1:
            torch.distributed.destroy_process_group()


def cpu_baseline_port(store, queries, seconds):
    """The C oracle (single-threaded restatement of the reference executor)."""
    from oracle import oracle as orc

    prep = orc.PreparedStore(store.matrices)
    rows = 0
    passes = 0
    t0 = time.perf_counter()
    while True:
        for name, q, plan in queries:
            _, srows, _ = orc.run(prep, [s.pattern for s in plan.steps], q.projection, q.distinct)
            rows += sum(srows[1:])
        passes += 1
        el = time.perf_counter() - t0
        if el >= seconds or passes >= 1000:
            break
    return {"value": round(rows / el, 1), "unit": "rows/s", "cores": 1, "kind": "port",
            "sample": f"{passes} passes of Q1-Q14 on the same store ({el:.1f} s, C oracle)"}


def run_reference(args):
    rank, world, local = _dist()
    if rank != 0:
        return
    ref = REPO / "oracle" / "_ref"
    if ref.exists() and str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        from gsmat import executor, planner, qparser, storage
    except Exception as exc:  # the reference package is not installed: time the C port
        print(json.dumps({"impl": "reference", "unavailable": f"reference not importable: {exc}"}))
        return
    cores = os.cpu_count() or 1
    with tempfile.TemporaryDirectory() as tmp:
        store_dir = _gen_store(Path(tmp), args.univ, args.seed)
        store = storage.load(store_dir)
        queries = []
        for name, text in _queries():
            q = qparser.bind_constants(qparser.parse_query(text), store.dictionary)
            queries.append((name, q, planner.make_plan(q, store.stats)))

        def one_step():
            rows = 0
            t0 = time.perf_counter()
            lat = {}
            for name, q, plan in queries:
                rep = executor.ExecutionReport()
                tq = time.perf_counter()
                executor.execute(q, plan, store, mode="parallel", worker_count=cores,
                                 row_budget=1 << 62, report=rep)
                lat[name] = time.perf_counter() - tq
                rows += sum(s.rows for s in rep.steps[1:])
            return time.perf_counter() - t0, rows, lat

        for _ in range(max(3, args.warmup)):
            one_step()
        res = [one_step() for _ in range(args.steps)]
        el = sum(r[0] for r in res)
        rows = sum(r[1] for r in res)
        value = rows / el
        lat = {n: round(1e3 * statistics.median(r[2][n] for r in res), 3) for n, *_ in queries}
        print(json.dumps({
            "impl": "reference",
            "metric": "LUBM-style join output rows/sec (per-query latency in latency_ms)",
            "value": round(value, 1), "unit": "rows/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": round(1e3 * el / args.steps, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (datagen/gsmgen lubm, seeded)",
            "config": {"workload": f"LUBM-style U={args.univ} ({store.triple_count} triples), "
                                   "Q1-Q14, one step = 14 queries",
                       "univ": args.univ, "seed": args.seed},
            "latency_ms": lat,
            "cpu_baseline": {"value": round(value, 1), "unit": "rows/s", "cores": cores,
                             "kind": "reference",
                             "sample": f"{args.steps} steps x Q1-Q14, gsmat.executor.execute "
                                       f"mode=parallel worker_count={cores}"},
            "e2e": {"value": round(value, 1), "unit": "rows/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
        }), flush=True)


def main():
    args = _args()
    _ensure_built()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
