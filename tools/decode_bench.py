#!/usr/bin/env python
"""Result decoding: `result_tsv` (device rendering)
against the CLI's per-cell loop (cli.py:101-105 with our dictionary and the
restated format_term) on LUBM results, output compared on a sample.
    python tools/decode_bench.py [--univ 10]
"""
from __future__ import annotations

import argparse
import json
import subprocess
import sys
import tempfile
import time
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

import paper_1807_07691_b200 as g  # noqa: E402

UB = "PREFIX ub: <http://swat.cse.lehigh.edu/onto/univ-bench.owl#> "
QUERIES = {
    "q14_all_students": UB + "PREFIX rdf: <http://www.w3.org/1999/02/22-rdf-syntax-ns#> "
    "SELECT ?x WHERE { ?x rdf:type ub:UndergraduateStudent . }",
    "classmates": UB + "SELECT ?x ?c ?y WHERE { ?x ub:takesCourse ?c . ?y ub:takesCourse ?c . }",
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--univ", type=int, default=10)
    args = ap.parse_args()
    with tempfile.TemporaryDirectory() as tmp:
        sd = f"{tmp}/lubm"
        subprocess.run([str(REPO / "oracle/_build/gsmgen"), "lubm", "--univ", str(args.univ), "--seed", "0",
                        "--out", sd], check=True, stdout=subprocess.DEVNULL)
        st = g.load(sd)
        dec = st.dictionary.decode_node
        for name, text in QUERIES.items():
            q = g.bind_constants(g.parse_query(text), st.dictionary)
            res = g.execute(q, g.make_plan(q, st.stats), st, row_budget=1 << 62)
            g.decode_rows(st, res.array[:10])  # dictionary upload + warm-up
            t0 = time.perf_counter()
            body = g.decode_rows(st, res.array)  # the TSV body as bytes
            ours = time.perf_counter() - t0
            import io, os
            with open(os.devnull, "wb") as fh:
                t0 = time.perf_counter()
                g.write_tsv(res, st, fh)  # straight from the library's buffer to the file
                ours_file = time.perf_counter() - t0
            out = ("\t".join(res.schema) + "\n").encode() + body
            arr = res.array
            n = len(arr)
            sample = min(n, 200_000)
            t0 = time.perf_counter()
            ref = "\t".join(res.schema) + "\n" + "".join(
                "\t".join(g.format_term(dec(int(v))) for v in row) + "\n" for row in arr[:sample].tolist())
            loop = time.perf_counter() - t0
            ref = ref.encode("utf-8")
            head = out[: len(ref)]
            print(json.dumps({"query": name, "rows": n, "bytes": len(out), "ours_s": round(ours, 4),
                              "ours_rows_per_s": round(n / ours, 1),
                              "write_tsv_s": round(ours_file, 4),
                              "write_tsv_rows_per_s": round(n / ours_file, 1),
                              "cli_loop_rows_per_s": round(sample / loop, 1), "cli_loop_sample": sample,
                              "sample_identical": head == ref}), flush=True)


if __name__ == "__main__":
    main()
