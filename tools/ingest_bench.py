#!/usr/bin/env python
"""Store build from N-Triples: our `build` (host
parse threads + GPU encode/sort) against the reference's `gsmat build`
(oracle/_ref, single Python process) on the same N-Triples file, with a
byte-for-byte comparison of the two store directories.

The input is a generated LUBM store written out as N-Triples in a shuffled
order (so the dictionary order is the file's, not the generator's).
    python tools/ingest_bench.py --univ 10 [--ref-univ 2]
The reference build is timed on --ref-univ (it needs ~13 s per million
triples), ours on both.
"""
from __future__ import annotations

import argparse
import json
import random
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
sys.path.append(str(REPO / "oracle" / "_ref"))

import paper_1807_07691_b200 as g  # noqa: E402


def write_nt(univ: int, out: Path, tmp: Path) -> int:
    sd = tmp / f"lubm{univ}"
    subprocess.run([str(REPO / "oracle/_build/gsmgen"), "lubm", "--univ", str(univ), "--seed", "0",
                    "--out", str(sd)], check=True, stdout=subprocess.DEVNULL)
    st = g.load(sd)
    dec, decp = st.dictionary.decode_node, st.dictionary.decode_predicate
    lines = []
    for pid, m in st.matrices.items():
        pt = f"<{decp(pid)}>"
        for s, o in np.asarray(m.so).tolist():
            lines.append(f"{g.format_term(dec(s))} {pt} {g.format_term(dec(o))} .")
    random.Random(univ).shuffle(lines)
    out.write_text("\n".join(lines) + "\n", encoding="utf-8")
    return len(lines)


def same_dirs(a: Path, b: Path) -> bool:
    na = sorted(p.name for p in a.iterdir())
    if na != sorted(p.name for p in b.iterdir()):
        return False
    return all((a / n).read_bytes() == (b / n).read_bytes() for n in na)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--univ", type=int, default=10)
    ap.add_argument("--ref-univ", type=int, default=2)
    args = ap.parse_args()
    subprocess.run(["make", "-s", "-C", str(REPO / "oracle")], check=True)
    with tempfile.TemporaryDirectory() as t:
        tmp = Path(t)
        for univ, with_ref in ((args.ref_univ, True), (args.univ, False)):
            nt = tmp / f"u{univ}.nt"
            n = write_nt(univ, nt, tmp)
            g.build(nt, tmp / f"warm{univ}")  # first call: CUDA context, module load
            t0 = time.perf_counter()
            counts = g.build(nt, tmp / f"ours{univ}")
            ours = time.perf_counter() - t0
            rec = {"univ": univ, "triples_in": n, "nt_bytes": nt.stat().st_size, "counts": counts,
                   "ours_s": round(ours, 3), "ours_triples_per_s": round(n / ours, 1)}
            if with_ref:
                try:
                    from gsmat import cli
                    t0 = time.perf_counter()
                    assert cli.main(["build", "--input", str(nt), "--out", str(tmp / f"ref{univ}")]) == 0
                    ref = time.perf_counter() - t0
                    rec["reference_s"] = round(ref, 3)
                    rec["reference_triples_per_s"] = round(n / ref, 1)
                    rec["byte_identical"] = same_dirs(tmp / f"ours{univ}", tmp / f"ref{univ}")
                except ImportError:
                    rec["reference_s"] = "reference package not installed"
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
