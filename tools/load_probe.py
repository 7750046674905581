#!/usr/bin/env python
"""Time the phases of storage.load on a generated store (loader fast-path
work): dictionary, pair-file reads, device upload
(gsm_store_put_predicate), device index build (gsm_store_finalize).
Usage: python tools/load_probe.py --univ 100 [--store DIR]"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import subprocess
import sys
import tempfile
import time
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--univ", type=int, default=100)
    ap.add_argument("--store", default=None)
    args = ap.parse_args()
    import numpy as np

    from paper_1807_07691_b200 import _lib, storage
    from paper_1807_07691_b200.dictionary import StoreDictionary

    subprocess.run(["make", "-s", "-C", str(REPO / "oracle")], check=True)
    d = Path(args.store) if args.store else Path(tempfile.mkdtemp(prefix="gsm_load_")) / "s"
    if not args.store:
        subprocess.run([str(REPO / "oracle/_build/gsmgen"), "lubm", "--univ", str(args.univ),
                        "--out", str(d)], check=True, stdout=subprocess.DEVNULL)
    L = _lib.lib()
    t = {}
    t0 = time.perf_counter()
    store = storage.load(d)
    t["load_total"] = time.perf_counter() - t0
    del store
    t0 = time.perf_counter()
    StoreDictionary(d)
    t["dictionary"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    pairs = {}
    for p in sorted(d.glob("p*.so")):
        pid = int(p.stem[1:])
        pairs[pid] = (np.fromfile(p, dtype="<u8").reshape(-1, 2),
                      np.fromfile(p.with_suffix(".os"), dtype="<u8").reshape(-1, 2))
    t["read_pairs"] = time.perf_counter() - t0
    nodes = int((d / "meta").read_text().split()[3])
    h = C.c_void_p()
    _lib.check(L.gsm_store_create(0, nodes, max(pairs), C.byref(h)))
    t0 = time.perf_counter()
    for pid in sorted(pairs):
        so, os_ = pairs[pid]
        _lib.check(L.gsm_store_put_predicate(h, pid, so.ctypes.data, os_.ctypes.data, so.shape[0]))
    t["put_predicates"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    _lib.check(L.gsm_store_finalize(h))
    t["finalize"] = time.perf_counter() - t0
    L.gsm_store_free(h)
    nbytes = sum(a.nbytes + b.nbytes for a, b in pairs.values())
    print(json.dumps({"univ": args.univ, "triples": sum(a.shape[0] for a, _ in pairs.values()),
                      "predicates": len(pairs), "pair_bytes": nbytes,
                      **{k: round(v, 3) for k, v in t.items()},
                      "upload_GBps": round(nbytes / t["put_predicates"] / 1e9, 2)}))


if __name__ == "__main__":
    main()
