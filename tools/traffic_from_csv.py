#!/usr/bin/env python
"""Per-launch DRAM traffic of the join kernels from an ncu --metrics CSV
(gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum over
every launch of a bench run): writes the mean read+write bytes per launch of
k_tilescan<FilterP> ("filter"), k_group ("group") and of all join kernels
("join") to profiles/ncu_traffic.json, which bench.py reports as
roofline.traffic.  Usage: python tools/traffic_from_csv.py launches.csv OUT.json"""
import collections
import csv
import json
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[ii]] = r[ki]
    cls = collections.defaultdict(list)
    for lid, m in per.items():
        n = names[lid]
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        if "k_group" in n:
            cls["group"].append(b)
            cls["join"].append(b)
        elif "k_tilescan" in n and "FilterP" in n:
            cls["filter"].append(b)
            cls["join"].append(b)
        elif "k_tilescan" in n and "ExpandP" in n:
            cls["expand"].append(b)
            cls["join"].append(b)
    out = {k: int(sum(v) / len(v)) for k, v in cls.items() if v}
    out["launches"] = {k: len(v) for k, v in cls.items()}
    out["_note"] = ("mean dram__bytes_read.sum + dram__bytes_write.sum per launch of the LUBM-10 "
                    "join kernels over every launch of `bench.py --steps 1 --warmup 3` under ncu "
                    "(cold caches, serialised launches): " + sys.argv[1].split("/")[-1])
    json.dump(out, open(sys.argv[2], "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
