#!/usr/bin/env python
"""Summarise ncu artefacts into profiles/: per-kernel launch table from a
--metrics launch list, and key metrics + top stall reasons from --set full
reports.  Usage: python tools/ncu_summary.py OUT.md [launches.csv] [*.ncu-rep]"""
from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
    ("smsp__inst_executed.sum", "instructions"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_st.sum", "global_store_requests"),
    ("lts__t_sectors_srcunit_tex_op_write.sum", "l2_write_sectors"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "l2_read_sectors"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if mi is not None and len(r) > mi and r[mi] != "gpu__time_duration.sum":
            continue
        if len(r) > vi:
            name = r[ki].split("(")[0].replace("void ", "")
            agg[name].append(float(r[vi].replace(",", "")) / 1e3)
    total = sum(sum(v) for v in agg.values())
    lines = ["| kernel | launches | total us | avg us | min us | max us | share |",
             "|---|---|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v):.1f} | {sum(v)/len(v):.2f} | {min(v):.2f} | "
                     f"{max(v):.2f} | {100*sum(v)/total:.1f}% |")
    return lines


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        rec = {"kernel": d.get("Kernel Name", "")[:60]}
        for k, short in KEYS:
            if k in d:
                rec[short] = f"{d[k]} {u.get(k, '')}".strip()
        stalls = [(float(d[k] or 0), k) for k in h
                  if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
        tot = sum(v for v, _ in stalls) or 1.0
        rec["top_stalls"] = [f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} "
                             f"{100*v/tot:.0f}%" for v, k in sorted(stalls, reverse=True)[:5] if v]
        out.append(rec)
    return out


def main():
    dst = sys.argv[1]
    md = []
    for a in sys.argv[2:]:
        if a.endswith(".csv"):
            md += [f"## Launch list: `{a.split('/')[-1]}`", ""] + launches(a) + [""]
        elif a.endswith(".ncu-rep"):
            md += [f"## ncu --set full: `{a.split('/')[-1]}`", ""]
            for rec in report(a):
                md.append("```")
                md.append(json.dumps(rec, indent=1))
                md.append("```")
            md.append("")
    open(dst, "w").write("\n".join(md))


if __name__ == "__main__":
    main()
