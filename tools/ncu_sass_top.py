#!/usr/bin/env python
"""Top stalled SASS instructions of one kernel in an ncu report (the source
page with warp-stall samples per instruction), with a few instructions of
context.  Usage: python tools/ncu_sass_top.py REPORT.ncu-rep [kernel_index] [N]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    top_n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdrs = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
    h = rows[hdrs[k]]
    si = h.index("Warp Stall Sampling (All Samples)")
    end = hdrs[k + 1] - 1 if k + 1 < len(hdrs) else len(rows)
    seg = [r for r in rows[hdrs[k] + 1:end] if len(r) > si and r[si].isdigit()]
    tot = sum(int(r[si]) for r in seg)
    print(f"kernel {k}: {len(seg)} instructions, {tot} stall samples")
    for r in sorted(seg, key=lambda r: -int(r[si]))[:top_n]:
        print(f"{int(r[si]):6d} {100.0 * int(r[si]) / max(tot, 1):5.1f}%  {r[1].strip()[:90]}")


if __name__ == "__main__":
    main()
