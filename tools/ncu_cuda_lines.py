#!/usr/bin/env python3
"""Warp-stall samples of an ncu report (--import-source on) aggregated per
CUDA source line, with the top stall reasons of each line.

  tools/ncu_cuda_lines.py REPORT.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(r for r in rows if r and r[0] == "Line No")
i_s = h.index("Warp Stall Sampling (All Samples)")
reasons = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
agg = []
for r in rows[rows.index(h) + 1:]:
    if len(r) > i_s and r[0] and r[i_s].strip() not in ("", "-"):
        try:
            n = int(float(r[i_s]))
        except ValueError:
            continue
        rs = sorted(((int(float(r[i] or 0)), c[6:]) for i, c in reasons if r[i] not in ("", "-")), reverse=True)[:3]
        agg.append((n, r[0], r[1].strip()[:80], rs))
tot = sum(a[0] for a in agg)
print(f"total samples {tot}")
for n, ln, src, rs in sorted(agg, reverse=True)[:top]:
    print(f"{n:7d} {100 * n / tot:5.1f}%  L{ln:5s} {src:80s} {rs}")
