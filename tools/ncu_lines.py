#!/usr/bin/env python3
"""Attribute ncu warp-stall samples of one kernel to CUDA source lines:
ncu's SASS page (absolute addresses) is matched to `nvdisasm -g` line info of
the same cubin by function-relative offset.

  tools/ncu_lines.py REPORT.ncu-rep LIB.so KERNEL_MANGLED_NAME [top]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, lib, kname = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
rows = list(csv.reader(io.StringIO(subprocess.run(
    ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
    capture_output=True, text=True).stdout)))
h = rows[1]
data = rows[2:]
i_s = h.index("Warp Stall Sampling (All Samples)")
i_e = h.index("Instructions Executed")
base = int(data[0][0], 16)
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
cubins = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")]
off2line = {}
for cb in cubins:
    out = subprocess.run(["nvdisasm", "-g", "-c", cb], capture_output=True, text=True).stdout
    inside = False
    line = None
    for ln in out.splitlines():
        if ln.startswith(".text."):
            inside = ln.strip().rstrip(":") == ".text." + kname
            line = None
            continue
        if not inside:
            continue
        m = re.search(r'//## File ".*/([^/"]+)", line (\d+)', ln)
        if m:
            line = f"{m.group(1)}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and line:
            off2line[int(m.group(1), 16)] = line
    if off2line:
        break
agg = collections.Counter()
ins = collections.Counter()
for r in data:
    off = int(r[0], 16) - base
    key = off2line.get(off, "?")
    agg[key] += int(r[i_s] or 0)
    ins[key] += int(r[i_e] or 0)
tot = sum(agg.values())
print(f"stall samples {tot}, mapped lines {len(off2line)}")
for k, v in agg.most_common(top):
    print(f"  {k:28s} {v:8d} {100 * v / tot:5.1f}%   insts {ins[k]}")
