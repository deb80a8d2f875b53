#!/usr/bin/env python3
"""Summarise an ncu report: key SOL/memory metrics, stall breakdown and the
hottest SASS lines (reads the .ncu-rep with the local ncu CLI)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20


def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
hdr, units, vals = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__t_sectors.sum", "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum",
        "lts__t_sectors_op_read.sum", "lts__t_sectors_op_write.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "lts__average_gcomp_input_sector_success_rate.pct"]
for w in want:
    if w in hdr:
        i = hdr.index(w)
        print(f"{w:60s} {vals[i]:>20s} {units[i]}")
rows = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source=sass"))))
h = rows[1]
data = rows[2:]
i_s = h.index("Warp Stall Sampling (All Samples)")
sc = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
tot = sum(int(r[i_s] or 0) for r in data)
agg = {}
for r in data:
    for i in sc:
        agg[h[i]] = agg.get(h[i], 0) + int(r[i] or 0)
print("stall samples", tot)
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]:
    print(f"  {k:28s} {v:8d} {100 * v / max(tot, 1):5.1f}%")
for r in sorted(data, key=lambda r: -int(r[i_s] or 0))[:top]:
    st = sorted([(int(r[i] or 0), h[i][6:]) for i in sc], reverse=True)[:2]
    print(f"  {r[0][-5:]} {r[i_s]:>6s} {r[1][:64]:64s} {st}")
