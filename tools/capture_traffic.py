#!/usr/bin/env python3
"""DRAM bytes actually moved per traversal, captured with ncu for the
CURRENT build, for bench.py's roofline.traffic / roofline.dram_frac.

  python tools/capture_traffic.py --workload rmat26 [--sources 64]
      runs ncu (dram__bytes_read.sum, dram__bytes_write.sum,
      gpu__time_duration.sum; --clock-control none) over one traversal from
      each of the first N bench sources and writes
      profiles/traffic_<workload>.json with the build hash (bench.build_hash:
      sha256 of the library sources) the numbers belong to. bench.py only
      reports a capture whose hash matches the library it runs.
  python tools/capture_traffic.py --inner ...   (what ncu runs)
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

METRICS = "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"


def inner(args):
    import paper_2503_00430_b200 as pb
    g = bench.build_graph(args.workload)
    cfg, _ = bench.kernel_config(g)
    cfg.variant = pb.parse_kernel_variant(args.variant)
    dg = g.device(0, bench.WORKLOADS[args.workload][3])
    srcs = [int(s) for s in bench.choose_sources(g, dg, cfg, args.workload)][:args.sources]
    for s in srcs:
        dg.bfs_async(s, cfg)
        dg.sync()
    print("SOURCES " + json.dumps(srcs), flush=True)


def outer(args):
    log = os.path.join(ROOT, "gpurun_out", f"traffic_{args.workload}.csv")
    os.makedirs(os.path.dirname(log), exist_ok=True)
    cmd = ["ncu", "--metrics", METRICS, "--clock-control", "none", "-k", "regex:bfs_(persistent|latency)",
           "--csv", "--log-file", log, sys.executable, os.path.abspath(__file__), "--inner",
           "--workload", args.workload, "--sources", str(args.sources), "--variant", args.variant]
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        sys.exit(f"ncu failed ({out.returncode}): {out.stderr[-2000:]}")
    srcs = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("SOURCES")][0][8:])
    rows = list(csv.DictReader(io.StringIO(
        "\n".join(ln for ln in open(log) if not ln.startswith("==")))))
    launches = {}
    for r in rows:
        lid = int(r["ID"])
        val = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
                 "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}.get(unit, 1.0)
        launches.setdefault(lid, {})[r["Metric Name"]] = val * scale
    # The first len(srcs) launches after the chooser's (mesh) are the sources.
    ids = sorted(launches)[-len(srcs):]
    per = []
    for s, lid in zip(srcs, ids):
        m = launches[lid]
        per.append({"source": s, "dram_bytes_read": m["dram__bytes_read.sum"],
                    "dram_bytes_write": m["dram__bytes_write.sum"],
                    "gpu_time_s": m["gpu__time_duration.sum"]})
    total = sum(p["dram_bytes_read"] + p["dram_bytes_write"] for p in per)
    res = {
        "workload": args.workload, "variant": args.variant, "build_hash": bench.build_hash(),
        "tool": f"ncu --metrics {METRICS} --clock-control none -k regex:bfs_(persistent|latency) "
                "(default cache control: caches flushed before each launch)",
        "sources": len(per),
        "dram_bytes_per_launch": total / len(per),
        "gpu_time_ms_per_launch": 1e3 * sum(p["gpu_time_s"] for p in per) / len(per),
        "per_source": per,
        "note": "bytes actually moved (read + write) per traversal; bench.py divides the sum "
                "over these sources by their live CUDA-event times and the measured HBM peak "
                "(roofline.dram_frac)",
    }
    path = os.path.join(ROOT, "profiles", f"traffic_{args.workload}.json")
    json.dump(res, open(path, "w"), indent=1)
    print(f"{path}: {res['dram_bytes_per_launch'] / 1e9:.3f} GB/launch over {len(per)} sources, "
          f"{res['gpu_time_ms_per_launch']:.3f} ms/launch (ncu, serialised)")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="rmat26")
    ap.add_argument("--sources", type=int, default=64)
    ap.add_argument("--variant", default="hybrid")
    ap.add_argument("--inner", action="store_true")
    a = ap.parse_args()
    inner(a) if a.inner else outer(a)
