"""bench.py's driver contract (task spec): one JSON line with the metric,
whole-job value, roofline, cpu_baseline, e2e, gpu_launches and clocks; the
reference arm's line. Run on a small config so the check costs seconds."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_help_lists_the_contract_flags():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"],
                         capture_output=True, text=True, timeout=120, cwd=ROOT)
    assert out.returncode == 0
    for flag in ("--gpus", "--steps", "--warmup", "--impl", "--workload", "--variant"):
        assert flag in out.stdout


@pytest.mark.gpu
def test_gpu_arm_json_line():
    d = run_bench("--workload", "rmat20", "--steps", "1", "--warmup", "3", "--cpu-budget", "2")
    assert d["metric"].startswith("GTEPS") and d["unit"] == "GTEPS" and d["value"] > 0
    assert d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 3
    assert d["higher_is_better"] is True and d["scaling"] in ("weak", "strong")
    assert d["vs_baseline"] is None and d["data"] == "synthetic" and d["dtype"] == "u32"
    assert d["config"]["workload"] == "rmat20" and d["ms_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    c = d["cpu_baseline"]
    assert c["kind"] in ("reference", "port") and c["cores"] >= 1 and c["value"] > 0
    # every source the CPU leg ran is checked against the GPU distances
    assert c["parity_checked_sources"] >= 1 and c["parity_mismatches"] == 0
    e = d["e2e"]
    assert e["unit"] == "GTEPS" and e["value"] > 0
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert d["clocks"]["sm_max_mhz"] > 0


def test_reference_arm_json_line_and_no_product_library():
    # The reference arm needs no GPU: the oracle builds the graph and the
    # reference's own bfs_hybrid (oracle/_ref) runs every one of the 64
    # sources over the timed steps; the product library is never loaded.
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--workload', "
            "'rmat20', '--steps', '8', '--warmup', '1']; "
            "runpy.run_path('bench.py', run_name='__main__'); "
            "maps = open('/proc/self/maps').read(); "
            "print('MAPS', int('libpbfs' in maps), int('libparbfs_ref' in maps or "
            "'liboracle_port' in maps))")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GTEPS"
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["config"]["sources_covered"] == 64 and d["config"]["same_config"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    maps = [ln for ln in out.stdout.splitlines() if ln.startswith("MAPS")][0].split()
    assert maps[1] == "0", "the reference arm loaded libpbfs.so"
    assert maps[2] == "1"
