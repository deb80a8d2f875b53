#!/bin/bash
# Two-level latency rounds: parity (latency-mode tests, mesh configs, smoke) + mesh A/B.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -k "latency or mesh or hand or criterion_1 or long_path or deeper" > gpurun_out/lat4_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/lat4_tests.log
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/lat4_tests.log 2>&1
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
ab() {
  local name=$1; shift
  r=$(env "$@" timeout 600 python bench.py --workload ${W:-mesh4096} --no-cpu-baseline --plugin-sources 0 --steps 2 --warmup 3 2>gpurun_out/ab_$name.err)
  echo "${W:-mesh4096} $name $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["config"].get("mean_bfs_ms"), d["roofline"]["frac"], d["e2e"]["value"])' 2>&1)" >> gpurun_out/lat4_ab.txt
}
ab lat2 PBFS_X=1
ab lat1 PBFS_LIB=$PWD/build/ab/libpbfs_lat1.so
ab lat2_grid74 PBFS_LATENCY_GRID=74
