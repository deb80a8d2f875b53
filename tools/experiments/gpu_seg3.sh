#!/bin/bash
# Owner-range hub split A/B round 3 (ranges shared by CTA groups).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "owner_range or golden" > gpurun_out/seg_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/seg_tests.log
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
ab() {
  local name=$1; shift
  r=$(env "$@" timeout 600 python bench.py --workload ${W:-rmat26} --no-cpu-baseline --plugin-sources 0 --steps 3 --warmup 3 2>gpurun_out/ab_$name.err)
  echo "${W:-rmat26} $name $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["config"].get("mean_bfs_ms"), d["roofline"]["frac"], d["e2e"]["value"])' 2>&1)" >> gpurun_out/seg_ab.txt
}
ab g3 PBFS_X=1
ab off PBFS_SEG=0
ab g1 PBFS_SEG_GROUP=1
ab g2 PBFS_SEG_GROUP=2
ab g6 PBFS_SEG_GROUP=6
ab g12 PBFS_SEG_GROUP=12
ab g3cw4096 PBFS_SEG_CW=4096
ab g3deg8192 PBFS_SEG_DEG=8192
ab g3deg1024 PBFS_SEG_DEG=1024
timeout 300 python tools/level_dump.py --sources 6 > gpurun_out/levels_seg_on.csv 2>/dev/null
