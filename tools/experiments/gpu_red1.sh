#!/bin/bash
# Reduction claim: parity (forced) + RMAT-26 / ER-24 A/B.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "owner_range or golden or reduction or size_gated" > gpurun_out/red_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/red_tests.log
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
ab() {
  local name=$1; shift
  r=$(env "$@" timeout 600 python bench.py --workload ${W:-rmat26} --no-cpu-baseline --plugin-sources 0 --steps 3 --warmup 3 2>gpurun_out/ab_$name.err)
  echo "${W:-rmat26} $name $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["config"].get("mean_bfs_ms"), d["roofline"]["frac"], d["e2e"]["value"])' 2>&1)" >> gpurun_out/red_ab.txt
}
ab red_noseg PBFS_SEG=0
ab nored_noseg PBFS_SEG=0 PBFS_RED_MINQ=0
ab red_seg PBFS_X=1
ab red_seg8192 PBFS_SEG_DEG=8192
ab red_noseg_q512 PBFS_SEG=0 PBFS_RED_MINQ=512
ab red_noseg_q65536 PBFS_SEG=0 PBFS_RED_MINQ=65536
W=er24 ab red PBFS_X=1
W=er24 ab nored PBFS_RED_MINQ=0
W=rmat20 ab red PBFS_X=1
W=rmat20 ab nored PBFS_RED_MINQ=0
PBFS_SEG=0 timeout 300 python tools/level_dump.py --sources 6 > gpurun_out/levels_red.csv 2>/dev/null
