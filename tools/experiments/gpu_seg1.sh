#!/bin/bash
# Owner-range hub split: parity on forced small graphs, then RMAT-26 A/B over
# the split knobs (graph cached once in /tmp).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "owner_range or golden or size_gated or criterion_1" > gpurun_out/seg_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/seg_tests.log
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
ab() {
  local name=$1; shift
  r=$(env "$@" timeout 600 python bench.py --workload ${W:-rmat26} --no-cpu-baseline --plugin-sources 0 --steps 3 --warmup 3 2>gpurun_out/ab_$name.err)
  echo "${W:-rmat26} $name $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["config"].get("mean_bfs_ms"), d["roofline"]["frac"], d["e2e"]["value"])' 2>&1)" >> gpurun_out/seg_ab.txt
}
ab seg_default PBFS_X=1
ab seg_off PBFS_SEG=0
ab seg_deg1024 PBFS_SEG_DEG=1024
ab seg_deg4096 PBFS_SEG_DEG=4096
ab seg_cw4096 PBFS_SEG_CW=4096
ab seg_cw12288 PBFS_SEG_CW=12288
ab seg_minq0 PBFS_SEG_MINQ=0
