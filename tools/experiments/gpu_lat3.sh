#!/bin/bash
# Latency-mode grid sweep on the mesh (config 3).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
ab() {
  local name=$1; shift
  r=$(env "$@" timeout 600 python bench.py --workload ${W:-mesh4096} --no-cpu-baseline --plugin-sources 0 --steps 2 --warmup 3 2>gpurun_out/ab_$name.err)
  echo "${W:-mesh4096} $name $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["config"].get("mean_bfs_ms"), d["roofline"]["frac"], d["e2e"]["value"])' 2>&1)" >> gpurun_out/lat3_ab.txt
}
for G in 148 111 74 56 37 24; do ab grid$G PBFS_LATENCY_GRID=$G; done
