#!/bin/bash
# Latency-mode A/B on the deep mesh (config 3): latency mode vs general path.
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
run() { # name, env...
  local name=$1; shift
  env "$@" timeout 900 python bench.py --workload mesh4096 --no-cpu-baseline --steps 1 --warmup 3 > gpurun_out/bench_mesh_$name.json 2> gpurun_out/bench_mesh_$name.err
  echo "$name $(python -c "import json;d=json.load(open('gpurun_out/bench_mesh_$name.json'));print(d['value'], d['config']['mean_bfs_ms'])" 2>&1 | tail -1)" >> gpurun_out/ab_mesh.txt
}
rm -f gpurun_out/ab_mesh.txt


run lat1_g148 PBFS_LATENCY=1
run lat0 PBFS_LATENCY=0
