#!/bin/bash
# Owner-range split with the L1 as the range cache (PBFS_SEG_CW=4: no smem).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
export PBFS_LIB=$PWD/build/ab/libpbfs_hot0.so
ab() {
  local name=$1; shift
  r=$(env "$@" timeout 600 python bench.py --workload ${W:-rmat26} --no-cpu-baseline --plugin-sources 0 --steps 3 --warmup 3 2>gpurun_out/ab_$name.err)
  echo "${W:-rmat26} $name $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["config"].get("mean_bfs_ms"), d["roofline"]["frac"], d["e2e"]["value"])' 2>&1)" >> gpurun_out/seg4_ab.txt
}
ab noseg PBFS_SEG=0
ab l1_g3 PBFS_SEG_CW=4
ab l1_g1 PBFS_SEG_CW=4 PBFS_SEG_GROUP=1
ab l1_g3_d8192 PBFS_SEG_CW=4 PBFS_SEG_DEG=8192
ab l1_g3_d32768 PBFS_SEG_CW=4 PBFS_SEG_DEG=32768
ab l1_g6 PBFS_SEG_CW=4 PBFS_SEG_GROUP=6
ab sm_g3_d32768 PBFS_SEG_DEG=32768
PBFS_SEG_CW=4 TAG=segl1 tools/gpu_ncu_src2.sh
