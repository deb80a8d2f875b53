#!/bin/bash
# ncu --set full of the current build: RMAT-26 hybrid from source index 2 (the
# 1.47 G-edge top-down level) and ER-24 from source index 0 (one dominant
# bottom-up level), each after a plain run of the same command.
cd "$(dirname "$0")/.."
OUT=gpurun_out/ncu3; mkdir -p $OUT
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
for spec in "rmat26 2" "er24 0"; do
  set -- $spec
  CMD="python tools/one_bfs.py --workload $1 --source-index $2 --repeat 2"
  $CMD > $OUT/one_$1.log 2>&1 || { cat $OUT/one_$1.log; exit 1; }
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:bfs_persistent -s 1 -c 1 \
      -o $OUT/$1_src$2 -f $CMD > $OUT/ncu_$1.log 2>&1
done
