#!/bin/bash
# ncu --set full of RMAT-26 traversals whose time sits in a mid-size top-down
# level (a few thousand hubs discovering ~1e7 fresh vertices): source index 1
# (6627 -> 10.7 M, 71 M edges), after a plain run of the same command.
cd "$(dirname "$0")/.."
OUT=gpurun_out/ncu_mid; mkdir -p $OUT
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
for idx in 1; do
  CMD="python tools/one_bfs.py --workload rmat26 --source-index $idx --repeat 2"
  $CMD > $OUT/one_$idx.log 2>&1 || { cat $OUT/one_$idx.log; exit 1; }
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:bfs_persistent -s 1 -c 1 \
      -o $OUT/rmat26_src$idx -f $CMD > $OUT/ncu_$idx.log 2>&1
done
python tools/level_dump.py --workload rmat26 --sources 8 > $OUT/levels8.csv 2> $OUT/levels8.err
