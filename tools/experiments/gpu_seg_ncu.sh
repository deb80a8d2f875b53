#!/bin/bash
# ncu --set full of one RMAT-26 traversal (source index 0) with the owner-range
# hub split on and off (each after a plain run of the same command).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
CMD="python tools/one_bfs.py --workload rmat26 --repeat 2"
for mode in on off; do
  if [ $mode = off ]; then export PBFS_SEG=0; else unset PBFS_SEG; fi
  $CMD > gpurun_out/one_$mode.log 2>&1 || { echo "plain run failed"; cat gpurun_out/one_$mode.log; exit 1; }
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:bfs_persistent -s 1 -c 1 \
      -o gpurun_out/seg_$mode -f $CMD > gpurun_out/ncu_seg_$mode.log 2>&1
done
