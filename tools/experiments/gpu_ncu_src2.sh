#!/bin/bash
# ncu --set full of the RMAT-26 traversal from source index 2 (one 1.47 G-edge
# top-down level = ~80 % of its time), after a plain run of the same command.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
CMD="python tools/one_bfs.py --workload rmat26 --source-index 2 --repeat 2"
$CMD > gpurun_out/one_src2.log 2>&1 || { cat gpurun_out/one_src2.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bfs_persistent -s 1 -c 1 \
    -o gpurun_out/src2_${TAG:-x} -f $CMD > gpurun_out/ncu_src2.log 2>&1
