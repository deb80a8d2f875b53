#!/bin/bash
# A/B the tunable builds in build/ab/ on one workload (graph cached once in /tmp).
# usage: tools/ab_bench.sh WORKLOAD NAME... (NAME "base" = the in-tree libpbfs.so)
# prints: workload name GTEPS mean-ms frac e2e-batch-GTEPS e2e-per-call-GTEPS
w=$1; shift
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
for n in "$@"; do
  if [ "$n" = base ]; then unset PBFS_LIB; else export PBFS_LIB=$PWD/build/ab/libpbfs_$n.so; fi
  r=$(timeout 600 python bench.py --workload $w --no-cpu-baseline --steps 3 --warmup 3 2>/dev/null)
  echo "$w $n $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["config"].get("mean_bfs_ms"), d["roofline"]["frac"], d["e2e"]["value"], d["e2e"].get("sync_per_call_value"))' 2>&1)"
done
