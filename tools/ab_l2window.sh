#!/bin/bash
# A/B of the persisting-L2 window (PBFS_L2_WINDOW=all|visited) on one workload.
#   tools/ab_l2window.sh WORKLOAD
w=${1:-rmat26}
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
for wv in all visited; do
  r=$(PBFS_L2_WINDOW=$wv timeout 900 python bench.py --workload $w --no-cpu-baseline --steps 3 --warmup 3 2>/dev/null)
  echo "$w window=$wv $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["config"].get("mean_bfs_ms"), d["roofline"]["frac"])' 2>&1)"
done
