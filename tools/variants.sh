#!/bin/bash
# The paper's kernel variants on the GPU (bench.py --variant): GTEPS, ms per BFS, roofline frac.
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
for w in ${@:-rmat26 er24}; do
  for v in hybrid hybrid-beamer visited-inline nonatomic conventional; do
    r=$(timeout 900 python bench.py --workload $w --variant $v --no-cpu-baseline --steps 2 --warmup 3 2>/dev/null)
    echo "$w $v $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["config"].get("mean_bfs_ms"), d["roofline"]["frac"], d["e2e"]["parity_last_source"])' 2>&1)"
  done
done
