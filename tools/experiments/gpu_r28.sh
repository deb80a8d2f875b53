#!/bin/bash
# RMAT-28 on one GPU: reduction-claim threshold A/B (PBFS_RED_MINQ; 0 = off).
OUT=gpurun_out/r28
mkdir -p $OUT
for q in 0 65536 1048576 4194304; do
  r=$(PBFS_RED_MINQ=$q timeout 1200 python bench.py --workload rmat28 --no-cpu-baseline --plugin-sources 0 --steps 2 --warmup 2 2>/dev/null)
  echo "rmat28 red_minq=$q $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["config"].get("mean_bfs_ms"), d["roofline"]["frac"], d["e2e"]["value"])' 2>&1)" | tee -a $OUT/ab_rmat28.txt
done
