#!/bin/bash
# Visited-probe L1 policy by word index (PBFS_HOT_MODE builds in build/ab) on
# RMAT-26 / RMAT-20 / ER-24, plus the plain-store variants on the base build.
cd "$(dirname "$0")/.."
OUT=gpurun_out/hot; mkdir -p $OUT
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
for w in rmat26 rmat20 er24; do
  bash tools/ab_bench.sh $w base hm1_4k hm1_16k hm2_16k hm3_16k hm1_64k base >> $OUT/ab.txt 2>&1
done
for var in hybrid-plain nonatomic conventional; do
  r=$(timeout 900 python bench.py --workload rmat26 --variant $var --no-cpu-baseline --plugin-sources 0 --steps 2 --warmup 3 2>>$OUT/var.err)
  echo "rmat26 $var $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["config"].get("mean_bfs_ms"), d["roofline"]["frac"])' 2>&1)" >> $OUT/ab.txt
done
echo done >> $OUT/ab.txt
