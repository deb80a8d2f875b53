#!/bin/bash
# Round-2 extras for the committed build (run under gpurun): the reference's
# kernel variants on RMAT-26 / ER-24 / RMAT-20, the loopback multi-partition
# bench lines, and RMAT-28 (config 5) on one GPU.
OUT=gpurun_out/extra
mkdir -p $OUT
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
bash tools/variants.sh rmat26 er24 rmat20 > $OUT/variants.txt 2>&1
for v in hybrid-plain; do
  for w in rmat26 er24 rmat20; do
    r=$(timeout 900 python bench.py --workload $w --variant $v --no-cpu-baseline --steps 2 --warmup 3 2>/dev/null)
    echo "$w $v $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["config"].get("mean_bfs_ms"), d["roofline"]["frac"], d["e2e"]["parity_last_source"])' 2>&1)" >> $OUT/variants.txt
  done
done
cat $OUT/variants.txt
for g in 2 4 8; do
  timeout 900 python bench.py --workload rmat26 --partitions $g --steps 2 --warmup 3 > $OUT/partitions${g}_rmat26.json 2> $OUT/partitions${g}_rmat26.err
done
unset PBFS_GRAPH_CACHE_DIR
timeout 1500 python bench.py --workload rmat28 --steps 2 --warmup 3 --cpu-budget 20 > $OUT/bench_rmat28.json 2> $OUT/bench_rmat28.err
tail -2 $OUT/bench_rmat28.err
