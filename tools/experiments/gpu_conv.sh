#!/bin/bash
# Top-down-only variants (Conventional CAS / NonAtomic plain store): dist probe
# A/B (PBFS_DIST_PROBE builds in build/ab) on RMAT-26 and ER-24, then one ncu
# --set full capture of Conventional from source index 2 (base build).
cd "$(dirname "$0")/.."
OUT=gpurun_out/conv; mkdir -p $OUT
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
for w in rmat26 er24; do
  for var in conventional nonatomic; do
    for n in base cad1 cad2; do
      if [ "$n" = base ]; then unset PBFS_LIB; else export PBFS_LIB=$PWD/build/ab/libpbfs_$n.so; fi
      r=$(timeout 900 python bench.py --workload $w --variant $var --no-cpu-baseline --plugin-sources 0 --steps 2 --warmup 3 2>>$OUT/ab.err)
      echo "$w $var $n $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["config"].get("mean_bfs_ms"), d["roofline"]["frac"])' 2>&1)" >> $OUT/ab.txt
    done
  done
done
unset PBFS_LIB
CMD="python tools/one_bfs.py --workload rmat26 --source-index 2 --repeat 2 --variant conventional"
$CMD > $OUT/one_conv.log 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:bfs_persistent -s 1 -c 1 \
    -o $OUT/conv_src2 -f $CMD > $OUT/ncu_conv.log 2>&1
echo done >> $OUT/ab.txt
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_rmat26.json 2> $OUT/bench_rmat26.err
