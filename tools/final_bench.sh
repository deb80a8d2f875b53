#!/bin/bash
# Round-end measurement set (run under gpurun): every config's bench line,
# the reference arm, a loopback partition run, the rmat26 launch list and
# one full ncu capture. Outputs under gpurun_out/final/.
OUT=gpurun_out/final
mkdir -p $OUT
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
for w in rmat20 er24 mesh4096 rmat26; do
  timeout 1200 python bench.py --workload $w --steps 3 --warmup 3 > $OUT/bench_$w.json 2> $OUT/bench_$w.err
done
timeout 900 python bench.py --impl reference --workload rmat26 --steps 1 --warmup 1 > $OUT/ref_rmat26.json 2> $OUT/ref_rmat26.err
timeout 900 python bench.py --workload rmat26 --partitions 2 --steps 1 --warmup 2 > $OUT/part2_rmat26.json 2> $OUT/part2_rmat26.err
bash tools/profile_bench.sh rmat26 $OUT/prof > $OUT/prof.log 2>&1
timeout 2400 python bench.py --workload rmat28 --steps 1 --warmup 3 > $OUT/bench_rmat28.json 2> $OUT/bench_rmat28.err
echo done > $OUT/DONE
