#!/bin/bash
# Round-2 measurement set (run under gpurun): traffic captures for the
# current build first (bench.py reports roofline.dram_frac only for a
# capture of the build it runs), then every config's bench line, the
# reference arm, the rmat26 / mesh launch lists and full ncu captures.
# Outputs under gpurun_out/final/ (traffic JSONs copied there too).
OUT=gpurun_out/final
mkdir -p $OUT
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
for w in rmat26 er24 rmat20 mesh4096; do
  timeout 1200 python tools/capture_traffic.py --workload $w > $OUT/traffic_$w.log 2>&1
  cp profiles/traffic_$w.json $OUT/ 2>/dev/null
done
for w in rmat26 er24 rmat20 mesh4096; do
  timeout 1200 python bench.py --workload $w --steps 3 --warmup 3 > $OUT/bench_$w.json 2> $OUT/bench_$w.err
done
timeout 900 python bench.py --impl reference --workload rmat26 --steps 2 --warmup 1 > $OUT/ref_rmat26.json 2> $OUT/ref_rmat26.err
bash tools/profile_bench.sh rmat26 $OUT/prof > $OUT/prof.log 2>&1
bash tools/profile_bench.sh mesh4096 $OUT/prof > $OUT/prof_mesh.log 2>&1
echo done > $OUT/DONE
