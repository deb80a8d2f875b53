#!/bin/bash
# A/B of the hub-pass reduction claim gated on the level's hub edges (in-tree)
# against the committed build (reduction for whole levels of >= 65536 frontier
# vertices): parity first, then bench lines and a threshold sweep.
OUT=gpurun_out/hubred
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -m gpu -x -q > $OUT/pytest.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
bash tools/ab_bench.sh rmat26 base head > $OUT/ab_rmat26.txt 2>&1
cat $OUT/ab_rmat26.txt
for e in 0 1048576 4194304 16777216 67108864; do
  echo "PBFS_RED_MIN_EDGES=$e $(PBFS_RED_MIN_EDGES=$e bash tools/ab_bench.sh rmat26 base)" >> $OUT/ab_sweep.txt
done
cat $OUT/ab_sweep.txt
bash tools/ab_bench.sh rmat20 base head > $OUT/ab_rmat20.txt 2>&1
bash tools/ab_bench.sh er24 base head > $OUT/ab_er24.txt 2>&1
cat $OUT/ab_rmat20.txt $OUT/ab_er24.txt
