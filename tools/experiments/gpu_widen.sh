#!/bin/bash
# A/B of the widening pool (dynamic pieces + blocking event waits, in-tree)
# against the committed build: batch parity tests, then bench lines.
OUT=gpurun_out/widen
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "batch or packed or pageable" > $OUT/pytest.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
bash tools/ab_bench.sh rmat26 base head base head > $OUT/ab_rmat26.txt 2>&1
cat $OUT/ab_rmat26.txt
for t in 15 14 12; do
  echo "PBFS_WIDEN_THREADS=$t $(PBFS_WIDEN_THREADS=$t bash tools/ab_bench.sh rmat26 base)" >> $OUT/ab_threads.txt
done
cat $OUT/ab_threads.txt
bash tools/ab_bench.sh er24 base head > $OUT/ab_er24.txt 2>&1
cat $OUT/ab_er24.txt
