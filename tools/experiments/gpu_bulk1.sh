#!/bin/bash
# A/B of the bulk-staged hub expansion and the split host transfers (run under
# gpurun): parity first, then bench lines for the in-tree build (bulk), the
# aligned item grid alone, and the previous behaviour; then the share of each
# distance array that travels as plain 4 B entries (PBFS_DIRECT_PCT).
OUT=gpurun_out/bulk1
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -m gpu -x -q > $OUT/pytest.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
bash tools/ab_bench.sh rmat26 base nobulk old base > $OUT/ab_rmat26.txt 2>&1
cat $OUT/ab_rmat26.txt
for pct in 0 15 35 50; do
  echo "PBFS_DIRECT_PCT=$pct $(PBFS_DIRECT_PCT=$pct bash tools/ab_bench.sh rmat26 base)" >> $OUT/ab_direct.txt
done
cat $OUT/ab_direct.txt
bash tools/ab_bench.sh rmat20 base old > $OUT/ab_rmat20.txt 2>&1
bash tools/ab_bench.sh er24 base old > $OUT/ab_er24.txt 2>&1
cat $OUT/ab_rmat20.txt $OUT/ab_er24.txt
