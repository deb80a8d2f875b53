#!/bin/bash
# Widening with whole-line AVX-512 non-temporal stores (default where the host
# has AVX-512) against the SSE2 loop (PBFS_NO_AVX512=1): batch parity tests,
# then alternating bench lines (GTEPS mean-ms frac e2e-batch e2e-per-call).
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "batch or packed or pageable" 2>&1 | tail -2
for i in 1 2 3; do
  echo "avx512 $(bash tools/ab_bench.sh rmat26 base)"
  echo "sse2   $(PBFS_NO_AVX512=1 bash tools/ab_bench.sh rmat26 base)"
done
echo "avx512 $(bash tools/ab_bench.sh rmat28 base)"
echo "sse2   $(PBFS_NO_AVX512=1 bash tools/ab_bench.sh rmat28 base)"
