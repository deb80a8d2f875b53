#!/bin/bash
# Single pbfs_bfs calls into pinned memory through the packed transfer
# (default) against the plain 4 B/vertex copy (PBFS_PINNED_PACKED=0).
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -m gpu -x -q -k "batch or packed or pageable or config4_rmat26_all or async" 2>&1 | tail -2
for i in 1 2; do
  echo "packed $(bash tools/ab_bench.sh rmat26 base)"
  echo "plain  $(PBFS_PINNED_PACKED=0 bash tools/ab_bench.sh rmat26 base)"
done
echo "packed $(bash tools/ab_bench.sh rmat28 base)"
