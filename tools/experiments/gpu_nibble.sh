#!/bin/bash
# 4-bit transfer codes (default where a traversal has < 15 levels) against
# 1 B codes (PBFS_PACK_MIN_BITS=8): batch / packed parity tests with the
# AVX-512 and the SSE2 widening loops, then alternating bench lines.
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_integration_cpp.py -m gpu -x -q -k "batch or packed or pageable or adapter or reference_drives" 2>&1 | tail -2
PBFS_NO_AVX512=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "batch or packed or pageable" 2>&1 | tail -2
PBFS_PACK_MIN_BITS=8 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pageable" 2>&1 | tail -2
for i in 1 2 3; do
  echo "nibble $(bash tools/ab_bench.sh rmat26 base)"
  echo "byte   $(PBFS_PACK_MIN_BITS=8 bash tools/ab_bench.sh rmat26 base)"
done
