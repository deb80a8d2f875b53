#!/bin/bash
# Full GPU suite + bench lines for the kept build.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests2.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gputests2.log
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
for W in rmat26 rmat20 er24 mesh4096; do
  timeout 900 python bench.py --workload $W --no-cpu-baseline --plugin-sources 0 --steps 3 --warmup 3 > gpurun_out/b2_$W.json 2> gpurun_out/b2_$W.err
done
