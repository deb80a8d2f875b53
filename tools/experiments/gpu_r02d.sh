#!/bin/bash
# GPU suite + RMAT-26 bench line on the current tree.
mkdir -p gpurun_out/r2d
PBFS_GEN_TIMING=1 timeout 3000 python -m pytest tests -m gpu -x -q --durations=30 > gpurun_out/r2d/gputests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2d/gputests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2d/bench.json 2> gpurun_out/r2d/bench.err
echo "bench rc=$?" >> gpurun_out/r2d/bench.err
