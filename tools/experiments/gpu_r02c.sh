#!/bin/bash
# Session-3 re-entry check: GPU test suite + default bench line on the rebuilt tree.
mkdir -p gpurun_out/r2c
nvidia-smi --query-gpu=name,clocks.sm,memory.total --format=csv > gpurun_out/r2c/smi.txt 2>&1
PBFS_GEN_TIMING=1 timeout 2700 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/r2c/gputests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2c/gputests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2c/bench.json 2> gpurun_out/r2c/bench.err
echo "bench rc=$?" >> gpurun_out/r2c/bench.err
