#!/bin/bash
# Final round-2 run of the committed build (under gpurun): the whole GPU test
# suite, then tools/final_r02.sh (traffic captures, bench lines of the four
# single-GPU configs, reference arm, launch lists, full ncu captures), then
# RMAT-28 (config 5) on one GPU.
mkdir -p gpurun_out/final
PBFS_GEN_TIMING=1 timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/final/gputests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/final/gputests.log
tail -3 gpurun_out/final/gputests.log
bash tools/final_r02.sh
timeout 1500 python bench.py --workload rmat28 --steps 2 --warmup 3 --cpu-budget 20 > gpurun_out/final/bench_rmat28.json 2> gpurun_out/final/bench_rmat28.err
tail -2 gpurun_out/final/bench_rmat28.err
