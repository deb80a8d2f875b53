cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,memory.total --format=csv > gpurun_out/r1_smi.txt 2>&1
nproc > gpurun_out/r1_nproc.txt; free -g >> gpurun_out/r1_nproc.txt
PBFS_GEN_TIMING=1 timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/r1_gputests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r1_gputests.log
PBFS_GEN_TIMING=1 timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r1_bench.json 2> gpurun_out/r1_bench.err
echo "bench rc=$?" >> gpurun_out/r1_bench.err
