cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -x -q --timeout 600 > gpurun_out/l1_tests.log 2>&1
echo "rc=$?" >> gpurun_out/l1_tests.log
timeout 900 python bench.py --workload mesh4096 --steps 2 --warmup 2 --no-cpu-baseline --plugin-sources 0 > gpurun_out/l1_mesh.json 2> gpurun_out/l1_mesh.err
timeout 900 python bench.py --workload rmat26 --steps 3 --warmup 3 --no-cpu-baseline --plugin-sources 0 > gpurun_out/l1_rmat26.json 2> gpurun_out/l1_rmat26.err
