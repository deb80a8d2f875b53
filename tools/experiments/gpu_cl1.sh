cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q --timeout 600 -k "latency or pageable or deep or mesh or config2" > gpurun_out/c1_tests.log 2>&1
echo "rc=$?" >> gpurun_out/c1_tests.log
timeout 900 python bench.py --workload mesh4096 --steps 2 --warmup 2 --no-cpu-baseline --plugin-sources 0 > gpurun_out/c1_mesh.json 2> gpurun_out/c1_mesh.err
PBFS_LATENCY_CLUSTER=0 timeout 900 python bench.py --workload mesh4096 --steps 2 --warmup 2 --no-cpu-baseline --plugin-sources 0 > gpurun_out/c1_mesh_nocl.json 2> gpurun_out/c1_mesh_nocl.err
