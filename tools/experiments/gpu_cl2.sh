cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "latency or pageable or deep" > gpurun_out/c2_tests.log 2>&1
echo "rc=$?" >> gpurun_out/c2_tests.log
B="python bench.py --workload mesh4096 --steps 2 --warmup 2 --no-cpu-baseline --plugin-sources 0"
timeout 900 $B > gpurun_out/c2_mesh_cl.json 2> gpurun_out/c2_mesh_cl.err
PBFS_LATENCY_CLUSTER=0 timeout 900 $B > gpurun_out/c2_mesh_spread.json 2> gpurun_out/c2_mesh_spread.err
PBFS_LATENCY_CLUSTER=0 PBFS_LIB=build/ab/libpbfs_nospread.so timeout 900 $B > gpurun_out/c2_mesh_base.json 2> gpurun_out/c2_mesh_base.err
