cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -k "latency or pageable or deep or mesh" > gpurun_out/l2_tests.log 2>&1
echo "rc=$?" >> gpurun_out/l2_tests.log
timeout 900 python bench.py --workload mesh4096 --steps 2 --warmup 2 --no-cpu-baseline --plugin-sources 0 > gpurun_out/l2_mesh.json 2> gpurun_out/l2_mesh.err

PBFS_LIB=build/ab/libpbfs_nolocal.so timeout 900 python bench.py --workload mesh4096 --steps 2 --warmup 2 --no-cpu-baseline --plugin-sources 0 > gpurun_out/l2_mesh_nolocal.json 2> gpurun_out/l2_mesh_nolocal.err
timeout 900 python bench.py --workload rmat26 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/l2_rmat26.json 2> gpurun_out/l2_rmat26.err
