cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_multi_engine.py tests/test_multigpu.py -x -q --timeout 300 > gpurun_out/m3_tests.log 2>&1
echo "rc=$?" >> gpurun_out/m3_tests.log
timeout 900 python tools/multi_profile.py rmat20 mesh4096 rmat26 > gpurun_out/m3_profile.txt 2> gpurun_out/m3_profile.err
echo "rc=$?" >> gpurun_out/m3_profile.txt
PBFS_MULTI_SYS_SCOPE=1 timeout 900 python tools/multi_profile.py rmat20 rmat26 > gpurun_out/m3_profile_sys.txt 2> gpurun_out/m3_profile_sys.err
