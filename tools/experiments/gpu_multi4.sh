cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_multi_engine.py tests/test_multigpu.py -x -q --timeout 300 > gpurun_out/m4_tests.log 2>&1
echo "rc=$?" >> gpurun_out/m4_tests.log
timeout 900 python tools/multi_profile.py rmat20 mesh4096 rmat26 > gpurun_out/m4_profile.txt 2> gpurun_out/m4_profile.err
echo "rc=$?" >> gpurun_out/m4_profile.txt
