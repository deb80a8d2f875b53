cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_multi_engine.py -x -q --timeout 120 > gpurun_out/m1_tests.log 2>&1
echo "rc=$?" >> gpurun_out/m1_tests.log
