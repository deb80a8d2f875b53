cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_cli.py -x -q --timeout 600 -s > gpurun_out/v1_tests.log 2>&1
echo "rc=$?" >> gpurun_out/v1_tests.log
