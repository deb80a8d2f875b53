cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_integration_cpp.py -x -q --timeout 800 > gpurun_out/b2_cpp.log 2>&1
echo "rc=$?" >> gpurun_out/b2_cpp.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/b2_bench.json 2> gpurun_out/b2_bench.err
for V in hybrid-plain nonatomic conventional hybrid-beamer; do
timeout 900 python bench.py --steps 2 --warmup 2 --variant $V --no-cpu-baseline --plugin-sources 0 > gpurun_out/b2_bench_$V.json 2> gpurun_out/b2_bench_$V.err
done
