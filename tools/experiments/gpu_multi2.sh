cd $GRAFT_REPO_ROOT
timeout 900 python tools/multi_profile.py rmat20 mesh4096 er24 rmat26 > gpurun_out/m2_profile.txt 2> gpurun_out/m2_profile.err
echo "rc=$?" >> gpurun_out/m2_profile.txt
for G in 2 8; do
timeout 600 python bench.py --partitions $G --steps 2 --warmup 1 > gpurun_out/m2_bench_p$G.json 2> gpurun_out/m2_bench_p$G.err
done
