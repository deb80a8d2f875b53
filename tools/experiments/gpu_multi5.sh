cd $GRAFT_REPO_ROOT
for W in all visited none; do for SC in 1 0; do
echo "== window=$W small_chunks=$SC" >> gpurun_out/m5_profile.txt
PBFS_MULTI_WINDOW=$W PBFS_MULTI_SMALL_CHUNKS=$SC timeout 600 python tools/multi_profile.py rmat26 >> gpurun_out/m5_profile.txt 2>> gpurun_out/m5_profile.err
done; done
