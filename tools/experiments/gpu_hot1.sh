#!/bin/bash
# Hot-word mirror + reduction claim: parity and RMAT-26 / RMAT-20 / ER-24 A/B.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "owner_range or golden or reduction or size_gated or criterion_1 or hand" > gpurun_out/hot_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/hot_tests.log
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
ab() {
  local name=$1; shift
  r=$(env "$@" timeout 600 python bench.py --workload ${W:-rmat26} --no-cpu-baseline --plugin-sources 0 --steps 3 --warmup 3 2>gpurun_out/ab_$name.err)
  echo "${W:-rmat26} $name $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["config"].get("mean_bfs_ms"), d["roofline"]["frac"], d["e2e"]["value"])' 2>&1)" >> gpurun_out/hot_ab.txt
}
L=$PWD/build/ab
for W in rmat26 rmat20 er24; do
  export W
  ab hot512_noseg PBFS_SEG=0
  ab hot0_noseg PBFS_SEG=0 PBFS_HOT=0
  ab hot0build_noseg PBFS_SEG=0 PBFS_LIB=$L/libpbfs_hot0.so
  ab hot2048_noseg PBFS_SEG=0 PBFS_LIB=$L/libpbfs_hot2048.so
  ab hot2048_noseg_nored PBFS_SEG=0 PBFS_RED_MINQ=0 PBFS_LIB=$L/libpbfs_hot2048.so
  ab hot512_seg PBFS_X=1
done
