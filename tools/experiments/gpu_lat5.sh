#!/bin/bash
# k-level latency rounds: parity (latency-mode tests, mesh configs, smoke) + mesh A/B over k.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -k "latency or mesh or hand or criterion_1 or long_path or deeper" > gpurun_out/lat5_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/lat5_tests.log
for L in 2 4 6; do
  PBFS_LIB=$PWD/build/ab/libpbfs_lv$L.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -k "latency or mesh or long_path or deeper" >> gpurun_out/lat5_tests.log 2>&1
  echo "tests lv$L rc=$?" >> gpurun_out/lat5_tests.log
done
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/lat5_tests.log 2>&1
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
ab() {
  local name=$1; shift
  r=$(env "$@" timeout 600 python bench.py --workload ${W:-mesh4096} --no-cpu-baseline --plugin-sources 0 --steps 2 --warmup 3 2>gpurun_out/ab_$name.err)
  echo "${W:-mesh4096} $name $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["config"].get("mean_bfs_ms"), d["roofline"]["frac"], d["e2e"]["value"])' 2>&1)" >> gpurun_out/lat5_ab.txt
}
ab lv3 PBFS_X=1
ab lv1 PBFS_LIB=$PWD/build/ab/libpbfs_lv1.so
ab lv2 PBFS_LIB=$PWD/build/ab/libpbfs_lv2.so
ab lv4 PBFS_LIB=$PWD/build/ab/libpbfs_lv4.so
ab lv5 PBFS_LIB=$PWD/build/ab/libpbfs_lv5.so
ab lv6 PBFS_LIB=$PWD/build/ab/libpbfs_lv6.so
