#!/bin/bash
# e2e (pbfs_bfs_batch) A/B: transfer slots in flight and widening threads.
# Prints: workload name value e2e batch-ms-per-source.
export PBFS_GRAPH_CACHE_DIR=/tmp/pbfs_graphs
w=${1:-rmat26}
run() { local name=$1; shift
  env "$@" timeout 900 python bench.py --workload $w --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/e2e_$name.json 2>/dev/null
  echo "$w $name $(python -c "import json;d=json.load(open('gpurun_out/e2e_$name.json'));e=d['e2e'];print(d['value'], e['value'], e['batch_ms_per_source'])")"
}
run s2 PBFS_BATCH_SLOTS=2
run s4 PBFS_BATCH_SLOTS=4
run s4t16 PBFS_BATCH_SLOTS=4 PBFS_WIDEN_THREADS=16
