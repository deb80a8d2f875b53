#!/usr/bin/env bash
# Profiles the bench command on a GPU box (run under gpurun). Each ncu pass
# follows a plain run of the identical command that exited 0.
#   tools/profile_bench.sh WORKLOAD OUTDIR
set -euo pipefail
W=${1:-rmat26}
OUT=${2:-gpurun_out}
CMD="python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline"
mkdir -p "$OUT"
$CMD > "$OUT/plain_$W.json" 2> "$OUT/plain_$W.log"
# 1) launch list: every traversal launch with its device time
ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:bfs_(persistent|latency)' -c 200 \
    --csv --log-file "$OUT/launches_$W.csv" $CMD > "$OUT/ncu_launches_$W.log" 2>&1
# 2) one full capture of the first warm-up launch (source index 0)
ncu --set full --clock-control none --import-source on -k 'regex:bfs_(persistent|latency)' -s 64 -c 1 \
    -o "$OUT/full_$W" $CMD > "$OUT/ncu_full_$W.log" 2>&1
echo done
