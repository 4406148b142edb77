#!/usr/bin/env bash
# Profiles the hot path under ncu on one GPU (run via gpurun). Outputs go to
# gpurun_out/; the summaries worth keeping are written to profiles/ by
# tools/summarize_ncu.py.
#   tools/profile.sh <tag> [config]
set -euo pipefail
TAG=${1:-r1}
CFG=${2:-c2}
OUT=gpurun_out
mkdir -p "$OUT"
# plain launches: ncu cannot profile kernel nodes of graphs with conditional nodes
BENCH="python bench.py --config $CFG --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-graph"
# 1) launch list with per-launch device time (cold-cache, serialised), past setup
ncu --metrics gpu__time_duration.sum --clock-control none -s ${SKIP:-700} -c 300 --csv \
    --log-file "$OUT/launches_${TAG}_${CFG}.csv" $BENCH > /dev/null
# 2) full sections of K3 / K1 / K2 on a live iterate: bench.py --profile-kernels
#    brackets exactly 2 launches of each with cudaProfilerStart/Stop
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -o "$OUT/prof_${TAG}_${CFG}" -f \
    python bench.py --config $CFG --warmup 2 --no-graph --profile-kernels 2 > /dev/null
echo "profile done: $OUT/launches_${TAG}_${CFG}.csv $OUT/prof_${TAG}_${CFG}.ncu-rep"
