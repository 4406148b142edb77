#!/bin/bash
# Round evidence on one GPU: full bench lines (product + reference arm) and
# ncu captures. Outputs in gpurun_out/ev_*; copy the keepers to profiles/.
#   tools/evidence.sh TAG "c2 c1 c3 c4"
cd "$(dirname "$0")/.."
TAG=${1:-r1}
for c in ${2:-c2 c1 c3 c4}; do
  timeout 1500 python bench.py --config $c > gpurun_out/ev_${TAG}_$c.json 2> gpurun_out/ev_${TAG}_$c.err
  tail -c 300 gpurun_out/ev_${TAG}_$c.json; echo
done
timeout 900 python bench.py --impl reference > gpurun_out/ev_${TAG}_c2_reference.json 2> gpurun_out/ev_${TAG}_c2_reference.err
tail -c 300 gpurun_out/ev_${TAG}_c2_reference.json; echo
for c in ${PROFILE_CONFIGS:-c2 c4}; do
  timeout 900 tools/profile.sh $TAG $c > gpurun_out/prof_${TAG}_$c.log 2>&1 || tail -5 gpurun_out/prof_${TAG}_$c.log
done
ls -la gpurun_out | tail -20
