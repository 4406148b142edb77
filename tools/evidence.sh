#!/bin/bash
# Round evidence on one GPU: GPU tests, full bench lines (product + reference
# arm) and ncu captures summarised ON THE BOX (the .ncu-rep files are deleted
# afterwards: gpurun copies back at most 64 MiB). Keepers go to profiles/.
#   tools/evidence.sh TAG "c2 c1 c3 c4 c5" "c2 c4 c5"
cd "$(dirname "$0")/.."
TAG=${1:-r1}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/ev_${TAG}_pytest.log 2>&1; tail -2 gpurun_out/ev_${TAG}_pytest.log
for c in ${2:-c2 c1 c3 c4 c5}; do
  extra=""
  # C5: 1e-8 is out of reach in a bench run; time to 1e-4 with a 30k-iteration cap
  [ $c = c5 ] && extra="--steps 5 --e2e-eps 1e-4 --e2e-cap 30000"
  timeout 1800 python bench.py --config $c $extra > gpurun_out/ev_${TAG}_$c.json 2> gpurun_out/ev_${TAG}_$c.err
  tail -c 200 gpurun_out/ev_${TAG}_$c.json; echo; tail -3 gpurun_out/ev_${TAG}_$c.err
done
if [ -n "${REF:-1}" ]; then
  timeout 900 python bench.py --impl reference > gpurun_out/ev_${TAG}_c2_reference.json 2> gpurun_out/ev_${TAG}_c2_reference.err
  tail -c 200 gpurun_out/ev_${TAG}_c2_reference.json; echo
fi
for c in ${3:-c2 c4 c5}; do
  case $c in c4) export SKIP=4000;; c5) export SKIP=8000;; *) export SKIP=700;; esac
  timeout 1200 tools/profile.sh $TAG $c > gpurun_out/prof_${TAG}_$c.log 2>&1 || tail -5 gpurun_out/prof_${TAG}_$c.log
  python tools/ncu_summary.py gpurun_out/prof_${TAG}_$c.ncu-rep --out gpurun_out/${TAG}_ncu_${c}_kernels.md > /dev/null 2>&1
  ncu -i gpurun_out/prof_${TAG}_$c.ncu-rep --page raw --csv > gpurun_out/${TAG}_ncu_${c}_raw.csv 2>/dev/null
  python tools/launch_share.py gpurun_out/launches_${TAG}_$c.csv --out gpurun_out/${TAG}_launches_$c.md > /dev/null 2>&1
  rm -f gpurun_out/prof_${TAG}_$c.ncu-rep
done
du -sh gpurun_out; ls gpurun_out | grep ${TAG}
