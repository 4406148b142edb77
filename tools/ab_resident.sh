#!/bin/bash
# C1 cluster-resident kernel: CTAs per cluster x threads per CTA.
#   tools/ab_resident.sh "default rt512 rt1024" "4 8 16"
cd "$(dirname "$0")/.."
for v in ${1:-default}; do
  if [ "$v" = default ]; then unset RHPDHG_LIB_DIR; else export RHPDHG_LIB_DIR=build/var_$v; fi
  for n in ${2:-16}; do
    RHP_RES_CTAS=$n timeout 300 python bench.py --config c1 --no-e2e --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/res_${v}_$n.json 2> gpurun_out/res_${v}_$n.err
    python -c "import json; d=json.loads(open('gpurun_out/res_${v}_$n.json').read().strip().splitlines()[-1]); print('$v ctas=$n', round(d['value']))" || tail -3 gpurun_out/res_${v}_$n.err
  done
done
