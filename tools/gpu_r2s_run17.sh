#!/bin/bash
# A/B: merge-path index/value stream with L1::no_allocate (RHP_STREAM_NA)
cd "$(dirname "$0")/.."
run() { # tag config libvariant
  tag=$1; cfg=$2; v=$3
  if [ "$v" = default ]; then unset RHPDHG_LIB_DIR; else export RHPDHG_LIB_DIR=build/var_$v; fi
  timeout 600 python bench.py --config $cfg --no-e2e --no-cpu-baseline --no-parity --steps 20 --warmup 3 > gpurun_out/r2s_ab_$tag.json 2> gpurun_out/r2s_ab_$tag.err
  python -c "
import json;d=json.loads(open('gpurun_out/r2s_ab_$tag.json').read().strip().splitlines()[-1]);k=d['roofline']['kernels']
print('$tag', round(d['value'],1), 'k1', round(k['k1_ms']*1e3,2), 'k2', round(k['k2_ms']*1e3,2), 'k3', round(k['k3_ms']*1e3,2))" || tail -3 gpurun_out/r2s_ab_$tag.err
}
for c in c4 c2; do
  run ${c}_def $c default; run ${c}_sna $c sna; run ${c}_defb $c default; run ${c}_snab $c sna
done
