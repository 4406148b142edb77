#!/bin/bash
# A/B: resident-kernel CTA size (C1); L1-allocating gathers on the relabelled A (C4)
cd "$(dirname "$0")/.."
run() { # tag config libvariant env...
  tag=$1; cfg=$2; v=$3; shift 3
  if [ "$v" = default ]; then unset RHPDHG_LIB_DIR; else export RHPDHG_LIB_DIR=build/var_$v; fi
  env "$@" timeout 600 python bench.py --config $cfg --no-e2e --no-cpu-baseline --no-parity --steps 20 --warmup 3 > gpurun_out/r2s_ab_$tag.json 2> gpurun_out/r2s_ab_$tag.err
  python -c "
import json;d=json.loads(open('gpurun_out/r2s_ab_$tag.json').read().strip().splitlines()[-1]);k=d['roofline']['kernels']
print('$tag', round(d['value'],1), 'k1', round(k['k1_ms']*1e3,2), 'k2', round(k['k2_ms']*1e3,2))" || tail -3 gpurun_out/r2s_ab_$tag.err
}
for v in default res512 res1024 default; do run c1_$v c1 $v; done
run c4_g0 c4 default
run c4_gA c4 default RHP_L1_GATHER=A
run c4_g0b c4 default
run c4_gAb c4 default RHP_L1_GATHER=A
