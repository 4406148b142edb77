#!/bin/bash
# A/B: chunk-level L2 prefetch in the merge-path walk (C4, C2, C3)
cd "$(dirname "$0")/.."
run() { # tag config libvariant
  tag=$1; cfg=$2; v=$3
  if [ "$v" = default ]; then unset RHPDHG_LIB_DIR; else export RHPDHG_LIB_DIR=build/var_$v; fi
  timeout 600 python bench.py --config $cfg --no-e2e --no-cpu-baseline --no-parity --steps 20 --warmup 3 > gpurun_out/r2s_ab_$tag.json 2> gpurun_out/r2s_ab_$tag.err
  python -c "
import json;d=json.loads(open('gpurun_out/r2s_ab_$tag.json').read().strip().splitlines()[-1]);k=d['roofline']['kernels'];g=d['roofline']['gather_ceiling'];l=d['config']['layout']
print('$tag', round(d['value'],1), 'k1', round(k['k1_ms']*1e3,1), 'k2', round(k['k2_ms']*1e3,1), 'k3', round(k['k3_ms']*1e3,1), 'gc', round(g['a_ms']*1e3,1), round(g['at_ms']*1e3,1))" || tail -3 gpurun_out/r2s_ab_$tag.err
}
for c in c4 c2; do
  for v in default pf1 pf2 default; do run ${c}_$v $c $v; done
done
for v in default pf1 pf2; do run c3_$v c3 $v; done
