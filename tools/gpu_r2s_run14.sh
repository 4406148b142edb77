#!/bin/bash
# A/B: programmatic dependent launch of the SpMVs (RHP_PDL=1) on the final build
cd "$(dirname "$0")/.."
run() { # tag config env...
  tag=$1; cfg=$2; shift 2
  env "$@" timeout 600 python bench.py --config $cfg --no-e2e --no-cpu-baseline --no-parity --steps 20 --warmup 3 > gpurun_out/r2s_ab_$tag.json 2> gpurun_out/r2s_ab_$tag.err
  python -c "
import json;d=json.loads(open('gpurun_out/r2s_ab_$tag.json').read().strip().splitlines()[-1]);k=d['roofline']['kernels'];l=d['config']['layout']
print('$tag', round(d['value'],1), 'k1', round(k['k1_ms']*1e3,2), 'k2', round(k['k2_ms']*1e3,2), 'pdl', l['pdl'])" || tail -3 gpurun_out/r2s_ab_$tag.err
}
for c in c3 c2 c4; do
  run ${c}_pdl0 $c
  run ${c}_pdl1 $c RHP_PDL=1
  run ${c}_pdl0b $c
  run ${c}_pdl1b $c RHP_PDL=1
done
