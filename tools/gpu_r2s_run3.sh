#!/bin/bash
# A/B: locality relabel x L1-allocating gathers (C4, C2, C3)
cd "$(dirname "$0")/.."
run() { # tag config env...
  tag=$1; cfg=$2; shift 2
  env "$@" timeout 600 python bench.py --config $cfg --no-e2e --no-cpu-baseline --no-parity --steps 20 --warmup 3 > gpurun_out/r2s_ab_$tag.json 2> gpurun_out/r2s_ab_$tag.err
  python -c "
import json;d=json.loads(open('gpurun_out/r2s_ab_$tag.json').read().strip().splitlines()[-1]);k=d['roofline']['kernels'];g=d['roofline']['gather_ceiling'];l=d['config']['layout']
print('$tag', round(d['value'],1), 'k1', round(k['k1_ms']*1e3,1), 'k2', round(k['k2_ms']*1e3,1), 'k3', round(k['k3_ms']*1e3,1), 'gc', round(g['a_ms']*1e3,1), round(g['at_ms']*1e3,1), 'relabel', l.get('relabel'), [round(x,3) for x in l.get('gather_sectors_per_nnz',[])], 'seg', l['segments'])" || tail -3 gpurun_out/r2s_ab_$tag.err
}
run c4_l0_g0 c4 RHP_LOCALITY=0
run c4_l0_gA c4 RHP_LOCALITY=0 RHP_L1_GATHER=A
run c4_l0_gT c4 RHP_LOCALITY=0 RHP_L1_GATHER=T
run c4_l0_g1 c4 RHP_LOCALITY=0 RHP_L1_GATHER=1
run c2_lm_g0 c2 RHP_LOCALITY=-1
run c2_l1_g0 c2 RHP_LOCALITY=1
run c2_l1_g1 c2 RHP_LOCALITY=1 RHP_L1_GATHER=1
run c3_lm_g0 c3 RHP_LOCALITY=-1
run c3_l1_g0 c3 RHP_LOCALITY=1
