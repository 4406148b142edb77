#!/bin/bash
# A/B: thread-per-row engine forced on C4's A (RHP_THREAD_ROWS cap)
cd "$(dirname "$0")/.."
run() { # tag config env...
  tag=$1; cfg=$2; shift 2
  env "$@" timeout 600 python bench.py --config $cfg --no-e2e --no-cpu-baseline --no-parity --steps 20 --warmup 3 > gpurun_out/r2s_ab_$tag.json 2> gpurun_out/r2s_ab_$tag.err
  python -c "
import json;d=json.loads(open('gpurun_out/r2s_ab_$tag.json').read().strip().splitlines()[-1]);k=d['roofline']['kernels'];g=d['roofline']['gather_ceiling'];l=d['config']['layout']
print('$tag', round(d['value'],1), 'k1', round(k['k1_ms']*1e3,1), 'k2', round(k['k2_ms']*1e3,1), 'k3', round(k['k3_ms']*1e3,1), 'gc', round(g['a_ms']*1e3,1), round(g['at_ms']*1e3,1), 'grids', l['grid_a'], l['grid_at'], l['thread_rows'])" || tail -3 gpurun_out/r2s_ab_$tag.err
}
run c4_tr_def c4
run c4_tr500 c4 RHP_THREAD_ROWS=500
