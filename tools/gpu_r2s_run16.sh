#!/bin/bash
# A/B: merge-path row ends one window ahead (RHP_RP_AHEAD) — speed and bitwise identity
cd "$(dirname "$0")/.."
run() { # tag config libvariant
  tag=$1; cfg=$2; v=$3
  if [ "$v" = default ]; then unset RHPDHG_LIB_DIR; else export RHPDHG_LIB_DIR=build/var_$v; fi
  timeout 600 python bench.py --config $cfg --no-e2e --no-cpu-baseline --no-parity --steps 20 --warmup 3 > gpurun_out/r2s_ab_$tag.json 2> gpurun_out/r2s_ab_$tag.err
  python -c "
import json;d=json.loads(open('gpurun_out/r2s_ab_$tag.json').read().strip().splitlines()[-1]);k=d['roofline']['kernels']
print('$tag', round(d['value'],1), 'k1', round(k['k1_ms']*1e3,2), 'k2', round(k['k2_ms']*1e3,2), 'k3', round(k['k3_ms']*1e3,2))" || tail -3 gpurun_out/r2s_ab_$tag.err
}
for c in c4 c2 c3; do
  run ${c}_rp1 $c default; run ${c}_rp0 $c rp0; run ${c}_rp1b $c default; run ${c}_rp0b $c rp0
done
for c in c2 c4; do
  unset RHPDHG_LIB_DIR; python tools/bitwise_check.py $c 200 /tmp/bw_${c}_1.npz
  RHPDHG_LIB_DIR=build/var_rp0 python tools/bitwise_check.py $c 200 /tmp/bw_${c}_0.npz
  python -c "
import numpy as np; a=np.load('/tmp/bw_${c}_1.npz'); b=np.load('/tmp/bw_${c}_0.npz')
print('$c bitwise x', np.array_equal(a['x'], b['x']), 'y', np.array_equal(a['y'], b['y']))"
done
