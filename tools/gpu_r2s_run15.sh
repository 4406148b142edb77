#!/bin/bash
# A/B on C4 K2 (thread-per-row, 4 CTAs/SM): 2 rows in flight; L1 gathers on A^T too
cd "$(dirname "$0")/.."
run() { # tag libvariant env...
  tag=$1; v=$2; shift 2
  if [ "$v" = default ]; then unset RHPDHG_LIB_DIR; else export RHPDHG_LIB_DIR=build/var_$v; fi
  env "$@" timeout 600 python bench.py --config c4 --no-e2e --no-cpu-baseline --no-parity --steps 20 --warmup 3 > gpurun_out/r2s_ab_$tag.json 2> gpurun_out/r2s_ab_$tag.err
  python -c "
import json;d=json.loads(open('gpurun_out/r2s_ab_$tag.json').read().strip().splitlines()[-1]);k=d['roofline']['kernels']
print('$tag', round(d['value'],1), 'k1', round(k['k1_ms']*1e3,2), 'k2', round(k['k2_ms']*1e3,2), 'k3', round(k['k3_ms']*1e3,2))" || tail -3 gpurun_out/r2s_ab_$tag.err
}
run c4_def default
run c4_rf2 rf2
run c4_l1both default RHP_L1_GATHER=1
run c4_def2 default
run c4_rf2b rf2
run c4_l1bothb default RHP_L1_GATHER=1
