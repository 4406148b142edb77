#!/bin/bash
# A/B: streaming (evict-first) epilogue-input loads (C4, C2, C5)
cd "$(dirname "$0")/.."
run() { # tag config steps libvariant
  tag=$1; cfg=$2; st=$3; v=$4
  if [ "$v" = default ]; then unset RHPDHG_LIB_DIR; else export RHPDHG_LIB_DIR=build/var_$v; fi
  timeout 900 python bench.py --config $cfg --no-e2e --no-cpu-baseline --no-parity --steps $st --warmup 3 > gpurun_out/r2s_ab_$tag.json 2> gpurun_out/r2s_ab_$tag.err
  python -c "
import json;d=json.loads(open('gpurun_out/r2s_ab_$tag.json').read().strip().splitlines()[-1]);k=d['roofline']['kernels']
print('$tag', round(d['value'],2), 'k1', round(k['k1_ms']*1e3,1), 'k2', round(k['k2_ms']*1e3,1), 'k3', round(k['k3_ms']*1e3,1))" || tail -3 gpurun_out/r2s_ab_$tag.err
}
for v in default epics default epics; do run c4_$v c4 20 $v; done
for v in default epics; do run c2_$v c2 20 $v; done
for v in default epics; do run c5_$v c5 5 $v; done
