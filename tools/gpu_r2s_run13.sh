#!/bin/bash
# A/B: forced column segments on the relabelled C4 (x = 200 MB > L2)
cd "$(dirname "$0")/.."
run() { # tag env...
  tag=$1; shift
  env "$@" timeout 600 python bench.py --config c4 --no-e2e --no-cpu-baseline --no-parity --steps 20 --warmup 3 > gpurun_out/r2s_ab_$tag.json 2> gpurun_out/r2s_ab_$tag.err
  python -c "
import json;d=json.loads(open('gpurun_out/r2s_ab_$tag.json').read().strip().splitlines()[-1]);k=d['roofline']['kernels'];l=d['config']['layout']
print('$tag', round(d['value'],1), 'k1', round(k['k1_ms']*1e3,1), 'k2', round(k['k2_ms']*1e3,1), 'seg', l['segments'])" || tail -3 gpurun_out/r2s_ab_$tag.err
}
run c4_seg1
run c4_seg2 RHP_SEG_FORCE=1 RHP_SEG_BYTES=104857600
run c4_seg3 RHP_SEG_FORCE=1 RHP_SEG_BYTES=70000000
run c4_seg4 RHP_SEG_FORCE=1 RHP_SEG_BYTES=52428800
