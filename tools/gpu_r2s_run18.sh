#!/bin/bash
# A/B: resident cluster size at 512 threads per CTA (C1)
cd "$(dirname "$0")/.."
run() { # tag env...
  tag=$1; shift
  env "$@" timeout 600 python bench.py --config c1 --no-e2e --no-cpu-baseline --no-parity --steps 20 --warmup 3 > gpurun_out/r2s_ab_$tag.json 2> gpurun_out/r2s_ab_$tag.err
  python -c "
import json;d=json.loads(open('gpurun_out/r2s_ab_$tag.json').read().strip().splitlines()[-1])
print('$tag', round(d['value'],1))" || tail -3 gpurun_out/r2s_ab_$tag.err
}
run c1_def; run c1_cta4 RHP_RES_CTAS=4; run c1_cta2 RHP_RES_CTAS=2; run c1_def2; run c1_cta4b RHP_RES_CTAS=4
