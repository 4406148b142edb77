#!/bin/bash
# A/B of one environment switch on the bench configs:
#   tools/ab_env.sh VAR "v1 v2" "c2 c3 c4"
cd "$(dirname "$0")/.."
var=$1
for c in ${3:-c2 c3}; do
  for v in $2; do
    env $var=$v timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 20 --warmup 5 \
      > gpurun_out/ab_${c}_${var}$v.json 2> gpurun_out/ab_${c}_${var}$v.err
    python -c "import json; d=json.loads(open('gpurun_out/ab_${c}_${var}$v.json').read().strip().splitlines()[-1]); L=d['config']['layout']; print('$c $var=$v', round(d['value']), L.get('gather_l1'), L.get('thread_rows'), {k: round(v, 4) for k, v in d['roofline']['kernels'].items()})" || tail -5 gpurun_out/ab_${c}_${var}$v.err
  done
done
