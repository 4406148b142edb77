#!/bin/bash
# A/B of programmatic dependent launch and the tuned gather policy on the
# bench configs:  tools/ab_pdl.sh "c2 c3 c4"
cd "$(dirname "$0")/.."
for c in ${1:-c2 c3}; do
  for pdl in 0 1; do
    RHP_PDL=$pdl timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 20 --warmup 5 \
      > gpurun_out/ab_${c}_pdl$pdl.json 2> gpurun_out/ab_${c}_pdl$pdl.err
    python -c "import json; d=json.loads(open('gpurun_out/ab_${c}_pdl$pdl.json').read().strip().splitlines()[-1]); print('$c pdl=$pdl', round(d['value']), d['config']['layout'].get('gather_l1'), {k: round(v, 4) for k, v in d['roofline']['kernels'].items()})" || tail -5 gpurun_out/ab_${c}_pdl$pdl.err
  done
done
