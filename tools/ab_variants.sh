#!/bin/bash
# A/B of library variants built by tools/build_variant.sh (run on the GPU box).
#   tools/ab_variants.sh default s2a1 ...   (default = the in-tree build)
cd "$(dirname "$0")/.."
for v in "$@"; do
  if [ "$v" = default ]; then unset RHPDHG_LIB_DIR; else export RHPDHG_LIB_DIR=build/var_$v; fi
  for c in ${AB_CONFIGS:-c2 c3}; do
    timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/ab_${v}_$c.json 2> gpurun_out/ab_${v}_$c.err
    python -c "import json; d=json.loads(open('gpurun_out/ab_${v}_$c.json').read().strip().splitlines()[-1]); k=d['roofline']['kernels']; print('$v','$c',round(d['value']),'k1',round(k['k1_ms']*1e3,1),'k2',round(k['k2_ms']*1e3,1),'k3',round(k['k3_ms']*1e3,1))" || tail -3 gpurun_out/ab_${v}_$c.err
  done
done
