#!/bin/bash
# A/B: long-row (CTA row run) engine batch / unroll / occupancy on C3 (K1 and plain A x vs cuSPARSE)
cd "$(dirname "$0")/.."
run() { # tag libvariant
  tag=$1; v=$2
  if [ "$v" = default ]; then unset RHPDHG_LIB_DIR; else export RHPDHG_LIB_DIR=build/var_$v; fi
  timeout 600 python bench.py --config c3 --no-e2e --no-cpu-baseline --no-parity --steps 20 --warmup 3 > gpurun_out/r2s_ab_c3_$tag.json 2> gpurun_out/r2s_ab_c3_$tag.err
  python -c "
import json;d=json.loads(open('gpurun_out/r2s_ab_c3_$tag.json').read().strip().splitlines()[-1]);k=d['roofline']['kernels'];g=d['roofline']['gather_ceiling']
print('c3 $tag', round(d['value'],1), 'k1', round(k['k1_ms']*1e3,2), 'k2', round(k['k2_ms']*1e3,2), 'k3', round(k['k3_ms']*1e3,2), 'gc', round(g['a_ms']*1e3,2))" || tail -3 gpurun_out/r2s_ab_c3_$tag.err
  timeout 600 python tools/cusparse_compare.py --configs c3 --out gpurun_out/r2s_cusp_c3_$tag.json > /dev/null 2>&1
  python -c "
import json;d=json.load(open('gpurun_out/r2s_cusp_c3_$tag.json'))
for r in d: print('   ', r['op'], 'ours', round(r['ours_us'],2), 'cusparse', round(r['cusparse_alg1_us'],2), round(r['speedup_vs_best_cusparse'],3))"
}
for v in default b4u2 b4u4 b3u4 b4u4k3 default; do run $v $v; done
