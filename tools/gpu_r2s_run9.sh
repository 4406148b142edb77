#!/bin/bash
# C5 (1B nnz, one GPU): column-segment size A/B, then ncu traffic of K1/K2/K3
cd "$(dirname "$0")/.."
OUT=gpurun_out/r2s_c5; mkdir -p $OUT
run() { # tag env...
  tag=$1; shift
  env "$@" timeout 900 python bench.py --config c5 --no-e2e --no-cpu-baseline --no-parity --steps 5 --warmup 3 > $OUT/ab_$tag.json 2> $OUT/ab_$tag.err
  python -c "
import json;d=json.loads(open('$OUT/ab_$tag.json').read().strip().splitlines()[-1]);k=d['roofline']['kernels'];l=d['config']['layout']
print('$tag', round(d['value'],2), 'k1', round(k['k1_ms']*1e3,1), 'k2', round(k['k2_ms']*1e3,1), 'k3', round(k['k3_ms']*1e3,1), 'seg', l['segments'], 'relabel', l.get('relabel'), 'setup', round(d['config']['setup_s'],1))" || tail -3 $OUT/ab_$tag.err
}
run default
run s48 RHP_SEG_BYTES=50331648
run s96 RHP_SEG_BYTES=100663296
run s128 RHP_SEG_BYTES=134217728
timeout 1500 ncu --set full --clock-control none --profile-from-start off \
    -o $OUT/prof_c5 -f python bench.py --config c5 --warmup 2 --no-graph --no-e2e \
    --no-cpu-baseline --no-parity --profile-kernels 2 > $OUT/prof_c5.log 2>&1
python tools/ncu_summary.py $OUT/prof_c5.ncu-rep --out $OUT/ncu_c5_kernels.md > /dev/null 2>&1
ncu -i $OUT/prof_c5.ncu-rep --page raw --csv > $OUT/ncu_c5_raw.csv 2>/dev/null
rm -f $OUT/prof_c5.ncu-rep
ls $OUT
