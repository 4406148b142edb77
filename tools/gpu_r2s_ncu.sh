#!/bin/bash
# C4 evidence on the relabelled layout: full bench line, launch list, ncu
# full sections of K3/K1/K2 (summarised on the box), K1/K2 source pages.
cd "$(dirname "$0")/.."
TAG=${1:-r2s}
OUT=gpurun_out/$TAG
mkdir -p $OUT
c=c4
timeout 1500 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
tail -c 400 $OUT/bench_$c.json; echo
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 6000 -c 400 --csv \
    --log-file $OUT/launches_$c.csv python bench.py --config $c --steps 2 --warmup 1 --no-e2e \
    --no-cpu-baseline --no-parity --no-graph > /dev/null 2>&1
python tools/launch_share.py $OUT/launches_$c.csv --out $OUT/launches_$c.md > /dev/null 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -o $OUT/prof_$c -f python bench.py --config $c --warmup 2 --no-graph --no-e2e \
    --no-cpu-baseline --no-parity --profile-kernels 2 > $OUT/prof_$c.log 2>&1
python tools/ncu_summary.py $OUT/prof_$c.ncu-rep --out $OUT/ncu_${c}_kernels.md > /dev/null 2>&1
ncu -i $OUT/prof_$c.ncu-rep --page raw --csv > $OUT/ncu_${c}_raw.csv 2>/dev/null
ncu -i $OUT/prof_$c.ncu-rep --page details --csv > $OUT/ncu_${c}_details.csv 2>/dev/null
ncu -i $OUT/prof_$c.ncu-rep --page source --csv --kernel-name regex:"spmv_fused<rhp::EpiDual" \
    --launch-count 1 > $OUT/ncu_${c}_k1_source.csv 2>/dev/null
ncu -i $OUT/prof_$c.ncu-rep --page source --csv --kernel-name regex:"spmv_rows<rhp::EpiAty" \
    --launch-count 1 > $OUT/ncu_${c}_k2_source.csv 2>/dev/null
rm -f $OUT/prof_$c.ncu-rep
du -sh $OUT; ls $OUT
