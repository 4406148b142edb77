#!/bin/bash
# Round-2 (final build) evidence on one GPU (run via gpurun): bench lines of every config,
# the reference arm, ncu launch lists and full captures of the hot kernels
# (summarised ON THE BOX; the .ncu-rep files are deleted), the cuSPARSE
# comparison. Keepers are copied into profiles/ afterwards.
#   tools/evidence_r2.sh TAG ["c4 c2 c3 c1 c5"] ["c4 c2 c3"]
cd "$(dirname "$0")/.."
TAG=${1:-r2s}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for c in ${2:-c4 c2 c3 c1 c5}; do
  extra=""
  [ $c = c5 ] && extra="--steps 5"
  [ $c = c2 ] && extra="--no-parity"
  timeout 1500 python bench.py --config $c $extra > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  tail -c 300 $OUT/bench_$c.json; echo; tail -2 $OUT/bench_$c.err
done
timeout 900 python bench.py --impl reference > $OUT/bench_c4_reference.json 2> $OUT/bench_c4_reference.err
for c in ${3:-c4 c2 c3}; do
  case $c in c4) SKIP=1200;; c5) SKIP=8000;; *) SKIP=700;; esac
  # launch list with per-launch device time of the bench command (plain
  # launches: ncu cannot time kernel nodes of conditional graphs), past setup
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s $SKIP -c 400 --csv \
      --log-file $OUT/launches_$c.csv python bench.py --config $c --steps 2 --warmup 1 --no-e2e \
      --no-cpu-baseline --no-parity --no-graph > /dev/null 2>&1
  python tools/launch_share.py $OUT/launches_$c.csv --out $OUT/launches_$c.md > /dev/null 2>&1
  # full sections of K3 / K1 / K2 on a live iterate (--profile-kernels brackets them)
  timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off \
      -o $OUT/prof_$c -f python bench.py --config $c --warmup 2 --no-graph --no-e2e \
      --no-cpu-baseline --no-parity --profile-kernels 2 > $OUT/prof_$c.log 2>&1
  python tools/ncu_summary.py $OUT/prof_$c.ncu-rep --out $OUT/ncu_${c}_kernels.md > /dev/null 2>&1
  ncu -i $OUT/prof_$c.ncu-rep --page raw --csv > $OUT/ncu_${c}_raw.csv 2>/dev/null
  ncu -i $OUT/prof_$c.ncu-rep --page source --csv --kernel-name regex:spmv_fused \
      --launch-count 1 > $OUT/ncu_${c}_k1_source.csv 2>/dev/null
  ncu -i $OUT/prof_$c.ncu-rep --page source --csv --kernel-name regex:spmv_rows \
      --launch-count 1 > $OUT/ncu_${c}_k2_source.csv 2>/dev/null
  ncu -i $OUT/prof_$c.ncu-rep --page details --csv > $OUT/ncu_${c}_details.csv 2>/dev/null
  rm -f $OUT/prof_$c.ncu-rep
done
timeout 900 python tools/cusparse_compare.py --configs c2,c3,c4 --out $OUT/cusparse_compare.json \
    > $OUT/cusparse.log 2>&1
du -sh $OUT; ls $OUT
