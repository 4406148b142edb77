export RHPDHG_SETUP_TRACE=0
for loc in -1 0; do
  RHP_LOCALITY=$loc timeout 600 python bench.py --config c4 --no-e2e --no-cpu-baseline --no-parity --steps 20 --warmup 3 > gpurun_out/r2s_ab_loc$loc.json 2> gpurun_out/r2s_ab_loc$loc.err
  echo loc=$loc rc=$?
done
timeout 900 python -m pytest tests/test_locality.py tests/test_sanitizer.py -m gpu -q > gpurun_out/r2s_loc_tests.log 2>&1; echo loctests rc=$?
timeout 1500 python -m pytest tests/test_bench_parity.py -m gpu -q -k c4 > gpurun_out/r2s_bp_c4.log 2>&1; echo bp rc=$?
