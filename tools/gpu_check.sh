#!/bin/bash
# GPU round trip used during development: GPU tests, then C2/C3 bench lines.
#   tools/gpu_check.sh [pytest-args]
cd "$(dirname "$0")/.."
timeout 1200 python -m pytest tests -m gpu -x -q ${@:--q} 2>&1 | tail -15
for c in c2 c3; do
  timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/chk_$c.json 2> gpurun_out/chk_$c.err
  python -c "import json; d=json.loads(open('gpurun_out/chk_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['value']), {k: round(v, 4) for k, v in d['roofline']['kernels'].items()})" || tail -5 gpurun_out/chk_$c.err
done
