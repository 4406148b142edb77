#!/bin/bash
# A/B of device variants on one GPU: each line "label ENV=... -- bench args".
# Prints value (iter/s), K1/K2/K3 ms and the dominant kernel's HBM fraction.
#   tools/ab_runs.sh "label1|ENV=1|--config c3" "label2||--config c3" ...
cd "$(dirname "$0")/.."
for spec in "$@"; do
  IFS='|' read -r label envs args <<< "$spec"
  env $envs timeout 900 python bench.py --no-e2e --no-cpu-baseline --no-parity $args \
      > gpurun_out/ab_$label.json 2> gpurun_out/ab_$label.err
  python - "$label" <<'PY'
import json, sys
label = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab_{label}.json").read().strip().splitlines()[-1])
    k = d["roofline"]["kernels"]
    print(f"{label:28s} {d['value']:10.1f} iter/s  K1 {k['k1_ms']*1e3:8.1f} us  K2 {k['k2_ms']*1e3:8.1f} us"
          f"  K3 {k['k3_ms']*1e3:7.1f} us  frac {d['roofline']['frac']:.3f}  layout {d['config']['layout'].get('segments')} {d['config']['layout'].get('cta_rows')}")
except Exception as e:
    print(label, "FAILED", e, open(f"gpurun_out/ab_{label}.err").read()[-800:])
PY
done
