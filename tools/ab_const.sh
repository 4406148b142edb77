#!/bin/bash
# A/B of the constant-bound epilogue inputs (RHP_CONST_INPUTS) on C3 and C4.
set -u
out=gpurun_out/${1:-ab_const}
mkdir -p $out
for cfg in c4 c3; do
  for f in 1 0 1 0; do
    RHP_CONST_INPUTS=$f python bench.py --config $cfg --no-e2e --no-cpu-baseline --no-parity \
      >> $out/${cfg}_$f.jsonl 2>> $out/err.log
  done
done
python - "$out" <<'PY'
import json, sys, glob, os
for f in sorted(glob.glob(sys.argv[1] + "/*.jsonl")):
    rows = [json.loads(l) for l in open(f) if l.startswith("{")]
    ks = [r["roofline"].get("kernels", {}) for r in rows]
    print(os.path.basename(f), [round(r["value"], 1) for r in rows],
          [(round(k["k1_ms"], 4), round(k["k2_ms"], 4)) for k in ks])
PY
