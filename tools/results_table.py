"""Markdown results table from a directory of bench.py JSON lines
(tools/evidence_r2s.sh output): python tools/results_table.py gpurun_out/r2s_final"""
import json
import sys
from pathlib import Path


def last(p):
    return json.loads(Path(p).read_text().strip().splitlines()[-1])


def main(d):
    d = Path(d)
    print("| config | GPU iter/s | K1 / K2 µs | dominant kernel HBM frac | iteration GB/s | e2e to tol | iterations | reference CPU iter/s |")
    print("|---|---|---|---|---|---|---|---|")
    for c in ("c4", "c2", "c3", "c1", "c5"):
        p = d / f"bench_{c}.json"
        if not p.exists():
            continue
        try:
            b = last(p)
        except Exception as e:  # noqa: BLE001
            print(f"| {c} | error {e} |")
            continue
        r = b.get("roofline", {})
        k = r.get("kernels", {})
        e = b.get("e2e") or {}
        cpu = b.get("cpu_baseline") or {}
        print(f"| {c.upper()} | {b['value']:.1f} | {k.get('k1_ms', 0) * 1e3:.1f} / {k.get('k2_ms', 0) * 1e3:.1f} | "
              f"{r.get('frac', 0):.3f} | {k.get('iteration_gbs_in_loop', 0):.0f} | "
              f"{e.get('time_to_tol_s', e.get('time_s', float('nan'))) if e else '—'} s ({e.get('status', '—')}) | "
              f"{e.get('iterations', '—')} | {cpu.get('value', float('nan')):.3g} |")


if __name__ == "__main__":
    main(sys.argv[1])
