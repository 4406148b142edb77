"""profiles/ncu_traffic.json entries from `ncu --page raw --csv` exports of a
`bench.py --profile-kernels 2` capture (K3, K1, K2 launched twice each on a
live iterate; a column-segmented operator's K1 / K2 is its segment launches
in order): DRAM read + write bytes per launch of K1, K2 and K3.

    python tools/traffic_from_ncu.py gpurun_out/r2m/ncu_c4_raw.csv c4 --source profiles/r2_ncu_c4_kernels.md
"""
import argparse
import csv
import io
import json
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def load(path):
    rows = list(csv.reader(io.StringIO(Path(path).read_text())))
    h = rows[0]
    out = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        rd = float(r[h.index("dram__bytes_read.sum")] or 0)
        wr = float(r[h.index("dram__bytes_write.sum")] or 0)
        ur = rows[1][h.index("dram__bytes_read.sum")]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(ur, 1)
        uw = rows[1][h.index("dram__bytes_write.sum")]
        scale_w = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(uw, 1)
        out.append((name, rd * scale + wr * scale_w))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("raw")
    ap.add_argument("config")
    ap.add_argument("--source", default="")
    a = ap.parse_args()
    launches = load(a.raw)
    # per kernel family: K3 = EpiPrimal walk, K1 = EpiDual (+ its preceding
    # EpiSegStore segments), K2 = EpiAty (+ its segments)
    k1 = k2 = k3 = 0.0
    n1 = n2 = n3 = 0
    pending = 0.0
    for name, b in launches:
        if "EpiPrimal" in name:
            k3 += b
            n3 += 1
        elif "EpiSegStore" in name or re.search(r"EpiStore", name):
            pending += b
        elif "EpiDual" in name:
            k1 += b + pending
            n1 += 1
            pending = 0.0
        elif "EpiAty" in name:
            k2 += b + pending
            n2 += 1
            pending = 0.0
    f = ROOT / "profiles" / "ncu_traffic.json"
    d = json.loads(f.read_text()) if f.exists() else {}
    d[a.config] = {"source": a.source or a.raw, "k1": round(k1 / max(n1, 1)),
                   "k2": round(k2 / max(n2, 1)), "k3": round(k3 / max(n3, 1))}
    f.write_text(json.dumps(d, indent=1) + "\n")
    print(a.config, d[a.config])


if __name__ == "__main__":
    main()
