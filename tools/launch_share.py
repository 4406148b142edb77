"""Per-kernel share of device time from an ncu launch list
(`ncu --metrics gpu__time_duration.sum --csv --log-file <csv>`), as markdown.

    python tools/launch_share.py gpurun_out/launches_<tag>_<cfg>.csv [--out profiles/<file>.md]
"""
import argparse
import collections
import csv
import re


def short(name):
    m = re.search(r"(spmv_fused|spmv_rows|spmv_cta_rows|epilogue_walk|k_\w+)<(?:rhp::)?(\w+)>", name)
    if m:
        return f"{m.group(1)}<{m.group(2)}>"
    return name.split("(")[0].replace("void ", "").replace("rhp::", "")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--out")
    ap.add_argument("--title", default="")
    args = ap.parse_args()
    rows = list(csv.reader(open(args.csv)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    d = collections.defaultdict(list)
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(r[ui], 1e-3)
        d[short(r[ki])].append(v * scale)
    tot = sum(sum(v) for v in d.values())
    out = [f"# Launch list share{(' — ' + args.title) if args.title else ''}", "",
           f"Source: `{args.csv}` (ncu gpu__time_duration.sum, --clock-control none; cold-cache, serialised "
           "launches, so only the shares are comparable with live timings).", "",
           "Profiled with plain launches (`--no-graph`): a block enqueues its iterations up to the next "
           "scheduled check, and launches past an earlier stop (a restart verdict) exit at entry — the "
           "short launches; 'working' = launches taking at least half of the kernel's maximum.", "",
           "| kernel | launches | working | mean us (working) | max us | share of device time |",
           "|---|---|---|---|---|---|"]
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        w = [t for t in v if t >= 0.5 * max(v)]
        out.append(f"| {k} | {len(v)} | {len(w)} | {sum(w) / len(w):.1f} | {max(v):.1f} | "
                   f"{sum(v) / tot:.3f} |")
    text = "\n".join(out) + "\n"
    if args.out:
        open(args.out, "w").write(text)
    print(text)


if __name__ == "__main__":
    main()
