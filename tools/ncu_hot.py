"""Hottest SASS instructions of a kernel in an ncu report (source page).

    python tools/ncu_hot.py gpurun_out/prof_x.ncu-rep [--kernel EpiDual] [--top 25] [--ctx 2]

Prints each hot instruction's share of the warp-stall samples, its address
and the preceding instructions (the stall is charged to the instruction that
waits, so the producer is usually just above it).
"""
import argparse
import csv
import io
import subprocess


def kernels(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    blocks, cur = [], None
    for line in out.splitlines():
        if line.startswith('"Kernel Name"'):
            cur = {"name": next(csv.reader(io.StringIO(line)))[1], "lines": []}
            blocks.append(cur)
        elif cur is not None:
            cur["lines"].append(line)
    res = []
    for b in blocks:
        rows = list(csv.DictReader(io.StringIO("\n".join(b["lines"]))))
        res.append((b["name"], rows))
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--kernel", default="")
    ap.add_argument("--top", type=int, default=25)
    ap.add_argument("--ctx", type=int, default=2)
    args = ap.parse_args()
    seen = set()
    for name, rows in kernels(args.rep):
        if args.kernel not in name or name in seen:
            continue
        seen.add(name)
        samp = [int(r.get("Warp Stall Sampling (All Samples)") or 0) for r in rows]
        total = sum(samp) or 1
        print(f"== {name}: {len(rows)} SASS lines, {total} samples")
        order = sorted(range(len(rows)), key=lambda i: -samp[i])[: args.top]
        for i in order:
            ctx = " | ".join(rows[j]["Source"].strip() for j in range(max(0, i - args.ctx), i))
            print(f"{samp[i] / total:6.3f} {rows[i]['Address'][-5:]} {rows[i]['Source'].strip():45s} <- {ctx}")


if __name__ == "__main__":
    main()
