"""Summarise an ncu report (read here, no GPU needed):

    python tools/ncu_summary.py gpurun_out/prof_<tag>.ncu-rep [--out profiles/<file>.md]

Prints per-kernel duration, DRAM bytes and throughput, L2/L1 hit rates,
occupancy and the dominant stall reasons.
"""
import argparse
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    # dram__throughput... is stored under a prefixed Triage name with empty
    # values in `--page raw`; the per-direction percentages are populated
    ("dram__bytes_read.sum.pct_of_peak_sustained_elapsed", "dram_rd_%pk"),
    ("dram__bytes_write.sum.pct_of_peak_sustained_elapsed", "dram_wr_%pk"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_%pk"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2_%pk"),
    ("lts__t_sector_hit_rate.pct", "L2_hit%"),
    ("l1tex__t_sector_hit_rate.pct", "L1_hit%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1_%pk"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "st_long"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "st_short"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "st_bar"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "st_mio"),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "st_lg"),
    ("smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio", "st_noinst"),
]


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"name": r[h.index("Kernel Name")]}
        for key, short in METRICS:
            if key in h:
                v = r[h.index(key)]
                d[short] = (v, units[h.index(key)])
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--out")
    a = ap.parse_args()
    res = load(a.rep)
    lines = [f"# ncu summary of `{a.rep}`", "",
             "| kernel | " + " | ".join(s for _, s in METRICS) + " |",
             "|---|" + "---|" * len(METRICS)]
    for d in res:
        name = d["name"].split("(")[0].replace("void ", "")[:48]
        cells = [f"{d[s][0]} {d[s][1]}".strip() if s in d else "" for _, s in METRICS]
        lines.append(f"| {name} | " + " | ".join(cells) + " |")
    text = "\n".join(lines) + "\n"
    if a.out:
        with open(a.out, "w") as f:
            f.write(text)
    sys.stdout.write(text)


if __name__ == "__main__":
    main()
