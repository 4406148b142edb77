"""Command-line entry points over the C ABI (no CPU fallback):

    python -m paper_2507_14051_b200 bench DIR [--json OUT] [--workers N] [--epsilon E]
                                     [--small-limit S] [--large-limit S]
        GPU directory benchmark with SGM10 scoring (rhpdhg::run_benchmark,
        reference bench.cpp:171-266; workers > 1 run concurrent solves, worker
        w on GPU w % device_count)
    python -m paper_2507_14051_b200 solve FILE.mps[.gz] [--epsilon E] [--out REPORT]
        one solve, the reference's key/value report on stdout or in REPORT
"""
import argparse
import sys

from .lp import SolverConfig, read_mps, run_benchmark, solve


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2507_14051_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("bench")
    b.add_argument("dir")
    b.add_argument("--json")
    b.add_argument("--workers", type=int, default=1)
    b.add_argument("--epsilon", type=float, default=1e-4)
    b.add_argument("--small-limit", type=float, default=3600.0)
    b.add_argument("--large-limit", type=float, default=18000.0)
    s = sub.add_parser("solve")
    s.add_argument("file")
    s.add_argument("--epsilon", type=float, default=1e-4)
    s.add_argument("--out")
    a = ap.parse_args(argv)
    if a.cmd == "bench":
        print(run_benchmark(a.dir, SolverConfig(epsilon=a.epsilon), a.small_limit,
                            a.large_limit, a.workers, a.json), end="")
        return 0
    lp, warnings = read_mps(a.file)
    for w in warnings:
        print(f"warning: {w}", file=sys.stderr)
    rep = solve(lp, SolverConfig(epsilon=a.epsilon))
    text = (f"status {rep.status}\nobjective {rep.objective!r}\niterations {rep.iterations}\n"
            f"restarts {rep.restart_count}\nwall_time_seconds {rep.wall_time_seconds!r}\n")
    if a.out:
        with open(a.out, "w") as f:
            f.write(text)
    else:
        print(text, end="")
    return 0 if rep.status == "optimal" else 2


if __name__ == "__main__":
    sys.exit(main())
