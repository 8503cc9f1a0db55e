"""Device time of the setup phase (assembly + Galerkin hierarchy) of a bench workload solve:
    python tools/setup_time.py --workload cfg4 --n 513"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg4")
    ap.add_argument("--n", type=int, default=513)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--opt", action="append", default=[], help="name=value runtime option")
    a = ap.parse_args()
    from paper_1712_06091_b200 import _lib, drivers, workloads

    for kv in a.opt:
        k, v = kv.split("=")
        _lib.set_option(k, float(v))

    wl = workloads.by_name(a.workload, a.n)
    cfg = drivers.StrategyConfig(strategy="adr_upwind_blend", tol=1e-6, max_iter=1)
    for r in range(a.reps):
        u, amp, rep = drivers.solve_adr_upwind(wl.medium, wl.grid, wl.source, wl.tt, cfg, wl.bc)
        print(f"{a.workload}_{a.n}: setup (assembly + hierarchy) {rep.setup_time * 1e3:.1f} ms device time")


if __name__ == "__main__":
    main()
