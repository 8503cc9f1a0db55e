"""standard_sl (shifted-Laplacian K-cycle on the 7-point Helmholtz operator) on the config-5
recipe, for A/B timing of library options:
    python tools/sl_solve.py --n 257 [name=value ...] [--sweep name=v1,v2]   (one process: tau is marched once)"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=257)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--sweep", default="", help="name=v1,v2,...: repeat the solves for each value of one option")
    a, extra = ap.parse_known_args()
    from paper_1712_06091_b200 import _lib, drivers, operators, workloads
    from paper_1712_06091_b200.fields import point_source

    for kv in extra:
        k, v = kv.split("=")
        _lib.set_option(k, float(v))
    wl = workloads.cfg5(a.n)
    q = point_source(wl.grid, wl.source)
    H = operators.assemble_helmholtz(wl.medium, wl.grid, wl.omega, wl.bc)
    cfg = drivers.StrategyConfig(strategy="standard_sl", alpha=0.5, tol=1e-6, max_iter=1000)
    name, vals = (a.sweep.split("=") + [""])[:2] if a.sweep else ("", "")
    for v in (vals.split(",") if vals else [None]):
        if v is not None:
            _lib.set_option(name, float(v))
            print(f"{name}={v}")
        for _ in range(a.reps + 1):
            u, rep = drivers.solve_standard(H, q, wl.medium, wl.omega, cfg)
            print(f"cfg5_{a.n} standard_sl: its={rep.iterations} fgmres {rep.device_time * 1e3:.1f} ms "
                  f"({wl.grid.n_nodes * rep.iterations / rep.device_time / 1e6:.0f} Mdof*it/s)", flush=True)


if __name__ == "__main__":
    main()
