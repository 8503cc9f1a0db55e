"""Share of the cluster engine in one bench-workload solve (real execution, no profiler):
engine cycles from CTA 0's clock64 counters (hadr_ce_profile) vs the solve's device time.

    python tools/engine_share.py [--n 1025]
"""

import argparse
import ctypes as C
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1025)
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--mhz", type=float, default=1965.0)
    a, extra = ap.parse_known_args()
    from paper_1712_06091_b200 import _lib, drivers, workloads

    L = _lib.lib()
    wl = workloads.by_name(a.workload, a.n)
    cfg = drivers.StrategyConfig(strategy="adr_upwind_blend", tol=1e-6, max_iter=1000)
    for opt in extra:
        if "=" in opt and not opt.startswith("--"):
            k, v = opt.split("=")
            _lib.set_option(k, float(v))
    _lib.set_option("ce_profile", 1)  # read when the K-cycle graphs are captured
    drivers.solve_adr_upwind(wl.medium, wl.grid, wl.source, wl.tt, cfg, wl.bc)
    prof = (C.c_ulonglong * 48)()
    L.hadr_ce_profile(prof, 1)
    u, amp, rep = drivers.solve_adr_upwind(wl.medium, wl.grid, wl.source, wl.tt, cfg, wl.bc)
    L.hadr_ce_profile(prof, 0)
    _lib.set_option("ce_profile", 0)
    eng_ms = prof[0] / (a.mhz * 1e3)
    print(f"its={rep.iterations} device_ms={rep.device_time*1e3:.1f} engine_ms={eng_ms:.1f} "
          f"engine_launches={prof[7]} per_launch_us={eng_ms*1e3/max(prof[7],1):.1f} counters={list(prof)}")


if __name__ == "__main__":
    main()
