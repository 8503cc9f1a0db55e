"""Golden solve for the config-3 recipe (down-scaled to 129 x 65: layered medium,
surface source, Neumann top, travel time from fast marching) by the REFERENCE.

    NUMBA_CACHE_DIR=/tmp/nbcache python tests/golden/make_golden_cfg3.py

Writes tests/golden/cfg3_65.npz (fields, fine operators, hierarchy, upwind solve).
"""

from __future__ import annotations

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as MG  # noqa: E402  (imports the reference in place)
import numpy as np  # noqa: E402
from helmadr import eikonal as heik, grid as hgrid  # noqa: E402

from paper_1712_06091_b200 import workloads  # noqa: E402


def main():
    wl = workloads.cfg3(65)
    # the travel time the reference's own fast marching produces for this medium
    g = hgrid.GridSpec(wl.grid.n1, wl.grid.n2, wl.grid.L1, wl.grid.L2)
    med = hgrid.Medium(g, wl.medium.kappa_sq, wl.medium.gamma)
    src = hgrid.SourceSpec(wl.source.i1, wl.source.i2, wl.source.omega)
    tt_ref = heik.compute_travel_time(med, g, src, "second")
    assert np.array_equal(tt_ref.tau1, wl.tt.tau1), "fast-marching restatement differs from the reference"
    out = {}
    MG.operator_case(wl, out, full_ops=False)
    MG.solve_case(wl, out, ("upwind",))
    out["tau1"] = wl.tt.tau1
    np.savez_compressed(os.path.join(HERE, "cfg3_65.npz"), **out)
    print("cfg3_65 upwind iterations", int(out["upwind_iterations"]))


if __name__ == "__main__":
    main()
