"""Golden travel times from the REFERENCE's fast marching (helmadr/eikonal.py
fast_march -> helmadr/_fmm.py, numba), run in this container.

    NUMBA_CACHE_DIR=/tmp/nbcache python tests/golden/make_golden_fmm.py

Writes tests/golden/fmm.npz: per case the slowness field kappa, the grid /
source, and the reference tau1 (orders 1 and 2).  The cases use this
repository's seeded config builders (config 3's layered medium with a surface
source, config 2's linear gradient with a buried source).
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from helmadr import eikonal, grid as hgrid  # noqa: E402

from paper_1712_06091_b200 import workloads  # noqa: E402
from paper_1712_06091_b200.fields import GridSpec, Medium, SourceSpec  # noqa: E402


def cases():
    # config 3 recipe, down-scaled (129 x 65 and 257 x 129), surface source
    for n in (65, 129):
        g = GridSpec(2 * (n - 1) + 1, n, 2.0, 1.0)
        v = workloads.cfg3_medium(g, max(1.0, 20.0 * (n - 1) / 2048))
        yield f"cfg3_{n}", g, 1.0 / v**2, ((g.n1 - 1) // 2, 0)
    # config 2 recipe (linear gradient), buried source
    n = 65
    g = GridSpec(n, n, 1.0, 1.0)
    _, x2 = g.coords()
    v = 1.5 + 2.5 * x2
    yield "cfg2_65", g, 1.0 / v**2, ((n - 1) // 2, round(0.05 * (n - 1)))


def main():
    out = {}
    for name, g, ksq, (i1, i2) in cases():
        hg = hgrid.GridSpec(g.n1, g.n2, g.L1, g.L2)
        med = hgrid.Medium(hg, ksq, np.zeros(g.shape))
        src = hgrid.SourceSpec(i1, i2, 1.0)
        out[f"{name}__shape"] = np.array(g.shape)
        out[f"{name}__L"] = np.array([g.L1, g.L2])
        out[f"{name}__src"] = np.array([i1, i2])
        out[f"{name}__kappa_sq"] = ksq
        for order in ("first", "second"):
            out[f"{name}__tau1_{order}"] = eikonal.fast_march(med, hg, src, order)
        print(name, g.shape, out[f"{name}__tau1_second"].min(), out[f"{name}__tau1_second"].max())
    np.savez_compressed(os.path.join(HERE, "fmm.npz"), **out)


if __name__ == "__main__":
    main()
