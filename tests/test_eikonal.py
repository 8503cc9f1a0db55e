"""Fast-marching travel time (setup input of the solve): libhadr's host marcher
(csrc/eikonal.cpp) against the reference's own fast_march output
(tests/golden/fmm.npz, made by tests/golden/make_golden_fmm.py).  No GPU."""

import os

import numpy as np
import pytest

from conftest import REPO

GOLD = os.path.join(REPO, "tests", "golden", "fmm.npz")


def _cases():
    z = np.load(GOLD)
    names = sorted({k.split("__")[0] for k in z.files})
    return z, names


@pytest.mark.parametrize("order", ["first", "second"])
def test_fast_march_bit_exact_vs_reference(order):
    from paper_1712_06091_b200.eikonal import fast_march
    from paper_1712_06091_b200.fields import GridSpec, Medium, SourceSpec

    z, names = _cases()
    assert names
    for name in names:
        n1, n2 = (int(x) for x in z[f"{name}__shape"])
        L1, L2 = (float(x) for x in z[f"{name}__L"])
        i1, i2 = (int(x) for x in z[f"{name}__src"])
        g = GridSpec(n1, n2, L1, L2)
        med = Medium(g, z[f"{name}__kappa_sq"], np.zeros((n1, n2)))
        t1 = fast_march(med, g, SourceSpec(i1, i2, 1.0), order)
        ref = z[f"{name}__tau1_{order}"]
        assert np.array_equal(t1, ref), (name, order, float(np.max(np.abs(t1 - ref))))


def test_fast_march_3d_linear_gradient():
    """3D extension (no reference counterpart): against the analytic linear-gradient travel time."""
    from paper_1712_06091_b200 import workloads
    from paper_1712_06091_b200.eikonal import fast_march

    errs = []
    for n in (33, 65):  # first-order-limited near the source: the error halves with h
        wl = workloads.cfg4(n)
        t1 = fast_march(wl.medium, wl.grid, wl.source, "second")
        exact = wl.tt.tau1
        assert np.all(t1 > 0)
        errs.append(float(np.max(np.abs(t1 - exact) / exact)))
    assert errs[1] < 1.5e-2 and errs[1] < 0.7 * errs[0], errs


def test_fast_march_errors():
    from paper_1712_06091_b200.eikonal import fast_march
    from paper_1712_06091_b200.fields import GridSpec, Medium, SourceSpec

    g = GridSpec(9, 9, 1.0, 1.0)
    med = Medium(g, np.ones((9, 9)), np.zeros((9, 9)))
    with pytest.raises(ValueError):
        fast_march(med, g, SourceSpec(4, 4, 1.0), order=3)
