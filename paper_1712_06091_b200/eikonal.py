"""Factored-eikonal travel times — mirror of helmadr/eikonal.py.

``fast_march`` runs the host marcher of libhadr (csrc/eikonal.cpp, a
restatement of helmadr/_fmm.py); ``tau_derivatives`` and
``compute_travel_time`` follow helmadr/eikonal.py:180-239.  This is setup: the
travel time is an input of the amplitude solve (north_star) and is timed
separately (``TravelTime.fm_time``).  3D grids use the marcher's 3D extension
(the reference has none).
"""

from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import _lib
from .fields import AnalyticBase, TravelTime


def _order_int(order) -> int:
    if order in (1, "first"):
        return 1
    if order in (2, "second"):
        return 2
    raise ValueError(f"order must be 'first'/'second' (or 1/2), got {order!r}")


def _base_fields(grid, source):
    """tau0 = |x - x0| and grad(tau0) (zero at the source), any dimension."""
    if grid.dim == 2:
        b = AnalyticBase(grid, source)
        return b.tau0, [b.grad1, b.grad2]
    X = grid.coords()
    pos = source.position(grid)
    e = [X[a] - pos[a] for a in range(3)]
    r = np.sqrt(e[0] ** 2 + e[1] ** 2 + e[2] ** 2)
    with np.errstate(divide="ignore", invalid="ignore"):
        g = [np.where(r > 0, ea / r, 0.0) for ea in e]
    return r, g


def fast_march(medium, grid, source, order="second") -> np.ndarray:
    """helmadr/eikonal.py:72-99: the factor tau1 (> 0 everywhere), tau = tau0 * tau1."""
    source.validate(grid)
    tau0, g0 = _base_fields(grid, source)
    dim = grid.dim
    n = np.array(list(grid.shape) + [1] * (3 - dim), dtype=np.int32)
    h = np.array(list(grid.hs) + [1.0] * (3 - dim), dtype=np.float64)
    src = np.array(list(source.index) + [0] * (3 - dim), dtype=np.int32)
    t0 = np.ascontiguousarray(tau0, dtype=np.float64)
    gs = [np.ascontiguousarray(x, dtype=np.float64) for x in g0] + [None] * (3 - dim)
    kap = np.ascontiguousarray(medium.kappa, dtype=np.float64)
    tau1 = np.empty(grid.shape, dtype=np.float64)
    nacc = C.c_longlong()
    L = _lib.load()
    _lib.check(L.hadr_fast_march(dim, _lib.cbuf(n), _lib.cbuf(h), _lib.cbuf(t0), _lib.cbuf(gs[0]), _lib.cbuf(gs[1]),
                                 _lib.cbuf(gs[2]) if gs[2] is not None else None, _lib.cbuf(kap), _lib.cbuf(src),
                                 _order_int(order), _lib.cbuf(tau1), C.byref(nacc)))
    if nacc.value != grid.n_nodes:
        raise RuntimeError(f"fast marching accepted {nacc.value} of {grid.n_nodes} nodes; "
                           "the update graph should be connected for positive kappa")
    return tau1


def tau_derivatives(tau1: np.ndarray, base, grid):
    """helmadr/eikonal.py:204-226 (2D): ((grad1, grad2), lap) of tau = tau0 * tau1."""
    from .workloads import travel_time_from_tau1

    tt = travel_time_from_tau1(grid, base.source, tau1)
    return (tt.grad1, tt.grad2), tt.lap


def compute_travel_time(medium, grid, source, order="second") -> TravelTime:
    """helmadr/eikonal.py:229-239: fast_march + tau_derivatives, with fm_time."""
    from .workloads import travel_time_from_tau1, travel_time_nd

    t0 = time.perf_counter()
    tau1 = fast_march(medium, grid, source, order)
    fm_time = time.perf_counter() - t0
    tt = travel_time_from_tau1(grid, source, tau1) if grid.dim == 2 else travel_time_nd(grid, source, tau1)
    tt.fm_time = fm_time
    return tt
