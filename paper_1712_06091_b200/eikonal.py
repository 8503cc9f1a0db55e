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


def _tau_fields_device(grid, src_index, tau1):
    """(tau, [grad per axis], lap) of tau = tau0*tau1 formed on the device (hadr_tau_derivatives)."""
    sh = tuple(int(v) for v in grid.shape)
    dim = len(sh)
    Ls = tuple(float(v) for v in getattr(grid, "Ls", (grid.L1, grid.L2)))
    t1 = np.ascontiguousarray(np.asarray(tau1, dtype=np.float64))
    if t1.shape != sh:
        raise ValueError(f"tau1 has shape {t1.shape}, grid is {sh}")
    n = np.asarray(sh, dtype=np.int32)
    L = np.asarray(Ls, dtype=np.float64)
    s = np.asarray(tuple(src_index), dtype=np.int32)
    tau = np.empty(sh)
    grads = np.empty((dim,) + sh)
    lap = np.empty(sh)
    _lib.check(_lib.lib().hadr_tau_derivatives(dim, _lib.cbuf(n), _lib.cbuf(L), _lib.cbuf(s), _lib.cbuf(t1),
                                               _lib.cbuf(tau), _lib.cbuf(grads), _lib.cbuf(lap), 0))
    return tau, [grads[a] for a in range(dim)], lap


def tau_derivatives(tau1: np.ndarray, base, grid):
    """helmadr/eikonal.py:180-226 on the device: ((grad1, grad2[, grad3]), lap) of
    tau = tau0 * tau1 (bit-identical to the reference's numpy arithmetic)."""
    _, grads, lap = _tau_fields_device(grid, base.source.index if hasattr(base.source, "index")
                                       else (base.source.i1, base.source.i2), tau1)
    return tuple(grads), lap


def compute_travel_time(medium, grid, source, order="second"):
    """helmadr/eikonal.py:229-239: fast_march (host, timed as fm_time), then the
    derivative fields of tau_derivatives — formed on the device where the solve needs
    them (``DeviceTravelTime``), so only tau1 is copied to the GPU."""
    from .fields import DeviceTravelTime

    t0 = time.perf_counter()
    tau1 = fast_march(medium, grid, source, order)
    fm_time = time.perf_counter() - t0
    return DeviceTravelTime(grid, source, tau1, fm_time)
