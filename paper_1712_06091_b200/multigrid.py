"""Geometric multigrid K-cycle on the B200 — drop-in mirror of helmadr/multigrid.py.

Hierarchy construction (Galerkin P^T A P, helmadr/multigrid.py:49-55, 113-129)
and the whole K-cycle recursion (helmadr/multigrid.py:132-171) run on the
device; one preconditioner application is a single CUDA-graph launch with all
data-dependent branches (breakdowns, re-orthogonalisation, the 0.1 early
exit of the inner FGMRES(2)) resolved on the GPU.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import as_c128, cbuf, check
from .stencil import Prolongation, StencilOperator, as_operator

COARSE_GMRES_STEPS = 10   # helmadr/multigrid.py:15
COARSE_FGMRES_TOL = 0.1   # helmadr/multigrid.py:16


def build_prolongation(fine_shape) -> Prolongation:
    """helmadr/multigrid.py:37-46 (matrix-free, device)."""
    return Prolongation(fine_shape)


def galerkin_coarsen(A, P: Prolongation) -> StencilOperator:
    """Coarse operator P^T A P on the device (helmadr/multigrid.py:49-55)."""
    op = as_operator(A, getattr(P, "fine_shape", None))
    if op.shape[1] != P.shape[0]:
        raise ValueError(f"dimension mismatch: A {op.shape}, P {P.shape}")
    h = C.c_void_p()
    check(_lib.lib().hadr_op_galerkin(op.handle, C.byref(h)))
    return StencilOperator(h)


def coarsenable_levels(shape, max_levels: int):
    """helmadr/multigrid.py:98-110 (per axis in 3D)."""
    shapes = [tuple(shape)]
    while len(shapes) < max_levels:
        m = shapes[-1]
        if any((mi - 1) % 2 for mi in m):
            break
        c = tuple((mi - 1) // 2 + 1 for mi in m)
        if any(ci < 3 for ci in c):
            break
        shapes.append(c)
    return shapes


class MGHierarchy:
    """Per-level device operators + K-cycle workspace (helmadr/multigrid.py:58-95).

    Constructed either as the reference does, ``MGHierarchy(ops=[...], prols=[...],
    shapes=[...], inv_diags=[], coarse_steps=10, coarse_tol=0.1)`` with per-level
    operators (scipy matrices or StencilOperators, finest first; the device keeps its
    own copies), or from a device hierarchy handle (``build_hierarchy``).
    ``prols`` must be the bilinear/trilinear prolongations of ``build_prolongation``
    (the device applies them matrix-free) and ``inv_diags``, when given, 1 / diag of
    each level (the device recomputes them bit-exactly); anything else raises."""

    def __init__(self, ops=None, prols=None, shapes=None, inv_diags=None, coarse_steps=COARSE_GMRES_STEPS,
                 coarse_tol=COARSE_FGMRES_TOL, *, handle=None, keepalive=()):
        if handle is None:
            if ops is None:
                raise TypeError("MGHierarchy needs ops (with prols and shapes) or a device handle")
            handle, keepalive = _hier_handle_from_levels(ops, prols, shapes, inv_diags, coarse_steps, coarse_tol)
        self._h = handle
        self._keep = tuple(keepalive)
        self.coarse_steps = coarse_steps
        self.coarse_tol = coarse_tol
        nl = C.c_int()
        shp = (C.c_int * 96)()
        check(_lib.lib().hadr_hier_info(self._h, C.byref(nl), shp))
        self.shapes = [(shp[3 * i], shp[3 * i + 1]) if shp[3 * i + 2] == 1 else
                       (shp[3 * i], shp[3 * i + 1], shp[3 * i + 2]) for i in range(nl.value)]
        self.ops = []
        for l in range(1, nl.value + 1):
            oh = C.c_void_p()
            check(_lib.lib().hadr_hier_level_op(self._h, l, C.byref(oh)))
            self.ops.append(StencilOperator(oh, owner=self))
        self.prols = [Prolongation(s) for s in self.shapes[:-1]]

    @property
    def handle(self):
        return self._h

    def __del__(self):
        try:
            if self._h:
                _lib._lib.hadr_hier_destroy(self._h)
                self._h = None
        except Exception:
            pass

    @property
    def n_levels(self) -> int:
        return len(self.shapes)

    @property
    def inv_diags(self):
        return [1.0 / A.diagonal() for A in self.ops]

    def relax_steps(self, level: int) -> int:
        return level + 1

    def summary(self) -> str:
        lines = []
        for l, (A, shape) in enumerate(zip(self.ops, self.shapes), start=1):
            relax = f"{self.relax_steps(l)} pre/post" if l < self.n_levels else f"{self.coarse_steps} coarsest"
            lines.append(f"level {l}: grid {'x'.join(map(str, shape))}, nnz {A.nnz}, relax {relax}")
        return "\n".join(lines)


def _hier_handle_from_levels(ops, prols, shapes, inv_diags, coarse_steps, coarse_tol):
    """Device hierarchy for the reference constructor MGHierarchy(ops, prols, shapes, ...)."""
    ops = list(ops)
    if shapes is None:
        shapes = [getattr(A, "grid_shape", None) for A in ops]
        if any(s_ is None for s_ in shapes):
            raise ValueError("scipy level operators need `shapes`")
    shapes = [tuple(int(v) for v in s_) for s_ in shapes]
    if len(shapes) != len(ops):
        raise ValueError(f"{len(ops)} operators but {len(shapes)} shapes")
    for l, (A, s_) in enumerate(zip(ops, shapes)):
        if A.shape[0] != int(np.prod(s_)):
            raise ValueError(f"level {l + 1}: operator {A.shape} does not match grid {s_}")
        if l + 1 < len(shapes) and tuple((n - 1) // 2 + 1 for n in s_) != shapes[l + 1]:
            raise ValueError(f"level {l + 2}: grid {shapes[l + 1]} is not the coarsening of {s_}")
    if prols is not None:
        prols = list(prols)
        if len(prols) != len(ops) - 1:
            raise ValueError(f"{len(ops)} levels need {len(ops) - 1} prolongations, got {len(prols)}")
        for l, P in enumerate(prols):
            if tuple(P.shape) != (int(np.prod(shapes[l])), int(np.prod(shapes[l + 1]))):
                raise ValueError(f"prolongation {l + 1} has shape {P.shape}")
            if isinstance(P, Prolongation):
                continue
            ref = Prolongation(shapes[l]).tocsr()
            Pc = P.tocsr() if hasattr(P, "tocsr") else None
            if Pc is None or (Pc != ref).nnz:
                raise ValueError(f"prolongation {l + 1} is not build_prolongation({shapes[l]}): the device applies "
                                 "the bilinear/trilinear P matrix-free")
    dev = [as_operator(A, shapes[i]) for i, A in enumerate(ops)]
    if inv_diags:
        for l, (A, d) in enumerate(zip(dev, inv_diags)):
            dg = A.diagonal()
            if np.any(dg == 0):
                raise ValueError("hierarchy operator has zero diagonal entries")
            if not np.array_equal(np.asarray(d), 1.0 / dg):
                raise ValueError(f"inv_diags[{l}] is not 1 / diag(ops[{l}])")
    arr = (C.c_void_p * len(dev))(*[d.handle.value for d in dev])
    h = C.c_void_p()
    check(_lib.lib().hadr_hier_from_ops(len(dev), arr, int(coarse_steps), float(coarse_tol), C.byref(h)))
    return h, tuple(dev)


def build_hierarchy(A0, grid, max_levels: int = 5, coarse_steps: int = COARSE_GMRES_STEPS,
                    coarse_tol: float = COARSE_FGMRES_TOL) -> MGHierarchy:
    """Chain of Galerkin operators on the device (helmadr/multigrid.py:113-129)."""
    shape = tuple(grid.shape) if hasattr(grid, "shape") else tuple(grid)
    if A0.shape[0] != int(np.prod(shape)):
        raise ValueError("operator dimension does not match the grid")
    if len(coarsenable_levels(shape, max_levels)) < 2:
        raise ValueError(
            f"grid {shape} cannot support two multigrid levels "
            f"((n_d - 1) must be even with at least 3 coarse nodes)"
        )
    fine = as_operator(A0, shape)
    h = C.c_void_p()
    check(_lib.lib().hadr_hier_create(fine.handle, int(max_levels), int(coarse_steps), float(coarse_tol),
                                      C.byref(h)))
    return MGHierarchy(handle=h, keepalive=(fine,), coarse_steps=coarse_steps, coarse_tol=coarse_tol)


def hierarchy_from_ops(ops, coarse_steps: int = COARSE_GMRES_STEPS, coarse_tol: float = COARSE_FGMRES_TOL,
                       shapes=None) -> MGHierarchy:
    """MGHierarchy(ops=...) from given per-level operators (finest first), e.g. the
    reference's own CSR hierarchy for bit-exact operator parity."""
    return MGHierarchy(ops=ops, prols=None, shapes=shapes, coarse_steps=coarse_steps, coarse_tol=coarse_tol)


def k_cycle(hier: MGHierarchy, level: int, b, x, stats: dict | None = None) -> np.ndarray:
    """One K-cycle at `level` (1 = finest) on the device (helmadr/multigrid.py:132-171)."""
    if not 1 <= level <= hier.n_levels:
        raise ValueError(f"level {level} outside 1..{hier.n_levels}")
    n = int(np.prod(hier.shapes[level - 1]))
    b = as_c128(b, n)
    x = as_c128(x, n)
    x_is_zero = not np.any(x)
    out = np.empty_like(b)
    visits = (C.c_int * hier.n_levels)()
    check(_lib.lib().hadr_kcycle(hier.handle, int(level), cbuf(b), None if x_is_zero else cbuf(x), cbuf(out),
                                 visits if stats is not None else None, 0))
    if stats is not None:
        for l in range(hier.n_levels):
            if visits[l]:
                stats[l + 1] = stats.get(l + 1, 0) + int(visits[l])
    return out


class KCyclePreconditioner:
    """apply(r) = k_cycle(hier, 1, r, 0) (helmadr/multigrid.py:174-184), one CUDA
    graph launch per application.  ``fgmres`` recognises it and keeps every
    vector on the device."""

    def __init__(self, hier: MGHierarchy):
        self.hier = hier

    def __call__(self, r) -> np.ndarray:
        n = int(np.prod(self.hier.shapes[0]))
        r = as_c128(r, n)
        z = np.empty_like(r)
        check(_lib.lib().hadr_precond_apply(self.hier.handle, cbuf(r), cbuf(z), 0))
        return z


def make_kcycle_preconditioner(hier: MGHierarchy) -> KCyclePreconditioner:
    return KCyclePreconditioner(hier)
