"""Krylov solvers on the B200 — drop-in mirror of helmadr/krylov.py.

Same names, arguments, defaults, error behaviour and report fields as the
reference (helmadr/krylov.py:16-242); the arithmetic runs in libhadr.so.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import HadrReport, as_c128, cbuf, check
from .stencil import StencilOperator, as_operator  # noqa: F401


@dataclass
class KrylovConfig:
    """helmadr/krylov.py:16-31."""

    restart: int = 5
    maxiter: int = 200
    tol: float = 1e-5
    flexible: bool = True
    collect_diagnostics: bool = False

    def __post_init__(self):
        if self.restart < 1:
            raise ValueError("restart must be >= 1")
        if self.tol <= 0:
            raise ValueError("tol must be positive")


@dataclass
class SolveReport:
    """helmadr/krylov.py:34-57, plus the device timing of the solve."""

    iterations: int
    history: np.ndarray
    converged: bool
    wall_time: float
    bnorm: float
    final_relres: float
    note: str = ""
    ortho_max: float = 0.0
    stage1: "SolveReport | None" = None
    stage2: "SolveReport | None" = None
    fm_time: float = 0.0
    device_time: float = 0.0   # CUDA-event time of the FGMRES solve
    setup_time: float = 0.0    # CUDA-event time of assembly + hierarchy (ADR drivers)

    def history_csv_lines(self) -> list[str]:
        scale = self.bnorm if self.bnorm > 0 else 1.0
        return [f"{i},{r / scale:.16e}" for i, r in enumerate(self.history)]


_NOTES = {0: "", 1: "numerical breakdown: non-finite Arnoldi vector"}


def grid_of(A, grid=None):
    """The structured grid a device stencil needs for ``A``: the operator's own grid, an
    explicit ``grid`` (shape tuple or object with ``.shape``), or — for a plain scipy
    matrix, the reference's documented argument type — the square (n = m^2) or cubic
    (n = m^3) grid its size implies.  Anything else must name its grid."""
    if grid is not None:
        return tuple(grid.shape) if hasattr(grid, "shape") and not isinstance(grid, tuple) else tuple(grid)
    g = getattr(A, "grid_shape", None)
    if g is not None:
        return tuple(g)
    n = int(A.shape[0])
    m = int(round(n ** 0.5))
    if m * m == n:
        return (m, m)
    m = int(round(n ** (1.0 / 3.0)))
    if m * m * m == n:
        return (m, m, m)
    raise ValueError(f"cannot infer the grid of a {A.shape} operator (not m^2 or m^3 points): pass grid=(n1, n2[, n3])"
                     " or wrap it with StencilOperator.from_csr(A, grid)")


def spmv(A, x, grid=None) -> np.ndarray:
    """y = A x with an explicit dimension check (helmadr/krylov.py:60-65)."""
    x = np.asarray(x)
    if A.shape[1] != x.shape[0]:
        raise ValueError(f"dimension mismatch: operator {A.shape}, vector {x.shape}")
    op = as_operator(A, grid_of(A, grid))
    return op.matvec(x)


def jacobi_apply(A, r, grid=None) -> np.ndarray:
    """z_j = r_j / A_jj (helmadr/krylov.py:68-73)."""
    op = as_operator(A, grid_of(A, grid))
    r = as_c128(r, op.shape[0])
    z = np.empty_like(r)
    check(_lib.lib().hadr_op_jacobi(op.handle, cbuf(r), cbuf(z), 0))
    return z


def gmres_relax(A, b, x, steps: int, grid=None) -> np.ndarray:
    """Fixed-length Jacobi-preconditioned GMRES from x (helmadr/krylov.py:82-119)."""
    op = as_operator(A, grid_of(A, grid))
    n = op.shape[0]
    b = as_c128(b, n)
    x = as_c128(x, n)
    out = np.empty_like(b)
    check(_lib.lib().hadr_gmres_relax(op.handle, cbuf(b), cbuf(x), int(steps), cbuf(out), 0))
    return out


def _report_from(rep: HadrReport, hist: np.ndarray) -> SolveReport:
    return SolveReport(
        iterations=int(rep.iterations),
        history=np.array(hist[: rep.history_len], copy=True),
        converged=bool(rep.converged),
        wall_time=float(rep.wall_time),
        bnorm=float(rep.bnorm),
        final_relres=float(rep.final_relres),
        note=_NOTES.get(int(rep.note), "breakdown"),
        device_time=float(rep.device_time),
        ortho_max=float(rep.ortho_max),
    )


def fgmres(A, b, x0=None, precond=None, cfg: KrylovConfig | None = None):
    """Restarted flexible GMRES (helmadr/krylov.py:122-242) on the device.

    ``A``: StencilOperator (or scipy matrix already wrapped); ``precond``: None
    or a K-cycle preconditioner from ``make_kcycle_preconditioner``.  Returns
    ``(x, SolveReport)``; inputs are not modified.
    """
    from .multigrid import KCyclePreconditioner  # local: multigrid imports krylov

    cfg = cfg or KrylovConfig()
    grid = getattr(A, "grid_shape", None)
    if grid is None and isinstance(precond, KCyclePreconditioner):
        grid = precond.hier.shapes[0]  # a scipy A on the hierarchy's finest grid
    op = as_operator(A, grid_of(A, grid))
    n = op.shape[0]
    b = as_c128(b, n)
    x0a = None if x0 is None else as_c128(x0, n)
    if precond is None:
        hh = None
    elif isinstance(precond, KCyclePreconditioner):
        hh = precond.hier.handle
    else:
        raise TypeError("precond must be None or make_kcycle_preconditioner(hier) (device K-cycle)")
    x = np.empty_like(b)
    rep = HadrReport()
    cap = max(int(cfg.maxiter), 0) + 2
    hist = np.zeros(cap)
    check(
        _lib.lib().hadr_fgmres_ex(op.handle, hh, cbuf(b), None if x0a is None else cbuf(x0a), int(cfg.restart),
                                  int(cfg.maxiter), float(cfg.tol), _flags(cfg), cbuf(x), C.byref(rep), cbuf(hist),
                                  cap, 0)
    )
    return x, _report_from(rep, hist)


def _flags(cfg: KrylovConfig) -> int:
    """KrylovConfig switches -> hadr_fgmres_ex flags (include/hadr.h)."""
    return (0 if cfg.flexible else 1) | (2 if cfg.collect_diagnostics else 0)


def fgmres_device(A, b_ptr: int, x_ptr: int, precond=None, cfg: KrylovConfig | None = None, x0_ptr: int | None = None):
    """fgmres on device-resident vectors (raw CUDA pointers, e.g. torch ``data_ptr()``).
    Returns the SolveReport; x is written in place."""
    cfg = cfg or KrylovConfig()
    op = as_operator(A, getattr(A, "grid_shape", None))
    hh = None if precond is None else precond.hier.handle
    rep = HadrReport()
    cap = max(int(cfg.maxiter), 0) + 2
    hist = np.zeros(cap)
    check(
        _lib.lib().hadr_fgmres_ex(op.handle, hh, C.c_void_p(b_ptr), None if x0_ptr is None else C.c_void_p(x0_ptr),
                                  int(cfg.restart), int(cfg.maxiter), float(cfg.tol), _flags(cfg), C.c_void_p(x_ptr),
                                  C.byref(rep), cbuf(hist), cap, 1)
    )
    return _report_from(rep, hist)


def launch_count() -> int:
    """Kernels libhadr.so has launched so far in this process."""
    return int(_lib.load().hadr_launch_count())
