"""Operator assembly on the device — mirror of helmadr/operators.py.

``assemble_adr`` / ``assemble_helmholtz`` build the stencil coefficients
directly into HBM planes (no CSR), term by term with the reference's numpy
expression semantics (helmadr/operators.py:85-234).  ``shift_operator``,
``similarity_conjugate`` and the blend are device-side plane arithmetic.
The phase factors (exp(+-i w tau)) are elementwise setup on the host inputs.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import cbuf, check
from .stencil import StencilOperator, as_operator

BC_KINDS = ("neumann", "sommerfeld")
ADR_SCHEMES = ("central", "upwind1", "upwind2")
_SCHEME_ID = {"central": 0, "upwind1": 1, "upwind2": 2, "helmholtz": 3}


@dataclass(frozen=True)
class BCSpec:
    """Boundary condition per side (helmadr/operators.py:30-51); front/back are the
    faces of the second lateral axis of 3D grids (restatement decision)."""

    top: str = "neumann"
    bottom: str = "sommerfeld"
    left: str = "sommerfeld"
    right: str = "sommerfeld"
    front: str = "sommerfeld"
    back: str = "sommerfeld"

    def __post_init__(self):
        for side in ("top", "bottom", "left", "right", "front", "back"):
            kind = getattr(self, side)
            if kind not in BC_KINDS:
                raise ValueError(f"{side} condition {kind!r} not in {BC_KINDS}")

    @classmethod
    def all_neumann(cls) -> "BCSpec":
        return cls(*(["neumann"] * 6))

    @classmethod
    def all_sommerfeld(cls) -> "BCSpec":
        return cls(*(["sommerfeld"] * 6))

    def codes(self):
        sides = (self.top, self.bottom, self.left, self.right, self.front, self.back)
        return np.array([BC_KINDS.index(k) for k in sides], dtype=np.int32)


def _bc(bc) -> BCSpec:
    if bc is None:
        return BCSpec()
    if isinstance(bc, BCSpec):
        return bc
    if isinstance(bc, (tuple, list)):
        return BCSpec(*bc)
    return BCSpec(bc.top, bc.bottom, bc.left, bc.right, getattr(bc, "front", "sommerfeld"),
                  getattr(bc, "back", "sommerfeld"))  # reference BCSpec (duck-typed)


def _f64(a, shape):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if a.shape != tuple(shape):
        raise ValueError(f"field has shape {a.shape}, expected {tuple(shape)}")
    return a


def _assemble(grid, omega, scheme, bc, kappa_sq, gamma, grads, lap, src):
    sh = tuple(grid.shape)
    dim = len(sh)
    n1, n2, n3 = sh[0], sh[1], (sh[2] if dim == 3 else 1)
    hs = tuple(getattr(grid, "hs", (grid.h1, grid.h2)))
    h3 = hs[2] if dim == 3 else 1.0
    ksq = _f64(kappa_sq, sh)
    gam = _f64(gamma, sh)
    zero = np.zeros(sh)
    g = [_f64(grads[a] if grads is not None else zero, sh) for a in range(dim)]
    g3 = g[2] if dim == 3 else zero
    lp = _f64(lap if lap is not None else zero, sh)
    codes = _bc(bc).codes()
    s = (-1, -1, -1) if src is None else (tuple(int(v) for v in src) + (0,))[:3]
    h = C.c_void_p()
    check(_lib.lib().hadr_assemble(dim, n1, n2, n3, float(hs[0]), float(hs[1]), float(h3), float(omega),
                                   _SCHEME_ID[scheme], cbuf(codes), s[0], s[1], s[2], cbuf(ksq), cbuf(gam),
                                   cbuf(g[0]), cbuf(g[1]), cbuf(g3), cbuf(lp), 0, C.byref(h)))
    return StencilOperator(h)


def _source_index(tt):
    base = getattr(tt, "base", None)
    if base is None:
        return None
    src = base.source
    return tuple(src.index) if hasattr(src, "index") else (src.i1, src.i2)


def assemble_helmholtz(medium, grid, omega: float, bc) -> StencilOperator:
    """Standard five-point Helmholtz operator (helmadr/operators.py:190-200)."""
    return _assemble(grid, omega, "helmholtz", bc, medium.kappa_sq, medium.gamma, None, None, None)


def assemble_adr(medium, grid, omega: float, tt, scheme: str, bc) -> StencilOperator:
    """Amplitude (ADR) operator (helmadr/operators.py:203-234)."""
    if scheme not in ADR_SCHEMES:
        raise ValueError(f"scheme {scheme!r} not in {ADR_SCHEMES}")
    if tuple(tt.grid.shape) != tuple(grid.shape):
        raise ValueError("travel time grid does not match")
    grads = list(getattr(tt, "grads", None) or [tt.grad1, tt.grad2])
    return _assemble(grid, omega, scheme, bc, medium.kappa_sq, medium.gamma, grads, tt.lap, _source_index(tt))


def shift_operator(A, alpha: float, omega: float, medium) -> StencilOperator:
    """A - i w^2 alpha diag(kappa^2) (helmadr/operators.py:237-244)."""
    op = as_operator(A, medium.grid.shape)
    if op.shape[0] != medium.grid.n_nodes:
        raise ValueError("operator dimension does not match the medium grid")
    s = -1j * omega**2 * alpha  # the reference's scalar, then times kappa^2 on the device
    ksq = np.ascontiguousarray(np.asarray(medium.kappa_sq, dtype=np.float64).reshape(-1))
    h = C.c_void_p()
    check(_lib.lib().hadr_op_add_diag(op.handle, float(s.real), float(s.imag), cbuf(ksq), C.byref(h)))
    return StencilOperator(h)


def blend_operator(A, B, beta: float) -> StencilOperator:
    """(1 - beta)*A + beta*B on the union pattern (helmadr/drivers.py:156)."""
    a = as_operator(A)
    b = as_operator(B)
    h = C.c_void_p()
    check(_lib.lib().hadr_op_axpby(1.0 - beta, 0.0, a.handle, float(beta), 0.0, b.handle, C.byref(h)))
    return StencilOperator(h)


def phase_scaling(tt, omega: float) -> np.ndarray:
    """M_jj = exp(-i w tau_j) (helmadr/operators.py:247-249)."""
    return np.exp(-1j * omega * tt.tau.reshape(-1))


def similarity_conjugate(A, m, direction: str) -> StencilOperator:
    """M A M^-1 or M^-1 A M (helmadr/operators.py:252-266), on the device."""
    op = as_operator(A)
    m = np.asarray(m).reshape(-1)
    if op.shape[0] != m.size:
        raise ValueError("dimension mismatch")
    if direction == "M_A_Minv":
        left, right = m, 1.0 / m
    elif direction == "Minv_A_M":
        left, right = 1.0 / m, m
    else:
        raise ValueError(f"direction {direction!r} not in ('M_A_Minv', 'Minv_A_M')")
    left = np.ascontiguousarray(left, dtype=np.complex128)
    right = np.ascontiguousarray(right, dtype=np.complex128)
    h = C.c_void_p()
    check(_lib.lib().hadr_op_similarity(op.handle, cbuf(left), cbuf(right), C.byref(h)))
    return StencilOperator(h)


def rhs_transform(q: np.ndarray, tt, omega: float, direction: str) -> np.ndarray:
    """helmadr/operators.py:269-278."""
    if q.shape != tt.tau.shape:
        raise ValueError("field/travel-time grid mismatch")
    if direction not in ("to_adr", "to_helmholtz"):
        raise ValueError(f"direction {direction!r} not in ('to_adr', 'to_helmholtz')")
    j = 1j if direction == "to_adr" else -1j
    nz = np.flatnonzero(q)
    if nz.size * 8 < q.size:  # a point source: the phase only where q is non-zero (same values there)
        out = np.zeros(q.shape, dtype=np.result_type(q.dtype, np.complex128))
        qf, tf, of = q.reshape(-1), tt.tau.reshape(-1), out.reshape(-1)
        of[nz] = qf[nz] * np.exp(j * omega * tf[nz])
        return out
    return q * np.exp(j * omega * tt.tau)


def max_nnz_per_row(A) -> int:
    csr = as_operator(A).tocsr()
    return int(np.diff(csr.indptr).max())


def export_operator_coo(A, path: str) -> None:
    """Debug dump: one 'row col re im' line per stored entry (helmadr/operators.py:281-286).

    The device operator is exported to canonical CSR (rows ascending, columns ascending
    within a row), the order the reference's ``A.tocoo()`` of a canonical CSR has.  A
    structured stencil stores no explicit zeros, so an entry the reference kept as an
    explicit 0 (e.g. cancelling duplicate COO terms) has no line here."""
    if isinstance(A, StencilOperator):
        A = A.tocsr()
    coo = A.tocoo()
    with open(path, "w", encoding="ascii") as fh:
        for r, c, v in zip(coo.row, coo.col, coo.data):
            fh.write(f"{r} {c} {v.real!r} {v.imag!r}\n")
