"""Device-resident structured operators — the B200 replacement for the scipy CSR
matrices the reference's solver consumes (helmadr/operators.py,
helmadr/multigrid.py:19-55).

``StencilOperator`` keeps an operator as union-offset coefficient planes in HBM
(complex128, plane-major: coef[o, k] multiplies x[k + d1*n2 + d2]).  It
supports the duck-typed surface the reference's solver uses on its matrices
(``@``, ``.shape``, ``.nnz``, ``.diagonal()``, ``.tocsr()``) so it can stand in
for the scipy objects in ``MGHierarchy.ops`` (helmadr/multigrid.py:58-72).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import scipy.sparse as sp

from . import _lib
from ._lib import as_c128, cbuf, check


class StencilOperator:
    """Complex128 2D stencil operator on an (n1, n2) nodal grid, on the GPU."""

    def __init__(self, handle, owner=None, keepalive=()):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle
        self._owner = owner            # hierarchy that owns a borrowed handle
        self._keep = tuple(keepalive)  # operators a derived handle depends on
        n1, n2, n3, no = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        offs = (C.c_int * 375)()
        check(_lib.lib().hadr_op_info(self._h, C.byref(n1), C.byref(n2), C.byref(n3), C.byref(no), offs))
        if n3.value == 1:  # 2D operator
            self.grid_shape = (n1.value, n2.value)
            self.offsets = [(offs[3 * i], offs[3 * i + 1]) for i in range(no.value)]
        else:
            self.grid_shape = (n1.value, n2.value, n3.value)
            self.offsets = [(offs[3 * i], offs[3 * i + 1], offs[3 * i + 2]) for i in range(no.value)]

    # ---- construction ----
    @classmethod
    def from_csr(cls, A, grid_shape) -> "StencilOperator":
        """Convert a square CSR matrix on the (n1, n2[, n3]) grid (bit-exact value copy)."""
        n1, n2, n3 = _dims(grid_shape)
        A = sp.csr_matrix(A)
        if A.shape != (n1 * n2 * n3, n1 * n2 * n3):
            raise ValueError(f"operator {A.shape} does not match grid {tuple(grid_shape)}")
        if not A.has_canonical_format:
            A = A.copy()
            A.sum_duplicates()
        indptr = np.ascontiguousarray(A.indptr, dtype=np.int64)
        indices = np.ascontiguousarray(A.indices, dtype=np.int32)
        data = np.ascontiguousarray(A.data, dtype=np.complex128)
        h = C.c_void_p()
        check(_lib.lib().hadr_op_from_csr(n1, n2, n3, int(A.nnz), cbuf(indptr), cbuf(indices), cbuf(data),
                                          C.byref(h)))
        return cls(h)

    @classmethod
    def from_planes(cls, grid_shape, offsets, coef) -> "StencilOperator":
        n1, n2, n3 = _dims(grid_shape)
        offs3 = [tuple(o) + (0,) * (3 - len(o)) for o in offsets]
        offs = np.ascontiguousarray(np.asarray(offs3, dtype=np.int32).reshape(-1))
        coef = np.ascontiguousarray(np.asarray(coef, dtype=np.complex128).reshape(len(offsets), n1 * n2 * n3))
        h = C.c_void_p()
        check(_lib.lib().hadr_op_from_planes(n1, n2, n3, len(offsets), cbuf(offs), cbuf(coef), C.byref(h)))
        return cls(h)

    def __del__(self):
        try:
            if self._owner is None and self._h:
                _lib._lib.hadr_op_destroy(self._h)
                self._h = None
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    # ---- duck-typed matrix surface ----
    @property
    def shape(self):
        n = int(np.prod(self.grid_shape))
        return (n, n)

    @property
    def dtype(self):
        return np.dtype(np.complex128)

    @property
    def storage_slots(self) -> int:
        """Coefficient planes the stencil kernel reads from the pair-compressed copy
        (0: the union planes).  Built by the first apply / solve."""
        import ctypes as C

        n = C.c_int()
        check(_lib.lib().hadr_op_storage(self._h, C.byref(n), None))
        return n.value

    @property
    def mixed_rows(self) -> int:
        """Rows of a class-compressed operator whose class holds both +-2 sides of an axis."""
        import ctypes as C

        n, ov = C.c_int(), C.c_longlong()
        check(_lib.lib().hadr_op_storage(self._h, C.byref(n), C.byref(ov)))
        return ov.value

    def planes(self) -> np.ndarray:
        n = self.shape[0]
        out = np.empty((len(self.offsets), n), dtype=np.complex128)
        check(_lib.lib().hadr_op_export(self._h, cbuf(out)))
        return out

    def tocsr(self) -> sp.csr_matrix:
        """Export to canonical scipy CSR (structural zeros dropped)."""
        n1, n2, n3 = _dims(self.grid_shape)
        n = n1 * n2 * n3
        P = self.planes()
        k = np.arange(n)
        i1, rem = k // (n2 * n3), k % (n2 * n3)
        i2, i3 = rem // n3, rem % n3
        rows, cols, vals = [], [], []
        for o, d in enumerate(self.offsets):
            d1, d2, d3 = tuple(d) + (0,) * (3 - len(d))
            j1, j2, j3 = i1 + d1, i2 + d2, i3 + d3
            ok = (j1 >= 0) & (j1 < n1) & (j2 >= 0) & (j2 < n2) & (j3 >= 0) & (j3 < n3) & (P[o] != 0)
            rows.append(k[ok])
            cols.append(((j1 * n2 + j2) * n3 + j3)[ok])
            vals.append(P[o][ok])
        A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))
        A.sort_indices()
        return A

    @property
    def nnz(self) -> int:
        return int(np.count_nonzero(self.planes()))

    def diagonal(self) -> np.ndarray:
        try:
            o = self.offsets.index((0,) * len(self.grid_shape))
        except ValueError:
            return np.zeros(self.shape[0], dtype=np.complex128)
        return self.planes()[o].copy()

    def matvec(self, x) -> np.ndarray:
        """y = A x on the GPU (scipy csr_matvec accumulation order: bit-exact)."""
        x = as_c128(x, self.shape[1])
        y = np.empty_like(x)
        check(_lib.lib().hadr_op_apply(self._h, cbuf(x), cbuf(y), 0))
        return y

    def __matmul__(self, x):
        if isinstance(x, np.ndarray) and x.ndim == 1:
            return self.matvec(x)
        return NotImplemented

    def __call__(self, x):
        return self.matvec(x)

    def __repr__(self):
        return f"<StencilOperator {'x'.join(map(str, self.grid_shape))}, {len(self.offsets)} offsets, device>"


def _dims(shape):
    shape = tuple(int(v) for v in shape)
    if len(shape) == 2:
        return shape[0], shape[1], 1
    if len(shape) == 3:
        return shape
    raise ValueError(f"grid shape must have 2 or 3 axes, got {shape}")


def as_operator(A, grid_shape=None) -> StencilOperator:
    """A StencilOperator for A (StencilOperator or scipy sparse on a known grid)."""
    if isinstance(A, StencilOperator):
        return A
    if sp.issparse(A):
        if grid_shape is None:
            raise ValueError("a scipy operator needs its grid shape to become a device stencil")
        return StencilOperator.from_csr(A, grid_shape)
    raise TypeError(
        f"unsupported operator type {type(A).__name__}: the B200 path needs a StencilOperator or a scipy sparse "
        "matrix on a structured grid (no CPU fallback for arbitrary callables)"
    )


class _TransposedProlongation:
    def __init__(self, P):
        self.P = P

    @property
    def shape(self):
        return (self.P.shape[1], self.P.shape[0])

    def __matmul__(self, r):
        r = as_c128(r, self.shape[1])
        out = np.empty(self.shape[0], dtype=np.complex128)
        check(_lib.lib().hadr_transfer(*_dims(self.P.fine_shape), 0, cbuf(r), cbuf(out), 0))
        return out


class Prolongation:
    """Bilinear (2D) / trilinear (3D) P = kron of 1D interpolations, applied
    matrix-free on the device (helmadr/multigrid.py:19-46).  ``P @ e`` prolongs,
    ``P.T @ r`` restricts."""

    def __init__(self, fine_shape):
        fine_shape = tuple(int(v) for v in fine_shape)
        if any((n - 1) % 2 for n in fine_shape):
            raise ValueError(f"cannot coarsen {fine_shape}: interval count is odd")
        self.fine_shape = fine_shape
        self.coarse_shape = tuple((n - 1) // 2 + 1 for n in fine_shape)

    @property
    def shape(self):
        return (int(np.prod(self.fine_shape)), int(np.prod(self.coarse_shape)))

    @property
    def T(self):
        return _TransposedProlongation(self)

    def __matmul__(self, e):
        e = as_c128(e, self.shape[1])
        out = np.empty(self.shape[0], dtype=np.complex128)
        check(_lib.lib().hadr_transfer(*_dims(self.fine_shape), 1, cbuf(e), cbuf(out), 0))
        return out

    def tocsr(self) -> sp.csr_matrix:
        def p1(nf):
            nc = (nf - 1) // 2 + 1
            r, c, v = [], [], []
            for i in range(nf):
                if i % 2 == 0:
                    r.append(i), c.append(i // 2), v.append(1.0)
                else:
                    r += [i, i]
                    c += [i // 2, i // 2 + 1]
                    v += [0.5, 0.5]
            return sp.csr_matrix((v, (r, c)), shape=(nf, nc))

        P = p1(self.fine_shape[0])
        for n in self.fine_shape[1:]:
            P = sp.kron(P, p1(n))
        P = P.tocsr()
        P.sort_indices()
        return P
