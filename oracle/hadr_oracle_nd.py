"""Dimension-generic (2D/3D) restatement of the reference's assembly, transfer
operators and hierarchy — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The reference is 2D-only (helmadr/grid.py:21-56); BASELINE
configs 4 and 5 are 3D, so the 3D oracle is a restatement of the 2D code
generalised per axis.  Every routine here is written once
for any number of axes and loops over the axes in the reference's order with
the reference's operations, so its **2D instantiation reproduces the reference
bit for bit** (tests/test_oracle_golden.py::test_nd_oracle_2d_is_bitexact) and
the 3D instantiation is the same code with a third axis.

3D decisions (not facts of the reference):
* axes: (x1, x2, depth); the last axis is depth (fastest in memory), as in 2D;
* boundary faces: axis 0 (left, right), axis 1 (front, back) in 3D, last axis (top, bottom);
* mass averaging weight 1/(2*dim) over the 2*dim axis neighbours (2D: 1/4);
* tau0 = |x - x0| with lap(tau0) = (dim - 1)/r (2D: 1/r);
* trilinear P = kron of three 1D interpolations (restriction P^T = 8x full weighting).
Krylov, relaxation and the K-cycle are dimension-agnostic: use hadr_oracle.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .hadr_oracle import Hier, _Triplets, interp_1d


def _strides(shape):
    st = []
    for ax in range(len(shape)):
        st.append(int(np.prod(shape[ax + 1:], dtype=np.int64)))
    return st


def _faces(dim, bc):
    """(low, high) face kinds per axis.  bc: dict of side -> kind."""
    if dim == 2:
        names = (("left", "right"), ("top", "bottom"))
    else:
        names = (("left", "right"), ("front", "back"), ("top", "bottom"))
    return [(bc[lo], bc[hi]) for lo, hi in names]


def bc_dict(dim, kinds):
    """kinds: 2D (top, bottom, left, right) like the reference BCSpec; 3D adds (front, back)."""
    keys = ("top", "bottom", "left", "right") + (("front", "back") if dim == 3 else ())
    return dict(zip(keys, kinds))


# --------------------------------------------------------------------------
# travel-time fields   (helmadr/eikonal.py:15-36, 180-226 per axis)
# --------------------------------------------------------------------------
def distance_factor(shape, Ls, src):
    dim = len(shape)
    hs = [L / (n - 1) for n, L in zip(shape, Ls)]
    X = np.meshgrid(*[np.linspace(0.0, L, n) for n, L in zip(shape, Ls)], indexing="ij")
    e = [X[a] - src[a] * hs[a] for a in range(dim)]
    r = np.hypot(e[0], e[1]) if dim == 2 else np.sqrt(e[0] ** 2 + e[1] ** 2 + e[2] ** 2)
    with np.errstate(divide="ignore", invalid="ignore"):
        g = [np.where(r > 0, ea / r, 0.0) for ea in e]
        l0 = np.where(r > 0, (dim - 1.0) / r, 0.0)
    return r, g, l0


def _d1(t, h, ax):
    out = np.empty_like(t)
    a = np.moveaxis(t, ax, 0)
    o = np.moveaxis(out, ax, 0)
    o[1:-1] = (a[2:] - a[:-2]) / (2.0 * h)
    o[0] = (a[1] - a[0]) / h
    o[-1] = (a[-1] - a[-2]) / h
    return out


def _d2(t, h, ax):
    out = np.empty_like(t)
    a = np.moveaxis(t, ax, 0)
    o = np.moveaxis(out, ax, 0)
    hh = h * h
    o[1:-1] = (a[2:] - 2.0 * a[1:-1] + a[:-2]) / hh
    o[0] = (2.0 * a[0] - 5.0 * a[1] + 4.0 * a[2] - a[3]) / hh
    o[-1] = (2.0 * a[-1] - 5.0 * a[-2] + 4.0 * a[-3] - a[-4]) / hh
    return out


def tau_fields(tau1, Ls, src):
    """Returns (grads list, lap, tau) (helmadr/eikonal.py:204-226, per axis)."""
    shape = tau1.shape
    dim = len(shape)
    hs = [L / (n - 1) for n, L in zip(shape, Ls)]
    tau0, g, l0 = distance_factor(shape, Ls, src)
    a = [_d1(tau1, hs[ax], ax) for ax in range(dim)]
    lap1 = _d2(tau1, hs[0], 0) + _d2(tau1, hs[1], 1)
    for ax in range(2, dim):
        lap1 = lap1 + _d2(tau1, hs[ax], ax)
    grads = [tau0 * a[ax] + tau1 * g[ax] for ax in range(dim)]
    s = g[0] * a[0] + g[1] * a[1]
    for ax in range(2, dim):
        s = s + g[ax] * a[ax]
    lap = tau1 * l0 + 2.0 * s + tau0 * lap1
    idx = tuple(src)
    for gr in grads:
        gr[idx] = 0.0
    lap[idx] = 2.0 * tau1[idx]
    return grads, lap, tau0 * tau1


# --------------------------------------------------------------------------
# assembly (helmadr/operators.py:85-234, per axis)
# --------------------------------------------------------------------------
def _lap_terms(T, shape, hs, omega, kappa, grads, bc):
    N = int(np.prod(shape))
    K = np.arange(N).reshape(shape)
    faces = _faces(len(shape), bc)
    for ax, (h, st, sz) in enumerate(zip(hs, _strides(shape), shape)):
        ih2 = 1.0 / (h * h)
        pos = np.indices(shape)[ax]
        sel = pos >= 1
        T.put(K[sel], K[sel] - st, np.full(sel.sum(), ih2))
        sel = pos <= sz - 2
        T.put(K[sel], K[sel] + st, np.full(sel.sum(), ih2))
        T.put(K, K, np.full(N, -2.0 * ih2))
        for low in (True, False):
            sel = pos == 0 if low else pos == sz - 1
            rows = K[sel]
            nb = rows + st if low else rows - st
            nd = grads[ax][sel]
            nd = -nd if low else nd
            if faces[ax][0 if low else 1] == "neumann":
                T.put(rows, nb, np.full(rows.size, ih2))
                T.put(rows, rows, 2j * omega * nd / h)
            else:
                T.put(rows, rows, (1.0 + 1j * omega * h * (nd - kappa[sel])) * ih2)


def _adv_terms(T, shape, hs, omega, c, ax, scheme, near):
    K = np.arange(int(np.prod(shape))).reshape(shape)
    h, st, sz = hs[ax], _strides(shape)[ax], shape[ax]
    pos = np.indices(shape)[ax]
    F = -2j * omega * c
    inner = (pos >= 1) & (pos <= sz - 2)
    cen = inner if scheme == "central" else inner & near
    chain = ~cen
    order = 1 if scheme == "upwind1" else 2
    T.put(K[cen], K[cen] + st, F[cen] / (2.0 * h))
    T.put(K[cen], K[cen] - st, -F[cen] / (2.0 * h))
    for sg in (1, -1):
        mc = chain & (c > 0 if sg == 1 else c < 0)
        if not mc.any():
            continue
        ok2 = (pos >= 2) if sg == 1 else (pos <= sz - 3)
        ok1 = (pos >= 1) if sg == 1 else (pos <= sz - 2)
        s2 = mc & ok2 if order == 2 else np.zeros_like(mc)
        s1 = mc & ok1 & ~s2
        s0 = mc & ~ok1
        s = sg * st
        if s2.any():
            T.put(K[s2], K[s2], sg * 3.0 * F[s2] / (2.0 * h))
            T.put(K[s2], K[s2] - s, -sg * 4.0 * F[s2] / (2.0 * h))
            T.put(K[s2], K[s2] - 2 * s, sg * F[s2] / (2.0 * h))
        if s1.any():
            T.put(K[s1], K[s1], sg * F[s1] / h)
            T.put(K[s1], K[s1] - s, -sg * F[s1] / h)
        if s0.any():
            T.put(K[s0], K[s0], -sg * F[s0] / h)
            T.put(K[s0], K[s0] + s, sg * F[s0] / h)


def mass_weight(dim):
    """-i/(2 dim): the 2D reference's -0.25j (helmadr/operators.py:179), 3D -i/6."""
    return -0.25j if dim == 2 else -1j / 6.0


def _mass_terms(T, shape, omega, lap_tau):
    K = np.arange(int(np.prod(shape))).reshape(shape)
    G = mass_weight(len(shape)) * omega * lap_tau
    for ax, (st, sz) in enumerate(zip(_strides(shape), shape)):
        pos = np.indices(shape)[ax]
        for sg in (1, -1):
            ins = (pos <= sz - 2) if sg == 1 else (pos >= 1)
            T.put(K[ins], K[ins] + sg * st, G[ins])
            T.put(K[~ins], K[~ins], G[~ins])


def helmholtz_csr(shape, hs, omega, kappa_sq, gamma, bc):
    N = int(np.prod(shape))
    T = _Triplets(N)
    z = np.zeros(shape)
    _lap_terms(T, shape, hs, omega, np.sqrt(kappa_sq), [z] * len(shape), bc)
    d = omega**2 * kappa_sq - 1j * omega * gamma * kappa_sq
    T.put(np.arange(N), np.arange(N), d.reshape(-1))
    return T.csr()


def adr_csr(shape, hs, omega, kappa_sq, gamma, grads, lap, src, scheme, bc):
    N = int(np.prod(shape))
    T = _Triplets(N)
    _lap_terms(T, shape, hs, omega, np.sqrt(kappa_sq), grads, bc)
    if src is not None:
        I = np.indices(shape)
        near = np.abs(I[0] - src[0]) <= 1
        for ax in range(1, len(shape)):
            near = near & (np.abs(I[ax] - src[ax]) <= 1)
    else:
        near = np.zeros(shape, dtype=bool)
    for ax in range(len(shape)):
        _adv_terms(T, shape, hs, omega, grads[ax], ax, scheme, near)
    _mass_terms(T, shape, omega, lap)
    gsq = grads[0] ** 2 + grads[1] ** 2
    for ax in range(2, len(shape)):
        gsq = gsq + grads[ax] ** 2
    react = -(omega**2) * (gsq - kappa_sq)
    att = -1j * omega * gamma * kappa_sq
    T.put(np.arange(N), np.arange(N), (react + att).reshape(-1))
    return T.csr()


def delta_source(shape, hs, src):
    q = np.zeros(shape, dtype=np.complex128)
    q[tuple(src)] = 1.0 / float(np.prod(hs))
    return q


# --------------------------------------------------------------------------
# multigrid (helmadr/multigrid.py:19-129, per axis)
# --------------------------------------------------------------------------
def prolongation(shape):
    P = interp_1d(shape[0])
    for n in shape[1:]:
        P = sp.kron(P, interp_1d(n))
    P = P.tocsr()
    P.sort_indices()
    return P


def level_shapes(shape, max_levels):
    out = [tuple(shape)]
    while len(out) < max_levels:
        m = out[-1]
        if any((mi - 1) % 2 for mi in m):
            break
        c = tuple((mi - 1) // 2 + 1 for mi in m)
        if any(ci < 3 for ci in c):
            break
        out.append(c)
    return out


def hierarchy(A0, shape, max_levels=5):
    from .hadr_oracle import galerkin

    shapes = level_shapes(shape, max_levels)
    if len(shapes) < 2:
        raise ValueError("fewer than two levels")
    ops = [A0.tocsr()]
    prols = []
    for fs in shapes[:-1]:
        P = prolongation(fs)
        prols.append(P)
        ops.append(galerkin(ops[-1], P))
    return Hier(ops=ops, prols=prols, shapes=shapes)


def solve_upwind(shape, hs, omega, src, kappa_sq, gamma, grads, lap, tau, bc, beta=0.25, tol=1e-6, maxiter=1000,
                 levels=5):
    """helmadr/drivers.py:136-168 in any dimension.  Returns (a, report)."""
    from .hadr_oracle import fgmres, kcycle_precond, to_adr

    q = delta_source(shape, hs, src)
    qh = to_adr(q, tau, omega).reshape(-1)
    H2 = adr_csr(shape, hs, omega, kappa_sq, gamma, grads, lap, src, "upwind2", bc)
    H1 = adr_csr(shape, hs, omega, kappa_sq, gamma, grads, lap, src, "upwind1", bc)
    B = ((1.0 - beta) * H2 + beta * H1).tocsr()
    Hi = hierarchy(B, shape, levels)
    a, rep = fgmres(H2, qh, None, kcycle_precond(Hi), 5, maxiter, tol)
    return a.reshape(shape), rep


def solve_sl(shape, hs, omega, src, kappa_sq, gamma, bc, alpha=0.5, tol=1e-6, maxiter=1000, levels=5):
    """helmadr/drivers.py:57-67 (standard_sl) in any dimension: FGMRES on the standard
    Helmholtz operator preconditioned by K-cycles on H - i alpha w^2 diag(kappa^2)
    (helmadr/operators.py:237-244).  Returns (u, report)."""
    from .hadr_oracle import fgmres, kcycle_precond, shifted

    H = helmholtz_csr(shape, hs, omega, kappa_sq, gamma, bc)
    Hi = hierarchy(shifted(H, alpha, omega, kappa_sq), shape, levels)
    q = delta_source(shape, hs, src).reshape(-1)
    u, rep = fgmres(H, q, None, kcycle_precond(Hi), 5, maxiter, tol)
    return u.reshape(shape), rep
