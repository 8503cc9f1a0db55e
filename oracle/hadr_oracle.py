"""numpy/scipy restatement of the reference amplitude solve — TEST INFRASTRUCTURE ONLY.

Header (see oracle/__init__.py): this module is the checker.  The product
(`paper_1712_06091_b200`) never imports it.  Every function cites the
reference line range it restates; the arithmetic is performed with the same
numpy/scipy primitives in the same order, so on the same machine the results
match the reference bit for bit (pinned by tests/test_oracle_golden.py against
fixtures generated from the reference by tests/golden/make_golden.py).

Reference root: /root/reference/pkg/src/helmadr  (cited as helmadr/<file>.py:L)
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

# helmadr/krylov.py:12-13
REORTH_RATIO = 1.0 / np.sqrt(2.0)
BREAKDOWN_TOL = 1e-14
# helmadr/multigrid.py:15-16
COARSEST_STEPS = 10
INNER_TOL = 0.1


# --------------------------------------------------------------------------
# plain containers (duck-compatible with the reference's types)
# --------------------------------------------------------------------------
@dataclass
class Report:
    """Mirror of helmadr/krylov.py:34-53 (SolveReport)."""

    iterations: int
    history: np.ndarray
    converged: bool
    wall_time: float
    bnorm: float
    final_relres: float
    note: str = ""
    ortho_max: float = 0.0
    stage1: "Report | None" = None
    stage2: "Report | None" = None


@dataclass
class Hier:
    """Mirror of helmadr/multigrid.py:58-88 (MGHierarchy)."""

    ops: list
    prols: list
    shapes: list
    inv_diags: list = field(default_factory=list)
    coarse_steps: int = COARSEST_STEPS
    coarse_tol: float = INNER_TOL

    def __post_init__(self):
        if not self.inv_diags:
            for op in self.ops:
                d = op.diagonal()
                if np.any(d == 0):
                    raise ValueError("zero diagonal")
                self.inv_diags.append(1.0 / d)

    @property
    def n_levels(self):
        return len(self.ops)


# --------------------------------------------------------------------------
# travel-time coefficient fields   (helmadr/eikonal.py:15-36, 180-226)
# --------------------------------------------------------------------------
def distance_factor(n1, n2, L1, L2, src):
    """tau0 = |x-x0| and its analytic gradient / Laplacian, zero at x0
    (helmadr/eikonal.py:23-36, coordinates helmadr/grid.py:52-56, x0 helmadr/grid.py:124-125).
    Returns (tau0, g1, g2, lap0)."""
    h1, h2 = L1 / (n1 - 1), L2 / (n2 - 1)
    X1, X2 = np.meshgrid(np.linspace(0.0, L1, n1), np.linspace(0.0, L2, n2), indexing="ij")
    e1 = X1 - src[0] * h1
    e2 = X2 - src[1] * h2
    r = np.hypot(e1, e2)
    with np.errstate(divide="ignore", invalid="ignore"):
        g1 = np.where(r > 0, e1 / r, 0.0)
        g2 = np.where(r > 0, e2 / r, 0.0)
        l0 = np.where(r > 0, 1.0 / r, 0.0)
    return r, g1, g2, l0


def _d1(t, h, ax):
    # helmadr/eikonal.py:180-188 : centred inside, one-sided first order at the ends
    out = np.empty_like(t)
    a = np.moveaxis(t, ax, 0)
    o = np.moveaxis(out, ax, 0)
    o[1:-1] = (a[2:] - a[:-2]) / (2.0 * h)
    o[0] = (a[1] - a[0]) / h
    o[-1] = (a[-1] - a[-2]) / h
    return out


def _d2(t, h, ax):
    # helmadr/eikonal.py:191-201 : 3-point inside, 4-point one-sided at the ends
    out = np.empty_like(t)
    a = np.moveaxis(t, ax, 0)
    o = np.moveaxis(out, ax, 0)
    hh = h * h
    o[1:-1] = (a[2:] - 2.0 * a[1:-1] + a[:-2]) / hh
    o[0] = (2.0 * a[0] - 5.0 * a[1] + 4.0 * a[2] - a[3]) / hh
    o[-1] = (2.0 * a[-1] - 5.0 * a[-2] + 4.0 * a[-3] - a[-4]) / hh
    return out


def tau_fields(tau1, L1, L2, src):
    """grad(tau), lap(tau) of tau = tau0*tau1 by the chain rule
    (helmadr/eikonal.py:204-226, tau = tau0*tau1 as helmadr/eikonal.py:238).
    Returns (grad1, grad2, lap, tau)."""
    n1, n2 = tau1.shape
    h1, h2 = L1 / (n1 - 1), L2 / (n2 - 1)
    tau0, g1, g2, l0 = distance_factor(n1, n2, L1, L2, src)
    a1 = _d1(tau1, h1, 0)
    a2 = _d1(tau1, h2, 1)
    lap1 = _d2(tau1, h1, 0) + _d2(tau1, h2, 1)
    grad1 = tau0 * a1 + tau1 * g1
    grad2 = tau0 * a2 + tau1 * g2
    lap = tau1 * l0 + 2.0 * (g1 * a1 + g2 * a2) + tau0 * lap1
    i1, i2 = src
    grad1[i1, i2] = 0.0
    grad2[i1, i2] = 0.0
    lap[i1, i2] = 2.0 * tau1[i1, i2]
    return grad1, grad2, lap, tau0 * tau1


# --------------------------------------------------------------------------
# operator assembly   (helmadr/operators.py)
# --------------------------------------------------------------------------
class _Triplets:
    """COO accumulation + canonical CSR (helmadr/operators.py:54-76)."""

    def __init__(self, n):
        self.n = n
        self.r, self.c, self.v = [], [], []

    def put(self, rows, cols, vals):
        rows = np.asarray(rows).reshape(-1)
        if rows.size == 0:
            return
        self.r.append(rows.astype(np.int64))
        self.c.append(np.asarray(cols).reshape(-1).astype(np.int64))
        self.v.append(np.asarray(vals, dtype=np.complex128).reshape(-1))

    def csr(self):
        out = sp.coo_matrix(
            (np.concatenate(self.v), (np.concatenate(self.r), np.concatenate(self.c))),
            shape=(self.n, self.n),
        ).tocsr()
        out.sum_duplicates()
        out.sort_indices()
        return out


def _bc_kind(bc, axis, low):
    # helmadr/operators.py:79-82 ; axis 0 = lateral (left/right), axis 1 = depth (top/bottom)
    if axis == 0:
        return bc[2] if low else bc[3]
    return bc[0] if low else bc[1]


def _axes(n1, n2, h1, h2):
    return ((h1, n2, n1), (h2, 1, n2))


def _lap_terms(T, n1, n2, h1, h2, omega, kappa, gr1, gr2, bc):
    """Five-point Laplacian + ghost-eliminated BC rows (helmadr/operators.py:85-120).
    bc = (top, bottom, left, right) strings."""
    K = np.arange(n1 * n2).reshape(n1, n2)
    grads = (gr1, gr2)
    for ax, (h, st, sz) in enumerate(_axes(n1, n2, h1, h2)):
        ih2 = 1.0 / (h * h)
        pos = np.indices((n1, n2))[ax]
        sel = pos >= 1
        T.put(K[sel], K[sel] - st, np.full(sel.sum(), ih2))
        sel = pos <= sz - 2
        T.put(K[sel], K[sel] + st, np.full(sel.sum(), ih2))
        T.put(K, K, np.full(n1 * n2, -2.0 * ih2))
        for low in (True, False):
            sel = pos == 0 if low else pos == sz - 1
            rows = K[sel]
            nb = rows + st if low else rows - st
            nd = grads[ax][sel]
            nd = -nd if low else nd
            if _bc_kind(bc, ax, low) == "neumann":
                T.put(rows, nb, np.full(rows.size, ih2))
                T.put(rows, rows, 2j * omega * nd / h)
            else:
                T.put(rows, rows, (1.0 + 1j * omega * h * (nd - kappa[sel])) * ih2)


def _adv_terms(T, n1, n2, h1, h2, omega, c, ax, scheme, near):
    """-2i w (dtau/dx_d)(da/dx_d), one axis (helmadr/operators.py:123-170)."""
    K = np.arange(n1 * n2).reshape(n1, n2)
    h, st, sz = _axes(n1, n2, h1, h2)[ax]
    pos = np.indices((n1, n2))[ax]
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


def _mass_terms(T, n1, n2, omega, lap_tau):
    """Neighbour-averaged -i w lap(tau) a (helmadr/operators.py:173-187)."""
    K = np.arange(n1 * n2).reshape(n1, n2)
    G = -0.25j * omega * lap_tau
    for ax, (st, sz) in enumerate(((n2, n1), (1, n2))):
        pos = np.indices((n1, n2))[ax]
        for sg in (1, -1):
            ins = (pos <= sz - 2) if sg == 1 else (pos >= 1)
            T.put(K[ins], K[ins] + sg * st, G[ins])
            T.put(K[~ins], K[~ins], G[~ins])


def helmholtz_csr(n1, n2, h1, h2, omega, kappa_sq, gamma, bc):
    """helmadr/operators.py:190-200."""
    n = n1 * n2
    T = _Triplets(n)
    z = np.zeros((n1, n2))
    _lap_terms(T, n1, n2, h1, h2, omega, np.sqrt(kappa_sq), z, z, bc)
    d = omega**2 * kappa_sq - 1j * omega * gamma * kappa_sq
    T.put(np.arange(n), np.arange(n), d.reshape(-1))
    return T.csr()


def adr_csr(n1, n2, h1, h2, omega, kappa_sq, gamma, grad1, grad2, lap, src, scheme, bc):
    """helmadr/operators.py:203-234.  src = (i1, i2) or None (no near-source set)."""
    n = n1 * n2
    T = _Triplets(n)
    _lap_terms(T, n1, n2, h1, h2, omega, np.sqrt(kappa_sq), grad1, grad2, bc)
    if src is not None:
        I1, I2 = np.indices((n1, n2))
        near = (np.abs(I1 - src[0]) <= 1) & (np.abs(I2 - src[1]) <= 1)
    else:
        near = np.zeros((n1, n2), dtype=bool)
    _adv_terms(T, n1, n2, h1, h2, omega, grad1, 0, scheme, near)
    _adv_terms(T, n1, n2, h1, h2, omega, grad2, 1, scheme, near)
    _mass_terms(T, n1, n2, omega, lap)
    gsq = grad1**2 + grad2**2
    react = -(omega**2) * (gsq - kappa_sq)
    att = -1j * omega * gamma * kappa_sq
    T.put(np.arange(n), np.arange(n), (react + att).reshape(-1))
    return T.csr()


def shifted(A, alpha, omega, kappa_sq):
    """A - i w^2 alpha diag(kappa^2)   (helmadr/operators.py:237-244)."""
    d = -1j * omega**2 * alpha * kappa_sq.reshape(-1)
    out = (A + sp.diags(d)).tocsr()
    out.sort_indices()
    return out


def phase(tau, omega):
    """helmadr/operators.py:247-249."""
    return np.exp(-1j * omega * tau.reshape(-1))


def conjugate_by(A, m, direction="M_A_Minv"):
    """helmadr/operators.py:252-266."""
    m = np.asarray(m).reshape(-1)
    if direction == "M_A_Minv":
        lft, rgt = m, 1.0 / m
    else:
        lft, rgt = 1.0 / m, m
    out = (sp.diags(lft) @ A @ sp.diags(rgt)).tocsr()
    out.sort_indices()
    return out


def to_adr(q, tau, omega):
    """helmadr/operators.py:274-275."""
    return q * np.exp(1j * omega * tau)


def to_helmholtz(q, tau, omega):
    """helmadr/operators.py:276-277 (also compose_waveform, helmadr/drivers.py:171-173)."""
    return q * np.exp(-1j * omega * tau)


def delta_source(n1, n2, h1, h2, src):
    """helmadr/grid.py:128-136."""
    q = np.zeros((n1, n2), dtype=np.complex128)
    q[src[0], src[1]] = 1.0 / (h1 * h2)
    return q


# --------------------------------------------------------------------------
# multigrid   (helmadr/multigrid.py)
# --------------------------------------------------------------------------
def interp_1d(nf):
    """helmadr/multigrid.py:19-34."""
    if (nf - 1) % 2:
        raise ValueError("odd interval count")
    nc = (nf - 1) // 2 + 1
    r, c, v = [], [], []
    for i in range(nf):
        if i % 2 == 0:
            r.append(i)
            c.append(i // 2)
            v.append(1.0)
        else:
            r += [i, i]
            c += [i // 2, i // 2 + 1]
            v += [0.5, 0.5]
    return sp.csr_matrix((v, (r, c)), shape=(nf, nc))


def prolongation(shape):
    """helmadr/multigrid.py:37-46."""
    P = sp.kron(interp_1d(shape[0]), interp_1d(shape[1])).tocsr()
    P.sort_indices()
    return P


def galerkin(A, P):
    """helmadr/multigrid.py:49-55."""
    if A.shape[1] != P.shape[0]:
        raise ValueError("dimension mismatch")
    Ac = (P.T @ (A @ P)).tocsr()
    Ac.sort_indices()
    return Ac


def level_shapes(shape, max_levels):
    """helmadr/multigrid.py:98-110."""
    out = [tuple(shape)]
    while len(out) < max_levels:
        m1, m2 = out[-1]
        if (m1 - 1) % 2 or (m2 - 1) % 2:
            break
        c1, c2 = (m1 - 1) // 2 + 1, (m2 - 1) // 2 + 1
        if c1 < 3 or c2 < 3:
            break
        out.append((c1, c2))
    return out


def hierarchy(A0, shape, max_levels=5):
    """helmadr/multigrid.py:113-129."""
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


def kcycle(H, lev, b, x, visits=None):
    """One K-cycle at level lev (1 = finest)   (helmadr/multigrid.py:132-171)."""
    if visits is not None:
        visits[lev] = visits.get(lev, 0) + 1
    A = H.ops[lev - 1]
    dinv = H.inv_diags[lev - 1]
    nsm = lev + 1
    x = relax(A, dinv, b, x, nsm)
    P = H.prols[lev - 1]
    rc = P.T @ (b - A @ x)
    if lev + 1 == H.n_levels:
        ec = relax(H.ops[lev], H.inv_diags[lev], rc, np.zeros_like(rc), H.coarse_steps)
        if visits is not None:
            visits[lev + 1] = visits.get(lev + 1, 0) + 1
    else:
        ec, _ = fgmres(
            H.ops[lev], rc, None,
            lambda v: kcycle(H, lev + 1, v, np.zeros_like(v), visits),
            restart=2, maxiter=2, tol=H.coarse_tol,
        )
    x = x + P @ ec
    return relax(A, dinv, b, x, nsm)


def kcycle_precond(H):
    """helmadr/multigrid.py:174-184."""
    return lambda r: kcycle(H, 1, r, np.zeros_like(r))


# --------------------------------------------------------------------------
# Krylov   (helmadr/krylov.py)
# --------------------------------------------------------------------------
def relax(A, dinv, b, x, steps):
    """Right-Jacobi-preconditioned GMRES(steps) from x (helmadr/krylov.py:91-119)."""
    x = np.array(x, dtype=np.complex128, copy=True)
    r = b - A @ x
    beta = np.linalg.norm(r)
    if beta == 0.0 or steps < 1:
        return x
    n = x.shape[0]
    s = min(steps, n)
    V = np.empty((s + 1, n), dtype=np.complex128)
    Hs = np.zeros((s + 1, s), dtype=np.complex128)
    V[0] = r / beta
    k = 0
    for j in range(s):
        w = A @ (dinv * V[j])
        for i in range(j + 1):
            hij = np.vdot(V[i], w)
            Hs[i, j] = hij
            w -= hij * V[i]
        hn = np.linalg.norm(w)
        Hs[j + 1, j] = hn
        k = j + 1
        if hn <= BREAKDOWN_TOL * beta:
            break
        V[j + 1] = w / hn
    rhs = np.zeros(k + 1, dtype=np.complex128)
    rhs[0] = beta
    y, *_ = np.linalg.lstsq(Hs[: k + 1, :k], rhs, rcond=None)
    return x + dinv * (V[:k].T @ y)


def _matvec_of(A):
    return A if callable(A) else (lambda v: A @ v)


def fgmres(A, b, x0=None, M=None, restart=5, maxiter=200, tol=1e-5, diagnostics=False, flexible=True):
    """Restarted (flexible) GMRES with MGS + one conditional re-orthogonalisation
    and complex Givens (helmadr/krylov.py:122-242).  flexible=False: x += M(V[:k]^T y)
    (helmadr/krylov.py:222-223).  Returns (x, Report)."""
    t0 = time.perf_counter()
    mv = _matvec_of(A)
    b = np.asarray(b, dtype=np.complex128).reshape(-1)
    n = b.shape[0]
    x = np.zeros(n, dtype=np.complex128) if x0 is None else np.array(x0, dtype=np.complex128, copy=True).reshape(-1)
    pc = M if M is not None else (lambda v: v)
    bn = float(np.linalg.norm(b))
    if bn == 0.0:
        return np.zeros(n, dtype=np.complex128), Report(0, np.array([0.0]), True, time.perf_counter() - t0, 0.0, 0.0)
    r = b - mv(x)
    rn = float(np.linalg.norm(r))
    hist = [rn]
    goal = tol * bn
    it = 0
    note = ""
    omax = 0.0
    while it < maxiter and rn > goal:
        m = min(restart, maxiter - it)
        V = np.empty((m + 1, n), dtype=np.complex128)
        Z = np.empty((m, n), dtype=np.complex128)
        Hm = np.zeros((m + 1, m), dtype=np.complex128)
        cs = np.zeros(m, dtype=np.complex128)
        sn = np.zeros(m, dtype=np.complex128)
        g = np.zeros(m + 1, dtype=np.complex128)
        g[0] = rn
        V[0] = r / rn
        k = 0
        broke = False
        for j in range(m):
            z = pc(V[j])
            Z[j] = z
            w = mv(z)
            w0 = np.linalg.norm(w)
            for i in range(j + 1):
                hij = np.vdot(V[i], w)
                Hm[i, j] = hij
                w -= hij * V[i]
            wn = np.linalg.norm(w)
            if wn < REORTH_RATIO * w0:
                for i in range(j + 1):
                    cor = np.vdot(V[i], w)
                    Hm[i, j] += cor
                    w -= cor * V[i]
                wn = np.linalg.norm(w)
            Hm[j + 1, j] = wn
            if not np.isfinite(wn):
                note = "numerical breakdown: non-finite Arnoldi vector"
                broke = True
                k = j
                break
            lucky = wn <= BREAKDOWN_TOL * max(bn, 1e-300)
            if not lucky:
                V[j + 1] = w / wn
            for i in range(j):
                t = cs[i] * Hm[i, j] + sn[i] * Hm[i + 1, j]
                Hm[i + 1, j] = -np.conj(sn[i]) * Hm[i, j] + np.conj(cs[i]) * Hm[i + 1, j]
                Hm[i, j] = t
            den = np.sqrt(np.abs(Hm[j, j]) ** 2 + np.abs(Hm[j + 1, j]) ** 2)
            if den == 0.0:
                cs[j], sn[j] = 1.0, 0.0
            else:
                cs[j] = np.conj(Hm[j, j]) / den
                sn[j] = np.conj(Hm[j + 1, j]) / den
            Hm[j, j] = cs[j] * Hm[j, j] + sn[j] * Hm[j + 1, j]
            Hm[j + 1, j] = 0.0
            g[j + 1] = -np.conj(sn[j]) * g[j]
            g[j] = cs[j] * g[j]
            it += 1
            k = j + 1
            hist.append(float(np.abs(g[j + 1])))
            if lucky or hist[-1] <= goal:
                break
        if diagnostics and k > 0:
            G = V[:k] @ V[:k].conj().T
            np.fill_diagonal(G, 0.0)
            omax = max(omax, float(np.abs(G).max()))
        if k > 0:
            y = np.linalg.solve(Hm[:k, :k], g[:k]) if k > 1 else g[:1] / Hm[0, 0]
            x = x + Z[:k].T @ y if flexible else x + pc(V[:k].T @ y)
        r = b - mv(x)
        rn = float(np.linalg.norm(r))
        if broke:
            break
    conv = rn <= goal * (1.0 + 1e-12) and not note
    rep = Report(it, np.asarray(hist), bool(conv), time.perf_counter() - t0, bn, rn / bn, note, omax)
    return x, rep


# --------------------------------------------------------------------------
# strategies   (helmadr/drivers.py)
# --------------------------------------------------------------------------
@dataclass
class Problem:
    """Everything a strategy needs; fields are (n1, n2) arrays."""

    n1: int
    n2: int
    h1: float
    h2: float
    omega: float
    src: tuple
    kappa_sq: np.ndarray
    gamma: np.ndarray
    tau: np.ndarray
    grad1: np.ndarray
    grad2: np.ndarray
    lap: np.ndarray
    bc: tuple = ("neumann", "sommerfeld", "sommerfeld", "sommerfeld")


def adr_of(p: Problem, scheme):
    return adr_csr(p.n1, p.n2, p.h1, p.h2, p.omega, p.kappa_sq, p.gamma,
                   p.grad1, p.grad2, p.lap, p.src, scheme, p.bc)


def helm_of(p: Problem):
    return helmholtz_csr(p.n1, p.n2, p.h1, p.h2, p.omega, p.kappa_sq, p.gamma, p.bc)


def solve_upwind(p: Problem, beta=0.25, restart=5, tol=1e-5, maxiter=400, levels=5):
    """helmadr/drivers.py:136-168.  Returns (u, a, report)."""
    q = delta_source(p.n1, p.n2, p.h1, p.h2, p.src)
    qh = to_adr(q, p.tau, p.omega).reshape(-1)
    t0 = time.perf_counter()
    H2 = adr_of(p, "upwind2")
    H1 = adr_of(p, "upwind1")
    B = ((1.0 - beta) * H2 + beta * H1).tocsr()
    Hi = hierarchy(B, (p.n1, p.n2), levels)
    a, rep = fgmres(H2, qh, None, kcycle_precond(Hi), restart, maxiter, tol)
    rep.wall_time = time.perf_counter() - t0
    a = a.reshape(p.n1, p.n2)
    return to_helmholtz(a, p.tau, p.omega), a, rep


def solve_sl(H, q, p: Problem, alpha=0.2, restart=5, tol=1e-5, maxiter=400, levels=5):
    """helmadr/drivers.py:57-67.  Returns (u, report)."""
    Hs = shifted(H, alpha, p.omega, p.kappa_sq)
    Hi = hierarchy(Hs, (p.n1, p.n2), levels)
    x, rep = fgmres(H, q.reshape(-1), None, kcycle_precond(Hi), restart, maxiter, tol)
    return x.reshape(p.n1, p.n2), rep


def solve_central(p: Problem, alpha=0.2, s1_cycles=5, s1_tol=1e-2, restart=5, tol=1e-5,
                  maxiter=400, levels=5):
    """Two-stage central ADR (helmadr/drivers.py:70-133).  Returns (u, a, report)."""
    q = delta_source(p.n1, p.n2, p.h1, p.h2, p.src).reshape(-1)
    qh = to_adr(q.reshape(p.n1, p.n2), p.tau, p.omega).reshape(-1)
    m = phase(p.tau, p.omega)
    t0 = time.perf_counter()
    H1 = adr_of(p, "upwind1")
    Hi1 = hierarchy(H1, (p.n1, p.n2), levels)
    a1, r1 = fgmres(H1, qh, None, kcycle_precond(Hi1), restart, s1_cycles, s1_tol)
    u0 = m * a1
    Hc = adr_of(p, "central")
    Ar = conjugate_by(Hc, m, "M_A_Minv")
    Hs = shifted(Ar, alpha, p.omega, p.kappa_sq)
    Hi2 = hierarchy(Hs, (p.n1, p.n2), levels)
    u, r2 = fgmres(Ar, q, u0, kcycle_precond(Hi2), restart, maxiter, tol)
    el = time.perf_counter() - t0
    a = to_adr(u.reshape(p.n1, p.n2), p.tau, p.omega)
    rep = Report(r1.iterations + r2.iterations, r2.history, r2.converged, el, r2.bnorm,
                 r2.final_relres, stage1=r1, stage2=r2)
    return u.reshape(p.n1, p.n2), a, rep


# --------------------------------------------------------------------------
# accuracy workflow and field dumps

def error_map(u, u_ref, floor=None):
    """helmadr/grid.py:175-191: |u - u_ref| / max(|u_ref|, floor), floor default
    1e-12 max|u_ref|."""
    u = np.asarray(u)
    u_ref = np.asarray(u_ref)
    if u.shape != u_ref.shape:
        raise ValueError("grid mismatch")
    mag = np.abs(u_ref)
    fl = 1e-12 * float(mag.max()) if floor is None else floor
    if fl < 0:
        raise ValueError("floor must be non-negative")
    return np.abs(u - u_ref) / np.where(mag < fl, fl, mag)


def compare(solutions, u_ref, floor=None):
    """helmadr/drivers.py:176-196: median / p95 / max of the error map over |u_ref| >= floor."""
    u_ref = np.asarray(u_ref)
    fl = 1e-12 * float(np.abs(u_ref).max()) if floor is None else floor
    keep = np.abs(u_ref) >= fl
    res = {}
    for name, u in solutions:
        e = error_map(u, u_ref, fl)
        v = e[keep]
        res[name] = {"median": float(np.median(v)), "p95": float(np.percentile(v, 95)), "max": float(v.max()),
                     "error_map": e}
    return res


def dump_bytes(values):
    """helmadr/models.py:100-113 payload: little-endian float64, complex as (re, im) pairs."""
    values = np.asarray(values)
    if np.iscomplexobj(values):
        flat = np.empty(2 * values.size)
        flat[0::2] = values.real.reshape(-1)
        flat[1::2] = values.imag.reshape(-1)
    else:
        flat = values.astype(np.float64).reshape(-1)
    return flat.astype("<f8").tobytes()
