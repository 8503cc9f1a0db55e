"""GPU tests of the drop-in surface beyond the solver kernels:

* ``tau_derivatives`` on the device (helmadr/eikonal.py:180-226, with AnalyticBase's
  distance factor, 15-36): bit-identical to the reference's fields (golden vectors) and to
  the ND oracle in 3D; a solve from tau1 alone equals the solve from host fields;
* ``KrylovConfig`` switches: ``collect_diagnostics`` -> ``ortho_max``
  (helmadr/krylov.py:214-217), ``flexible=False`` (222-223), ``maxiter < 0``;
* the reference's documented argument types: scipy matrices into ``spmv`` /
  ``jacobi_apply`` / ``gmres_relax`` (helmadr/krylov.py:60-88), the
  ``MGHierarchy(ops, prols, shapes)`` constructor (helmadr/multigrid.py:58-81),
  ``export_operator_coo`` (helmadr/operators.py:281-286);
* INTEGRATION.md §1's monkey-patch: the reference's ``solve_adr_upwind`` call sequence
  (helmadr/drivers.py:146-168) with the three names it binds at import
  (helmadr/drivers.py:14-15) re-bound to this package, on reference-shaped inputs
  (scipy CSR operators, a GridSpec-like grid, the reference's KrylovConfig fields).
"""

import types

import numpy as np
import pytest
from conftest import csr_from, oracle_problem
from parity_util import protocol_bar, rel, self_floor

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hadr():
    import paper_1712_06091_b200 as H

    H._lib.lib()  # raises if no device / no library: no fallback
    return H


# --------------------------------------------------------------------------
# tau_derivatives on the device
# --------------------------------------------------------------------------
@pytest.mark.parametrize("case", ["g33", "g65", "gcfg3"])
def test_tau_derivatives_device_bitexact(hadr, case, request):
    """Device tau = tau0 tau1, grad(tau), lap(tau) from tau1 == the reference's own
    tau_derivatives output (golden vectors made by helmadr/eikonal.py), bit for bit."""
    from paper_1712_06091_b200 import eikonal, fields, workloads
    from paper_1712_06091_b200.eikonal import _tau_fields_device

    g = request.getfixturevalue(case)
    wl = {"g33": lambda: workloads.cfg1(33), "g65": lambda: workloads.cfg2(65),
          "gcfg3": lambda: workloads.cfg3(65)}[case]()
    tau1 = wl.tt.tau1
    tau, grads, lap = _tau_fields_device(wl.grid, wl.source.index, tau1)
    for k, v in (("grad1", grads[0]), ("grad2", grads[1]), ("lap", lap), ("tau", tau)):
        assert np.array_equal(v, g[k]), k
    (g1, g2), lp = eikonal.tau_derivatives(tau1, fields.AnalyticBase(wl.grid, wl.source), wl.grid)
    assert np.array_equal(g1, g["grad1"]) and np.array_equal(g2, g["grad2"]) and np.array_equal(lp, g["lap"])


@pytest.mark.parametrize("which", ["cfg4_17", "cfg4_33", "cfg5_33"])
def test_tau_derivatives_device_3d(hadr, which):
    """3D (per-axis restatement, lap(tau0) = 2/r): device fields == the ND oracle's."""
    from oracle import hadr_oracle_nd as ND
    from paper_1712_06091_b200 import workloads
    from paper_1712_06091_b200.eikonal import _tau_fields_device

    name, n = which.split("_")
    wl = workloads.by_name(name, int(n))
    tau, grads, lap = _tau_fields_device(wl.grid, wl.source.index, wl.tt.tau1)
    g_ref, lap_ref, tau_ref = ND.tau_fields(wl.tt.tau1, wl.grid.Ls, wl.source.index)
    for a, b in zip(grads, g_ref):
        assert np.array_equal(a, b)
    assert np.array_equal(lap, lap_ref) and np.array_equal(tau, tau_ref)


@pytest.mark.parametrize("n", [65, 129])
def test_solve_from_tau1_only_identical(hadr, n):
    """drivers.solve_adr_upwind with a DeviceTravelTime (only tau1 crosses the link, the
    derivative fields are formed on the device) == the solve from host-formed fields."""
    from paper_1712_06091_b200 import drivers, fields, workloads

    wl = workloads.cfg2(n)
    cfg = drivers.StrategyConfig(strategy="adr_upwind_blend", tol=1e-6, max_iter=1000)
    u0, a0, r0 = drivers.solve_adr_upwind(wl.medium, wl.grid, wl.source, wl.tt, cfg, wl.bc)
    dtt = fields.DeviceTravelTime(wl.grid, wl.source, wl.tt.tau1)
    u1, a1, r1 = drivers.solve_adr_upwind(wl.medium, wl.grid, wl.source, dtt, cfg, wl.bc)
    assert r1.iterations == r0.iterations
    assert np.array_equal(a1, a0) and np.array_equal(u1, u0)
    # host reads of a DeviceTravelTime's fields are the same values
    assert np.array_equal(dtt.lap, wl.tt.lap) and np.array_equal(dtt.grad2, wl.tt.grad2)


# --------------------------------------------------------------------------
# KrylovConfig switches
# --------------------------------------------------------------------------
def _g65_problem(hadr):
    from oracle import hadr_oracle as O
    from paper_1712_06091_b200 import workloads

    p = oracle_problem(workloads.cfg2(65))
    q = O.delta_source(p.n1, p.n2, p.h1, p.h2, p.src)
    qh = O.to_adr(q, p.tau, p.omega).reshape(-1)
    H2 = O.adr_of(p, "upwind2")
    B = (0.75 * H2 + 0.25 * O.adr_of(p, "upwind1")).tocsr()
    return p, qh, H2, B


def test_collect_diagnostics_ortho_max(hadr):
    """collect_diagnostics: ortho_max = max |<v_i, v_j>| (i != j) of the Arnoldi basis
    over the cycles (helmadr/krylov.py:214-217) — rounding-level, like the oracle's;
    without the flag it is 0 as in the reference."""
    from oracle import hadr_oracle as O

    p, qh, H2, B = _g65_problem(hadr)
    _, r_or = O.fgmres(H2, qh, None, O.kcycle_precond(O.hierarchy(B, (p.n1, p.n2), 5)), 5, 1000, 1e-6,
                       diagnostics=True)
    A = hadr.StencilOperator.from_csr(H2, (p.n1, p.n2))
    M = hadr.make_kcycle_preconditioner(hadr.build_hierarchy(B, (p.n1, p.n2), 5))
    x0, r0 = hadr.fgmres(A, qh, None, M, hadr.KrylovConfig(restart=5, maxiter=1000, tol=1e-6))
    x1, r1 = hadr.fgmres(A, qh, None, M, hadr.KrylovConfig(restart=5, maxiter=1000, tol=1e-6,
                                                           collect_diagnostics=True))
    assert r0.ortho_max == 0.0
    assert 0.0 < r1.ortho_max <= 1e-12 and 0.0 < r_or.ortho_max <= 1e-12
    assert np.array_equal(x0, x1) and r0.iterations == r1.iterations  # diagnostics do not perturb the solve


def test_nonflexible_fgmres(hadr):
    """flexible=False: x += M(V[:k]^T y) per cycle (helmadr/krylov.py:222-223).  Without a
    preconditioner it is the flexible solve; with the K-cycle it matches the oracle's
    non-flexible solve (tol 1e-10: <= 1e-8 strictly, iterations +-1)."""
    from oracle import hadr_oracle as O

    p, qh, H2, B = _g65_problem(hadr)
    A = hadr.StencilOperator.from_csr(H2, (p.n1, p.n2))
    cf = hadr.KrylovConfig(restart=5, maxiter=60, tol=1e-6)
    cn = hadr.KrylovConfig(restart=5, maxiter=60, tol=1e-6, flexible=False)
    xa, ra = hadr.fgmres(A, qh, None, None, cf)
    xb, rb = hadr.fgmres(A, qh, None, None, cn)
    assert np.array_equal(xa, xb) and ra.iterations == rb.iterations
    a_or, r_or = O.fgmres(H2, qh, None, O.kcycle_precond(O.hierarchy(B, (p.n1, p.n2), 5)), 5, 1000, 1e-10,
                          flexible=False)
    M = hadr.make_kcycle_preconditioner(hadr.build_hierarchy(B, (p.n1, p.n2), 5))
    x, rep = hadr.fgmres(A, qh, None, M, hadr.KrylovConfig(restart=5, maxiter=1000, tol=1e-10, flexible=False))
    assert rep.converged and abs(rep.iterations - r_or.iterations) <= 1
    assert rel(x, a_or) <= 1e-8


def test_negative_maxiter(hadr, g33):
    """maxiter < 0: no iteration, x0 returned, history [||r0||] (helmadr/krylov.py:154)."""
    A = csr_from(g33, "blend")
    op = hadr.StencilOperator.from_csr(A, (33, 33))
    b = np.ones(A.shape[0], complex)
    x, rep = hadr.fgmres(op, b, None, None, hadr.KrylovConfig(restart=5, maxiter=-3, tol=1e-6))
    assert rep.iterations == 0 and not np.any(x) and len(rep.history) == 1 and not rep.converged


# --------------------------------------------------------------------------
# reference argument types
# --------------------------------------------------------------------------
def test_scipy_inputs(hadr, g33):
    """spmv / jacobi_apply / gmres_relax take plain scipy matrices (the reference's
    documented type): the grid is inferred for square (m^2) operators or passed."""
    A = csr_from(g33, "lev0")
    b, x = g33["rnd_b"], g33["rnd_x"]
    assert np.array_equal(hadr.spmv(A, b), A @ b)
    assert np.array_equal(hadr.jacobi_apply(A, b), b / A.diagonal())
    assert rel(hadr.gmres_relax(A, b, x, 2), g33["relax2"]) <= 1e-12
    assert rel(hadr.gmres_relax(A, b, x, 2, grid=(33, 33)), g33["relax2"]) <= 1e-12
    import scipy.sparse as sp

    R = sp.random(33 * 17, 33 * 17, density=0.0, format="csr") + sp.identity(33 * 17, format="csr")
    with pytest.raises(ValueError):
        hadr.spmv(R, np.ones(33 * 17))  # neither m^2 nor m^3 points, no grid
    assert np.array_equal(hadr.spmv(R, np.ones(33 * 17), grid=(33, 17)), np.ones(33 * 17))


def test_mghierarchy_reference_constructor(hadr, g33):
    """MGHierarchy(ops=..., prols=..., shapes=...) as the reference builds it
    (helmadr/multigrid.py:126-129), from the reference's own CSR levels and scipy
    prolongations: the K-cycle equals the reference's (golden) to rounding."""
    from oracle import hadr_oracle as O

    n = int(g33["n_levels"])
    shapes = [tuple(int(v) for v in s) for s in g33["shapes"]]
    ops = [csr_from(g33, f"lev{l}") for l in range(n)]
    prols = [O.prolongation(s) for s in shapes[:-1]]
    H = hadr.MGHierarchy(ops=ops, prols=prols, shapes=shapes)
    assert H.n_levels == n and H.shapes == shapes
    b = g33["rnd_b"]
    assert rel(hadr.k_cycle(H, 1, b, np.zeros_like(b)), g33["kcycle"]) <= 1e-12
    H2 = hadr.MGHierarchy(ops=ops, prols=prols, shapes=shapes, inv_diags=[1.0 / A.diagonal() for A in ops])
    assert rel(hadr.make_kcycle_preconditioner(H2)(b), g33["kcycle"]) <= 1e-12
    bad = list(prols)
    bad[0] = 2.0 * bad[0]
    with pytest.raises(ValueError):
        hadr.MGHierarchy(ops=ops, prols=bad, shapes=shapes)


def test_export_operator_coo(hadr, g33, tmp_path):
    """export_operator_coo writes the reference's 'row col re im' lines (repr floats) in
    canonical CSR order (helmadr/operators.py:281-286)."""
    from paper_1712_06091_b200.operators import export_operator_coo

    A = csr_from(g33, "blend")
    A.eliminate_zeros()
    op = hadr.StencilOperator.from_csr(A, (33, 33))
    path = tmp_path / "op.txt"
    export_operator_coo(op, str(path))
    coo = A.tocoo()
    want = "".join(f"{r} {c} {v.real!r} {v.imag!r}\n" for r, c, v in zip(coo.row, coo.col, coo.data))
    assert path.read_text() == want


def test_integration_monkeypatch(hadr, g65):
    """the reference driver's body (helmadr/drivers.py:146-168) looks up
    ``fgmres``, ``build_hierarchy`` and ``make_kcycle_preconditioner`` as module globals
    bound at import (helmadr/drivers.py:14-15).  Re-binding exactly those three names to
    this package runs the reference's own call sequence on the GPU with reference-shaped
    inputs: scipy CSR operators, a GridSpec-like grid object, a KrylovConfig-like cfg."""
    from oracle import hadr_oracle as O
    from paper_1712_06091_b200 import workloads

    wl = workloads.cfg2(65)
    p = oracle_problem(wl)

    class GridSpec:  # helmadr/grid.py:21-56 surface the hierarchy needs
        shape = (p.n1, p.n2)
        n_nodes = p.n1 * p.n2

    class KrylovConfig:  # helmadr/krylov.py:16-31 fields
        restart, maxiter, tol, flexible, collect_diagnostics = 5, 1000, 1e-6, True, False

    def solve_adr_upwind_body(mod):  # helmadr/drivers.py:148-165, names resolved through `mod`
        q = O.delta_source(p.n1, p.n2, p.h1, p.h2, p.src)
        qhat = O.to_adr(q, p.tau, p.omega).reshape(-1)
        H2up = O.adr_of(p, "upwind2")
        H1up = O.adr_of(p, "upwind1")
        blend = ((1.0 - 0.25) * H2up + 0.25 * H1up).tocsr()
        hier = mod.build_hierarchy(blend, GridSpec(), 5)
        return mod.fgmres(H2up, qhat, x0=None, precond=mod.make_kcycle_preconditioner(hier), cfg=KrylovConfig())

    D = types.SimpleNamespace()
    D.fgmres = hadr.fgmres                                            # helmadr/krylov.py:122
    D.build_hierarchy = hadr.build_hierarchy                          # helmadr/multigrid.py:113
    D.make_kcycle_preconditioner = hadr.make_kcycle_preconditioner    # helmadr/multigrid.py:174
    a, rep = solve_adr_upwind_body(D)
    floor, base = self_floor(O, lambda: O.solve_upwind(p, tol=1e-6, maxiter=1000)[1])
    assert np.array_equal(base.reshape(-1), g65["upwind_a"].reshape(-1))
    assert rep.converged and abs(rep.iterations - int(g65["upwind_iterations"])) <= 1
    assert rel(a, g65["upwind_a"]) <= protocol_bar(floor)
