"""Pin the CPU oracle against golden vectors produced by the reference itself.

Everything here is bit-exact (np.array_equal): the oracle restates the
reference with the same numpy/scipy primitives in the same order, and the
fixtures were generated single-threaded on this image (tests/golden/make_golden.py).
"""

import numpy as np
import pytest

from conftest import csr_from, oracle_problem
from oracle import hadr_oracle as O
from paper_1712_06091_b200 import workloads

CASES = {"g33": (lambda: workloads.cfg1(33)), "g65": (lambda: workloads.cfg2(65))}


def _same_csr(A, g, key):
    B = csr_from(g, key)
    A = A.tocsr()
    assert np.array_equal(A.indptr, B.indptr), key
    assert np.array_equal(A.indices, B.indices), key
    assert np.array_equal(A.data, B.data), key


@pytest.mark.parametrize("case", ["g33", "g65"])
def test_travel_time_fields_bitexact(case, request):
    g = request.getfixturevalue(case)
    wl = CASES[case]()
    p = oracle_problem(wl)
    gr1, gr2, lap, tau = O.tau_fields(wl.tt.tau1, wl.grid.L1, wl.grid.L2, p.src)
    for k, v in (("grad1", gr1), ("grad2", gr2), ("lap", lap), ("tau", tau)):
        assert np.array_equal(v, g[k]), k
        # the package's setup path computes the identical fields
        assert np.array_equal(getattr(wl.tt, k), g[k]), k
    assert np.array_equal(wl.medium.kappa_sq, g["kappa_sq"])
    assert np.array_equal(wl.medium.gamma, g["gamma"])


def test_assembly_bitexact(g33):
    p = oracle_problem(workloads.cfg1(33))
    H2 = O.adr_of(p, "upwind2")
    H1 = O.adr_of(p, "upwind1")
    _same_csr(H2, g33, "H2up")
    _same_csr(H1, g33, "H1up")
    _same_csr((0.75 * H2 + 0.25 * H1).tocsr(), g33, "blend")
    Hc = O.adr_of(p, "central")
    _same_csr(Hc, g33, "Hcen")
    H = O.helm_of(p)
    _same_csr(H, g33, "H")
    _same_csr(O.shifted(H, 0.2, p.omega, p.kappa_sq), g33, "Hs")
    _same_csr(O.conjugate_by(Hc, O.phase(p.tau, p.omega)), g33, "Aresc")


def test_assembly_linear_bitexact(g65):
    p = oracle_problem(workloads.cfg2(65))
    _same_csr(O.adr_of(p, "upwind2"), g65, "H2up")


@pytest.mark.parametrize("case", ["g33", "g65"])
def test_hierarchy_and_kcycle_bitexact(case, request):
    g = request.getfixturevalue(case)
    B = csr_from(g, "blend")
    n1, n2 = int(g["meta"][0]), int(g["meta"][1])
    H = O.hierarchy(B, (n1, n2), 5)
    assert H.n_levels == int(g["n_levels"])
    assert [list(s) for s in H.shapes] == g["shapes"].tolist()
    for l, A in enumerate(H.ops):
        _same_csr(A, g, f"lev{l}")
    b, x = g["rnd_b"], g["rnd_x"]
    assert np.array_equal(O.relax(H.ops[0], H.inv_diags[0], b, x, 2), g["relax2"])
    nc = H.ops[-1].shape[0]
    assert np.array_equal(
        O.relax(H.ops[-1], H.inv_diags[-1], b[:nc], np.zeros(nc, complex), 10), g["relax10_coarsest"])
    visits = {}
    assert np.array_equal(O.kcycle(H, 1, b, np.zeros_like(b), visits), g["kcycle"])
    assert [visits.get(l, 0) for l in range(1, H.n_levels + 1)] == g["kcycle_visits"].tolist()
    P = H.prols[0]
    assert np.array_equal(P.T @ b, g["restrict"])
    assert np.array_equal(P @ b[: P.shape[1]], g["prolong"])


@pytest.mark.parametrize("case", ["g33", "g65", "gcfg1"])
def test_strategies_bitexact(case, request):
    g = request.getfixturevalue(case)
    wl = {"g33": lambda: workloads.cfg1(33), "g65": lambda: workloads.cfg2(65),
          "gcfg1": lambda: workloads.cfg1(129)}[case]()
    p = oracle_problem(wl)
    u, a, rep = O.solve_upwind(p, tol=1e-6, maxiter=1000)
    assert rep.iterations == int(g["upwind_iterations"])
    assert np.array_equal(rep.history, g["upwind_history"])
    assert np.array_equal(a, g["upwind_a"])
    H = O.helm_of(p)
    q = O.delta_source(p.n1, p.n2, p.h1, p.h2, p.src)
    u, rep = O.solve_sl(H, q, p, tol=1e-6, maxiter=1000)
    assert rep.iterations == int(g["standard_iterations"])
    assert np.array_equal(u, g["standard_u"])
    u, a, rep = O.solve_central(p, tol=1e-6, maxiter=1000)
    assert rep.iterations == int(g["central_iterations"])
    assert rep.stage1.iterations == int(g["central_stage1_iterations"])
    assert np.array_equal(u, g["central_u"])


def test_cfg3_recipe_bitexact(gcfg3):
    """Config-3 recipe at 129 x 65 (layered medium, surface source, Neumann top, travel
    time from the fast-marching restatement == the reference's, checked when the fixture
    was made): fields, fine operators, hierarchy and the upwind solve are bit-exact."""
    g = gcfg3
    wl = workloads.cfg3(65)
    assert np.array_equal(wl.tt.tau1, g["tau1"])
    p = oracle_problem(wl)  # the oracle's tau_derivatives of the fast-marching tau1
    for k, v in (("grad1", p.grad1), ("grad2", p.grad2), ("lap", p.lap), ("tau", p.tau)):
        assert np.array_equal(v, g[k]), k
    assert np.array_equal(wl.medium.kappa_sq, g["kappa_sq"]) and np.array_equal(wl.medium.gamma, g["gamma"])
    H2, H1 = O.adr_of(p, "upwind2"), O.adr_of(p, "upwind1")
    _same_csr(H2, g, "H2up")
    B = (0.75 * H2 + 0.25 * H1).tocsr()
    _same_csr(B, g, "blend")
    Hi = O.hierarchy(B, (p.n1, p.n2), 5)
    for l, A in enumerate(Hi.ops):
        _same_csr(A, g, f"lev{l}")
    u, a, rep = O.solve_upwind(p, tol=1e-6, maxiter=1000)
    assert rep.iterations == int(g["upwind_iterations"])
    assert np.array_equal(a, g["upwind_a"])


def test_cfg1_iteration_counts_match_survey(gcfg1):
    # SURVEY.md §6 measured-here table: upwind 18, central 19, standard 20
    assert int(gcfg1["upwind_iterations"]) == 18
    assert int(gcfg1["central_iterations"]) == 19
    assert int(gcfg1["standard_iterations"]) == 20


@pytest.mark.parametrize("case", ["g33", "g65"])
def test_nd_oracle_2d_is_bitexact(case, request):
    """The dimension-generic oracle (used for 3D) reproduces the reference in 2D bit for bit."""
    from oracle import hadr_oracle_nd as ND

    g = request.getfixturevalue(case)
    wl = CASES[case]()
    shape, Ls = wl.grid.shape, (wl.grid.L1, wl.grid.L2)
    src = (wl.source.i1, wl.source.i2)
    grads, lap, tau = ND.tau_fields(wl.tt.tau1, Ls, src)
    assert np.array_equal(grads[0], g["grad1"]) and np.array_equal(grads[1], g["grad2"])
    assert np.array_equal(lap, g["lap"]) and np.array_equal(tau, g["tau"])
    hs = (wl.grid.h1, wl.grid.h2)
    bc = ND.bc_dict(2, wl.bc)
    H2 = ND.adr_csr(shape, hs, wl.omega, wl.medium.kappa_sq, wl.medium.gamma, grads, lap, src, "upwind2", bc)
    _same_csr(H2, g, "H2up")
    B = csr_from(g, "blend")
    Hi = ND.hierarchy(B, shape, 5)
    for l, A in enumerate(Hi.ops):
        _same_csr(A, g, f"lev{l}")
    if case == "g33":
        _same_csr(ND.helmholtz_csr(shape, hs, wl.omega, wl.medium.kappa_sq, wl.medium.gamma, bc), g, "H")
        for scheme, key in (("upwind1", "H1up"), ("central", "Hcen")):
            A = ND.adr_csr(shape, hs, wl.omega, wl.medium.kappa_sq, wl.medium.gamma, grads, lap, src, scheme, bc)
            _same_csr(A, g, key)


def test_nd_oracle_3d_structure():
    """3D instantiation: stencil reach, Galerkin identity, P partition of unity, a converging solve."""
    from oracle import hadr_oracle as O
    from oracle import hadr_oracle_nd as ND
    from paper_1712_06091_b200 import workloads

    wl = workloads.cfg4(17)
    shape = wl.grid.shape
    hs = wl.grid.hs
    src = wl.source.index
    bc = ND.bc_dict(3, wl.bc)
    grads, lap, tau = ND.tau_fields(wl.tt.tau1, wl.grid.Ls, src)
    for a, b_ in zip(grads, wl.tt.grads):
        assert np.array_equal(a, b_)
    H2 = ND.adr_csr(shape, hs, wl.omega, wl.medium.kappa_sq, wl.medium.gamma, grads, lap, src, "upwind2", bc)
    assert np.diff(H2.indptr).max() <= 13
    P = ND.prolongation(shape)
    assert np.allclose(P @ np.ones(P.shape[1]), 1.0)
    B = (0.75 * H2 + 0.25 * ND.adr_csr(shape, hs, wl.omega, wl.medium.kappa_sq, wl.medium.gamma, grads, lap,
                                         src, "upwind1", bc)).tocsr()
    Hi = ND.hierarchy(B, shape, 5)
    Ac = (P.T @ B @ P).toarray()
    assert np.abs(Hi.ops[1].toarray() - Ac).max() <= 1e-12 * np.abs(Ac).max()
    assert max(np.diff(A.indptr).max() for A in Hi.ops[1:]) <= 81
    a, rep = ND.solve_upwind(shape, hs, wl.omega, src, wl.medium.kappa_sq, wl.medium.gamma, grads, lap, tau, bc)
    assert rep.converged and rep.iterations < 60
