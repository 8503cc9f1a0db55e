"""Generate golden fixtures by running the REFERENCE (helmadr) in this container.

    NUMBA_CACHE_DIR=/tmp/nbcache python tests/golden/make_golden.py

Reads /root/reference/pkg/src (read-only, imported in place); writes
tests/golden/*.npz.  Inputs are built with the reference's own types and
``tau_derivatives`` from the analytic tau1 of ``paper_1712_06091_b200.workloads``
(the synthetic-config recipe).  Nothing here runs on the GPU box.
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")  # BLAS thread count moves results

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import helmadr  # noqa: E402
from helmadr import drivers, eikonal, grid as hgrid, krylov, multigrid, operators  # noqa: E402

from paper_1712_06091_b200 import workloads  # noqa: E402

TOL = 1e-6
MAXIT = 1000


def ref_inputs(wl):
    """Reference-typed inputs for a workload: same kappa^2, gamma, tau1."""
    g = hgrid.GridSpec(wl.grid.n1, wl.grid.n2, wl.grid.L1, wl.grid.L2)
    med = hgrid.Medium(g, wl.medium.kappa_sq, wl.medium.gamma)
    src = hgrid.SourceSpec(wl.source.i1, wl.source.i2, wl.source.omega)
    base = eikonal.AnalyticBase(g, src)
    (g1, g2), lap = eikonal.tau_derivatives(wl.tt.tau1, base, g)
    tt = eikonal.TravelTime(g, wl.tt.tau1, base.tau0 * wl.tt.tau1, g1, g2, lap, base)
    bc = operators.BCSpec(*wl.bc)
    return g, med, src, tt, bc


def put_csr(out, key, A):
    A = A.tocsr()
    out[key + "_indptr"] = A.indptr.astype(np.int64)
    out[key + "_indices"] = A.indices.astype(np.int32)
    out[key + "_data"] = A.data.astype(np.complex128)


def put_report(out, key, rep):
    out[key + "_iterations"] = np.int64(rep.iterations)
    out[key + "_history"] = np.asarray(rep.history)
    out[key + "_converged"] = np.bool_(rep.converged)
    out[key + "_final_relres"] = np.float64(rep.final_relres)
    out[key + "_bnorm"] = np.float64(rep.bnorm)


def operator_case(wl, out, full_ops=True):
    g, med, src, tt, bc = ref_inputs(wl)
    out["tau"] = tt.tau
    out["grad1"] = tt.grad1
    out["grad2"] = tt.grad2
    out["lap"] = tt.lap
    out["kappa_sq"] = med.kappa_sq
    out["gamma"] = med.gamma
    out["meta"] = np.array([g.n1, g.n2, g.L1, g.L2, src.i1, src.i2, src.omega])
    om = src.omega
    H2 = operators.assemble_adr(med, g, om, tt, "upwind2", bc)
    H1 = operators.assemble_adr(med, g, om, tt, "upwind1", bc)
    blend = (0.75 * H2 + 0.25 * H1).tocsr()
    put_csr(out, "H2up", H2)
    put_csr(out, "blend", blend)
    if full_ops:
        Hc = operators.assemble_adr(med, g, om, tt, "central", bc)
        H = operators.assemble_helmholtz(med, g, om, bc)
        Hs = operators.shift_operator(H, 0.2, om, med)
        m = operators.phase_scaling(tt, om)
        Ar = operators.similarity_conjugate(Hc, m, "M_A_Minv")
        put_csr(out, "H1up", H1)
        put_csr(out, "Hcen", Hc)
        put_csr(out, "H", H)
        put_csr(out, "Hs", Hs)
        put_csr(out, "Aresc", Ar)
    hier = multigrid.build_hierarchy(blend, g, 5)
    out["n_levels"] = np.int64(hier.n_levels)
    out["shapes"] = np.array(hier.shapes, dtype=np.int64)
    for l, A in enumerate(hier.ops):
        put_csr(out, f"lev{l}", A)
    rng = np.random.default_rng(1712)
    n0 = g.n_nodes
    b = rng.standard_normal(n0) + 1j * rng.standard_normal(n0)
    x = rng.standard_normal(n0) + 1j * rng.standard_normal(n0)
    out["rnd_b"] = b
    out["rnd_x"] = x
    out["relax2"] = krylov._gmres_relax_pre(hier.ops[0], hier.inv_diags[0], b, x, 2)
    nc = hier.ops[-1].shape[0]
    bc_ = b[:nc]
    out["relax10_coarsest"] = krylov._gmres_relax_pre(hier.ops[-1], hier.inv_diags[-1], bc_, np.zeros(nc, complex), 10)
    stats = {}
    out["kcycle"] = multigrid.k_cycle(hier, 1, b, np.zeros(n0, complex), stats)
    out["kcycle_visits"] = np.array([stats.get(l, 0) for l in range(1, hier.n_levels + 1)])
    # restriction / prolongation of the first level on the random vectors
    P = hier.prols[0]
    out["restrict"] = P.T @ b
    out["prolong"] = P @ b[: P.shape[1]]
    out["spmv_blend"] = blend @ x
    return g, med, src, tt, bc


def solve_case(wl, out, strategies=("upwind", "standard", "central")):
    g, med, src, tt, bc = ref_inputs(wl)
    if "upwind" in strategies:
        cfg = drivers.StrategyConfig(strategy="adr_upwind_blend", tol=TOL, max_iter=MAXIT)
        u, a, rep = drivers.solve_adr_upwind(med, g, src, tt, cfg, bc)
        out["upwind_a"] = a
        put_report(out, "upwind", rep)
    if "standard" in strategies:
        cfg = drivers.StrategyConfig(strategy="standard_sl", tol=TOL, max_iter=MAXIT)
        H = operators.assemble_helmholtz(med, g, src.omega, bc)
        q = hgrid.point_source(g, src)
        u, rep = drivers.solve_standard(H, q, med, src.omega, cfg)
        out["standard_u"] = u
        put_report(out, "standard", rep)
    if "central" in strategies:
        cfg = drivers.StrategyConfig(strategy="adr_central_two_stage", tol=TOL, max_iter=MAXIT)
        u, a, rep = drivers.solve_adr_central(med, g, src, tt, cfg, bc)
        out["central_u"] = u
        put_report(out, "central", rep)
        out["central_stage1_iterations"] = np.int64(rep.stage1.iterations)


def main():
    cases = {
        "g33_const": (workloads.cfg1(33), True, ("upwind", "standard", "central")),
        "g65_linear": (workloads.cfg2(65), False, ("upwind", "standard", "central")),
    }
    for name, (wl, full, strat) in cases.items():
        out = {}
        operator_case(wl, out, full)
        solve_case(wl, out, strat)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
        print(name, {k: out[k] for k in out if k.endswith("_iterations")})
    # full BASELINE config 1 (129^2): solution fields + histories only
    out = {}
    solve_case(workloads.cfg1(129), out)
    np.savez_compressed(os.path.join(HERE, "cfg1_129.npz"), **out)
    print("cfg1_129", {k: out[k] for k in out if k.endswith("_iterations")})


if __name__ == "__main__":
    main()
