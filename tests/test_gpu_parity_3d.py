"""3D GPU parity (BASELINE configs 4/5 have no reference: the oracle is the
dimension-generic restatement oracle/hadr_oracle_nd.py, whose 2D instantiation
is pinned bit-exact to the reference).  Tolerances as in test_gpu_parity.py."""

import numpy as np
import pytest
from parity_util import protocol_bar, self_floor

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


@pytest.fixture(scope="module")
def hadr():
    import paper_1712_06091_b200 as H

    H._lib.lib()
    return H


@pytest.fixture(scope="module", params=[17, 33])
def case3d(request):
    from oracle import hadr_oracle_nd as ND
    from paper_1712_06091_b200 import workloads

    wl = workloads.cfg4(request.param)
    g = wl.grid
    shape, hs, src = g.shape, g.hs, wl.source.index
    bc = ND.bc_dict(3, wl.bc)
    grads, lap, tau = ND.tau_fields(wl.tt.tau1, g.Ls, src)
    args = (shape, hs, wl.omega, wl.medium.kappa_sq, wl.medium.gamma, grads, lap, src)
    H2 = ND.adr_csr(*args, "upwind2", bc)
    H1 = ND.adr_csr(*args, "upwind1", bc)
    B = (0.75 * H2 + 0.25 * H1).tocsr()
    return dict(wl=wl, shape=shape, hs=hs, src=src, bc=bc, grads=grads, lap=lap, tau=tau, H2=H2, H1=H1, B=B,
                Hi=ND.hierarchy(B, shape, 5))


def test_spmv_and_transfer_bitexact_3d(hadr, case3d):
    from oracle import hadr_oracle_nd as ND

    shape, H2 = case3d["shape"], case3d["H2"]
    op = hadr.StencilOperator.from_csr(H2, shape)
    assert len(op.offsets) <= 13
    rng = np.random.default_rng(5)
    x = rng.standard_normal(H2.shape[0]) + 1j * rng.standard_normal(H2.shape[0])
    assert np.array_equal(op @ x, H2 @ x)
    P = ND.prolongation(shape)
    Pd = hadr.build_prolongation(shape)
    assert np.array_equal(Pd.T @ x, P.T @ x)
    e = x[: P.shape[1]]
    assert np.array_equal(Pd @ e, P @ e)
    # coarse 81-offset operator: chunked stencil path
    A1 = case3d["Hi"].ops[1]
    op1 = hadr.StencilOperator.from_csr(A1, case3d["Hi"].shapes[1])
    x1 = x[: A1.shape[0]]
    assert np.array_equal(op1 @ x1, A1 @ x1)


def test_pair_compressed_stencil_bitexact_3d(hadr, case3d):
    """3D fine upwind operators pair-compressed (13 -> 10 planes) reproduce csr_matvec."""
    rng = np.random.default_rng(9)
    for key in ("H2", "B"):
        A = case3d[key]
        x = rng.standard_normal(A.shape[0]) + 1j * rng.standard_normal(A.shape[0])
        op = hadr.StencilOperator.from_csr(A, case3d["shape"])
        y = op @ x
        assert op.storage_slots == 10, key
        assert np.array_equal(y, A @ x), key


@pytest.mark.parametrize("tile", [0, 2])
def test_stencil_kernels_bitexact_3d(hadr, case3d, tile):
    """Flat and shared-memory-tiled stencil kernels (option stencil_tile 0 / 2 = always)
    both reproduce csr_matvec bit for bit, fine 13-offset and coarse 81-offset."""
    from oracle import hadr_oracle as O

    hadr._lib.set_option("stencil_tile", tile)
    hadr._lib.set_option("ce_max_n", 0)
    try:
        rng = np.random.default_rng(7)
        for l in (0, 1):
            A = case3d["Hi"].ops[l] if l else case3d["H2"]
            op = hadr.StencilOperator.from_csr(A, case3d["Hi"].shapes[l])
            x = rng.standard_normal(A.shape[0]) + 1j * rng.standard_normal(A.shape[0])
            assert np.array_equal(op @ x, A @ x), l
        Hi = case3d["Hi"]
        H = hadr.hierarchy_from_ops(Hi.ops, shapes=Hi.shapes)
        b = rng.standard_normal(Hi.ops[0].shape[0]) + 1j * rng.standard_normal(Hi.ops[0].shape[0])
        assert rel(hadr.make_kcycle_preconditioner(H)(b), O.kcycle(Hi, 1, b, np.zeros_like(b))) <= 1e-12
    finally:
        hadr._lib.set_option("stencil_tile", 1)
        hadr._lib.set_option("ce_max_n", 32768)


def test_device_assembly_3d(hadr, case3d):
    from paper_1712_06091_b200 import operators

    wl = case3d["wl"]
    for scheme, ref in (("upwind2", case3d["H2"]), ("upwind1", case3d["H1"])):
        got = operators.assemble_adr(wl.medium, wl.grid, wl.omega, wl.tt, scheme, wl.bc).tocsr()
        assert np.array_equal(got.indptr, ref.indptr) and np.array_equal(got.indices, ref.indices)
        assert np.abs(got.data - ref.data).max() <= 4e-16 * np.abs(ref.data).max()


def test_galerkin_3d(hadr, case3d):
    Hi = case3d["Hi"]
    H = hadr.build_hierarchy(case3d["B"], case3d["shape"], 5)
    assert [tuple(s) for s in H.shapes] == [tuple(s) for s in Hi.shapes]
    for l in range(1, H.n_levels):
        ref = Hi.ops[l]
        err = abs(H.ops[l].tocsr() - ref).max()
        assert err <= 1e-12 * abs(ref).max(), (l, err)


@pytest.mark.parametrize("engine", ["cluster", "cluster_gmem", "graph"])
def test_kcycle_3d(hadr, case3d, engine):
    from oracle import hadr_oracle as O

    hadr._lib.set_option("ce_max_n", 0 if engine == "graph" else 32768)
    hadr._lib.set_option("ce_smem_relax", 0 if engine == "cluster_gmem" else 1)
    try:
        Hi = case3d["Hi"]
        H = hadr.hierarchy_from_ops(Hi.ops, shapes=Hi.shapes)
        n = Hi.ops[0].shape[0]
        rng = np.random.default_rng(9)
        b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        ref = O.kcycle(Hi, 1, b, np.zeros_like(b))
        assert rel(hadr.k_cycle(H, 1, b, np.zeros_like(b)), ref) <= 1e-12
        assert rel(hadr.make_kcycle_preconditioner(H)(b), ref) <= 1e-12
    finally:
        hadr._lib.set_option("ce_max_n", 32768)
        hadr._lib.set_option("ce_smem_relax", 1)


def _nd_upwind(c, tol):
    from oracle import hadr_oracle_nd as ND

    wl = c["wl"]
    return ND.solve_upwind(c["shape"], c["hs"], wl.omega, c["src"], wl.medium.kappa_sq, wl.medium.gamma, c["grads"],
                           c["lap"], c["tau"], c["bc"], tol=tol)


def _nd_sl(c, tol):
    from oracle import hadr_oracle_nd as ND

    wl = c["wl"]
    return ND.solve_sl(c["shape"], c["hs"], wl.omega, c["src"], wl.medium.kappa_sq, wl.medium.gamma, c["bc"],
                       alpha=0.5, tol=tol)


def test_solve_upwind_3d(hadr, case3d):
    """Public driver (3D device assembly, hierarchy, FGMRES) vs the ND oracle at the parity
    protocol's bar: iterations +-1, amplitude <= max(1e-8, 3x the oracle self-floor)."""
    from oracle import hadr_oracle_nd as ND
    from paper_1712_06091_b200 import drivers

    wl = case3d["wl"]
    a_ref, rep_ref = _nd_upwind(case3d, 1e-6)
    floor, _ = self_floor(ND, lambda: _nd_upwind(case3d, 1e-6)[0])
    cfg = drivers.StrategyConfig(strategy="adr_upwind_blend", tol=1e-6, max_iter=1000)
    u, a, rep = drivers.solve_adr_upwind(wl.medium, wl.grid, wl.source, wl.tt, cfg, wl.bc)
    assert rep.converged and abs(rep.iterations - rep_ref.iterations) <= 1
    assert rel(a, a_ref) <= protocol_bar(floor), (rel(a, a_ref), floor)


@pytest.mark.parametrize("solver", ["upwind", "standard_sl"])
def test_solve_3d_tight_tol_strict(hadr, solver):
    """Protocol step 3 in 3D (33^3-class grid, config-4 recipe; standard_sl with alpha 0.5
    on the config-5 recipe): at tol 1e-10 the public drivers and the ND oracle agree to
    <= 1e-8 strictly."""
    from oracle import hadr_oracle_nd as ND
    from paper_1712_06091_b200 import drivers, operators, workloads
    from paper_1712_06091_b200.fields import point_source

    wl = workloads.cfg4(33) if solver == "upwind" else workloads.cfg5(33)
    g = wl.grid
    grads, lap, tau = ND.tau_fields(wl.tt.tau1, g.Ls, wl.source.index)
    c = dict(wl=wl, shape=g.shape, hs=g.hs, src=wl.source.index, bc=ND.bc_dict(3, wl.bc), grads=grads, lap=lap,
             tau=tau)
    if solver == "upwind":
        ref, _ = _nd_upwind(c, 1e-10)
        cfg = drivers.StrategyConfig(strategy="adr_upwind_blend", tol=1e-10, max_iter=1000)
        _, x, rep = drivers.solve_adr_upwind(wl.medium, wl.grid, wl.source, wl.tt, cfg, wl.bc)
    else:
        ref, _ = _nd_sl(c, 1e-10)
        H = operators.assemble_helmholtz(wl.medium, wl.grid, wl.omega, wl.bc)
        cfg = drivers.StrategyConfig(strategy="standard_sl", alpha=0.5, tol=1e-10, max_iter=1000)
        x, rep = drivers.solve_standard(H, point_source(wl.grid, wl.source), wl.medium, wl.omega, cfg)
    assert rep.converged
    assert rel(x, ref) <= 1e-8


@pytest.fixture(scope="module")
def cfg5_small():
    """BASELINE config 5 recipe at 33 x 33 x 17: Gaussian random medium, tau from the 3D
    fast marcher (setup), all-Sommerfeld, 2-cell layer."""
    from oracle import hadr_oracle_nd as ND
    from paper_1712_06091_b200 import workloads

    wl = workloads.cfg5(33)
    g = wl.grid
    grads, lap, tau = ND.tau_fields(wl.tt.tau1, g.Ls, wl.source.index)
    return dict(wl=wl, shape=g.shape, hs=g.hs, src=wl.source.index, bc=ND.bc_dict(3, wl.bc), grads=grads, lap=lap,
                tau=tau)


def test_device_assembly_helmholtz_3d(hadr, cfg5_small):
    """3D standard Helmholtz (7-point) and its shift on the device equal the ND oracle."""
    from oracle import hadr_oracle as O
    from oracle import hadr_oracle_nd as ND
    from paper_1712_06091_b200 import operators

    c = cfg5_small
    wl = c["wl"]
    ref = ND.helmholtz_csr(c["shape"], c["hs"], wl.omega, wl.medium.kappa_sq, wl.medium.gamma, c["bc"])
    H = operators.assemble_helmholtz(wl.medium, wl.grid, wl.omega, wl.bc)
    got = H.tocsr()
    assert np.array_equal(got.indptr, ref.indptr) and np.array_equal(got.indices, ref.indices)
    assert np.abs(got.data - ref.data).max() <= 4e-16 * np.abs(ref.data).max()
    Hs = operators.shift_operator(H, 0.5, wl.omega, wl.medium).tocsr()
    Hs_ref = O.shifted(ref, 0.5, wl.omega, wl.medium.kappa_sq)
    assert np.abs(Hs - Hs_ref).max() <= 4e-16 * np.abs(Hs_ref).max()


def test_cfg5_recipe_solves(hadr, cfg5_small):
    """Config 5's two solvers on its recipe (fast-marching tau, random medium):
    adr_upwind and standard_sl with alpha = 0.5 vs the ND oracle — iterations within 1,
    amplitude within the protocol bar (upwind; as test_solve_upwind_3d), wavefield within
    1e-8 (SL)."""
    from oracle import hadr_oracle_nd as ND
    from paper_1712_06091_b200 import drivers, operators
    from paper_1712_06091_b200.fields import point_source

    c = cfg5_small
    wl = c["wl"]
    a_ref, rep_ref = _nd_upwind(c, 1e-6)
    floor, _ = self_floor(ND, lambda: _nd_upwind(c, 1e-6)[0])
    cfg = drivers.StrategyConfig(strategy="adr_upwind_blend", tol=1e-6, max_iter=1000)
    u, a, rep = drivers.solve_adr_upwind(wl.medium, wl.grid, wl.source, wl.tt, cfg, wl.bc)
    assert rep.converged and abs(rep.iterations - rep_ref.iterations) <= 1
    assert rel(a, a_ref) <= protocol_bar(floor), (rel(a, a_ref), floor)
    u_ref, rs_ref = _nd_sl(c, 1e-6)
    H = operators.assemble_helmholtz(wl.medium, wl.grid, wl.omega, wl.bc)
    q = point_source(wl.grid, wl.source)
    cfg_sl = drivers.StrategyConfig(strategy="standard_sl", alpha=0.5, tol=1e-6, max_iter=1000)
    u_sl, rs = drivers.solve_standard(H, q, wl.medium, wl.omega, cfg_sl)
    assert rs.converged and abs(rs.iterations - rs_ref.iterations) <= 1
    assert rel(u_sl, u_ref) <= 1e-8


def test_class_compressed_coarse_bitexact_3d(hadr, case3d):
    """Coarse 81-offset Galerkin operators stored class-compressed (each row reads the
    slots of its upwind sign class: 54 planes in the interior, more where the upwind
    side changes) reproduce csr_matvec bit for bit, and equal the union-plane kernel."""
    A1 = case3d["Hi"].ops[1]
    shape1 = case3d["Hi"].shapes[1]
    rng = np.random.default_rng(13)
    x = rng.standard_normal(A1.shape[0]) + 1j * rng.standard_normal(A1.shape[0])
    ys = {}
    try:
        for cc in (0, 1):
            hadr._lib.set_option("class_compress", cc)
            op = hadr.StencilOperator.from_csr(A1, shape1)
            ys[cc] = op @ x
            assert (54 <= op.storage_slots <= 81) if cc else op.storage_slots == 0
    finally:
        hadr._lib.set_option("class_compress", 2)
    assert np.array_equal(ys[1], A1 @ x)
    assert np.array_equal(ys[0], ys[1])


@pytest.mark.parametrize("c64", [0, 1])
def test_compressed_solve_identical_3d(hadr, c64):
    """A 3D solve whose coarse levels take the graph path (cl_max_n lowered) with the
    pair-compressed fine and class-compressed coarse operators is bit-identical to the
    union-plane solve (complex128 and mixed precision)."""
    from paper_1712_06091_b200 import drivers, workloads

    wl = workloads.cfg4(33)
    cfg = drivers.StrategyConfig(strategy="adr_upwind_blend", tol=1e-6, max_iter=1000)
    out = {}
    hadr._lib.set_option("cl_max_n", 1000)
    hadr._lib.set_option("ce_max_n", 1000)
    hadr._lib.set_option("kcycle_c64", c64)
    try:
        for cmp in (0, 1):
            hadr._lib.set_option("class_compress", cmp)
            hadr._lib.set_option("pair_compress", cmp)
            u, a, rep = drivers.solve_adr_upwind(wl.medium, wl.grid, wl.source, wl.tt, cfg, wl.bc)
            out[cmp] = (a, rep.iterations, list(rep.history))
    finally:
        for k, v in (("class_compress", 2), ("pair_compress", 1), ("cl_max_n", 32768), ("ce_max_n", 32768),
                     ("kcycle_c64", 0)):
            hadr._lib.set_option(k, v)
    assert out[0][1] == out[1][1]
    assert np.array_equal(out[0][0], out[1][0])
    assert out[0][2] == out[1][2]


def test_solve_upwind_3d_c64_mixed(hadr, case3d):
    """BASELINE config 4's complex64 variant (mixed precision: complex64 K-cycle operators,
    complex128 vectors and outer FGMRES) vs the complex128 ND oracle: iterations within 1,
    amplitude within 1e-4 (north_star's complex64 bar)."""
    from oracle import hadr_oracle_nd as ND
    from paper_1712_06091_b200 import drivers

    wl = case3d["wl"]
    a_ref, rep_ref = ND.solve_upwind(case3d["shape"], case3d["hs"], wl.omega, case3d["src"], wl.medium.kappa_sq,
                                     wl.medium.gamma, case3d["grads"], case3d["lap"], case3d["tau"], case3d["bc"])
    cfg = drivers.StrategyConfig(strategy="adr_upwind_blend", tol=1e-6, max_iter=1000)
    hadr._lib.set_option("kcycle_c64", 1)
    try:
        u, a, rep = drivers.solve_adr_upwind(wl.medium, wl.grid, wl.source, wl.tt, cfg, wl.bc)
    finally:
        hadr._lib.set_option("kcycle_c64", 0)
    assert rep.converged and abs(rep.iterations - rep_ref.iterations) <= 1
    assert rel(a, a_ref) <= 1e-4


def test_relax_split_solve_identical_3d(hadr):
    """Large 3D levels form the relaxation input D^-1 (s w) once per point (a scale kernel,
    then a plain stencil) instead of per neighbour inside the stencil: bit-identical solve
    (forced on a small grid with relax_split lowered and the coarse levels on the graph path)."""
    from paper_1712_06091_b200 import drivers, workloads

    wl = workloads.cfg4(33)
    cfg = drivers.StrategyConfig(strategy="adr_upwind_blend", tol=1e-6, max_iter=1000)
    out = {}
    hadr._lib.set_option("cl_max_n", 1000)
    hadr._lib.set_option("ce_max_n", 1000)
    try:
        for split in (0, 1000):
            hadr._lib.set_option("relax_split", split)
            u, a, rep = drivers.solve_adr_upwind(wl.medium, wl.grid, wl.source, wl.tt, cfg, wl.bc)
            out[split] = (a, rep.iterations, list(rep.history))
    finally:
        for k, v in (("relax_split", 8192), ("cl_max_n", 32768), ("ce_max_n", 32768)):
            hadr._lib.set_option(k, v)
    assert out[0][1] == out[1000][1]
    assert np.array_equal(out[0][0], out[1000][0])
    assert out[0][2] == out[1000][2]


@pytest.mark.parametrize("shape", [(9, 7, 6), (19, 47, 75), (33, 16, 35), (40, 31, 129)])
def test_march_stencil_bitexact_3d(hadr, shape):
    """The plane-marching bulk-copy kernel (option stencil_march = 2: always) on the
    pair-compressed 3D fine operator reproduces csr_matvec bit for bit, as the flat kernel
    does, on grids with ragged tiles, several column tiles and several plane chunks."""
    rng = np.random.default_rng(41)
    from parity_util import plus2_operator

    offs, coef, A = plus2_operator(shape, rng)
    N = A.shape[0]
    x = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    ref = A @ x
    out = {}
    try:
        for mode in (0, 2):
            hadr._lib.set_option("stencil_march", mode)
            hadr._lib.set_option("cl_max_n", 0)
            op = hadr.StencilOperator.from_planes(shape, offs, coef)
            out[mode] = op @ x
            assert op.storage_slots == 10
    finally:
        hadr._lib.set_option("stencil_march", 1)
        hadr._lib.set_option("cl_max_n", 32768)
    assert np.array_equal(out[0], ref)
    assert np.array_equal(out[2], ref)


@pytest.mark.parametrize("c64", [0, 1])
def test_march_solve_3d(hadr, c64):
    """A 3D solve with every fine-level sweep on the marching kernel (residuals and the
    dot / norm reductions included) equals the flat-kernel solve: same iterations, amplitude
    within 1e-8 (the reductions sum per-block partials of a different grid; the solve amplifies rounding to ~1e-9)."""
    from paper_1712_06091_b200 import drivers, workloads

    wl = workloads.cfg4(33)
    cfg = drivers.StrategyConfig(strategy="adr_upwind_blend", tol=1e-6, max_iter=1000)
    out = {}
    hadr._lib.set_option("kcycle_c64", c64)
    hadr._lib.set_option("relax_split", 1000)
    hadr._lib.set_option("cl_max_n", 1000)
    try:
        for mode in (0, 2):
            hadr._lib.set_option("stencil_march", mode)
            u, a, rep = drivers.solve_adr_upwind(wl.medium, wl.grid, wl.source, wl.tt, cfg, wl.bc)
            out[mode] = (a, rep.iterations)
    finally:
        for k, v in (("stencil_march", 1), ("kcycle_c64", 0), ("cl_max_n", 32768), ("relax_split", 8192)):
            hadr._lib.set_option(k, v)
    assert out[0][1] == out[2][1]
    assert rel(out[2][0], out[0][0]) <= 1e-8


@pytest.mark.parametrize("shape", [(9, 7, 6), (21, 40, 71), (40, 31, 129)])
def test_march_stencil_7point_bitexact_3d(hadr, shape):
    """The marching kernel's 7-point instantiation (3D plus of radius 1 from its union planes:
    the standard Helmholtz / shifted-Laplacian fine operators of standard_sl) reproduces
    csr_matvec bit for bit, as the flat kernel does."""
    from parity_util import plus1_operator

    rng = np.random.default_rng(47)
    offs, coef, A = plus1_operator(shape, rng)
    N = A.shape[0]
    x = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    ref = A @ x
    out = {}
    try:
        for mode in (0, 2):
            hadr._lib.set_option("stencil_march", mode)
            hadr._lib.set_option("cl_max_n", 0)
            op = hadr.StencilOperator.from_planes(shape, offs, coef)
            out[mode] = op @ x
    finally:
        hadr._lib.set_option("stencil_march", 1)
        hadr._lib.set_option("cl_max_n", 32768)
    assert np.array_equal(out[0], ref)
    assert np.array_equal(out[2], ref)


@pytest.mark.parametrize("c64", [0, 1])
def test_march_solve_sl_3d(hadr, c64):
    """standard_sl in 3D (config-5 recipe at 33 x 33 x 17) with every fine-level sweep of the
    Helmholtz operator and of the shifted operator's K-cycle on the marching kernel equals the
    flat-kernel solve: same iterations, wavefield within 1e-8."""
    from paper_1712_06091_b200 import drivers, operators, workloads
    from paper_1712_06091_b200.fields import point_source

    wl = workloads.cfg5(33)
    q = point_source(wl.grid, wl.source)
    cfg = drivers.StrategyConfig(strategy="standard_sl", alpha=0.5, tol=1e-6, max_iter=1000)
    out = {}
    hadr._lib.set_option("kcycle_c64", c64)
    hadr._lib.set_option("relax_split", 1000)
    hadr._lib.set_option("cl_max_n", 1000)
    try:
        for mode in (0, 2):
            hadr._lib.set_option("stencil_march", mode)
            H = operators.assemble_helmholtz(wl.medium, wl.grid, wl.omega, wl.bc)
            u, rep = drivers.solve_standard(H, q, wl.medium, wl.omega, cfg)
            out[mode] = (u, rep.iterations)
    finally:
        for k, v in (("stencil_march", 1), ("kcycle_c64", 0), ("cl_max_n", 32768), ("relax_split", 8192)):
            hadr._lib.set_option(k, v)
    assert out[0][1] == out[2][1]
    assert rel(out[2][0], out[0][0]) <= 1e-8
