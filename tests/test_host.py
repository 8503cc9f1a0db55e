"""CPU-only tests: the C-ABI library loads and exports every declared symbol,
and the host-side logic mirrors the reference (no GPU calls here)."""

import os
import re

import numpy as np
import pytest

from conftest import REPO


def _header_functions():
    src = open(os.path.join(REPO, "include", "hadr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hadr_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_1712_06091_b200 import _lib

    L = _lib.load()  # dlopen only; no device needed
    declared = _header_functions()
    assert declared, "no functions parsed from include/hadr.h"
    for name in declared:
        assert hasattr(L, name), f"libhadr.so does not export {name}"
    assert sorted(_lib.EXPORTS) == declared  # the Python binding covers the whole ABI


def test_library_is_sm100a():
    import subprocess

    so = os.path.join(REPO, "paper_1712_06091_b200", "libhadr.so")
    out = subprocess.run(["cuobjdump", "-lelf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_coarsenable_levels_matches_oracle():
    from oracle import hadr_oracle as O
    from paper_1712_06091_b200 import coarsenable_levels

    for shape in [(1025, 1025), (4097, 2049), (257, 129), (9, 9), (33, 17), (10, 9), (769, 257)]:
        assert coarsenable_levels(shape, 5) == O.level_shapes(shape, 5)
    # SPEC.md:461-462 examples
    assert coarsenable_levels((257, 257), 5) == [(257, 257), (129, 129), (65, 65), (33, 33), (17, 17)]
    assert coarsenable_levels((9, 9), 5) == [(9, 9), (5, 5), (3, 3)]


def test_configs_and_validation():
    from paper_1712_06091_b200 import KrylovConfig, drivers, operators, workloads

    with pytest.raises(ValueError):
        KrylovConfig(restart=0)
    with pytest.raises(ValueError):
        KrylovConfig(tol=0)
    with pytest.raises(ValueError):
        drivers.StrategyConfig(strategy="nope")
    with pytest.raises(ValueError):
        drivers.StrategyConfig(alpha=2.0)
    with pytest.raises(ValueError):
        operators.BCSpec(top="dirichlet")
    assert drivers.StrategyConfig().krylov().restart == 5
    wl = workloads.cfg2(1025)
    assert (wl.source.i1, wl.source.i2) == (512, 51)
    assert abs(wl.omega - 2 * np.pi * 1.5 * 1024 / 12) < 1e-9
    wl1 = workloads.cfg1(129)
    assert (wl1.source.i1, wl1.source.i2) == (64, 64)
    assert abs(wl1.omega - 2 * np.pi * 128 / 10) < 1e-9
    # gamma ramps 0 -> omega over the layer, max at the corners
    g = wl1.medium.gamma
    assert g[64, 64] == 0 and abs(g[0, 64] - wl1.omega) < 1e-9 and abs(g.max() - wl1.omega) < 1e-9


def test_linear_gradient_tau_is_an_eikonal_solution():
    """|grad tau|^2 ~= kappa^2 for the analytic linear-gradient travel time (FD check)."""
    from paper_1712_06091_b200 import workloads

    wl = workloads.cfg2(257)
    tt, ksq = wl.tt, wl.medium.kappa_sq
    res = np.abs(tt.grad_sq - ksq) / ksq
    s = (wl.source.i1, wl.source.i2)
    mask = np.ones_like(res, bool)
    mask[s[0] - 3:s[0] + 4, s[1] - 3:s[1] + 4] = False
    assert np.median(res[mask]) < 1e-3


def test_bench_cpu_baseline_helpers_import():
    import bench

    assert bench.B_OP_2D_UPWIND_C128 == 7726.0
    hbm, src = bench.peaks()
    assert hbm > 1000


def test_grid_inference_for_scipy_operators():
    """spmv / jacobi_apply / gmres_relax accept plain scipy matrices (helmadr/krylov.py:60-88):
    the grid is the operator's own, an explicit one, or the square / cubic grid its size implies."""
    import scipy.sparse as sp

    from paper_1712_06091_b200.krylov import grid_of

    assert grid_of(sp.identity(33 * 33, format="csr")) == (33, 33)
    assert grid_of(sp.identity(9 * 9 * 9, format="csr")) == (27, 27)  # m^2 wins over m^3 (729 = 27^2)
    assert grid_of(sp.identity(5 * 5 * 5, format="csr")) == (5, 5, 5)
    assert grid_of(sp.identity(65 * 33, format="csr"), (65, 33)) == (65, 33)

    class G:
        shape = (65, 33)

    assert grid_of(sp.identity(65 * 33, format="csr"), G()) == (65, 33)
    with pytest.raises(ValueError):
        grid_of(sp.identity(65 * 33, format="csr"))


def test_krylov_flags():
    from paper_1712_06091_b200 import KrylovConfig
    from paper_1712_06091_b200.krylov import _flags

    assert _flags(KrylovConfig()) == 0
    assert _flags(KrylovConfig(flexible=False)) == 1
    assert _flags(KrylovConfig(collect_diagnostics=True)) == 2


def test_bench_op_stream_model_reproduces_survey_b_op():
    """bench.py's algorithmic-bytes model (the reference's op stream, SURVEY.md §8(d)
    counting) reproduces SURVEY's B_op for config 2 (7,726 B/dof/iteration) within 1%, and
    gives the cluster engine's per-launch bytes (inner FGMRES(2) at 129^2 with everything
    below) that the bench line's roofline uses."""
    import sys

    sys.path.insert(0, REPO)
    import bench

    Ns = [1025 ** 2, 513 ** 2, 257 ** 2, 129 ** 2, 65 ** 2]
    S = [7.0, 14.96, 14.91, 14.82, 14.64]
    lev, inner = bench.op_stream_model(Ns, S, 7.0)
    assert abs(sum(lev) / Ns[0] - 7726.0) / 7726.0 < 0.01
    # 4 engine launches per outer iteration carry levels 4-5's bytes
    assert abs(4 * inner(3) - (lev[3] + lev[4])) / (lev[3] + lev[4]) < 0.02


def test_bench_arms_share_the_config_dict():
    """Both bench arms print the same `config` (the driver compares them)."""
    import argparse
    import sys

    sys.path.insert(0, REPO)
    import bench
    from paper_1712_06091_b200 import workloads

    wl = workloads.cfg2(65)
    a = argparse.Namespace(tol=1e-6)
    c1, c2 = bench.bench_config(wl, a, 1), bench.bench_config(wl, a, 1)
    assert c1 == c2 and c1["grid"] == [65, 65] and c1["tol"] == 1e-6
    assert "outer_iterations" not in c1 and "t_setup_ms" not in c1


@pytest.mark.parametrize("shape", [(513, 513, 257), (65, 513, 257), (129, 1025, 513), (257, 257, 129), (33, 16, 35),
                                   (9, 7, 6), (40, 31, 129), (4097, 2049, 1), (37, 1300, 1), (9, 7, 1)])
@pytest.mark.parametrize("jac", [0, 1])
def test_march_plan_covers_the_slab(shape, jac):
    """Host logic of the plane-marching stencil kernel (hadr_march_plan, no device): its tiles and
    plane chunks cover every owned point exactly once, a tile holds at most one point per compute
    thread, the ring fits shared memory and the reduction scratch (8192 blocks) is respected —
    on the BASELINE grids (config 4, an 8-rank slab of it, a slab of config 5), ragged 3D grids
    and 2D grids (marched row by row)."""
    import ctypes as C

    from paper_1712_06091_b200 import _lib

    L = _lib.load()
    out = (C.c_int * 10)()
    n1, n2, n3 = shape
    assert L.hadr_march_plan(n1, n2, n3, jac, out) == 0, L.hadr_last_error()
    nty, ntx, nch, pc, pitch, slot, hy, blocks, smem, cap = list(out)
    d3 = n3 > 1
    nY, nX = (n2, n3) if d3 else (1, n2)
    assert blocks == nty * ntx * nch <= 8192
    assert smem == 6 * slot * 16 * (2 if jac else 1) <= 200 * 1024
    cover = np.zeros((nY, nX), dtype=np.int32)
    for ty in range(nty):
        y0, y1 = ty * nY // nty, (ty + 1) * nY // nty
        for tx in range(ntx):
            x0, x1 = tx * nX // ntx, (tx + 1) * nX // ntx
            assert 0 < (y1 - y0) * (x1 - x0) <= cap
            assert x1 - x0 + 4 <= pitch and (y1 - y0 + 2 * hy) * pitch <= slot
            cover[y0:y1, x0:x1] += 1
    assert (cover == 1).all()
    planes = np.zeros(n1, dtype=np.int32)
    for c in range(nch):
        planes[c * pc:min((c + 1) * pc, n1)] += 1
    assert (planes == 1).all() and (nch - 1) * pc < n1
