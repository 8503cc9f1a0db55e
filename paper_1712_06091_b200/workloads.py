"""Seeded synthetic workloads with BASELINE.json's shapes.

BASELINE.json names no public dataset; these builders generate the configs'
media, sources, attenuation layers and analytic travel times.  Decisions that
are not facts of the reference are marked.

* cfg1 : 129^2 on [0,1]^2, kappa = 1, 10 ppw, source at the centre, 16-cell layer,
         tau = kappa*r (tau1 = 1), all-Sommerfeld.
* cfg2 : 1025^2, v = 1.5 + 2.5 x2, 12 ppw at v_min, source (0.5, 0.05),
         20-cell layer, analytic linear-gradient tau, all-Sommerfeld.
* cfg3 : 4097 x 2049, seeded smooth layered velocity, surface source, tau from
         the fast-marching restatement (csrc/eikonal.cpp), Neumann top.
* cfg4 : 3D 513^2 x 257, linear gradient, analytic tau.
Both accept ``n=`` for down-scaled parity cases (same physics, ppw kept).

The coefficient fields grad(tau), lap(tau) follow the reference's
``tau_derivatives`` (helmadr/eikonal.py:180-226) applied to the analytic tau1.
This is setup (the travel time is an input of the solve, north_star) and is
not timed.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .fields import AnalyticBase, GridSpec, Medium, SourceSpec, TravelTime

ALL_SOMMERFELD = ("sommerfeld", "sommerfeld", "sommerfeld", "sommerfeld")  # (top, bottom, left, right)


@dataclass
class Workload:
    name: str
    grid: GridSpec
    medium: Medium
    source: SourceSpec
    tt: TravelTime
    bc: tuple  # (top, bottom, left, right)

    @property
    def omega(self) -> float:
        return self.source.omega

    @property
    def n_dof(self) -> int:
        return self.grid.n_nodes


def cell_layer_gamma(grid: GridSpec, omega: float, cells: int, sides) -> np.ndarray:
    """gamma = omega*(d/W)^2 ramp of helmadr/grid.py:158-171 with the band width W
    given in cells instead of one wavelength (decision)."""
    x1, x2 = grid.coords()
    w1, w2 = cells * grid.h1, cells * grid.h2
    g = np.zeros(grid.shape)
    ramps = []
    if "left" in sides:
        ramps.append((w1 - x1, w1))
    if "right" in sides:
        ramps.append((x1 - (grid.L1 - w1), w1))
    if "top" in sides:
        ramps.append((w2 - x2, w2))
    if "bottom" in sides:
        ramps.append((x2 - (grid.L2 - w2), w2))
    for depth, width in ramps:
        d = np.clip(depth, 0.0, width)
        g = np.maximum(g, omega * (d / width) ** 2)
    return g


def _d1(t, h, ax):
    out = np.empty_like(t)
    a, o = np.moveaxis(t, ax, 0), np.moveaxis(out, ax, 0)
    o[1:-1] = (a[2:] - a[:-2]) / (2.0 * h)
    o[0] = (a[1] - a[0]) / h
    o[-1] = (a[-1] - a[-2]) / h
    return out


def _d2(t, h, ax):
    out = np.empty_like(t)
    a, o = np.moveaxis(t, ax, 0), np.moveaxis(out, ax, 0)
    hh = h * h
    o[1:-1] = (a[2:] - 2.0 * a[1:-1] + a[:-2]) / hh
    o[0] = (2.0 * a[0] - 5.0 * a[1] + 4.0 * a[2] - a[3]) / hh
    o[-1] = (2.0 * a[-1] - 5.0 * a[-2] + 4.0 * a[-3] - a[-4]) / hh
    return out


def travel_time_from_tau1(grid: GridSpec, source: SourceSpec, tau1: np.ndarray) -> TravelTime:
    """Chain rule on tau = tau0*tau1 (helmadr/eikonal.py:204-226, 236-239): central
    first differences, 3-/4-point second differences, grad = 0 and lap = 2 tau1
    at the source node."""
    base = AnalyticBase(grid, source)
    a1 = _d1(tau1, grid.h1, 0)
    a2 = _d1(tau1, grid.h2, 1)
    lap1 = _d2(tau1, grid.h1, 0) + _d2(tau1, grid.h2, 1)
    grad1 = base.tau0 * a1 + tau1 * base.grad1
    grad2 = base.tau0 * a2 + tau1 * base.grad2
    lap = tau1 * base.lap + 2.0 * (base.grad1 * a1 + base.grad2 * a2) + base.tau0 * lap1
    i1, i2 = source.i1, source.i2
    grad1[i1, i2] = 0.0
    grad2[i1, i2] = 0.0
    lap[i1, i2] = 2.0 * tau1[i1, i2]
    return TravelTime(grid, tau1, base.tau0 * tau1, grad1, grad2, lap, base)


def linear_gradient_tau1(grid: GridSpec, source: SourceSpec, v0: float, g: float) -> np.ndarray:
    """tau1 = tau/tau0 for v(x2) = v0 + g*x2, tau = arccosh(1 + g^2 r^2/(2 v v_s))/g,
    with tau1(x0) := kappa(x0) = 1/v(x0) (the limit)  (SURVEY.md §8(d) cfg 2)."""
    x1, x2 = grid.coords()
    p1, p2 = source.position(grid)
    v = v0 + g * x2
    vs = v0 + g * p2
    r = np.hypot(x1 - p1, x2 - p2)
    tau = np.arccosh(1.0 + (g * r) ** 2 / (2.0 * v * vs)) / g
    with np.errstate(divide="ignore", invalid="ignore"):
        t1 = np.where(r > 0, tau / r, 1.0 / vs)
    t1[source.i1, source.i2] = 1.0 / vs
    return t1


def cfg1(n: int = 129, ppw: float = 10.0, layer: int | None = None) -> Workload:
    """BASELINE config 1 (n=129): constant kappa, centre source."""
    grid = GridSpec(n, n, 1.0, 1.0)
    omega = 2.0 * np.pi / (ppw * grid.h1)
    layer = layer if layer is not None else max(2, round(16 * (n - 1) / 128))
    src = SourceSpec((n - 1) // 2, (n - 1) // 2, omega)
    ksq = np.ones(grid.shape)
    gam = cell_layer_gamma(grid, omega, layer, ("top", "bottom", "left", "right"))
    med = Medium(grid, ksq, gam)
    tt = travel_time_from_tau1(grid, src, np.ones(grid.shape))
    return Workload(f"cfg1_{n}", grid, med, src, tt, ALL_SOMMERFELD)


def cfg2(n: int = 1025, ppw: float = 12.0, layer: int | None = None) -> Workload:
    """BASELINE config 2 (n=1025): linear-gradient velocity 1.5 + 2.5 x2."""
    grid = GridSpec(n, n, 1.0, 1.0)
    vmin, g = 1.5, 2.5
    omega = 2.0 * np.pi * vmin / (ppw * grid.h1)
    layer = layer if layer is not None else max(3, round(20 * (n - 1) / 1024))
    i2 = max(layer + 2, round(0.05 * (n - 1)))
    src = SourceSpec((n - 1) // 2, i2, omega)
    x1, x2 = grid.coords()
    v = vmin + g * x2
    ksq = 1.0 / v**2
    gam = cell_layer_gamma(grid, omega, layer, ("top", "bottom", "left", "right"))
    med = Medium(grid, ksq, gam)
    tt = travel_time_from_tau1(grid, src, linear_gradient_tau1(grid, src, vmin, g))
    return Workload(f"cfg2_{n}", grid, med, src, tt, ALL_SOMMERFELD)


class _Base3:
    def __init__(self, source):
        self.source = source


def travel_time_nd(grid, source, tau1) -> TravelTime:
    """3D chain rule on tau = tau0*tau1: the per-axis generalisation of
    helmadr/eikonal.py:204-226 (lap(tau0) = 2/r in 3D; grad = 0 and lap = 2 tau1
    at the source node)."""
    X = grid.coords()
    pos = source.position(grid)
    e = [X[a] - pos[a] for a in range(3)]
    r = np.sqrt(e[0] ** 2 + e[1] ** 2 + e[2] ** 2)
    with np.errstate(divide="ignore", invalid="ignore"):
        g = [np.where(r > 0, ea / r, 0.0) for ea in e]
        l0 = np.where(r > 0, 2.0 / r, 0.0)
    hs = grid.hs
    a = [_d1(tau1, hs[ax], ax) for ax in range(3)]
    lap1 = _d2(tau1, hs[0], 0) + _d2(tau1, hs[1], 1)
    lap1 = lap1 + _d2(tau1, hs[2], 2)
    grads = [r * a[ax] + tau1 * g[ax] for ax in range(3)]
    s = g[0] * a[0] + g[1] * a[1]
    s = s + g[2] * a[2]
    lap = tau1 * l0 + 2.0 * s + r * lap1
    idx = source.index
    for gr in grads:
        gr[idx] = 0.0
    lap[idx] = 2.0 * tau1[idx]
    return TravelTime(grid, tau1, r * tau1, grads[0], grads[1], lap, _Base3(source), 0.0, grads[2])


def cfg4(n: int = 513, ppw: float = 10.0, layer: int | None = None) -> Workload:
    """BASELINE config 4 (n=513): 513 x 513 x 257 on [0,1]^2 x [0,0.5], h = 1/512,
    v = 1.5 + 2.5 z (z = depth, the last axis), source (0.5, 0.5, 0.05), 10 ppw at
    v = 1.5, 16-cell layer on all six faces, all-Sommerfeld, analytic tau."""
    from .fields import GridSpec3, SourceSpec3

    n3 = (n - 1) // 2 + 1
    grid = GridSpec3(n, n, n3, 1.0, 1.0, 0.5)
    h = grid.h1
    vmin, g = 1.5, 2.5
    omega = 2.0 * np.pi * vmin / (ppw * h)
    layer = layer if layer is not None else max(2, round(16 * (n - 1) / 512))
    i3 = max(layer + 2, round(0.05 / grid.h3))
    src = SourceSpec3((n - 1) // 2, (n - 1) // 2, i3, omega)
    X = grid.coords()
    v = vmin + g * X[2]
    ksq = 1.0 / v**2
    gam = np.zeros(grid.shape)
    for ax in range(3):
        w = layer * grid.hs[ax]
        for depth in (w - X[ax], X[ax] - (grid.Ls[ax] - w)):
            d = np.clip(depth, 0.0, w)
            gam = np.maximum(gam, omega * (d / w) ** 2)
    med = Medium(grid, ksq, gam)
    pos = src.position(grid)
    vs = vmin + g * pos[2]
    r = np.sqrt((X[0] - pos[0]) ** 2 + (X[1] - pos[1]) ** 2 + (X[2] - pos[2]) ** 2)
    tau = np.arccosh(1.0 + (g * r) ** 2 / (2.0 * v * vs)) / g
    with np.errstate(divide="ignore", invalid="ignore"):
        t1 = np.where(r > 0, tau / r, 1.0 / vs)
    t1[src.index] = 1.0 / vs
    tt = travel_time_nd(grid, src, t1)
    bc = ("sommerfeld",) * 6  # (top, bottom, left, right, front, back)
    return Workload(f"cfg4_{n}", grid, med, src, tt, bc)


def cfg3_medium(grid: GridSpec, sigma_cells: float) -> np.ndarray:
    """Seeded smooth layered velocity (SURVEY.md §8(d) config 3 recipe): 8 random planar
    interfaces, 9 layer velocities in [1.5, 4.5], Gaussian smoothing sigma (cells),
    affine rescale to [1.5, 4.5]."""
    from scipy.ndimage import gaussian_filter

    rng = np.random.default_rng(1712)
    z0 = np.sort(rng.uniform(0.08, 0.95, 8))
    slope = rng.uniform(-0.15, 0.15, 8)
    vel = rng.uniform(1.5, 4.5, 9)
    x1, x2 = grid.coords()
    layer = np.zeros(grid.shape, dtype=np.int64)
    for k in range(8):
        layer += (x2 > z0[k] + slope[k] * (x1 - 1.0)).astype(np.int64)
    v = gaussian_filter(vel[layer], sigma=sigma_cells, mode="nearest")
    vmin, vmax = v.min(), v.max()
    return 1.5 + 3.0 * (v - vmin) / (vmax - vmin)


def cfg3(n: int = 2049, ppw: float = 10.0, layer: int | None = None, tt=None) -> Workload:
    """BASELINE config 3 (n=2049): 4097 x 2049 on [0,2] x [0,1], h = 1/2048, seeded smooth
    layered velocity 1.5-4.5, 10 ppw at v = 1.5, source at the top centre (2048, 0),
    tau from fast marching (eikonal.compute_travel_time, setup), reference default
    boundary (Neumann top, Sommerfeld elsewhere) with the 20-cell layer on the bottom,
    left and right.  ``n`` scales the grid (2n-1) x n, smoothing and
    layer in proportion."""
    from .eikonal import compute_travel_time

    grid = GridSpec(2 * (n - 1) + 1, n, 2.0, 1.0)
    h = grid.h1
    omega = 2.0 * np.pi * 1.5 / (ppw * h)
    scale = (n - 1) / 2048
    layer = layer if layer is not None else max(2, round(20 * scale))
    src = SourceSpec((grid.n1 - 1) // 2, 0, omega)
    v = cfg3_medium(grid, max(1.0, 20.0 * scale))
    ksq = 1.0 / v**2
    gam = cell_layer_gamma(grid, omega, layer, ("bottom", "left", "right"))
    med = Medium(grid, ksq, gam)
    if tt is None:
        tt = compute_travel_time(med, grid, src, "second")
    bc = ("neumann", "sommerfeld", "sommerfeld", "sommerfeld")  # reference BCSpec() default
    return Workload(f"cfg3_{n}", grid, med, src, tt, bc)


def _lerp_axis(a: np.ndarray, m: int, ax: int) -> np.ndarray:
    """Nodal linear interpolation by an integer factor m along one axis: coarse node j
    lands on fine node j*m (exact nodal alignment)."""
    if m == 1:
        return a
    nc = a.shape[ax]
    nf = (nc - 1) * m + 1
    pos = np.arange(nf) / m
    j0 = np.minimum(np.floor(pos).astype(np.int64), nc - 2)
    t = pos - j0
    shp = [1] * a.ndim
    shp[ax] = nf
    t = t.reshape(shp)
    return np.take(a, j0, axis=ax) * (1.0 - t) + np.take(a, j0 + 1, axis=ax) * t


def cfg5_medium(grid, corr_cells: float, vmin: float = 2.0, vmax: float = 4.0) -> np.ndarray:
    """Seeded smooth Gaussian random velocity (BASELINE config 5): white noise
    (numpy default_rng(1712)) filtered by a Gaussian of sigma = corr/2 cells, whose
    autocorrelation exp(-r^2 / (4 sigma^2)) falls to 1/e at corr cells (decision), then
    an affine map to [vmin, vmax].  The noise lives on a lattice m = (n1-1)//128 fine
    cells apart (m = 8 at 1025^2 x 513; sigma/m = 2.5 lattice cells, smooth at that
    scale) and is interpolated trilinearly to the grid, so building the 539 M-node field
    costs seconds instead of a 539 M-point filter."""
    from scipy.ndimage import gaussian_filter

    m = max(1, (grid.n1 - 1) // 128)
    while any((n - 1) % m for n in grid.shape):
        m //= 2
    cshape = tuple((n - 1) // m + 1 for n in grid.shape)
    rng = np.random.default_rng(1712)
    w = rng.standard_normal(cshape)
    f = gaussian_filter(w, sigma=0.5 * corr_cells / m, mode="reflect")
    for ax in range(f.ndim):
        f = _lerp_axis(f, m, ax)
    lo, hi = f.min(), f.max()
    return vmin + (vmax - vmin) * (f - lo) / (hi - lo)


def cfg5(n: int = 1025, ppw: float = 10.0, layer: int | None = None, tt=None) -> Workload:
    """BASELINE config 5 (n=1025): 1025 x 1025 x 513 on [0,1]^2 x [0,0.5], h = 1/1024,
    seeded Gaussian random velocity 2-4 km/s with a 40-cell correlation length
    (cfg5_medium), 10 ppw at v = 2 (decision), source (0.5, 0.5, 0.05), 16-cell layer
    on all six faces, all-Sommerfeld, tau from the 3D fast marcher at setup.  Solved
    with adr_upwind and with standard_sl at alpha = 0.5 ("shift 1+0.5i", SURVEY.md
    Appendix B4).  ``n`` scales grid, correlation length and layer in proportion."""
    from .eikonal import compute_travel_time
    from .fields import GridSpec3, SourceSpec3

    n3 = (n - 1) // 2 + 1
    grid = GridSpec3(n, n, n3, 1.0, 1.0, 0.5)
    h = grid.h1
    vmin = 2.0
    omega = 2.0 * np.pi * vmin / (ppw * h)
    scale = (n - 1) / 1024
    layer = layer if layer is not None else max(2, round(16 * scale))
    i3 = max(layer + 2, round(0.05 / grid.h3))
    src = SourceSpec3((n - 1) // 2, (n - 1) // 2, i3, omega)
    v = cfg5_medium(grid, max(2.0, 40.0 * scale))
    ksq = 1.0 / v**2
    X = grid.coords()
    gam = np.zeros(grid.shape)
    for ax in range(3):
        wl = layer * grid.hs[ax]
        for depth in (wl - X[ax], X[ax] - (grid.Ls[ax] - wl)):
            d = np.clip(depth, 0.0, wl)
            gam = np.maximum(gam, omega * (d / wl) ** 2)
    med = Medium(grid, ksq, gam)
    if tt is None:
        tt = compute_travel_time(med, grid, src, "second")
    bc = ("sommerfeld",) * 6
    return Workload(f"cfg5_{n}", grid, med, src, tt, bc)


def by_name(name: str, n: int | None = None) -> Workload:
    builders = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5}
    if name not in builders:
        raise ValueError(f"unknown workload {name!r}; known: {sorted(builders)}")
    return builders[name]() if n is None else builders[name](n)
