"""Host-side inputs of the amplitude solve: grid, medium, source, travel time.

These are plain containers with the attribute names of the reference types
(helmadr/grid.py:21-56 GridSpec, 78-98 Medium, 101-136 SourceSpec;
helmadr/eikonal.py:15-61 AnalyticBase/TravelTime), so the drivers in
``drivers.py`` accept either the reference's objects or these.  Nothing here
is on the timed path: the travel time is an input of the solve (north_star),
produced once at setup.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class GridSpec:
    """Nodal grid on [0, L1] x [0, L2]; k = i1*n2 + i2, i2 (depth) fastest
    (helmadr/grid.py:3-9, 21-56)."""

    n1: int
    n2: int
    L1: float
    L2: float

    def __post_init__(self):
        if self.n1 < 5 or self.n2 < 5:
            raise ValueError(f"grid needs at least 5 nodes per dimension, got {self.n1}x{self.n2}")
        if self.L1 <= 0 or self.L2 <= 0:
            raise ValueError("domain lengths must be positive")

    @property
    def h1(self) -> float:
        return self.L1 / (self.n1 - 1)

    @property
    def h2(self) -> float:
        return self.L2 / (self.n2 - 1)

    @property
    def shape(self) -> tuple[int, int]:
        return (self.n1, self.n2)

    @property
    def n_nodes(self) -> int:
        return self.n1 * self.n2

    def coords(self):
        return np.meshgrid(np.linspace(0.0, self.L1, self.n1), np.linspace(0.0, self.L2, self.n2), indexing="ij")

    @property
    def hs(self):
        return (self.h1, self.h2)

    @property
    def Ls(self):
        return (self.L1, self.L2)

    @property
    def dim(self) -> int:
        return 2


@dataclass(frozen=True)
class GridSpec3:
    """3D nodal grid on [0,L1]x[0,L2]x[0,L3]; the last axis is depth (fastest),
    k = (i1*n2 + i2)*n3 + i3 — the 2D convention of helmadr/grid.py:5-9 with a
    second lateral axis (3D restatement decision)."""

    n1: int
    n2: int
    n3: int
    L1: float
    L2: float
    L3: float

    def __post_init__(self):
        if min(self.n1, self.n2, self.n3) < 5:
            raise ValueError("grid needs at least 5 nodes per dimension")
        if min(self.L1, self.L2, self.L3) <= 0:
            raise ValueError("domain lengths must be positive")

    @property
    def hs(self):
        return (self.L1 / (self.n1 - 1), self.L2 / (self.n2 - 1), self.L3 / (self.n3 - 1))

    @property
    def h1(self):
        return self.hs[0]

    @property
    def h2(self):
        return self.hs[1]

    @property
    def h3(self):
        return self.hs[2]

    @property
    def Ls(self):
        return (self.L1, self.L2, self.L3)

    @property
    def shape(self):
        return (self.n1, self.n2, self.n3)

    @property
    def n_nodes(self) -> int:
        return self.n1 * self.n2 * self.n3

    @property
    def dim(self) -> int:
        return 3

    def coords(self):
        return np.meshgrid(*[np.linspace(0.0, L, n) for n, L in zip(self.shape, self.Ls)], indexing="ij")


@dataclass
class Medium:
    """kappa^2 > 0 and gamma >= 0 on the grid (helmadr/grid.py:78-98)."""

    grid: GridSpec
    kappa_sq: np.ndarray
    gamma: np.ndarray | None = None

    def __post_init__(self):
        self.kappa_sq = np.asarray(self.kappa_sq, dtype=np.float64)
        if self.kappa_sq.shape != self.grid.shape or not np.all(np.isfinite(self.kappa_sq)):
            raise ValueError("kappa_sq must be a finite field on the grid")
        if np.min(self.kappa_sq) <= 0:
            raise ValueError("kappa_sq must be strictly positive everywhere")
        if self.gamma is None:
            self.gamma = np.zeros(self.grid.shape)
        self.gamma = np.asarray(self.gamma, dtype=np.float64)
        if self.gamma.shape != self.grid.shape or np.min(self.gamma) < 0:
            raise ValueError("gamma must be a non-negative field on the grid")

    @property
    def kappa(self) -> np.ndarray:
        return np.sqrt(self.kappa_sq)


@dataclass(frozen=True)
class SourceSpec:
    """Point source at node (i1, i2), angular frequency omega (helmadr/grid.py:101-125)."""

    i1: int
    i2: int
    omega: float

    def validate(self, grid: GridSpec) -> None:
        if self.omega <= 0:
            raise ValueError("omega must be positive")
        on_top = self.i2 == 0 and 0 <= self.i1 <= grid.n1 - 1
        inside = 1 <= self.i1 <= grid.n1 - 2 and 1 <= self.i2 <= grid.n2 - 2
        if not (on_top or inside):
            raise ValueError(f"source node ({self.i1}, {self.i2}) must be inside the grid or on the top row")

    def position(self, grid: GridSpec):
        return (self.i1 * grid.h1, self.i2 * grid.h2)

    @property
    def index(self):
        return (self.i1, self.i2)


@dataclass(frozen=True)
class SourceSpec3:
    """Point source at node (i1, i2, i3) of a 3D grid."""

    i1: int
    i2: int
    i3: int
    omega: float

    def validate(self, grid) -> None:
        if self.omega <= 0:
            raise ValueError("omega must be positive")
        on_top = self.i3 == 0 and 0 <= self.i1 < grid.n1 and 0 <= self.i2 < grid.n2
        inside = all(1 <= i <= n - 2 for i, n in zip(self.index, grid.shape))
        if not (on_top or inside):
            raise ValueError(f"source node {self.index} must be inside the grid or on the top face")

    @property
    def index(self):
        return (self.i1, self.i2, self.i3)

    def position(self, grid):
        return tuple(i * h for i, h in zip(self.index, grid.hs))


class AnalyticBase:
    """tau0 = |x - x0| with analytic gradient and Laplacian, zeroed at x0
    (helmadr/eikonal.py:15-36)."""

    def __init__(self, grid: GridSpec, source: SourceSpec):
        source.validate(grid)
        self.grid = grid
        self.source = source
        x1, x2 = grid.coords()
        p1, p2 = source.position(grid)
        e1, e2 = x1 - p1, x2 - p2
        r = np.hypot(e1, e2)
        self.tau0 = r
        with np.errstate(divide="ignore", invalid="ignore"):
            self.grad1 = np.where(r > 0, e1 / r, 0.0)
            self.grad2 = np.where(r > 0, e2 / r, 0.0)
            self.lap = np.where(r > 0, 1.0 / r, 0.0)


@dataclass
class TravelTime:
    """tau = tau0*tau1 plus grad(tau), lap(tau) (helmadr/eikonal.py:39-61)."""

    grid: GridSpec
    tau1: np.ndarray
    tau: np.ndarray
    grad1: np.ndarray
    grad2: np.ndarray
    lap: np.ndarray
    base: AnalyticBase | None = None
    fm_time: float = 0.0

    grad3: np.ndarray | None = None

    @property
    def grads(self):
        return [self.grad1, self.grad2] + ([self.grad3] if self.grad3 is not None else [])

    @property
    def grad_sq(self) -> np.ndarray:
        s = self.grad1**2 + self.grad2**2
        if self.grad3 is not None:
            s = s + self.grad3**2
        return s


class _SourceOnly:
    """``base`` of a DeviceTravelTime: the source (the distance factor lives on the device)."""

    def __init__(self, source):
        self.source = source


class DeviceTravelTime:
    """A TravelTime given by tau1 alone: tau = tau0*tau1, grad(tau) and lap(tau) are formed
    on the device (``hadr_tau_derivatives``, helmadr/eikonal.py:180-226) — inside the solve
    by the drivers, so only tau1 crosses the host link (8 B/dof instead of the 32-40 B/dof
    of tau, the gradients and the Laplacian).  Reading ``tau`` / ``grad1`` / ``lap`` / ...
    on the host forms them on the device once and copies them back (same values)."""

    def __init__(self, grid, source, tau1, fm_time: float = 0.0):
        source.validate(grid)
        tau1 = np.asarray(tau1)
        if tau1.shape != tuple(grid.shape):
            raise ValueError(f"tau1 has shape {tau1.shape}, grid is {tuple(grid.shape)}")
        self.grid = grid
        self.source = source
        self.tau1 = tau1
        self.base = _SourceOnly(source)
        self.fm_time = fm_time
        self._host = None

    device_derivatives = True

    def _fields(self):
        if self._host is None:
            from .eikonal import _tau_fields_device

            self._host = _tau_fields_device(self.grid, self.source.index, self.tau1)
        return self._host

    @property
    def tau(self):
        return self._fields()[0]

    @property
    def grads(self):
        return list(self._fields()[1])

    @property
    def grad1(self):
        return self._fields()[1][0]

    @property
    def grad2(self):
        return self._fields()[1][1]

    @property
    def grad3(self):
        g = self._fields()[1]
        return g[2] if len(g) > 2 else None

    @property
    def lap(self):
        return self._fields()[2]

    @property
    def grad_sq(self) -> np.ndarray:
        s = self.grad1**2 + self.grad2**2
        if self.grad3 is not None:
            s = s + self.grad3**2
        return s


def point_source(grid, source) -> np.ndarray:
    """1/(h1 h2 [h3]) at the source node (helmadr/grid.py:128-136)."""
    source.validate(grid)
    q = np.zeros(grid.shape, dtype=np.complex128)
    if len(grid.shape) == 2:
        q[source.i1, source.i2] = 1.0 / (grid.h1 * grid.h2)
    else:
        q[tuple(source.index)] = 1.0 / float(np.prod(grid.hs))
    return q
