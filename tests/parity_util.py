"""Parity-protocol helpers shared by the GPU tests.

The protocol's end-to-end bar at the BASELINE tolerance is: iterations within +-1 and
relative L2 of the amplitude <= max(1e-8, 3 x the oracle's own self-floor).  The floor is
measured here, on the same inputs, by re-running the oracle with a 1e-15 relative
perturbation of one level of its preconditioner hierarchy at a time (SURVEY.md §8(c),
Appendix A step 6) and taking the largest amplitude change.  The oracle (test
infrastructure) is the checker only.
"""

from contextlib import contextmanager

import numpy as np


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


@contextmanager
def perturbed_hierarchy(mod, level, seed):
    """Every hierarchy ``mod.hierarchy`` builds inside the block has level ``level``'s
    operator multiplied entrywise by (1 + 1e-15 N(0, 1)) (and its inverse diagonal redone)."""
    orig = mod.hierarchy
    rng = np.random.default_rng(seed)

    def build(*a, **k):
        Hi = orig(*a, **k)
        if level < Hi.n_levels:
            A = Hi.ops[level]
            A.data = A.data * (1 + 1e-15 * rng.standard_normal(A.data.size))
            Hi.inv_diags[level] = 1.0 / A.diagonal()
        return Hi

    mod.hierarchy = build
    try:
        yield
    finally:
        mod.hierarchy = orig


def self_floor(mod, solve, levels=5):
    """(floor, unperturbed result) of ``solve()`` -> amplitude array."""
    base = solve()
    worst = 0.0
    for lev in range(levels):
        with perturbed_hierarchy(mod, lev, 3 + lev):
            worst = max(worst, rel(solve(), base))
    return worst, base


def protocol_bar(floor):
    return max(1e-8, 3.0 * floor)


def plus2_operator(shape, rng):
    """Random operator on the plus-radius-2 union of a 2D / 3D grid (9 / 13 offsets, sorted):
    one of the two +-2 entries of every axis zeroed per row (the upwind pair property).
    Out-of-grid entries are zero for the +-2 pairs but left non-zero for the +-1 offsets — a
    kernel must skip them by position, not rely on a zero coefficient.
    Returns (offsets, planes, csr)."""
    import scipy.sparse as sp

    dim = len(shape)
    N = int(np.prod(shape))
    offs = sorted([(0,) * dim] + [tuple(d if a == ax else 0 for a in range(dim)) for ax in range(dim)
                                  for d in (-2, -1, 1, 2)])
    idx = np.meshgrid(*[np.arange(n) for n in shape], indexing="ij")
    strides = [int(np.prod(shape[a + 1:])) for a in range(dim)]
    coef = rng.standard_normal((len(offs), N)) + 1j * rng.standard_normal((len(offs), N))
    side = rng.integers(0, 2, size=(dim, N))
    rows, cols, vals = [], [], []
    k = np.arange(N)
    for o, d in enumerate(offs):
        ok = np.ones(shape, dtype=bool)
        for ax in range(dim):
            ok &= (idx[ax] + d[ax] >= 0) & (idx[ax] + d[ax] < shape[ax])
        ok = ok.ravel()
        present = ok.copy()
        for ax in range(dim):
            if abs(d[ax]) == 2:
                present &= side[ax] == (1 if d[ax] > 0 else 0)
        if max(abs(x) for x in d) != 1:
            coef[o, ~present] = 0.0
        rows.append(k[present])
        cols.append((k + sum(d[ax] * strides[ax] for ax in range(dim)))[present])
        vals.append(coef[o, present])
    A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(N, N))
    return offs, coef, A


def plus1_operator(shape, rng):
    """Random operator on the 3D plus of radius 1 (7 offsets, sorted); out-of-grid entries are
    left non-zero in the planes (a kernel must skip them by position).  Returns (offsets,
    planes, csr)."""
    import scipy.sparse as sp

    N = int(np.prod(shape))
    offs = sorted([(0, 0, 0)] + [tuple(d if a == ax else 0 for a in range(3)) for ax in range(3) for d in (-1, 1)])
    idx = np.meshgrid(*[np.arange(n) for n in shape], indexing="ij")
    strides = [shape[1] * shape[2], shape[2], 1]
    coef = rng.standard_normal((7, N)) + 1j * rng.standard_normal((7, N))
    rows, cols, vals = [], [], []
    k = np.arange(N)
    for o, d in enumerate(offs):
        ok = np.ones(shape, dtype=bool)
        for ax in range(3):
            ok &= (idx[ax] + d[ax] >= 0) & (idx[ax] + d[ax] < shape[ax])
        ok = ok.ravel()
        rows.append(k[ok])
        cols.append((k + sum(d[ax] * strides[ax] for ax in range(3)))[ok])
        vals.append(coef[o, ok])
    A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(N, N))
    return offs, coef, A
