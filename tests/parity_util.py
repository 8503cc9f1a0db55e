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
