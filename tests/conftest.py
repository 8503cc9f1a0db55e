"""Shared test setup.

* ``gpu`` marker: tests that need a B200 (run on the GPU box with ``-m gpu``).
* OPENBLAS_NUM_THREADS=1 before numpy is imported: the oracle is pinned bit for
  bit against fixtures generated single-threaded (SURVEY.md §8(c) shows BLAS
  thread count moves the reference's own results).
"""

import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import pytest  # noqa: E402
from threadpoolctl import threadpool_limits  # noqa: E402

# a pytest plugin may have imported numpy before the env var above was set
threadpool_limits(1)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def csr_from(g, key):
    import scipy.sparse as sp

    indptr = g[key + "_indptr"]
    n = indptr.size - 1
    return sp.csr_matrix((g[key + "_data"], g[key + "_indices"], indptr), shape=(n, n))


def oracle_problem(wl):
    """oracle.Problem for a workloads.Workload (same arrays, reference bc order)."""
    from oracle import hadr_oracle as O

    g = wl.grid
    src = (wl.source.i1, wl.source.i2)
    if getattr(wl.tt, "device_derivatives", False):  # tau1 only: the checker forms the fields itself
        gr1, gr2, lap, tau = O.tau_fields(wl.tt.tau1, g.L1, g.L2, src)
    else:
        gr1, gr2, lap, tau = wl.tt.grad1, wl.tt.grad2, wl.tt.lap, wl.tt.tau
    return O.Problem(g.n1, g.n2, g.h1, g.h2, wl.omega, src, wl.medium.kappa_sq, wl.medium.gamma, tau, gr1, gr2, lap,
                     wl.bc)


@pytest.fixture(scope="session")
def g33():
    return load_golden("g33_const")


@pytest.fixture(scope="session")
def g65():
    return load_golden("g65_linear")


@pytest.fixture(scope="session")
def gcfg1():
    return load_golden("cfg1_129")


@pytest.fixture(scope="session")
def gcfg3():
    return load_golden("cfg3_65")
