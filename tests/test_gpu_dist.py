"""Slab-decomposed (multi-rank) amplitude solve on the B200.

The box has one GPU, so the multi-rank path runs R processes on it with the
host communicator (gloo callbacks: nothing on the device waits for another
rank), and the NCCL communicator is exercised at world size 1 (graph-captured
NCCL all-gather / broadcast).  Each case compares the collective solve with
the single-GPU path, itself pinned to the oracle in test_gpu_parity*.py:
same iteration count, amplitudes within the north-star 1e-8 relative L2.
"""

import json
import os
import subprocess
import sys

import pytest

from conftest import REPO
from test_dist import _free_port

CASES = [
    # (ranks, args)
    (2, ["--case", "cfg1:65", "--backend", "host"]),                      # 2D, 2 slab levels, CE coarse
    (2, ["--case", "cfg4:33", "--backend", "host", "--levels", "3"]),     # 3D, slab inner FGMRES, gathered coarsest
    (3, ["--case", "cfg4:33", "--backend", "host", "--levels", "2"]),     # uneven slabs
    (1, ["--case", "cfg1:65", "--backend", "nccl"]),                      # NCCL, captured in the K-cycle graph
    (2, ["--case", "cfg4:65", "--backend", "host", "--levels", "2", "--c64", "1"]),  # mixed precision
    (2, ["--case", "cfg3:65", "--backend", "host", "--levels", "2"]),     # Neumann top, non-square, FM tau
    (2, ["--case", "cfg4:33", "--backend", "host", "--levels", "2", "--opt", "relax_split=1000"]),  # split relax, z halos
    (2, ["--case", "cfg4:33", "--backend", "host", "--levels", "2", "--opt", "stencil_march=2"]),   # marching kernel on slabs
    (3, ["--case", "cfg4:65", "--backend", "host", "--levels", "2", "--opt", "stencil_march=2"]),   # ... uneven slabs, chunks
]


@pytest.mark.gpu
@pytest.mark.parametrize("ranks,args", CASES, ids=[f"r{r}-" + "-".join(a[1::2]) for r, a in CASES])
def test_slab_solve_matches_single_gpu(ranks, args, tmp_path):
    out = tmp_path / "res.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(ranks),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "tools/dist_check.py", *args,
           "--out", str(out)]
    p = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, OMP_NUM_THREADS="1"))
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    r = json.loads(out.read_text())
    assert r["ranks"] == ranks and r["converged"]
    assert r["dist_levels"] >= 1
    assert abs(r["iterations"] - r["iterations_single"]) <= 1
    tol = 1e-4 if "--c64" in args else 1e-8
    assert r["rel_l2_vs_single"] <= tol, r
