"""K1 (fine-level relaxation stencil) microbenchmark on the bench workload, for
the roofline line of bench.py and the ncu --set full capture.

    python tools/k1_kernel.py [--reps 50] [--variant 1]
"""

import argparse
import ctypes as C
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def k1_measure(wl, reps=50, variant=1):
    import torch

    from paper_1712_06091_b200 import _lib, operators

    L = _lib.lib()
    g = wl.grid
    H2 = operators.assemble_adr(wl.medium, g, wl.omega, wl.tt, "upwind2", wl.bc)
    H1 = operators.assemble_adr(wl.medium, g, wl.omega, wl.tt, "upwind1", wl.bc)
    B = operators.blend_operator(H2, H1, 0.25)
    N = g.n_nodes
    x = torch.randn(N, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    torch.cuda.synchronize()
    ms = C.c_double()
    _lib.check(L.hadr_op_bench(B.handle, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), reps, variant,
                               C.byref(ms)))
    nnz = B.nnz
    per_point = 5 if variant == 1 else 2  # x, dinv, y, V, V0  |  x, y
    alg = (nnz + per_point * N) * 16
    layout = (len(B.offsets) + per_point) * N * 16
    return {"avg_launch_ms": ms.value, "algorithmic_bytes_per_launch": alg, "layout_bytes_per_launch": layout,
            "nnz": nnz, "planes": len(B.offsets), "N": N}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--variant", type=int, default=1)
    ap.add_argument("--size", type=int, default=1025)
    ap.add_argument("--pc", type=int, default=1, help="option pair_compress")
    a = ap.parse_args()
    from paper_1712_06091_b200 import _lib, workloads

    _lib.set_option("pair_compress", a.pc)

    print(json.dumps(k1_measure(workloads.cfg2(a.size), a.reps, a.variant)))
