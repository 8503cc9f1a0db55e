"""Per-level stencil microbenchmark of the bench hierarchy (cfg2 / cfg4): for every level
operator, hadr_op_bench's plain apply (variant 0) and the relaxation Arnoldi input
(variant 1: y = A D^-1 (s x), basis write, fused dot + finalize) — live CUDA events,
back to back; bytes = stored planes (layout) and non-zeros (algorithmic).

    python tools/level_bench.py [--workload cfg4] [--n 513] [--reps 20]
"""

import argparse
import ctypes as C
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg4")
    ap.add_argument("--n", type=int, default=513)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--levels", type=int, default=99, help="bench the first N levels only")
    ap.add_argument("--variants", default="0,1", help="hadr_op_bench variants (0 apply, 1 fused relaxation input, "
                    "2 apply + dot, 3 split relaxation step: scale/Jacobi kernel + apply + dot)")
    a, extra = ap.parse_known_args()
    import torch

    from paper_1712_06091_b200 import _lib, multigrid, operators, workloads

    for opt in extra:
        k, v = opt.split("=")
        _lib.set_option(k, float(v))
    L = _lib.lib()
    wl = workloads.by_name(a.workload, a.n)
    g = wl.grid
    H2 = operators.assemble_adr(wl.medium, g, wl.omega, wl.tt, "upwind2", wl.bc)
    H1 = operators.assemble_adr(wl.medium, g, wl.omega, wl.tt, "upwind1", wl.bc)
    B = operators.blend_operator(H2, H1, 0.25)
    del H1
    hier = multigrid.build_hierarchy(B, g.shape, 5)
    out = []
    for lev, op in enumerate(hier.ops[: a.levels]):
        N = op.shape[0]
        x = torch.randn(N, dtype=torch.complex128, device="cuda")
        y = torch.empty_like(x)
        nnz = op.nnz if N * len(op.offsets) <= 2e8 else float('nan')  # export is host-side
        for var in [int(v) for v in a.variants.split(",")]:
            ms = C.c_double()
            _lib.check(L.hadr_op_bench(op.handle, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), a.reps, var,
                                       C.byref(ms)))
            per = {0: 2, 1: 5, 2: 3, 3: 9}[var]  # vector streams of 16 B per point
            planes = op.storage_slots or len(op.offsets)
            lay = (planes + per) * N * 16
            alg = (nnz + per * N) * 16
            out.append({"level": lev, "N": N, "offsets": len(op.offsets), "slots": op.storage_slots, "mixed": op.mixed_rows,
                        "nnz_per_row": nnz / N, "variant": var, "us": ms.value * 1e3,
                        "layout_GBs": lay / ms.value / 1e6, "alg_GBs": alg / ms.value / 1e6})
            print(json.dumps(out[-1]))
        del x, y


if __name__ == "__main__":
    main()
