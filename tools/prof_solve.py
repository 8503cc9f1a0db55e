"""Small driver for ncu launch lists: one warm-up solve, then one profiled solve
of the bench workload with a capped outer iteration count.

    python tools/prof_solve.py --n 1025 --its 2
"""

import argparse
import ctypes as C
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1025)
    ap.add_argument("--its", type=int, default=2)
    ap.add_argument("--warm", type=int, default=1)
    args = ap.parse_args()
    from paper_1712_06091_b200 import _lib, workloads
    from paper_1712_06091_b200.fields import point_source
    from paper_1712_06091_b200.operators import rhs_transform

    L = _lib.lib()
    for opt in ("pdl", "ce_max_n", "kcycle_c64", "stencil_tile", "ce_smem_relax", "cl_max_n", "ce_cgs2", "defer_mgs", "ce_smem_coef", "mid_ppt", "mid_max_n", "mid_min_n", "class_compress", "pair_compress", "relax_split", "stencil_march", "march_min_n", "small_max_work"):
        if os.environ.get("HADR_" + opt.upper()) is not None:
            _lib.set_option(opt, float(os.environ["HADR_" + opt.upper()]))
    wl = workloads.by_name(os.environ.get("HADR_WORKLOAD", "cfg2"), args.n)
    g = wl.grid
    dim = len(g.shape)
    n1, n2, n3 = g.shape[0], g.shape[1], (g.shape[2] if dim == 3 else 1)
    hs = tuple(g.hs) + (1.0,)
    src = tuple(wl.source.index) + (0,)
    qhat = rhs_transform(point_source(g, wl.source), wl.tt, wl.omega, "to_adr").reshape(-1)
    codes = np.array([1] * 6, dtype=np.int32)
    grads = list(wl.tt.grads) + [np.zeros(g.shape)] * (3 - dim)
    f = [np.ascontiguousarray(x, dtype=np.float64) for x in [wl.medium.kappa_sq, wl.medium.gamma] + grads +
         [wl.tt.lap]]
    a = np.empty(n1 * n2 * n3, complex)
    rep = _lib.HadrReport()
    hist = np.zeros(2000)
    ts = C.c_double()

    def solve(its):
        _lib.check(L.hadr_solve_adr_upwind(dim, n1, n2, n3, hs[0], hs[1], hs[2], wl.omega, _lib.cbuf(codes),
                                           src[0], src[1], src[2], *[_lib.cbuf(x) for x in f], _lib.cbuf(qhat),
                                           0.25, 5, 5, its, 1e-6, _lib.cbuf(a), C.byref(rep), _lib.cbuf(hist),
                                           2000, C.byref(ts), 0))
        return rep.device_time

    for _ in range(args.warm):
        solve(args.its)
    k0 = L.hadr_launch_count()
    t = solve(args.its)
    if os.environ.get("HADR_PRINT_MEM"):  # device memory held with the hierarchy pooled (nvidia-smi, MiB)
        import subprocess

        used = subprocess.run(["nvidia-smi", "--query-gpu=memory.used", "--format=csv,noheader,nounits"],
                              capture_output=True, text=True).stdout.split()[0]
        print(f"device memory in use after the solve: {used} MiB")
    print(f"profiled solve: its={rep.iterations} device_time={t*1e3:.3f} ms kernels={L.hadr_launch_count()-k0}")




def ce_breakdown(n=1025, its=1000):
    """Phase breakdown of the cluster engine over one solve."""
    from paper_1712_06091_b200 import _lib

    L = _lib.lib()
    _lib.set_option("ce_profile", 1)
    out = (C.c_ulonglong * 48)()
    L.hadr_ce_profile(out, 1)
    sys.argv = [sys.argv[0], "--n", str(n), "--its", str(its), "--warm", "0"]
    main()
    L.hadr_ce_profile(out, 1)
    v = list(out)
    f = 1.9e3  # cycles per us
    print(f"CE launches={v[7]} total={v[0]/f:.0f}us")
    for name, i in (("allreduce", 1), ("relax control", 3), ("stencil", 5), ("vector ops", 8), ("barriers", 10),
                    ("transfers", 12), ("relax update", 14), ("stencil big", 16), ("smrelax stage big", 18),
                    ("smrelax rows big", 20), ("smrelax stage sm", 22), ("smrelax rows sm", 24),
                    ("allred barrier", 26), ("fg control", 28), ("cgs2", 30), ("cg dots1", 32),
                    ("cg allred1", 34), ("cg update1", 36), ("cg dots2", 38), ("cg allred2", 40),
                    ("cg update2", 42), ("cg final sync", 44)):
        print(f"  {name:13s} {v[i]/f:9.0f} us  n={v[i+1]:7d}  {v[i]/max(v[i+1],1)/1.9:7.0f} ns/op")


def sweep_ce(n=1025, values=(0, 32768, 70000, 270000)):
    from paper_1712_06091_b200 import _lib

    for v in values:
        _lib.set_option("ce_max_n", v)
        sys.argv = [sys.argv[0], "--n", str(n), "--its", "1000", "--warm", "1"]
        print(f"ce_max_n={v}: ", end="")
        main()


if __name__ == "__main__":
    if "--sweep" in sys.argv:
        sweep_ce()
    elif "--ce" in sys.argv:
        sys.argv.remove("--ce")
        ce_breakdown(int(sys.argv[sys.argv.index("--n") + 1]) if "--n" in sys.argv else 1025)
    else:
        main()
