"""Multi-rank check of the slab-decomposed solve (run under torchrun).

  torchrun --nproc-per-node R --master-addr 127.0.0.1 --master-port P tools/dist_check.py \
      --case cfg4:33 --backend host [--levels L] [--min-planes M] [--out file.json]

Every rank runs drivers.solve_adr_upwind collectively (slab path); rank 0 then
detaches the communicator, solves the same problem on its own GPU (single-GPU
path) and writes both reports plus the relative L2 difference of the
amplitudes as JSON.  With --backend host, the ranks may share one GPU (gloo
host callbacks, nothing on the device waits for another rank).
"""

from __future__ import annotations

import argparse
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="cfg4:33")
    ap.add_argument("--backend", default="host", choices=("host", "nccl", "auto"))
    ap.add_argument("--levels", type=int, default=0)
    ap.add_argument("--min-planes", type=int, default=16)
    ap.add_argument("--c64", type=int, default=0)
    ap.add_argument("--opt", action="append", default=[], help="library option name=value (repeatable)")
    ap.add_argument("--out", default="")
    args = ap.parse_args()

    import numpy as np
    import torch.distributed as dist

    dist.init_process_group("gloo" if args.backend == "host" else "nccl")
    rank, size = dist.get_rank(), dist.get_world_size()
    if args.backend == "host":
        os.environ["HADR_DEVICE"] = "0"

    import paper_1712_06091_b200 as H
    from paper_1712_06091_b200 import distributed as D, drivers, workloads

    name, n = args.case.split(":")
    wl = workloads.by_name(name, int(n))
    backend = D.init(args.backend)
    D.set_policy(min_planes=args.min_planes, levels=args.levels)
    if args.c64:
        H._lib.set_option("kcycle_c64", 1)
    for o in args.opt:
        k, v = o.split("=")
        H._lib.set_option(k, float(v))
    bounds, nd, nl = D.plan(wl.grid.shape, 5)
    cfg = drivers.StrategyConfig(strategy="adr_upwind_blend", tol=1e-6, max_iter=1000)
    u, a, rep = drivers.solve_adr_upwind(wl.medium, wl.grid, wl.source, wl.tt, cfg, wl.bc)
    D.finalize()
    dist.barrier()
    if rank == 0:
        u1, a1, rep1 = drivers.solve_adr_upwind(wl.medium, wl.grid, wl.source, wl.tt, cfg, wl.bc)
        rel = float(np.linalg.norm(a.reshape(-1) - a1.reshape(-1)) / np.linalg.norm(a1))
        out = {
            "case": args.case, "ranks": size, "backend": backend, "bounds": bounds, "dist_levels": nd,
            "levels": nl, "iterations": rep.iterations, "iterations_single": rep1.iterations,
            "converged": bool(rep.converged), "final_relres": rep.final_relres, "rel_l2_vs_single": rel,
            "history": [float(h) for h in rep.history], "history_single": [float(h) for h in rep1.history],
            "device_time_s": rep.device_time, "device_time_single_s": rep1.device_time,
        }
        line = json.dumps(out)
        print(line, flush=True)
        if args.out:
            with open(args.out, "w") as f:
                f.write(line + "\n")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
