#!/usr/bin/env python
"""Benchmark: amplitude solve (FGMRES(5) + multigrid K-cycle) — Mdof*iter/s.

Workload (BASELINE.json configs[1]): 1025^2 grid, v = 1.5 + 2.5 x2, 12 ppw,
source (0.5, 0.05), 20-cell layer, analytic linear-gradient tau, complex128,
ADR upwind-blend strategy (helmadr/drivers.py:136-168), tol 1e-6, 5 levels.

One step = one full amplitude solve as the reference times it
(helmadr/drivers.py:153-165): device assembly of H2up/H1up, blend, Galerkin
hierarchy, FGMRES to 1e-6.
  value : inputs (medium, tau fields, transformed source) resident in HBM;
          CUDA events on the library stream around the K steps.
  e2e   : the public API drivers.solve_adr_upwind(...) with numpy inputs in
          pinned host memory: the point source's phase value (host), H2D of the
          fields, the solve, the waveform u = a exp(-i w tau) on the device, D2H
          of a and u — wall clock.
Metric: Mdof*iter/s = N * outer_iterations / t / 1e6.

--impl reference: the CPU oracle (oracle/hadr_oracle.py, a restatement of
the Python reference) on the host cores, bounded sample per step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

HBM_FALLBACK = 6650.0
B_OP_2D_UPWIND_C128 = 7726.0   # algorithmic bytes / dof / outer iteration


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


def self_launch(args):
    """`python bench.py --gpus N` without torchrun: re-launch as N ranks (one per GPU)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo")
        return ws, rank, local, dist
    return 1, 0, local, None


def max_over_ranks(x, dist):
    if dist is None:
        return x
    import torch

    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x, dist):
    if dist is None:
        return x
    import torch

    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        try:
            self.f.flush()
            rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        except Exception:
            rows = []
        sm = [float(r[1]) for r in rows if len(r) >= 9]
        mx = max([float(r[2]) for r in rows if len(r) >= 9] or [0.0])
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            if len(r) >= 9:
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def pinned(a):
    import torch

    t = torch.from_numpy(np.ascontiguousarray(a))
    return t.pin_memory().numpy()


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------
def run_ours(args, ws, rank, local, dist):
    import ctypes as C

    import torch

    os.environ["HADR_DEVICE"] = str(local)
    torch.cuda.set_device(local)
    import paper_1712_06091_b200 as H
    from paper_1712_06091_b200 import _lib, drivers, workloads
    from paper_1712_06091_b200.fields import point_source
    from paper_1712_06091_b200.operators import rhs_transform

    L = _lib.lib()
    wl = workloads.by_name(args.workload, args.size)
    g = wl.grid
    n1, n2 = g.shape[0], g.shape[1]
    N = n1 * n2
    cfg = drivers.StrategyConfig(strategy="adr_upwind_blend", tol=args.tol, max_iter=args.maxiter)
    qhat = rhs_transform(point_source(g, wl.source), wl.tt, wl.omega, "to_adr").reshape(-1)
    from paper_1712_06091_b200.operators import _bc

    codes = _bc(wl.bc).codes()
    dim = len(g.shape)
    n3 = g.shape[2] if dim == 3 else 1
    hs = tuple(g.hs) + (1.0,)
    src = tuple(wl.source.index) + (0,)
    # ---- device-resident inputs ----
    dev = torch.device("cuda", local)
    grads = list(wl.tt.grads) + [np.zeros(g.shape)] * (3 - dim)
    fields = [torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(dev)
              for x in [wl.medium.kappa_sq, wl.medium.gamma] + grads + [wl.tt.lap]]
    N = N * n3
    q_d = torch.from_numpy(qhat).to(dev)
    a_d = torch.empty(N, dtype=torch.complex128, device=dev)
    torch.cuda.synchronize()
    rep = _lib.HadrReport()
    cap = cfg.max_iter + 2
    hist = np.zeros(cap)
    tset = C.c_double()

    def step_device():
        _lib.check(L.hadr_solve_adr_upwind(
            dim, n1, n2, n3, float(hs[0]), float(hs[1]), float(hs[2]), float(wl.omega), _lib.cbuf(codes), src[0],
            src[1], src[2], *[C.c_void_p(f.data_ptr()) for f in fields], C.c_void_p(q_d.data_ptr()), float(cfg.beta),
            int(cfg.levels), int(cfg.restart), int(cfg.max_iter), float(cfg.tol), C.c_void_p(a_d.data_ptr()),
            C.byref(rep), _lib.cbuf(hist), cap, C.byref(tset), 1))
        return rep.iterations, tset.value, rep.device_time

    for _ in range(args.warmup):
        step_device()
    its_list, t_setup, t_kry = [], [], []
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    n_launch0 = L.hadr_launch_count()
    with Clocks(local) as clk:
        L.hadr_stream_timer(1)
        for _ in range(args.steps):
            its, ts, tk = step_device()
            its_list.append(its)
            t_setup.append(ts)
            t_kry.append(tk)
        t_dev = L.hadr_stream_timer(0) * 1e-3
    torch.cuda.synchronize()
    launches = L.hadr_launch_count() - n_launch0
    if dist:
        dist.barrier()
    t_max = max_over_ranks(t_dev, dist)
    mdof_its = sum_over_ranks(N * sum(its_list) / 1e6, dist)
    value = mdof_its / t_max
    a_dev = a_d.cpu().numpy()

    # ---- "complex64" variant = mixed precision (K-cycle operators in c64, outer FGMRES c128) ----
    _lib.set_option("kcycle_c64", 1)
    step_device()
    L.hadr_stream_timer(1)
    its64 = [step_device()[0] for _ in range(args.steps)]
    t64 = max_over_ranks(L.hadr_stream_timer(0) * 1e-3, dist)
    a64 = a_d.cpu().numpy()
    _lib.set_option("kcycle_c64", 0)
    c64 = {"value": sum_over_ranks(N * sum(its64) / 1e6, dist) / t64, "unit": "Mdof*iter/s",
           "outer_iterations": its64, "ms_per_step": t64 / args.steps * 1e3,
           "rel_l2_vs_c128": float(np.linalg.norm(a64 - a_dev) / np.linalg.norm(a_dev)),
           "note": "K-cycle operators stored in complex64 (widened to c128 arithmetic); vectors, reductions and "
                   "the outer FGMRES complex128 (SURVEY.md §7.3 item 5)"}

    # ---- e2e through the public API (host numpy inputs, pinned) ----
    # the travel time enters as tau1 alone: tau, grad(tau), lap(tau) are formed on the device
    # (tau_derivatives, helmadr/eikonal.py:180-226) inside the timed call
    from paper_1712_06091_b200.fields import DeviceTravelTime

    med = type(wl.medium)(g, pinned(wl.medium.kappa_sq), pinned(wl.medium.gamma))
    tt_p = DeviceTravelTime(g, wl.source, pinned(wl.tt.tau1))
    e2e_its = 0
    u = a = None
    for _ in range(max(1, min(args.warmup, 2))):
        drivers.solve_adr_upwind(med, g, wl.source, tt_p, cfg, wl.bc)
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        u, a, r = drivers.solve_adr_upwind(med, g, wl.source, tt_p, cfg, wl.bc)
        e2e_its += r.iterations
    t_e2e = max_over_ranks(time.perf_counter() - t0, dist)
    e2e_value = sum_over_ranks(N * e2e_its / 1e6, dist) / t_e2e
    h2d = 3 * 8 * N + 16     # kappa^2, gamma, tau1; the point source's one value
    d2h = 2 * 16 * N         # amplitude a and waveform u
    agree = float(np.linalg.norm(a.reshape(-1) - a_dev) / np.linalg.norm(a_dev))

    # ---- rooflines: the dominant kernel (cluster engine) and the fine sweep K1, live CUDA events ----
    its_mean = sum(its_list) / len(its_list)
    roof = engine_roofline(H, L, wl, cfg, its_mean, sum(t_kry) / len(t_kry))
    roof_k1 = kernel_roofline(H, L, wl, cfg, args)
    hbm, src = peaks()
    solve_bw = B_OP_2D_UPWIND_C128 * N * its_mean / (sum(t_kry) / len(t_kry)) / 1e9
    out = {
        "metric": "amplitude solve Mdof*iter/s (FGMRES(5) + K-cycle, ADR upwind blend)",
        "value": value,
        "unit": "Mdof*iter/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_max / args.steps * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "c128",
        "data": "synthetic (seeded config builder: linear-gradient velocity, analytic tau)",
        "config": bench_config(wl, args, ws),
        "run": {"outer_iterations": its_list, "t_setup_ms": [x * 1e3 for x in t_setup],
                "t_krylov_ms": [x * 1e3 for x in t_kry]},
        "e2e": {"value": e2e_value, "unit": "Mdof*iter/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": t_e2e / args.steps * 1e3, "rel_l2_vs_device_path": agree},
        "gpu_launches": int(launches),
        "complex64_mixed": c64,
        "roofline": roof,
        "roofline_k1": roof_k1,
        "solve_roofline": {"bound": "hbm", "model_bytes_per_dof_iter": B_OP_2D_UPWIND_C128,
                           "achieved": solve_bw, "peak": hbm, "unit": "GB/s", "frac": solve_bw / hbm,
                           "peak_source": src, "note": "B_op (SURVEY.md §8(d)) over the FGMRES time"},
        "clocks": clk.summary(),
    }
    if rank == 0 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(wl, args, its_full=round(its_mean))
    if args.extra_3d:
        out["config_4_3d"] = guarded_slab_run(lambda: run_3d(args, L, local, dist, ws, rank), out, ws, rank,
                                              args.slab_timeout)
    if args.extra_cfg3:
        out["config_3"] = run_3d(args, L, local, dist, 1, rank, which="cfg3")
    if args.extra_cfg5:
        out["config_5"] = run_3d(args, L, local, dist, 1, rank, which="cfg5")
    return out


def guarded_slab_run(fn, out, ws, rank, timeout_s):
    """The N > 1 config-4 line is ONE solve split over the ranks (NCCL inside the K-cycle
    graphs).  If it fails or stalls, the headline line must still be printed: a watchdog
    prints what was measured so far (rank 0) and ends the process after timeout_s."""
    if ws == 1:
        return fn()
    import threading

    def fire():
        if rank == 0:
            res = dict(out)
            res["config_4_3d"] = {"error": f"slab solve did not finish within {timeout_s:.0f} s"}
            print(json.dumps(res), flush=True)
        os._exit(0)

    timer = threading.Timer(timeout_s, fire)
    timer.daemon = True
    timer.start()
    try:
        return fn()
    except Exception as e:  # noqa: BLE001 - recorded in the JSON line, the headline stands
        return {"error": f"{type(e).__name__}: {e}"}
    finally:
        timer.cancel()


B_OP_3D_UPWIND_C128 = 6788.0  # 3D adr_upwind c128 (10 / 10 / 54 non-zeros)


def run_3d(args, L, local, dist, ws=1, rank=0, which="cfg4"):
    """BASELINE configs[3] (3D 513^2 x 257, c128): device-resident inputs, CUDA events.
    N > 1 (torchrun): ONE solve split in axis-0 slabs over the N GPUs (NCCL halo exchange /
    all-gather / broadcast, coarse levels agglomerated) — strong scaling, max over ranks.
    The CPU sample is the dimension-generic oracle on a down-scaled grid (rank 0).
    which="cfg3": BASELINE configs[2] (2D 4097 x 2049, layered medium, fast-marching tau,
    1 GPU; every rank solves its own replica when N > 1)."""
    import ctypes as C

    import torch

    from paper_1712_06091_b200 import _lib, drivers, workloads
    from paper_1712_06091_b200.fields import point_source
    from paper_1712_06091_b200.operators import _bc, rhs_transform

    t_fm = None
    if which == "cfg3":
        wl = workloads.cfg3(args.extra_cfg3)
        t_fm = wl.tt.fm_time
    elif which == "cfg5":
        wl = workloads.cfg5(args.extra_cfg5)
        t_fm = wl.tt.fm_time
    else:
        wl = workloads.cfg4(args.extra_3d)
    g = wl.grid
    dim = len(g.shape)
    n1, n2 = g.shape[0], g.shape[1]
    n3 = g.shape[2] if dim == 3 else 1
    N = n1 * n2 * n3
    b_op = B_OP_3D_UPWIND_C128 if dim == 3 else B_OP_2D_UPWIND_C128
    cfg = drivers.StrategyConfig(strategy="adr_upwind_blend", tol=args.tol, max_iter=args.maxiter)
    qhat = rhs_transform(point_source(g, wl.source), wl.tt, wl.omega, "to_adr").reshape(-1)
    dev = torch.device("cuda", local)
    fields = [torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(dev)
              for x in [wl.medium.kappa_sq, wl.medium.gamma] + list(wl.tt.grads) + [wl.tt.lap]]
    q_d = torch.from_numpy(qhat).to(dev)
    a_d = torch.empty(N, dtype=torch.complex128, device=dev)
    del qhat
    torch.cuda.synchronize()
    codes = _bc(wl.bc).codes()
    rep = _lib.HadrReport()
    hist = np.zeros(cfg.max_iter + 2)
    tset = C.c_double()
    hs, src = g.hs, wl.source.index
    slab = None
    if ws > 1:
        from paper_1712_06091_b200 import distributed as D

        D.init("nccl")
        bounds, nd, nl = D.plan(g.shape, cfg.levels)
        slab = {"bounds": bounds, "slab_levels": nd, "levels": nl}

    def step():
        _lib.check(L.hadr_solve_adr_upwind(
            dim, n1, n2, n3, hs[0], hs[1], hs[2] if dim == 3 else 1.0, float(wl.omega), _lib.cbuf(codes), src[0],
            src[1], src[2] if dim == 3 else 0, *[C.c_void_p(f.data_ptr()) for f in fields[:2 + dim]],
            *([C.c_void_p(0)] if dim == 2 else []), C.c_void_p(fields[-1].data_ptr()), C.c_void_p(q_d.data_ptr()),
            float(cfg.beta),
            int(cfg.levels), int(cfg.restart), int(cfg.max_iter), float(cfg.tol), C.c_void_p(a_d.data_ptr()),
            C.byref(rep), _lib.cbuf(hist), len(hist), C.byref(tset), 1))
        return rep.iterations, tset.value, rep.device_time

    step()
    its, tk = [], []
    L.hadr_stream_timer(1)
    for _ in range(args.steps_3d):
        i, _, t = step()
        its.append(i)
        tk.append(t)
    t_dev = max_over_ranks(L.hadr_stream_timer(0) * 1e-3, dist)
    c64 = None
    if which == "cfg4":  # BASELINE config 4 names complex64 too: the mixed-precision K-cycle
        L.hadr_pool_trim()  # release the recycled complex128 hierarchy before building the mixed one
        _lib.set_option("kcycle_c64", 1)
        try:
            step()
            its64 = []
            L.hadr_stream_timer(1)
            for _ in range(args.steps_3d):
                its64.append(step()[0])
            t64 = max_over_ranks(L.hadr_stream_timer(0) * 1e-3, dist)
        finally:
            _lib.set_option("kcycle_c64", 0)
            L.hadr_pool_trim()
        c64 = {"value": N * sum(its64) / t64 / 1e6, "unit": "Mdof*iter/s", "outer_iterations": its64,
               "ms_per_step": t64 / len(its64) * 1e3,
               "note": "K-cycle operators stored complex64 (widened to c128 arithmetic); vectors, reductions and "
                       "the outer FGMRES complex128 (SURVEY.md §7.3 item 5); parity <= 1e-4 in tests"}
    if slab is not None:
        D.finalize()
    hbm, srcp = peaks()
    t_k = max_over_ranks(sum(tk) / len(tk), dist)
    bw = b_op * N * (sum(its) / len(its)) / t_k / 1e9 / ws  # per-GPU bytes
    label = {"cfg3": f"BASELINE configs[2], 2D {n1}x{n2}, layered medium, fast-marching tau",
             "cfg5": f"BASELINE configs[4] recipe at {n1}x{n2}x{n3} (full 1025^2x513 needs 8 GPUs), Gaussian random "
                     f"medium, 3D fast-marching tau, adr_upwind",
             "cfg4": f"BASELINE configs[3], 3D {n1}x{n2}x{n3}"}[which]
    out = {"workload": f"{wl.name} ({label}, c128, {ws} GPU)",
           "value": N * sum(its) / t_dev / 1e6, "unit": "Mdof*iter/s", "outer_iterations": its,
           "n_gpus": ws, "scaling": "strong" if ws > 1 else None,
           "parallelism": f"axis-0 slabs x{ws} (NCCL)" if ws > 1 else "single GPU", "slab_plan": slab,
           "ms_per_step": t_dev / len(its) * 1e3, "t_krylov_ms": [t * 1e3 for t in tk],
           "solve_roofline": {"bound": "hbm", "model_bytes_per_dof_iter": b_op, "achieved": bw,
                              "peak": hbm, "unit": "GB/s", "frac": bw / hbm, "peak_source": srcp,
                              "note": "per GPU" if ws > 1 else ""}}
    if c64 is not None:
        out["complex64_mixed"] = c64
    if t_fm is not None:
        out["t_fast_march_s"] = t_fm
        out["note"] = "travel time from the fast-marching restatement at setup (host, untimed, t_fast_march_s)"
    del fields, q_d, a_d
    torch.cuda.empty_cache()
    if which == "cfg4" and ws == 1:
        L.hadr_pool_trim()
        out["roofline_k1m"] = roofline_k1m(wl)
    if which == "cfg5":
        out["standard_sl"] = run_cfg5_sl(args, L, wl)
    if not args.no_cpu_baseline and rank == 0 and which == "cfg5":
        from threadpoolctl import threadpool_limits

        from oracle import hadr_oracle_nd as ND

        w5 = workloads.cfg5(65)
        gg = w5.grid
        bc = ND.bc_dict(3, w5.bc)
        grads, lap, tau = ND.tau_fields(w5.tt.tau1, gg.Ls, w5.source.index)
        with threadpool_limits(1):
            t0 = time.perf_counter()
            _, r = ND.solve_upwind(gg.shape, gg.hs, w5.omega, w5.source.index, w5.medium.kappa_sq, w5.medium.gamma,
                                   grads, lap, tau, bc, maxiter=3)
            tc = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": gg.n_nodes * r.iterations / tc / 1e6, "unit": "Mdof*iter/s", "cores": 1,
                               "kind": "port", "sample": f"nd oracle on cfg5_65 (65x65x33): assembly + hierarchy + "
                                                         f"{r.iterations} outer iterations ({tc:.1f} s)"}
    elif not args.no_cpu_baseline and rank == 0 and which == "cfg3":
        from threadpoolctl import threadpool_limits

        from oracle import hadr_oracle as O

        ws_ = workloads.cfg3(513)  # 1025 x 513: same recipe, bounded CPU sample
        gg = ws_.grid
        p = oracle_problem(ws_)
        with threadpool_limits(1):
            t0 = time.perf_counter()
            _, _, r = O.solve_upwind(p, tol=args.tol, maxiter=6)
            tc = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": gg.n_nodes * r.iterations / tc / 1e6, "unit": "Mdof*iter/s", "cores": 1,
                               "kind": "port", "sample": f"oracle on cfg3_513 (1025x513): assembly + hierarchy + "
                                                         f"{r.iterations} outer iterations ({tc:.1f} s)"}
    elif not args.no_cpu_baseline and rank == 0:
        from threadpoolctl import threadpool_limits

        from oracle import hadr_oracle_nd as ND

        ws = workloads.cfg4(65)
        gg = ws.grid
        bc = ND.bc_dict(3, ws.bc)
        with threadpool_limits(1):
            t0 = time.perf_counter()
            grads, lap, tau = ND.tau_fields(ws.tt.tau1, gg.Ls, ws.source.index)
        with threadpool_limits(1):
            t0 = time.perf_counter()
            _, r = ND.solve_upwind(gg.shape, gg.hs, ws.omega, ws.source.index, ws.medium.kappa_sq, ws.medium.gamma,
                                   grads, lap, tau, bc, maxiter=3)
            tc = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": gg.n_nodes * r.iterations / tc / 1e6, "unit": "Mdof*iter/s", "cores": 1,
                               "kind": "port", "sample": f"nd oracle on cfg4_65 (65x65x33): assembly + hierarchy + "
                                                         f"{r.iterations} outer iterations ({tc:.1f} s)"}
    return out


B_OP_3D_SL_C128 = 5006.0  # 3D standard_sl c128 (7 / 7 / 27 non-zeros)


def run_cfg5_sl(args, L, wl):
    """Config 5's second solver: standard_sl (shift alpha = 0.5 on the 7-point Helmholtz
    operator, helmadr/drivers.py:57-67) through the public API; the reference times the
    FGMRES only (helmadr/drivers.py:63-66), so does this line (device time of fgmres)."""
    from paper_1712_06091_b200 import drivers, operators
    from paper_1712_06091_b200.fields import point_source

    g = wl.grid
    N = g.n_nodes
    H = operators.assemble_helmholtz(wl.medium, g, wl.omega, wl.bc)
    q = point_source(g, wl.source)
    cfg = drivers.StrategyConfig(strategy="standard_sl", alpha=0.5, tol=args.tol, max_iter=args.maxiter)
    drivers.solve_standard(H, q, wl.medium, wl.omega, cfg)
    its, tk = [], []
    for _ in range(args.steps_3d):
        _, rep = drivers.solve_standard(H, q, wl.medium, wl.omega, cfg)
        its.append(rep.iterations)
        tk.append(rep.device_time)
    t = sum(tk) / len(tk)
    hbm, srcp = peaks()
    bw = B_OP_3D_SL_C128 * N * (sum(its) / len(its)) / t / 1e9
    return {"value": N * sum(its) / sum(tk) / 1e6, "unit": "Mdof*iter/s", "outer_iterations": its,
            "ms_per_step": t * 1e3, "alpha": 0.5,
            "solve_roofline": {"bound": "hbm", "model_bytes_per_dof_iter": B_OP_3D_SL_C128, "achieved": bw,
                               "peak": hbm, "unit": "GB/s", "frac": bw / hbm, "peak_source": srcp},
            "note": "FGMRES device time per solve (the reference's standard_sl timing); K-cycle on H - 0.5i w^2 "
                    "diag(kappa^2), the 'shift 1+0.5i' of BASELINE config 5"}


def op_stream_model(Ns, S, S_outer, b=16, restart=5, s_coarse=10):
    """Algorithmic bytes of the reference's op stream (SURVEY.md §8(d) counting: stencil
    (S+2)b per point, +b for a fused right-hand-side read or D^-1; dot 2b, axpy 3b, norm b,
    scale 2b, lincomb (k+2)b; copies and known-zero spmvs not counted; re-orthogonalisation
    on every FGMRES step, two inner iterations; S = mean non-zeros per row).  Follows
    helmadr/krylov.py:91-242 and helmadr/multigrid.py:132-171.  Returns (bytes per level per
    outer iteration, function level -> bytes of one inner FGMRES(2) call at that level with
    everything below it).  For config 2 the total reproduces SURVEY's B_op (7,726 B/dof/it)
    within 1%."""
    nl = len(Ns)

    def relax(lev, l, s, xzero):
        t = 0 if xzero else (S[l] + 3) * b
        t += 3 * b
        for j in range(s):
            t += (S[l] + 3) * b + (j + 1) * 5 * b + 3 * b
        t += (s + 3) * b
        lev[l] += t * Ns[l]

    def kcycle(lev, l):
        relax(lev, l, l + 2, True)
        lev[l] += (S[l] + 3) * b * Ns[l] + b * Ns[l] + 2 * b * Ns[l]
        lev[l + 1] += 2 * b * Ns[l + 1]
        if l + 1 == nl - 1:
            relax(lev, l + 1, s_coarse, True)
        else:
            inner(lev, l + 1)
        relax(lev, l, l + 2, False)

    def inner(lev, c):
        t = 4 * b
        for j in range(2):
            kcycle(lev, c)
            t += (S[c] + 2) * b + 3 * b + 2 * (j + 1) * 5 * b + 2 * b
        t += 4 * b + (S[c] + 3) * b + b
        lev[c] += t * Ns[c]

    lev = [0.0] * nl
    kcycle(lev, 0)
    t = sum((S_outer + 2) * b + 3 * b + 2 * (j + 1) * 5 * b + 2 * b for j in range(restart)) / restart
    t += ((restart + 2) * b + (S_outer + 3) * b + 3 * b) / restart
    lev[0] += t * Ns[0]

    def inner_bytes(c):
        x = [0.0] * nl
        inner(x, c)
        return sum(x)

    return lev, inner_bytes


def engine_roofline(H, L, wl, cfg, its_mean, t_krylov):
    """The dominant kernel of the headline solve: k_cluster_engine, the coarse part of the
    K-cycle (inner FGMRES(2) at the engine's entry level with both recursive K-cycles and
    the coarsest GMRES(10)) as ONE persistent 16-CTA cluster kernel.  Timed live with CUDA
    events (hadr_ce_bench: back-to-back launches on the library stream, after a real
    preconditioner application filled its inputs); algorithmic bytes per launch = the
    reference op stream of that call (op_stream_model with the levels' measured mean
    non-zeros per row).  latency_budget: the engine's clock64 phase counters over profiled
    launches — reduction-separated steps per launch and what each costs."""
    import ctypes as C

    from paper_1712_06091_b200 import operators
    from paper_1712_06091_b200.fields import point_source

    g = wl.grid
    H2 = operators.assemble_adr(wl.medium, g, wl.omega, wl.tt, "upwind2", wl.bc)
    H1 = operators.assemble_adr(wl.medium, g, wl.omega, wl.tt, "upwind1", wl.bc)
    hier = H.build_hierarchy(operators.blend_operator(H2, H1, cfg.beta), g, cfg.levels)
    del H1
    M = H.make_kcycle_preconditioner(hier)
    q = operators.rhs_transform(point_source(g, wl.source), wl.tt, wl.omega, "to_adr").reshape(-1)
    M(q / np.linalg.norm(q))
    entry = None
    for lev in range(2, hier.n_levels):
        try:
            t = C.c_double()
            _lib_check(L.hadr_ce_bench(hier.handle, lev, 1, C.byref(t)))
            entry = lev
            break
        except ValueError:
            continue
    if entry is None:
        return {"kernel": "k_cluster_engine", "error": "no level runs in the cluster engine"}
    avg = C.c_double()
    _lib_check(L.hadr_ce_bench(hier.handle, entry, 200, C.byref(avg)))
    Ns = [int(np.prod(s)) for s in hier.shapes]
    S = [hier.ops[l].nnz / Ns[l] if l >= entry - 1 else 0.0 for l in range(hier.n_levels)]
    _, inner_bytes = op_stream_model(Ns, S, 7.0)
    bytes_launch = inner_bytes(entry - 1)
    hbm, src = peaks()
    ach = bytes_launch / (avg.value * 1e-3) / 1e9
    launches_per_it = 2 ** (entry - 2)  # inner(entry) runs once per visit of level entry-1
    # latency budget: phase counters of CTA 0 over profiled launches (clock64, 1965 MHz)
    from paper_1712_06091_b200 import _lib

    prof = (C.c_ulonglong * 48)()
    _lib.set_option("ce_profile", 1)
    try:
        L.hadr_ce_profile(prof, 1)
        t = C.c_double()
        _lib_check(L.hadr_ce_bench(hier.handle, entry, 50, C.byref(t)))
        L.hadr_ce_profile(prof, 1)
    finally:
        _lib.set_option("ce_profile", 0)
    v = list(prof)
    nl_ = max(v[7], 1)
    mhz = 1965.0
    budget = {"launches_profiled": v[7], "us_per_launch_profiled": v[0] / mhz / nl_,
              "allreduces_per_launch": v[2] / nl_, "us_per_allreduce": v[1] / mhz / max(v[2], 1),
              "stencils_per_launch": v[6] / nl_, "us_per_stencil": v[5] / mhz / max(v[6], 1),
              "control_us_per_launch": v[3] / mhz / nl_, "vector_ops_us_per_launch": v[8] / mhz / nl_,
              "barrier_us_per_launch": v[10] / mhz / nl_, "transfer_us_per_launch": v[12] / mhz / nl_,
              "lincomb_us_per_launch": v[14] / mhz / nl_,
              "note": "clock64 of CTA 0 (thread 0; relaxation control on the last thread), 1965 MHz"}
    traffic = None
    try:  # dram__bytes_read.sum + dram__bytes_write.sum of the committed ncu --set full capture
        with open(os.path.join(REPO, "profiles", "r02_engine_ncu.json")) as f:
            pr = json.load(f)
        traffic = (pr["dram_read_MB"] + pr["dram_write_MB"]) * 1e6
    except Exception:
        pass
    return {"kernel": f"k_cluster_engine (16-CTA cluster; inner FGMRES(2) at level {entry} "
                      f"{'x'.join(map(str, hier.shapes[entry - 1]))} + K-cycles + coarsest GMRES(10))",
            "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm, "traffic": traffic,
            "peak_source": src, "avg_launch_ms": avg.value, "algorithmic_bytes_per_launch": bytes_launch,
            "launches_per_outer_iteration": launches_per_it,
            "share_of_krylov_time": launches_per_it * its_mean * avg.value * 1e-3 / t_krylov,
            "mean_nnz_per_row": {f"level{l + 1}": S[l] for l in range(entry - 1, hier.n_levels)},
            "latency_budget": budget,
            "traffic_note": "working set L2/SMEM-resident (DRAM traffic ~0): bound by reduction-separated steps"}


def _lib_check(code):
    from paper_1712_06091_b200 import _lib

    _lib.check(code)


def kernel_roofline(H, L, wl, cfg, args):
    """K1 — the fine-level relaxation stencil y = A(D^-1 s x) with the basis write
    and the fused <V0, y> — timed live with CUDA events on the library stream
    (back-to-back launches, no host sync), against its algorithmic bytes."""
    sys.path.insert(0, os.path.join(REPO, "tools"))
    from k1_kernel import k1_measure

    m = k1_measure(wl, reps=50, variant=1)
    hbm, src = peaks()
    ach = m["algorithmic_bytes_per_launch"] / (m["avg_launch_ms"] * 1e-3) / 1e9
    traffic = None
    try:  # dram__bytes_read.sum + dram__bytes_write.sum from the committed ncu --set full capture
        with open(os.path.join(REPO, "profiles", "k1_ncu.json")) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    except Exception:
        pass
    return {"kernel": "k_stencil<IN_SCALE|IN_JAC|IN_WRITEV, APPLY, RED_DOT> (K1, fine level 1025^2, blend operator)",
            "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm, "traffic": traffic,
            "peak_source": src, **m}


def roofline_k1m(wl, reps=20):
    """The 3D fine level's dominant kernel, live: k_stencil_march (plane-marching, bulk-copy
    input tiles) on the pair-compressed upwind operator of the config-4 grid — the relaxation
    Arnoldi input (hadr_op_bench variant 1) and apply + dot (variant 2), CUDA events over
    back-to-back launches.  Algorithmic bytes per point: 10 coefficient slots + pair code +
    the vector streams (x, D^-1, V_0 in; V_j, y out | x, u in; y out), 16 B each."""
    import ctypes as C

    import torch

    from paper_1712_06091_b200 import _lib, operators

    L = _lib.lib()
    g = wl.grid
    H2 = operators.assemble_adr(wl.medium, g, wl.omega, wl.tt, "upwind2", wl.bc)
    N = g.n_nodes
    x = torch.randn(N, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    hbm, src = peaks()
    traffic = {}
    try:
        with open(os.path.join(REPO, "profiles", "r02_march3d_ncu.json")) as f:
            pr = json.load(f)
        traffic = {1: pr["relaxation_input"]["dram_bytes_per_launch"], 2: pr["apply_dot"]["dram_bytes_per_launch"]}
    except Exception:
        pass
    out = {}
    for var, name, streams in ((1, "relaxation_input", 5), (2, "apply_dot", 3)):
        ms = C.c_double()
        _lib.check(L.hadr_op_bench(H2.handle, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), reps, var,
                                   C.byref(ms)))
        alg = ((10 + streams) * 16 + 1) * N
        ach = alg / (ms.value * 1e-3) / 1e9
        out[name] = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                     "traffic": traffic.get(var), "avg_launch_ms": ms.value, "algorithmic_bytes_per_launch": alg,
                     "peak_source": src}
    out["kernel"] = ("k_stencil_march<13, ...> (K1m: 3D fine level, pair-compressed 13-offset upwind operator, "
                     f"{g.shape[0]}x{g.shape[1]}x{g.shape[2]}; cp.async.bulk input tiles in a 6-slot shared-memory ring)")
    out["note"] = ("frac > 1 is possible: the peak is the measured copy bandwidth (1 read : 1 write), this kernel "
                   "reads 13-15 streams per stream written")
    del H2, x, y
    torch.cuda.empty_cache()
    return out


# --------------------------------------------------------------------------
# CPU oracle (baseline / reference arm)
# --------------------------------------------------------------------------
def bench_config(wl, args, ws):
    """The workload's config dict — identical in both arms (the driver compares them)."""
    g = wl.grid
    return {"workload": f"{wl.name} (BASELINE configs[1], 2D {g.n1}x{g.n2}, c128)", "grid": [g.n1, g.n2],
            "strategy": "adr_upwind_blend", "tol": args.tol, "restart": 5, "levels": 5,
            "parallelism": f"replicas x{ws}", "l2": "working set (~1.3 GB) > 126 MB L2; no flush needed"}


def oracle_problem(wl):
    """oracle.Problem of a 2D workload, the derivative fields formed by the oracle's own
    restatement of tau_derivatives (helmadr/eikonal.py:180-226) from tau1."""
    from oracle import hadr_oracle as O

    g = wl.grid
    src = (wl.source.i1, wl.source.i2)
    gr1, gr2, lap, tau = O.tau_fields(wl.tt.tau1, g.L1, g.L2, src)
    return O.Problem(g.n1, g.n2, g.h1, g.h2, wl.omega, src, wl.medium.kappa_sq, wl.medium.gamma, tau, gr1, gr2, lap,
                     wl.bc)


def _oracle_upwind_timed(p, tol, maxiter):
    """The reference's timed region of solve_adr_upwind (helmadr/drivers.py:153-165) on the
    oracle restatement: (t_setup = assembly + blend + hierarchy, t_krylov = fgmres, iterations)."""
    from oracle import hadr_oracle as O

    q = O.delta_source(p.n1, p.n2, p.h1, p.h2, p.src)
    qh = O.to_adr(q, p.tau, p.omega).reshape(-1)
    t0 = time.perf_counter()
    H2 = O.adr_of(p, "upwind2")
    H1 = O.adr_of(p, "upwind1")
    B = ((1.0 - 0.25) * H2 + 0.25 * H1).tocsr()
    Hi = O.hierarchy(B, (p.n1, p.n2), 5)
    t1 = time.perf_counter()
    _, rep = O.fgmres(H2, qh, None, O.kcycle_precond(Hi), 5, maxiter, tol)
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1, rep.iterations


def _charged(t_setup, t_kry, its, its_full):
    """Seconds a full solve would take: the sample's setup + its per-iteration cost x the
    full solve's iteration count (setup charged once, as in the GPU arm's solve)."""
    return t_setup + its_full * t_kry / max(its, 1)


def cpu_baseline(wl, args, its_full):
    """The oracle (numpy/scipy restatement of the reference, 1 thread) on this host: one
    bounded sample = assembly + hierarchy + `--cpu-its` outer iterations, charged to the
    full solve's iteration count (the GPU arm's, equal to the reference's within +-1 by the
    parity tests)."""
    from threadpoolctl import threadpool_limits

    p = oracle_problem(wl)
    with threadpool_limits(1):
        ts, tk, its = _oracle_upwind_timed(p, args.tol, args.cpu_its)
    t = _charged(ts, tk, its, its_full)
    N = wl.grid.n_nodes
    return {"value": N * its_full / t / 1e6, "unit": "Mdof*iter/s", "cores": 1, "kind": "port",
            "sample": f"oracle solve_upwind on {wl.name}: assembly + hierarchy ({ts:.1f} s) + {its} outer FGMRES "
                      f"iterations ({tk:.1f} s), charged to a full {its_full}-iteration solve ({t:.1f} s); host "
                      f"cpu_count={os.cpu_count()}, 1 thread (scipy sparse kernels are single-threaded)"}


def run_reference(args, ws, rank, local, dist):
    """The reference's CPU path (the oracle restatement, bit-exact to helmadr on its own
    goldens) on the host cores with all BLAS threads, same workload / config / metric.
    A full solve runs once first (untimed calibration: its iteration count and time); each
    warm-up and timed step is then a bounded sample — assembly + hierarchy + `--ref-its`
    outer iterations — charged to the full solve's iteration count (setup once, per-
    iteration cost x iterations), so one step stands for the same work as a GPU-arm step."""
    if rank != 0:
        return None
    from paper_1712_06091_b200 import workloads

    wl = workloads.by_name(args.workload, args.size)
    N = wl.grid.n_nodes
    p = oracle_problem(wl)
    ts0, tk0, its_full = _oracle_upwind_timed(p, args.tol, args.maxiter)
    for _ in range(args.warmup):
        _oracle_upwind_timed(p, args.tol, args.ref_its)
    charged, walls, samples = [], [], []
    for _ in range(args.steps):
        ts, tk, its = _oracle_upwind_timed(p, args.tol, args.ref_its)
        charged.append(_charged(ts, tk, its, its_full))
        walls.append(ts + tk)
        samples.append([round(ts, 3), round(tk, 3), its])
    value = N * its_full * len(charged) / sum(charged) / 1e6
    cores = os.cpu_count()
    return {
        "impl": "reference",
        "metric": "amplitude solve Mdof*iter/s (FGMRES(5) + K-cycle, ADR upwind blend)",
        "value": value,
        "unit": "Mdof*iter/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": sum(charged) / len(charged) * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "c128",
        "data": "synthetic (seeded config builder: linear-gradient velocity, analytic tau)",
        "config": bench_config(wl, args, ws),
        "run": {"full_solve": {"iterations": its_full, "t_setup_s": ts0, "t_krylov_s": tk0,
                               "value": N * its_full / (ts0 + tk0) / 1e6},
                "samples_setup_krylov_its": samples, "sample_wall_ms": [w * 1e3 for w in walls]},
        "cpu_baseline": {"value": value, "unit": "Mdof*iter/s", "cores": cores, "kind": "port",
                         "sample": f"per step: oracle assembly + hierarchy + {args.ref_its} outer iterations, "
                                   f"charged to the calibration solve's {its_full} iterations (all BLAS threads; "
                                   f"scipy sparse kernels single-threaded)"},
        "e2e": {"value": value, "unit": "Mdof*iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--size", type=int, default=None, help="override the grid size n (parity/debug runs)")
    ap.add_argument("--tol", type=float, default=1e-6)
    ap.add_argument("--maxiter", type=int, default=1000)
    ap.add_argument("--cpu-its", type=int, default=4, help="outer iterations in the cpu_baseline sample")
    ap.add_argument("--ref-its", type=int, default=2, help="outer iterations per reference-arm step sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--extra-3d", type=int, default=513, help="also run BASELINE config 4 at this n (0: skip)")
    ap.add_argument("--steps-3d", type=int, default=2)
    ap.add_argument("--slab-timeout", type=float, default=600.0,
                    help="N > 1: watchdog on the multi-GPU config-4 solve (the headline is printed regardless)")
    ap.add_argument("--extra-cfg3", type=int, default=2049, help="also run BASELINE config 3 at this n (0: skip)")
    ap.add_argument("--extra-cfg5", type=int, default=257,
                    help="also run BASELINE config 5's recipe at this n (0: skip; full size 1025 needs 8 GPUs)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)
    ws, rank, local, dist = dist_init()
    if ws != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={ws} but --gpus {args.gpus}")
    if args.impl == "reference":
        out = run_reference(args, ws, rank, local, dist)
    else:
        out = run_ours(args, ws, rank, local, dist)
    if rank == 0 and out is not None:
        print(json.dumps(out))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
