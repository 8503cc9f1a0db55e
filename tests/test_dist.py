"""Multi-process (world_size 2, gloo on 127.0.0.1) coverage of the N>1 host
logic: max/sum-over-ranks timing reductions used by bench.py, and the
reference arm under torchrun (rank 0 runs and prints, rank 1 exits 0)."""

import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import REPO


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, REPO)
    import bench

    dist.init_process_group("gloo", rank=rank, world_size=world)
    mx = bench.max_over_ranks(1.0 + rank, dist)
    sm = bench.sum_over_ranks(10.0 * (rank + 1), dist)
    q.put((rank, mx, sm))
    dist.destroy_process_group()


def test_rank_reductions_gloo():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [2.0, 2.0]      # max over ranks
    assert [r[2] for r in res] == [30.0, 30.0]    # sum over ranks


def test_reference_arm_under_torchrun():
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--impl", "reference",
           "--gpus", "2", "--size", "33", "--steps", "1", "--warmup", "0", "--ref-its", "2"]
    out = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    rec = json.loads(lines[0])
    assert rec["impl"] == "reference" and rec["n_gpus"] == 2 and rec["value"] > 0
    assert rec["e2e"]["h2d_bytes_per_step"] == 0


def test_bench_gpus_flag_self_launches():
    """`python bench.py --gpus 2` without torchrun re-launches itself as 2 ranks (one JSON
    line from rank 0 with n_gpus 2); a WORLD_SIZE that contradicts --gpus is refused."""
    cmd = [sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--size", "33", "--steps", "1",
           "--warmup", "0", "--ref-its", "2"]
    out = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1 and json.loads(lines[0])["n_gpus"] == 2
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    bad = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=120, env=env)
    assert bad.returncode != 0 and "WORLD_SIZE" in (bad.stderr + bad.stdout)


# ---------------------------------------------------------------------------
# multi-GPU slab decomposition: host logic (no device)
# ---------------------------------------------------------------------------
def test_slab_bounds():
    sys.path.insert(0, REPO)
    from paper_1712_06091_b200 import distributed as D

    for n1, size, align in [(513, 8, 8), (513, 2, 16), (33, 2, 8), (1025, 4, 8), (65, 3, 4), (257, 8, 1)]:
        b = D.slab_bounds(n1, size, align)
        assert len(b) == size + 1 and b[0] == 0 and b[-1] == n1
        assert all(b[r] % align == 0 for r in range(size))
        assert all(b[r + 1] > b[r] for r in range(size))
        # nested coarse slabs: level l owns [b >> l) with the same rank order
        for l in range(1, max(1, align.bit_length() - 1) + 1):
            bl = [x >> l for x in b[:-1]] + [(n1 - 1) // (1 << l) + 1]
            assert all(bl[r + 1] >= bl[r] for r in range(size))
    assert D.slab_bounds(33, 2, 8) == [0, 16, 33]
    with pytest.raises(ValueError):
        D.slab_bounds(9, 8, 8)


def _comm_worker(rank, world, port, q):
    import ctypes as C

    import numpy as np
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, REPO)
    from paper_1712_06091_b200 import distributed as D

    dist.init_process_group("gloo", rank=rank, world_size=world)
    ag, sr, bc = D._host_callbacks()
    out = {}
    # allgather: recv = every rank's bytes in rank order
    send = (C.c_double * 4)(*[rank * 10.0 + q for q in range(4)])
    recv = (C.c_double * (4 * world))()
    assert ag(C.addressof(send), C.addressof(recv), 32) == 0
    out["allgather"] = list(recv)
    # the halo exchange's two sendrecv phases (Comm::halo): first planes down / last planes up
    lo, hi = (rank - 1 if rank > 0 else -1), (rank + 1 if rank < world - 1 else -1)
    first = (C.c_double * 2)(rank + 0.25, rank + 0.5)
    last = (C.c_double * 2)(rank + 0.75, rank + 0.875)
    above = (C.c_double * 2)(-1.0, -1.0)
    below = (C.c_double * 2)(-1.0, -1.0)
    assert sr(C.addressof(first), 16 if lo >= 0 else 0, lo, C.addressof(above), 16 if hi >= 0 else 0, hi) == 0
    assert sr(C.addressof(last), 16 if hi >= 0 else 0, hi, C.addressof(below), 16 if lo >= 0 else 0, lo) == 0
    out["above"], out["below"] = list(above), list(below)
    # bcast from the last rank
    buf = (C.c_double * 3)(*([7.0, 8.0, 9.0] if rank == world - 1 else [0.0, 0.0, 0.0]))
    assert bc(C.addressof(buf), 24, world - 1) == 0
    out["bcast"] = list(buf)
    q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_host_communicator_callbacks_gloo(world):
    """The gloo host callbacks libhadr's host communicator calls (dist.h kind 2)."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_comm_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=180) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect_ag = [r * 10.0 + k for r in range(world) for k in range(4)]
    for r in range(world):
        o = res[r]
        assert o["allgather"] == expect_ag
        assert o["above"] == ([r + 1 + 0.25, r + 1 + 0.5] if r < world - 1 else [-1.0, -1.0])
        assert o["below"] == ([r - 1 + 0.75, r - 1 + 0.875] if r > 0 else [-1.0, -1.0])
        assert o["bcast"] == [7.0, 8.0, 9.0]


def test_bench_slab_watchdog_prints_headline():
    """bench.py's multi-GPU config-4 line runs under a watchdog: if the slab solve stalls,
    rank 0 still prints the JSON line measured so far (with the stall recorded) and the
    process exits 0; an exception is recorded instead of propagating."""
    import json
    import subprocess

    code = ("import sys, time; sys.path.insert(0, %r); import bench; "
            "bench.guarded_slab_run(lambda: time.sleep(30), {'metric': 'm', 'value': 1.0}, 2, 0, 1.0)") % REPO
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stderr
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["value"] == 1.0 and "error" in line["config_4_3d"]
    sys.path.insert(0, REPO)
    import bench

    def boom():
        raise RuntimeError("nccl")

    assert "nccl" in bench.guarded_slab_run(boom, {}, 2, 0, 60.0)["error"]


def test_slab_plan_agglomerates_small_levels():
    """SURVEY.md §8(e) with the cost model of DESIGN.md §7: split the levels whose per-step
    bytes saved exceed a collective's cost, agglomerate (replicate) the rest — config 4
    (513^2 x 257): 513^2x257, 257^2x129 and 129^2x65 split, 65^2x33 down replicated at 2, 4
    and 8 ranks; config 5 (1025^2 x 513): four levels split at 8 ranks."""
    sys.path.insert(0, REPO)
    from paper_1712_06091_b200 import distributed as D

    for R in (2, 4, 8):
        b, nd, nl = D.plan_for((513, 513, 257), 5, R)
        assert nl == 5 and nd == 3, (R, nd)
        assert b[0] == 0 and b[-1] == 513 and len(b) == R + 1
        assert all((x % 8) == 0 for x in b[:-1])  # slabs nest on the 3 split levels
    b, nd, nl = D.plan_for((1025, 1025, 513), 5, 8)
    assert (nd, nl) == (4, 5)
    b, nd, nl = D.plan_for((65, 65, 33), 5, 2)  # coarse levels too small to pay for a split
    assert nd == 1
