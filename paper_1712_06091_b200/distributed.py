"""Multi-GPU slab decomposition of the amplitude solve.

The reference (helmadr) is a single-process CPU package; this module adds the
data-parallel layout the build targets: one process per GPU, the fine grid and
the larger coarse levels split into axis-0 slabs (halo exchange per stencil,
one all-gather of 4 doubles per Krylov reduction), the small coarse levels
agglomerated (replicated on every rank).  After :func:`init`, the public
drivers (``drivers.solve_adr_upwind``) run collectively and return the global
amplitude on every rank.

Backends
--------
* ``"nccl"``  one GPU per rank (``LOCAL_RANK`` selects it); the communicator
  is NCCL, opened by libhadr itself (the torch process group, of any backend,
  only carries the unique id), and the exchanges are captured in the K-cycle
  CUDA graph.
* ``"host"``  blocking host callbacks over a ``torch.distributed`` process
  group (gloo).  Ranks may share one GPU — nothing on the device waits for
  another rank — which is how the multi-rank path is tested on a 1-GPU box.
"""

from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

from . import _lib

_keep = []  # ctypes callbacks must outlive the communicator


def _u8(ptr: int, n: int):
    import torch

    if n <= 0:
        return torch.empty(0, dtype=torch.uint8)
    return torch.from_numpy(np.ctypeslib.as_array((C.c_uint8 * n).from_address(ptr)))


def _host_callbacks(group=None):
    import torch
    import torch.distributed as dist

    size = dist.get_world_size(group)

    def allgather(send, recv, nbytes):
        try:
            t = _u8(send, nbytes).clone()
            out = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(size)]
            dist.all_gather(out, t, group=group)
            for r in range(size):
                C.memmove(recv + r * nbytes, out[r].data_ptr(), nbytes)
            return 0
        except Exception as e:  # noqa: BLE001 - reported through the C return code
            print(f"hadr host allgather failed: {e!r}", file=sys.stderr)
            return 1

    def sendrecv(send, sbytes, dst, recv, rbytes, src):
        try:
            reqs = []
            if dst >= 0 and sbytes > 0:
                reqs.append(dist.isend(_u8(send, sbytes).clone(), dst, group=group))
            if src >= 0 and rbytes > 0:
                reqs.append(dist.irecv(_u8(recv, rbytes), src, group=group))
            for q in reqs:
                q.wait()
            return 0
        except Exception as e:  # noqa: BLE001
            print(f"hadr host sendrecv failed: {e!r}", file=sys.stderr)
            return 1

    def bcast(buf, nbytes, root):
        try:
            dist.broadcast(_u8(buf, nbytes), src=root, group=group)
            return 0
        except Exception as e:  # noqa: BLE001
            print(f"hadr host bcast failed: {e!r}", file=sys.stderr)
            return 1

    return (_lib.HOST_ALLGATHER(allgather), _lib.HOST_SENDRECV(sendrecv), _lib.HOST_BCAST(bcast))


def init(backend: str = "auto", group=None) -> str:
    """Attach libhadr to the initialised ``torch.distributed`` process group.

    backend "auto": NCCL when every rank can have its own GPU, else host callbacks.
    Returns the backend used.
    """
    import torch
    import torch.distributed as dist

    if not dist.is_initialized():
        raise RuntimeError("torch.distributed is not initialised")
    rank, size = dist.get_rank(group), dist.get_world_size(group)
    if backend == "auto":
        ndev = torch.cuda.device_count() if torch.cuda.is_available() else 0
        backend = "nccl" if ndev >= size else "host"
    if backend == "nccl":
        local = int(os.environ.get("LOCAL_RANK", rank))
        dev = int(os.environ.get("HADR_DEVICE", local))
        L = _lib.lib(dev)  # binds the device now; raises if the library already sits on another one
        uid = C.create_string_buffer(128)
        if rank == 0:
            _lib.check(L.hadr_dist_nccl_id(uid))
        obj = [bytes(uid.raw) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        uid = C.create_string_buffer(obj[0], 128)
        _lib.check(L.hadr_dist_init_nccl(rank, size, uid))
    elif backend == "host":
        L = _lib.lib()
        cbs = _host_callbacks(group)
        _keep.append(cbs)
        _lib.check(L.hadr_dist_init_host(rank, size, *cbs))
    else:
        raise ValueError(f"unknown backend {backend!r}")
    return backend


def finalize() -> None:
    _lib.check(_lib.lib().hadr_dist_finalize())


def info() -> tuple[int, int, str]:
    """(rank, size, backend) of the active communicator ("none" when single-process)."""
    r, s, k = C.c_int(), C.c_int(), C.c_int()
    _lib.load().hadr_dist_info(C.byref(r), C.byref(s), C.byref(k))
    return r.value, s.value, {0: "none", 1: "nccl", 2: "host"}[k.value]


def plan(shape, levels: int = 5):
    """Slab plan of a global grid under the active communicator: (bounds, n_dist_levels, n_levels)."""
    n1, n2 = int(shape[0]), int(shape[1])
    n3 = int(shape[2]) if len(shape) > 2 else 1
    _, size, _ = info()
    b = np.zeros(size + 1, dtype=np.int32)
    nd, nl = C.c_int(), C.c_int()
    _lib.check(_lib.lib().hadr_dist_plan(n1, n2, n3, int(levels), b.ctypes.data, C.byref(nd), C.byref(nl)))
    return b.tolist(), nd.value, nl.value


def slab_bounds(n1: int, size: int, align: int = 1) -> list[int]:
    """Split n1 planes into `size` slabs with interior boundaries multiples of `align` (host only)."""
    b = np.zeros(size + 1, dtype=np.int32)
    _lib.check(_lib.load().hadr_slab_bounds(int(n1), int(size), int(align), b.ctypes.data))
    return b.tolist()


def set_policy(min_planes: int | None = None, levels: int | None = None) -> None:
    """Slab-level policy: keep a coarse level distributed while every slab has >= min_planes planes;
    levels > 0 forces exactly that many distributed levels (0 restores the plane rule)."""
    if min_planes is not None:
        _lib.set_option("dist_min_planes", min_planes)
    if levels is not None:
        _lib.set_option("dist_levels", levels)


def plan_for(shape, levels: int = 5, size: int = 1):
    """The slab plan ``plan`` would make with ``size`` ranks (host logic, no device):
    (bounds, n_dist_levels, n_levels).  Coarse levels whose split saves less per step than
    a collective costs (points x planes < 8e6 x R/(R-1)) or that would keep fewer than
    dist_min_planes (16) planes per slab are agglomerated (replicated)."""
    n1, n2 = int(shape[0]), int(shape[1])
    n3 = int(shape[2]) if len(shape) > 2 else 1
    b = np.zeros(size + 1, dtype=np.int32)
    nd, nl = C.c_int(), C.c_int()
    _lib.check(_lib.load().hadr_slab_plan(n1, n2, n3, int(levels), int(size), b.ctypes.data, C.byref(nd),
                                          C.byref(nl)))
    return [int(x) for x in b], nd.value, nl.value
