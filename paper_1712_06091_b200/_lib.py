"""ctypes binding of libhadr.so (include/hadr.h).

The CUDA library is the product path: there is no CPU fallback.  If the
shared object is missing, or no CUDA device is visible when a solver entry
point is first used, this module raises instead of computing anything.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HADR_LIB_PATH") or os.path.join(_HERE, "libhadr.so")

HADR_OK, HADR_EVALUE, HADR_ERUNTIME, HADR_ECUDA = 0, 1, 2, 3

# every symbol include/hadr.h declares (checked by tests/test_lib_abi.py)
EXPORTS = (
    "hadr_last_error", "hadr_init", "hadr_device_sync", "hadr_device_malloc", "hadr_device_free", "hadr_memcpy",
    "hadr_op_from_csr", "hadr_op_from_planes", "hadr_op_info", "hadr_op_export", "hadr_op_apply",
    "hadr_op_jacobi", "hadr_op_axpby", "hadr_op_add_diag", "hadr_op_similarity", "hadr_op_galerkin",
    "hadr_op_destroy", "hadr_transfer", "hadr_hier_create", "hadr_hier_from_ops", "hadr_hier_info",
    "hadr_hier_level_op", "hadr_kcycle", "hadr_precond_apply", "hadr_hier_destroy", "hadr_gmres_relax",
    "hadr_fgmres", "hadr_launch_count", "hadr_assemble", "hadr_solve_adr_upwind", "hadr_pool_trim",
    "hadr_stream_timer", "hadr_set_option", "hadr_ce_profile", "hadr_op_bench",
    "hadr_dist_nccl_id", "hadr_dist_init_nccl", "hadr_dist_init_host", "hadr_dist_finalize", "hadr_dist_info",
    "hadr_dist_plan", "hadr_slab_bounds", "hadr_fast_march", "hadr_phase_transform", "hadr_op_storage",
    "hadr_relative_error", "hadr_memset", "hadr_fgmres_ex",
    "hadr_tau_derivatives", "hadr_ce_bench", "hadr_slab_plan", "hadr_march_plan",
)

# host-communicator callbacks (include/hadr.h hadr_host_*)
HOST_ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_longlong)
HOST_SENDRECV = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_longlong, C.c_int, C.c_void_p, C.c_longlong, C.c_int)
HOST_BCAST = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_longlong, C.c_int)


class HadrReport(C.Structure):
    _fields_ = [
        ("iterations", C.c_int),
        ("converged", C.c_int),
        ("note", C.c_int),
        ("history_len", C.c_int),
        ("bnorm", C.c_double),
        ("final_relres", C.c_double),
        ("wall_time", C.c_double),
        ("device_time", C.c_double),
        ("ortho_max", C.c_double),
    ]


_vp, _i, _d, _i64 = C.c_void_p, C.c_int, C.c_double, C.c_int64
_SIGS = {
    "hadr_last_error": (C.c_char_p, []),
    "hadr_init": (_i, [_i]),
    "hadr_device_sync": (_i, []),
    "hadr_device_malloc": (_i, [C.POINTER(_vp), C.c_size_t]),
    "hadr_device_free": (_i, [_vp]),
    "hadr_memcpy": (_i, [_vp, _vp, C.c_size_t, _i]),
    "hadr_op_from_csr": (_i, [_i, _i, _i, _i64, _vp, _vp, _vp, C.POINTER(_vp)]),
    "hadr_op_from_planes": (_i, [_i, _i, _i, _i, _vp, _vp, C.POINTER(_vp)]),
    "hadr_op_info": (_i, [_vp, C.POINTER(_i), C.POINTER(_i), C.POINTER(_i), C.POINTER(_i), _vp]),
    "hadr_op_export": (_i, [_vp, _vp]),
    "hadr_op_apply": (_i, [_vp, _vp, _vp, _i]),
    "hadr_op_jacobi": (_i, [_vp, _vp, _vp, _i]),
    "hadr_op_axpby": (_i, [_d, _d, _vp, _d, _d, _vp, C.POINTER(_vp)]),
    "hadr_op_add_diag": (_i, [_vp, _d, _d, _vp, C.POINTER(_vp)]),
    "hadr_op_similarity": (_i, [_vp, _vp, _vp, C.POINTER(_vp)]),
    "hadr_op_galerkin": (_i, [_vp, C.POINTER(_vp)]),
    "hadr_op_destroy": (None, [_vp]),
    "hadr_assemble": (_i, [_i, _i, _i, _i, _d, _d, _d, _d, _i, _vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _i,
                           C.POINTER(_vp)]),
    "hadr_solve_adr_upwind": (_i, [_i, _i, _i, _i, _d, _d, _d, _d, _vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp,
                                   _vp, _d, _i, _i, _i, _d, _vp, C.POINTER(HadrReport), _vp, _i, C.POINTER(_d), _i]),
    "hadr_pool_trim": (_i, []),
    "hadr_stream_timer": (_d, [_i]),
    "hadr_set_option": (_i, [C.c_char_p, _d]),
    "hadr_ce_profile": (_i, [_vp, _i]),
    "hadr_op_bench": (_i, [_vp, _vp, _vp, _i, _i, C.POINTER(_d)]),
    "hadr_ce_bench": (_i, [_vp, _i, _i, C.POINTER(_d)]),
    "hadr_transfer": (_i, [_i, _i, _i, _i, _vp, _vp, _i]),
    "hadr_hier_create": (_i, [_vp, _i, _i, _d, C.POINTER(_vp)]),
    "hadr_hier_from_ops": (_i, [_i, _vp, _i, _d, C.POINTER(_vp)]),
    "hadr_hier_info": (_i, [_vp, C.POINTER(_i), _vp]),
    "hadr_hier_level_op": (_i, [_vp, _i, C.POINTER(_vp)]),
    "hadr_kcycle": (_i, [_vp, _i, _vp, _vp, _vp, _vp, _i]),
    "hadr_precond_apply": (_i, [_vp, _vp, _vp, _i]),
    "hadr_hier_destroy": (None, [_vp]),
    "hadr_launch_count": (C.c_longlong, []),
    "hadr_gmres_relax": (_i, [_vp, _vp, _vp, _i, _vp, _i]),
    "hadr_fgmres": (_i, [_vp, _vp, _vp, _vp, _i, _i, _d, _vp, C.POINTER(HadrReport), _vp, _i, _i]),
    "hadr_fgmres_ex": (_i, [_vp, _vp, _vp, _vp, _i, _i, _d, _i, _vp, C.POINTER(HadrReport), _vp, _i, _i]),
    "hadr_dist_nccl_id": (_i, [_vp]),
    "hadr_dist_init_nccl": (_i, [_i, _i, _vp]),
    "hadr_dist_init_host": (_i, [_i, _i, HOST_ALLGATHER, HOST_SENDRECV, HOST_BCAST]),
    "hadr_dist_finalize": (_i, []),
    "hadr_dist_info": (_i, [C.POINTER(_i), C.POINTER(_i), C.POINTER(_i)]),
    "hadr_dist_plan": (_i, [_i, _i, _i, _i, _vp, C.POINTER(_i), C.POINTER(_i)]),
    "hadr_slab_bounds": (_i, [_i, _i, _i, _vp]),
    "hadr_slab_plan": (_i, [_i, _i, _i, _i, _i, _vp, C.POINTER(_i), C.POINTER(_i)]),
    "hadr_march_plan": (_i, [_i, _i, _i, _i, _vp]),
    "hadr_fast_march": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _vp, C.POINTER(C.c_longlong)]),
    "hadr_phase_transform": (_i, [C.c_longlong, _vp, _vp, _d, _i, _vp, _i]),
    "hadr_op_storage": (_i, [_vp, C.POINTER(_i), C.POINTER(C.c_longlong)]),
    "hadr_memset": (_i, [_vp, _i, C.c_size_t]),
    "hadr_tau_derivatives": (_i, [_i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i]),
    "hadr_relative_error": (_i, [C.c_longlong, _vp, _vp, _d, _vp, C.POINTER(_d), C.POINTER(C.c_longlong), _vp, _i,
                                 _vp, _i]),
}

_lib = None
_initialised = False


def load(path: str = LIB_PATH):
    """dlopen libhadr.so and declare signatures (no device needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(make -C paper_1712_06091_b200/csrc). There is no CPU fallback."
        )
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


_device = None  # the CUDA device the library was bound to (hadr_init binds once)


def lib(device=None):
    """The library with a CUDA device initialised (raises if none).  The first call binds the
    device (`device`, else HADR_DEVICE, else 0); a later call that names a different device
    raises instead of silently staying on the first one."""
    global _initialised, _device
    L = load()
    if not _initialised:
        dev = int(device) if device is not None else int(os.environ.get("HADR_DEVICE", "0"))
        check(L.hadr_init(dev))
        _initialised = True
        _device = dev
    elif device is not None and int(device) != _device:
        raise RuntimeError(f"libhadr is already bound to CUDA device {_device}; cannot rebind to {int(device)} "
                           "(call distributed.init() before any other library call)")
    return L


def set_option(name: str, value: float) -> None:
    """Runtime switches of libhadr.so, e.g. set_option("ce_max_n", 0) disables the cluster engine."""
    check(lib().hadr_set_option(name.encode(), float(value)))


def check(code: int) -> None:
    if code == HADR_OK:
        return
    msg = (_lib.hadr_last_error() or b"").decode(errors="replace")
    if code == HADR_EVALUE:
        raise ValueError(msg)
    raise RuntimeError(f"libhadr: {msg}")


def cbuf(a: np.ndarray) -> int:
    """Pointer of a C-contiguous numpy array."""
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def as_c128(v, n: int | None = None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(v, dtype=np.complex128).reshape(-1))
    if n is not None and a.shape[0] != n:
        raise ValueError(f"dimension mismatch: operator {n}, vector {a.shape}")
    return a
