"""B200-native amplitude solve of arXiv 1712.06091 (Treister & Haber).

Drop-in for the hot path of the reference package ``helmadr``: flexible GMRES
preconditioned by the geometric-multigrid K-cycle, run as hand-written sm_100a
CUDA kernels in ``libhadr.so`` (C ABI: include/hadr.h) behind a Python API with
the reference's names and semantics.  Importing needs no GPU; the first solver
call initialises the device and raises if the library or the device is missing.
"""

from . import _lib
from .krylov import (KrylovConfig, SolveReport, fgmres, fgmres_device, gmres_relax, jacobi_apply, launch_count,
                     spmv)
from .multigrid import (COARSE_FGMRES_TOL, COARSE_GMRES_STEPS, KCyclePreconditioner, MGHierarchy,
                        build_hierarchy, build_prolongation, coarsenable_levels, galerkin_coarsen,
                        hierarchy_from_ops, k_cycle, make_kcycle_preconditioner)
from .stencil import Prolongation, StencilOperator, as_operator
from .accuracy import accuracy_compare, read_field, read_meta, relative_error_map, write_field, write_meta

__all__ = [
    "KrylovConfig", "SolveReport", "fgmres", "fgmres_device", "gmres_relax", "jacobi_apply", "spmv", "launch_count",
    "COARSE_FGMRES_TOL", "COARSE_GMRES_STEPS", "KCyclePreconditioner", "MGHierarchy", "build_hierarchy",
    "build_prolongation", "coarsenable_levels", "galerkin_coarsen", "hierarchy_from_ops", "k_cycle",
    "make_kcycle_preconditioner", "Prolongation", "StencilOperator", "as_operator",
    "accuracy_compare", "read_field", "read_meta", "relative_error_map", "write_field", "write_meta",
]
