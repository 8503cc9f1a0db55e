"""Field dumps and the accuracy workflow.

* ``write_field`` / ``read_field`` / ``write_meta`` / ``read_meta``: the reference's
  wire format for nodal fields (helmadr/models.py:76-120): a headerless
  little-endian float64 file, row-major in the solver's point order (depth
  fastest), complex fields as interleaved (re, im) pairs, plus a ``<path>.meta``
  ASCII sidecar of ``key=value`` lines (n1, n2, L1, L2, complex).  3D grids add
  ``n3`` / ``L3`` lines (this build's extension; a 2D sidecar is byte-identical
  to the reference's).  Amplitudes exchanged with the reference go through it.
* ``relative_error_map`` (helmadr/grid.py:175-191) and ``accuracy_compare``
  (helmadr/drivers.py:176-196) run on the device through ``hadr_relative_error``:
  one streaming pass for the map, a device compaction + radix sort of the
  masked errors, and numpy's own median / linear-percentile arithmetic on the
  few order statistics read back.  Same errors as the reference (grid mismatch,
  negative floor).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .fields import GridSpec, GridSpec3


def _meta_path(path: str) -> str:
    return path if path.endswith(".meta") else path + ".meta"


def write_meta(path: str, grid, complex_: bool) -> None:
    lines = [f"n1={grid.n1}", f"n2={grid.n2}"]
    if getattr(grid, "dim", 2) == 3:
        lines.append(f"n3={grid.n3}")
    lines += [f"L1={grid.L1!r}", f"L2={grid.L2!r}"]
    if getattr(grid, "dim", 2) == 3:
        lines.append(f"L3={grid.L3!r}")
    lines.append(f"complex={'true' if complex_ else 'false'}")
    with open(_meta_path(path), "w", encoding="ascii") as fh:
        fh.write("\n".join(lines) + "\n")


def read_meta(path: str):
    kv = {}
    with open(_meta_path(path), encoding="ascii") as fh:
        for line in fh:
            line = line.strip()
            if line:
                key, _, value = line.partition("=")
                kv[key.strip()] = value.strip()
    if "n3" in kv:
        grid = GridSpec3(int(kv["n1"]), int(kv["n2"]), int(kv["n3"]), float(kv["L1"]), float(kv["L2"]),
                         float(kv["L3"]))
    else:
        grid = GridSpec(int(kv["n1"]), int(kv["n2"]), float(kv["L1"]), float(kv["L2"]))
    return grid, kv.get("complex", "false").lower() == "true"


def write_field(path: str, grid, values) -> None:
    """Dump a nodal field with its .meta sidecar (complex: interleaved re/im)."""
    values = np.asarray(values)
    if values.shape != tuple(grid.shape):
        raise ValueError(f"field shape {values.shape} does not match grid {tuple(grid.shape)}")
    cplx = np.iscomplexobj(values)
    if cplx:
        # complex128 memory already is the interleaved (re, im) float64 stream
        flat = np.ascontiguousarray(values, dtype=np.complex128).reshape(-1).view(np.float64)
    else:
        flat = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
    flat.astype("<f8", copy=False).tofile(path)
    write_meta(path, grid, cplx)


def read_field(path: str):
    grid, cplx = read_meta(path)
    flat = np.fromfile(path, dtype="<f8")
    n = grid.n_nodes
    want = 2 * n if cplx else n
    if flat.size != want:
        raise ValueError(f"field file {path!r} holds {flat.size} floats, expected {want}")
    if cplx:
        values = flat.astype(np.float64, copy=False).view(np.complex128).reshape(grid.shape).copy()
    else:
        values = flat.reshape(grid.shape)
    return values, grid


def _device_errors(u, u_ref, floor, want_map: bool, order_idx=()):
    u = np.asarray(u)
    u_ref = np.asarray(u_ref)
    if u.shape != u_ref.shape:
        raise ValueError(f"grid mismatch: {u.shape} vs {u_ref.shape}")
    if floor is not None and floor < 0:
        raise ValueError("floor must be non-negative")
    uc = _lib.as_c128(u)
    rc = _lib.as_c128(u_ref)
    n = uc.size
    err = np.empty(n, dtype=np.float64) if want_map else None
    idx = np.ascontiguousarray(order_idx, dtype=np.int64)
    vals = np.zeros(max(idx.size, 1), dtype=np.float64)
    used, count = C.c_double(), C.c_longlong()
    L = _lib.lib()
    _lib.check(L.hadr_relative_error(n, _lib.cbuf(uc), _lib.cbuf(rc), -1.0 if floor is None else float(floor),
                                     _lib.cbuf(err) if err is not None else None, C.byref(used), C.byref(count),
                                     _lib.cbuf(idx) if idx.size else None, int(idx.size), _lib.cbuf(vals), 0))
    return (None if err is None else err.reshape(u.shape)), used.value, count.value, vals[: idx.size]


def relative_error_map(u, u_ref, floor: float | None = None) -> np.ndarray:
    """|u - u_ref| / |u_ref|, with |u_ref| < floor replaced by floor (default
    1e-12 * max|u_ref|)."""
    err, _, _, _ = _device_errors(u, u_ref, floor, True)
    return err


def _percentile_linear(lo: float, hi: float, gamma: float) -> float:
    # numpy's _lerp (method 'linear'): a + (b - a) t, or b - (b - a)(1 - t) for t >= 0.5
    d = np.float64(hi) - np.float64(lo)
    if gamma >= 0.5:
        return float(np.float64(hi) - d * (1.0 - gamma))
    return float(np.float64(lo) + d * gamma)


def _stats(u, u_ref, floor):
    # the masked count first decides which order statistics numpy's median and p95 read
    _, used, m, _ = _device_errors(u, u_ref, floor, False)
    if m == 0:
        raise ValueError("no reference values above the floor")
    vi = np.float64(0.95) * np.float64(m - 1)  # numpy virtual index for q = 95 / 100
    lo = int(np.floor(vi))
    gamma = float(vi - lo)
    mid = [(m - 1) // 2, m // 2]
    idx = mid + [lo, min(lo + 1, m - 1), m - 1]
    err, _, m2, v = _device_errors(u, u_ref, floor, True, idx)
    assert m2 == m
    median = float(v[0]) if m % 2 else float((np.float64(v[0]) + np.float64(v[1])) / 2.0)
    return err, median, _percentile_linear(v[2], v[3], gamma), float(v[4])


def accuracy_compare(solutions, u_ref, floor: float | None = None) -> dict:
    """Per-solution relative-error maps and their median / 95th percentile / max over
    the nodes where |u_ref| >= floor (default 1e-12 * max|u_ref|)."""
    out = {}
    for name, u in solutions:
        err, median, p95, mx = _stats(u, u_ref, floor)
        out[name] = {"median": median, "p95": p95, "max": mx, "error_map": err}
    return out


__all__ = ["write_meta", "read_meta", "write_field", "read_field", "relative_error_map", "accuracy_compare"]
