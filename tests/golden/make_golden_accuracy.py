"""Golden vectors for the accuracy workflow and the field-dump format, produced by
the REFERENCE (helmadr.drivers.accuracy_compare, helmadr.grid.relative_error_map,
helmadr.models.write_field) in this container.

    python tests/golden/make_golden_accuracy.py

Writes tests/golden/accuracy.npz: a seeded complex reference field on a 33x17 grid
(with a patch of exact zeros so the floor mask matters), two perturbed solutions,
their error maps and median / p95 / max (default floor and an explicit floor), and
the raw bytes of the reference's field dump + .meta sidecar of one of them.
"""

from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from helmadr import drivers, models  # noqa: E402
from helmadr.grid import GridSpec, relative_error_map  # noqa: E402


def main():
    rng = np.random.default_rng(20171215)
    g = GridSpec(33, 17, 2.0, 1.0)
    u_ref = rng.standard_normal(g.shape) + 1j * rng.standard_normal(g.shape)
    u_ref[3:6, 4:9] = 0.0
    u_ref[10, :] *= 1e-14
    u1 = u_ref * (1 + 1e-3 * rng.standard_normal(g.shape)) + 1e-6 * rng.standard_normal(g.shape)
    u2 = u_ref + 1e-2 * (rng.standard_normal(g.shape) + 1j * rng.standard_normal(g.shape))
    out = {"u_ref": u_ref, "u1": u1, "u2": u2}
    for tag, floor in (("def", None), ("fl", 0.5)):
        res = drivers.accuracy_compare([("u1", u1), ("u2", u2)], u_ref, floor)
        for name in ("u1", "u2"):
            for k in ("median", "p95", "max"):
                out[f"{tag}_{name}_{k}"] = np.float64(res[name][k])
            out[f"{tag}_{name}_map"] = res[name]["error_map"]
    out["map_fl_u1_direct"] = relative_error_map(u1, u_ref, 0.5)
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "u1.bin")
        models.write_field(p, g, u1)
        out["dump_bin"] = np.frombuffer(open(p, "rb").read(), dtype=np.uint8)
        out["dump_meta"] = np.frombuffer(open(p + ".meta", "rb").read(), dtype=np.uint8)
        q = os.path.join(d, "vel.bin")
        models.write_field(q, g, np.abs(u_ref))
        out["dump_real_bin"] = np.frombuffer(open(q, "rb").read(), dtype=np.uint8)
        out["dump_real_meta"] = np.frombuffer(open(q + ".meta", "rb").read(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "accuracy.npz"), **out)


if __name__ == "__main__":
    main()
