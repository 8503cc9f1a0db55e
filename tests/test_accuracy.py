"""Field dumps and the accuracy workflow.

CPU: the oracle restatement against the reference's own outputs
(tests/golden/make_golden_accuracy.py), the dump format byte for byte, round
trips and errors.  GPU: the device error map / masked statistics
(hadr_relative_error) against the golden vectors.  Tolerance: the device |z| is
CUDA's hypot (<= 1 ulp from glibc's), so maps and statistics agree to 4 ulp
relative (rtol 1e-15); the masks are identical on these inputs.
"""

import os

import numpy as np
import pytest

from conftest import load_golden


@pytest.fixture(scope="module")
def acc():
    return load_golden("accuracy")


def _stats_of(g, tag, name):
    return {k: float(g[f"{tag}_{name}_{k}"]) for k in ("median", "p95", "max")}


def test_oracle_accuracy_bitexact(acc):
    from oracle import hadr_oracle as O

    for tag, floor in (("def", None), ("fl", 0.5)):
        res = O.compare([("u1", acc["u1"]), ("u2", acc["u2"])], acc["u_ref"], floor)
        for name in ("u1", "u2"):
            assert {k: res[name][k] for k in ("median", "p95", "max")} == _stats_of(acc, tag, name)
            assert np.array_equal(res[name]["error_map"], acc[f"{tag}_{name}_map"])
    assert O.dump_bytes(acc["u1"]) == bytes(acc["dump_bin"])


def test_field_dump_format(acc, tmp_path):
    from paper_1712_06091_b200 import accuracy
    from paper_1712_06091_b200.fields import GridSpec, GridSpec3

    g = GridSpec(33, 17, 2.0, 1.0)
    p = str(tmp_path / "u1.bin")
    accuracy.write_field(p, g, acc["u1"])
    assert open(p, "rb").read() == bytes(acc["dump_bin"])
    assert open(p + ".meta", "rb").read() == bytes(acc["dump_meta"])
    q = str(tmp_path / "v.bin")
    accuracy.write_field(q, g, np.abs(acc["u_ref"]))
    assert open(q, "rb").read() == bytes(acc["dump_real_bin"])
    assert open(q + ".meta", "rb").read() == bytes(acc["dump_real_meta"])
    v, g2 = accuracy.read_field(p)
    assert g2 == g and np.array_equal(v, acc["u1"])
    # 3D extension: n3 / L3 sidecar lines, round trip
    g3 = GridSpec3(5, 6, 7, 1.0, 1.0, 0.5)
    w = np.random.default_rng(1).standard_normal(g3.shape) * (1 + 1j)
    r = str(tmp_path / "w.bin")
    accuracy.write_field(r, g3, w)
    w2, g4 = accuracy.read_field(r)
    assert g4 == g3 and np.array_equal(w2, w)
    with pytest.raises(ValueError):
        accuracy.write_field(r, g, w)
    with open(r, "ab") as fh:
        fh.write(b"\0" * 8)
    with pytest.raises(ValueError):
        accuracy.read_field(r)
    assert os.path.exists(r + ".meta")


@pytest.mark.gpu
def test_device_accuracy_compare(acc):
    from paper_1712_06091_b200 import accuracy

    for tag, floor in (("def", None), ("fl", 0.5)):
        res = accuracy.accuracy_compare([("u1", acc["u1"]), ("u2", acc["u2"])], acc["u_ref"], floor)
        for name in ("u1", "u2"):
            want = _stats_of(acc, tag, name)
            for k in ("median", "p95", "max"):
                assert res[name][k] == pytest.approx(want[k], rel=1e-15, abs=0), (tag, name, k)
            np.testing.assert_allclose(res[name]["error_map"], acc[f"{tag}_{name}_map"], rtol=1e-15, atol=0)
    m = accuracy.relative_error_map(acc["u1"], acc["u_ref"], 0.5)
    np.testing.assert_allclose(m, acc["map_fl_u1_direct"], rtol=1e-15, atol=0)
    with pytest.raises(ValueError):
        accuracy.relative_error_map(acc["u1"][:-1], acc["u_ref"])
    with pytest.raises(ValueError):
        accuracy.relative_error_map(acc["u1"], acc["u_ref"], -1.0)
    # odd / even mask sizes exercise both median branches
    for n in (101, 100):
        rng = np.random.default_rng(n)
        ur = rng.standard_normal(n) + 1j
        u = ur + 1e-3 * rng.standard_normal(n)
        r = accuracy.accuracy_compare([("u", u)], ur)["u"]
        e = np.abs(u - ur) / np.abs(ur)
        assert r["median"] == pytest.approx(float(np.median(e)), rel=1e-15)
        assert r["p95"] == pytest.approx(float(np.percentile(e, 95)), rel=1e-15)
