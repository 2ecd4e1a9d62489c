"""On-disk formats next to the hot path: splat PLY import
(io.hpp:493-637) and the visibility-field JSON (io.hpp:255-295). Host-only code in
the native library, so these run on CPU."""
import json
import math

import numpy as np
import pytest

from paper_2605_30342_b200 import api
from paper_2605_30342_b200.model import K_Y00, ParameterError, VisibilityField, VmfParams


def write_ply(path, n, rest_per_channel=15, extra_element=False, ascii=False, drop=None, header_extra=""):
    rng = np.random.default_rng(3)
    props = ["x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2"]
    props += [f"f_rest_{i}" for i in range(3 * rest_per_channel)]
    props += ["opacity", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"]
    if drop:
        props = [p for p in props if p != drop]
    data = rng.normal(size=(n, len(props))).astype(np.float32)
    lines = ["ply", f"format {'ascii' if ascii else 'binary_little_endian'} 1.0", "comment test"]
    if extra_element:
        lines += ["element face 2", "property float a"]
    lines += [f"element vertex {n}"] + [f"property float {p}" for p in props]
    if header_extra:
        lines.append(header_extra)
    lines.append("end_header")
    with open(path, "wb") as f:
        f.write(("\n".join(lines) + "\n").encode())
        if extra_element:
            f.write(np.zeros(2, np.float32).tobytes())
        f.write(data.astype("<f4").tobytes())
    return props, data


def test_splat_ply_activations_and_layout(tmp_path):
    path = str(tmp_path / "s.ply")
    props, data = write_ply(path, 7, extra_element=True)
    sc = api.load_splat_ply(path)
    col = {p: data[:, i].astype(np.float64) for i, p in enumerate(props)}
    assert sc.num_particles == 7 and sc.color_degree == 3
    assert np.array_equal(sc.positions, np.stack([col["x"], col["y"], col["z"]], 1).astype(np.float32))
    assert np.allclose(sc.opacities, 1.0 / (1.0 + np.exp(-col["opacity"])), rtol=1e-6)
    assert np.allclose(sc.scales, np.exp(np.stack([col[f"scale_{k}"] for k in range(3)], 1)), rtol=1e-6)
    q = np.stack([col[f"rot_{k}"] for k in range(4)], 1)
    assert np.allclose(sc.rotations, q / np.linalg.norm(q, axis=1, keepdims=True), atol=1e-6)
    for c in range(3):
        assert np.allclose(sc.colors[:, c, 0], col[f"f_dc_{c}"] + 0.5 / K_Y00, rtol=1e-6)  # io.hpp:620
        for k in range(15):
            assert np.array_equal(sc.colors[:, c, 1 + k], data[:, props.index(f"f_rest_{c * 15 + k}")])
    assert np.allclose(sc.bounds_min, sc.positions.min(0)) and np.allclose(sc.bounds_max, sc.positions.max(0))


def test_splat_ply_degree_zero_and_errors(tmp_path):
    p0 = str(tmp_path / "d0.ply")
    write_ply(p0, 3, rest_per_channel=0)
    assert api.load_splat_ply(p0).color_degree == 0
    bad = [dict(ascii=True), dict(drop="rot_2"), dict(rest_per_channel=2), dict(header_extra="bogus line")]
    for i, kw in enumerate(bad):
        p = str(tmp_path / f"bad{i}.ply")
        write_ply(p, 3, **kw)
        with pytest.raises(ParameterError):
            api.load_splat_ply(p)
    trunc = str(tmp_path / "trunc.ply")
    write_ply(trunc, 5)
    raw = open(trunc, "rb").read()
    open(trunc, "wb").write(raw[:-10])
    with pytest.raises(ParameterError):
        api.load_splat_ply(trunc)
    with pytest.raises(ParameterError):
        api.load_splat_ply(str(tmp_path / "missing.ply"))


def test_field_json_round_trip_and_schema(tmp_path):
    rng = np.random.default_rng(5)
    g = rng.normal(size=(6, 9))
    f = VisibilityField(2, VmfParams(1.25), 17, g, np.zeros(0, np.uint8))
    virt = np.array([0, 1, 0, 0, 1, 0], np.uint8)
    path = str(tmp_path / "field.json")
    api.save_field_json(path, f, virt)
    doc = json.load(open(path))
    assert doc["L"] == 2 and doc["kappa"] == 1.25 and doc["num_views"] == 17
    assert len(doc["gamma"]) == 6 and len(doc["gamma"][0]) == 9 and doc["virtual"][1] is True
    back = api.load_field_json(path)
    assert back.degree == 2 and back.num_views == 17 and back.vmf.kappa == 1.25
    assert np.array_equal(back.gamma, g) and np.array_equal(back.virtual_mask, virt)
    bad = dict(doc)
    del bad["virtual"]
    json.dump(bad, open(path, "w"))
    with pytest.raises(ParameterError):
        api.load_field_json(path)
    bad = dict(doc)
    bad["gamma"] = doc["gamma"][:5]
    json.dump(bad, open(path, "w"))
    with pytest.raises(ParameterError):
        api.load_field_json(path)
