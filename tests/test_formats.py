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
    # ragged rows with the right total are still rejected row by row (io.hpp:290)
    bad = dict(doc)
    bad["gamma"] = [doc["gamma"][0][:8], doc["gamma"][1] + [0.5]] + doc["gamma"][2:]
    json.dump(bad, open(path, "w"))
    with pytest.raises(ParameterError, match="row"):
        api.load_field_json(path)


# ---- ports of the reference's io tests (R/tests/test_io.cpp) -----------------
REQ = ["x", "y", "z", "opacity", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3",
       "f_dc_0", "f_dc_1", "f_dc_2"]


def splat_ply(path, vertices, n_rest=0, fmt="binary_little_endian", leading=b"", leading_header=""):
    """Minimal splat PLY in the reference fixture's property order (test_io.cpp:49-65)."""
    head = f"ply\nformat {fmt} 1.0\n{leading_header}element vertex {len(vertices)}\n"
    head += "".join(f"property float {n}\n" for n in REQ)
    head += "".join(f"property float f_rest_{i}\n" for i in range(n_rest))
    head += "end_header\n"
    body = b"".join(np.asarray(v, "<f4").tobytes() for v in vertices)
    with open(path, "wb") as f:
        f.write(head.encode() + leading + body)


def vertex(x, y, z):
    """opacity logit 0, log-scale 0, identity quaternion, zero DC (test_io.cpp:67-70)."""
    return [x, y, z, 0, 0, 0, 0, 1, 0, 0, 0, 0, 0, 0]


def test_ref_splat_ply_standard_activations(tmp_path):
    """test_io.cpp:321-368"""
    path = str(tmp_path / "splats.ply")
    v = [vertex(0.125, -2.5, 3.75), vertex(1.0, 2.0, 3.0), vertex(-0.5, 0.25, 9.0)]
    v[1][3] = 2.0    # opacity logit
    v[1][4] = -1.0   # log scale x
    v[1][7] = 0.0    # quaternion (0, 2, 0, 0): renormalised
    v[1][8] = 2.0
    v[2][11] = 0.5   # red DC
    splat_ply(path, v)
    sc = api.load_splat_ply(path)
    assert sc.num_particles == 3 and sc.color_degree == 0
    assert list(sc.positions[0]) == [0.125, -2.5, 3.75]          # bit-exact
    assert sc.opacities[0] == pytest.approx(0.5, rel=1e-12)
    assert sc.opacities[1] == pytest.approx(1.0 / (1.0 + math.exp(-2.0)), rel=1e-7)
    assert sc.scales[0, 0] == pytest.approx(1.0, rel=1e-12)
    assert sc.scales[1, 0] == pytest.approx(math.exp(-1.0), rel=1e-7)
    assert float(np.linalg.norm(sc.rotations[1].astype(np.float64))) == pytest.approx(1.0, rel=1e-7)
    assert list(sc.rotations[1]) == [0.0, 1.0, 0.0, 0.0]
    # zero DC decodes to mid-grey, the offset folded into the coefficient (io.hpp:620)
    assert K_Y00 * float(sc.colors[0, 0, 0]) == pytest.approx(0.5, rel=1e-7)
    assert K_Y00 * float(sc.colors[2, 0, 0]) == pytest.approx(0.5 + K_Y00 * 0.5, rel=1e-6)
    assert sc.bounds_min[0] == -0.5 and sc.bounds_max[2] == 9.0


def test_ref_splat_ply_f_rest_channel_major(tmp_path):
    """test_io.cpp:370-384"""
    path = str(tmp_path / "rest.ply")
    v = vertex(0, 0, 1) + [0.1 * (i + 1) for i in range(9)]
    splat_ply(path, [v], n_rest=9)
    sc = api.load_splat_ply(path)
    assert sc.num_particles == 1 and sc.color_degree == 1
    for c in range(3):
        for k in range(3):
            assert float(sc.colors[0, c, 1 + k]) == pytest.approx(0.1 * (3 * c + k + 1), rel=1e-6)


def test_ref_splat_ply_rejects_malformed_inputs_by_name(tmp_path):
    """test_io.cpp:386-434: the messages name what is wrong."""
    path = str(tmp_path / "missing_prop.ply")
    head = "ply\nformat binary_little_endian 1.0\nelement vertex 0\n"
    head += "".join(f"property float {n}\n" for n in REQ if n != "opacity") + "end_header\n"
    open(path, "w").write(head)
    with pytest.raises(ParameterError, match="'opacity'"):
        api.load_splat_ply(path)
    path = str(tmp_path / "ascii.ply")
    splat_ply(path, [], fmt="ascii")
    with pytest.raises(ParameterError, match="ASCII"):
        api.load_splat_ply(path)
    path = str(tmp_path / "nan.ply")
    v = [vertex(0, 0, 0), vertex(1, 1, 1)]
    v[1][0] = float("nan")
    splat_ply(path, v)
    with pytest.raises(ParameterError) as e:
        api.load_splat_ply(path)
    assert "vertex 1" in str(e.value) and "'x'" in str(e.value)
    path = str(tmp_path / "bad_rest.ply")
    splat_ply(path, [vertex(0, 0, 0) + [0.0] * 6], n_rest=6)
    with pytest.raises(ParameterError):
        api.load_splat_ply(path)
    path = str(tmp_path / "not_a.ply")
    open(path, "w").write("OFF\n0 0 0\n")
    with pytest.raises(ParameterError):
        api.load_splat_ply(path)


def test_ref_splat_ply_skips_unknown_leading_elements(tmp_path):
    """test_io.cpp:436-455"""
    path = str(tmp_path / "extra_element.ply")
    splat_ply(path, [vertex(1, 2, 3)], leading_header="element camera 2\nproperty float cx\n",
              leading=np.array([7.0, 8.0], "<f4").tobytes())
    sc = api.load_splat_ply(path)
    assert sc.num_particles == 1 and sc.positions[0, 2] == 3.0


@pytest.mark.gpu
def test_ref_field_json_round_trip_preserves_queries(tmp_path):
    """test_io.cpp:191-221: a device-built field saved and re-loaded keeps its
    coefficients bit for bit, its metadata, the virtual mask and its queries."""
    from paper_2605_30342_b200.model import Scene, make_lookat
    parts = [dict(pos=(x, 1.0, 1.0), scale=0.05, opacity=0.6, color_sh=[[0.5 / K_Y00]] * 3) for x in (0.8, 1.2)]
    parts[1]["virtual"] = True
    parts[1]["opacity"] = 0.0
    sc = Scene.from_particles(parts, 0, bounds=((0, 0, 0), (2, 2, 2)))
    cam = make_lookat((0.2, 1.0, 1.0), (2.0, 1.0, 1.0))
    with api.Context(0) as ctx:
        ds = ctx.upload(sc)
        f = api.construct_field(ctx, ds, [cam], VmfParams(1.3), 2)
        host = f.download()
        path = str(tmp_path / "field.json")
        api.save_field_json(path, host, sc.is_virtual)
        back = api.load_field_json(path)
        assert back.degree == 2 and back.num_views == 1 and back.vmf.kappa == 1.3
        assert np.array_equal(back.virtual_mask, sc.is_virtual.astype(np.uint8))
        assert np.array_equal(back.gamma, host.gamma)
        assert np.any(host.gamma[0] != 0) and not np.any(host.gamma[1])
        f2 = api.upload_field(ctx, ds, back)
        d = np.array([1.0, 0.2, -0.1])
        d /= np.linalg.norm(d)
        q1 = api.query_visibility(ctx, f, [0, 1], [d, d])
        q2 = api.query_visibility(ctx, f2, [0, 1], [d, d])
        assert np.array_equal(q1, q2) and q1[1] == 0.0
