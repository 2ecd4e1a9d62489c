"""ctypes front-end of the CPU ORACLE (liboracle.so). TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module. The product path
(paper_2605_30342_b200) never does.

Every function mirrors one reference entry point (file:line in
gavis_oracle.c). The scene is fed in double: parity runs pass the exact fp32
values the CUDA path consumes.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


class Camera(C.Structure):
    _fields_ = [("rotation", C.c_double * 9), ("position", C.c_double * 3), ("width", C.c_int32),
                ("height", C.c_int32), ("fov_h", C.c_double), ("fov_v", C.c_double),
                ("near_plane", C.c_double)]


class Raster(C.Structure):
    _fields_ = [("tile_size", C.c_int32), ("_pad", C.c_int32), ("transmittance_cutoff", C.c_double),
                ("dilation", C.c_double), ("alpha_clamp_max", C.c_double)]


class Unc(C.Structure):
    _fields_ = [("beta", C.c_double), ("prior_opacity", C.c_double), ("color_sigma", C.c_double),
                ("prior_cov", C.c_double * 9), ("variance_provider", C.c_int32),
                ("correlation", C.c_int32), ("correlation_lambda", C.c_double)]


class SceneC(C.Structure):
    _fields_ = [("num_particles", C.c_int64), ("color_degree", C.c_int32), ("_pad", C.c_int32),
                ("positions", C.c_void_p), ("rotations", C.c_void_p), ("scales", C.c_void_p),
                ("opacities", C.c_void_p), ("colors", C.c_void_p), ("is_virtual", C.c_void_p)]


class Splat(C.Structure):
    _fields_ = [("particle_index", C.c_int32), ("_pad", C.c_int32), ("mean_x", C.c_double),
                ("mean_y", C.c_double), ("conic_a", C.c_double), ("conic_b", C.c_double),
                ("conic_c", C.c_double), ("depth", C.c_double), ("radius", C.c_double),
                ("opacity", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.gor_bessel_i.restype = C.c_double
        _lib.gor_query_visibility.restype = C.c_double
        _lib.gor_image_entropy.restype = C.c_double
        _lib.gor_raymarch_transmittance.restype = C.c_double
        _lib.gor_project_scene.restype = C.c_int64
        _lib.gor_splat_binning.restype = C.c_int64
        _lib.gor_query_view.restype = C.c_int64
        _lib.gor_select_nbv.restype = C.c_int
        _lib.gor_project_particle.restype = C.c_int
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def camera_struct(cam) -> Camera:
    c = Camera()
    rot = np.asarray(cam.rotation, np.float64).reshape(9)
    for i in range(9):
        c.rotation[i] = float(rot[i])
    for i in range(3):
        c.position[i] = float(cam.position[i])
    c.width, c.height = int(cam.width), int(cam.height)
    c.fov_h, c.fov_v, c.near_plane = float(cam.fov_h), float(cam.fov_v), float(cam.near)
    return c


def cameras_array(cams: Sequence) -> C.Array:
    arr = (Camera * max(1, len(cams)))()
    for i, cam in enumerate(cams):
        arr[i] = camera_struct(cam)
    return arr


def raster_struct(rc) -> Raster:
    return Raster(int(rc.tile_size), 0, float(rc.transmittance_cutoff), float(rc.dilation),
                  float(rc.alpha_clamp_max))


def unc_struct(uc) -> Unc:
    u = Unc()
    u.beta, u.prior_opacity, u.color_sigma = float(uc.beta), float(uc.prior_opacity), float(uc.color_sigma)
    q = np.asarray(uc.prior_cov, np.float64).reshape(9)
    for i in range(9):
        u.prior_cov[i] = float(q[i])
    u.variance_provider = int(getattr(uc, "variance_provider", 0))
    u.correlation = int(getattr(uc, "correlation", 0))
    u.correlation_lambda = float(getattr(uc, "correlation_lambda", 1.0))
    return u


_var_keepalive = None


def set_coeff_variances(variances, degree: int) -> None:
    """Coefficient variances [N][3][(degree+1)^2] used when variance_provider == 1."""
    global _var_keepalive
    _var_keepalive = None if variances is None else np.ascontiguousarray(variances, np.float64).reshape(-1)
    lib().gor_set_coeff_variances(_p(_var_keepalive), degree)


def image_entropy_hook(H, depth, lam: float) -> float:
    lib().gor_image_entropy_hook.restype = C.c_double
    h = np.ascontiguousarray(H, np.float64)
    d = np.ascontiguousarray(depth, np.float64)
    return lib().gor_image_entropy_hook(_p(h), _p(d), h.size, C.c_double(lam))


class OracleScene:
    """Holds double copies of a model.Scene and the C struct pointing at them."""

    def __init__(self, scene):
        self.scene = scene
        n = scene.num_particles
        self.pos = np.ascontiguousarray(scene.positions, np.float64).reshape(-1)
        self.rot = np.ascontiguousarray(scene.rotations, np.float64).reshape(-1)
        self.scl = np.ascontiguousarray(scene.scales, np.float64).reshape(-1)
        self.op = np.ascontiguousarray(scene.opacities, np.float64).reshape(-1)
        self.col = np.ascontiguousarray(scene.colors, np.float64).reshape(-1)
        self.virt = np.ascontiguousarray(scene.is_virtual, np.uint8).reshape(-1)
        # keep non-empty buffers so pointers are valid
        for name in ("pos", "rot", "scl", "op", "col", "virt"):
            if getattr(self, name).size == 0:
                setattr(self, name, np.zeros(1, getattr(self, name).dtype))
        self.c = SceneC(n, scene.color_degree, 0, _p(self.pos), _p(self.rot), _p(self.scl),
                        _p(self.op), _p(self.col), _p(self.virt))
        self.n = n


def _scene(s) -> OracleScene:
    return s if isinstance(s, OracleScene) else OracleScene(s)


def eval_sh(degree: int, d) -> np.ndarray:
    out = np.zeros((degree + 1) ** 2)
    dd = np.asarray(d, np.float64)
    lib().gor_eval_sh(degree, _p(dd), _p(out))
    return out


def bessel_i(l: int, x: float) -> float:
    return lib().gor_bessel_i(l, C.c_double(x))


def vmf_scales(kappa: float, degree: int) -> np.ndarray:
    out = np.zeros(degree + 1)
    lib().gor_vmf_scales(C.c_double(kappa), degree, _p(out))
    return out


def project_scene(scene, cam, dilation: float = 0.3):
    s = _scene(scene)
    buf = (Splat * max(1, s.n))()
    n = lib().gor_project_scene(C.byref(s.c), C.byref(camera_struct(cam)), C.c_double(dilation), buf)
    return [buf[i] for i in range(n)]


def covered_pixel_range(m: float, r: float, n: int):
    lo, hi = C.c_int(), C.c_int()
    lib().gor_covered_pixel_range(C.c_double(m), C.c_double(r), n, C.byref(lo), C.byref(hi))
    return lo.value, hi.value


def splat_binning(splats, width: int, height: int, tile_size: int):
    arr = (Splat * max(1, len(splats)))(*splats)
    tiles = ((width + tile_size - 1) // tile_size) * ((height + tile_size - 1) // tile_size)
    off = np.zeros(tiles + 1, np.int64)
    total = lib().gor_splat_binning(arr, len(splats), width, height, tile_size, _p(off), None)
    ent = np.zeros(max(1, total), np.int32)
    lib().gor_splat_binning(arr, len(splats), width, height, tile_size, _p(off), _p(ent))
    return off, ent[:total]


def rasterize(scene, cam, rc, contrib: bool = False):
    s = _scene(scene)
    P = cam.width * cam.height
    rgb, depth, T = np.zeros(P * 3), np.zeros(P), np.zeros(P)
    cc = np.zeros(P, np.int32) if contrib else None
    lib().gor_rasterize(C.byref(s.c), C.byref(camera_struct(cam)), C.byref(raster_struct(rc)),
                        _p(rgb), _p(depth), _p(T), _p(cc))
    return (rgb, depth, T, cc) if contrib else (rgb, depth, T)


def rasterize_brute(scene, cam, rc):
    s = _scene(scene)
    P = cam.width * cam.height
    rgb, depth, T = np.zeros(P * 3), np.zeros(P), np.zeros(P)
    lib().gor_rasterize_brute(C.byref(s.c), C.byref(camera_struct(cam)), C.byref(raster_struct(rc)),
                              _p(rgb), _p(depth), _p(T))
    return rgb, depth, T


def single_view_visibility(scene, cam, rc, with_counts: bool = False):
    s = _scene(scene)
    v = np.zeros(max(1, s.n))
    touch = np.zeros(max(1, s.n), np.int64)
    cc = np.zeros(cam.width * cam.height, np.int32)
    lib().gor_single_view_visibility(C.byref(s.c), C.byref(camera_struct(cam)),
                                     C.byref(raster_struct(rc)), _p(v), _p(touch), _p(cc))
    if with_counts:
        return v[: s.n], touch[: s.n], cc
    return v[: s.n]


def accumulate_view(gamma: np.ndarray, degree: int, kappa: float, scene, cam, vis) -> None:
    s = _scene(scene)
    vv = np.ascontiguousarray(vis, np.float64)
    lib().gor_accumulate_view(_p(gamma), degree, C.c_double(kappa), C.byref(s.c),
                              C.byref(camera_struct(cam)), _p(vv))


def construct_field(scene, views, kappa: float, degree: int, rc, threads: int = 1) -> np.ndarray:
    s = _scene(scene)
    nb = (degree + 1) ** 2
    gamma = np.zeros(max(1, s.n) * nb)
    cams = cameras_array(views)
    lib().gor_construct_field(C.byref(s.c), cams, len(views), C.c_double(kappa), degree,
                              C.byref(raster_struct(rc)), threads, _p(gamma))
    return gamma[: s.n * nb].reshape(s.n, nb)


def query_visibility(row, degree: int, num_views: int, is_virtual: bool, d) -> float:
    r = np.ascontiguousarray(row, np.float64)
    dd = np.ascontiguousarray(d, np.float64)
    return lib().gor_query_visibility(_p(r), degree, num_views, int(is_virtual), _p(dd))


def query_view(gamma, degree: int, num_views: int, scene, cam, dilation: float = 0.3):
    s = _scene(scene)
    g = np.ascontiguousarray(gamma, np.float64)
    idx = np.zeros(max(1, s.n), np.int32)
    vis = np.zeros(max(1, s.n))
    n = lib().gor_query_view(_p(g), degree, num_views, C.byref(s.c), C.byref(camera_struct(cam)),
                             C.c_double(dilation), _p(idx), _p(vis))
    return idx[:n], vis[:n]


def splat_visibility(gamma, degree: int, num_views: int, scene, cam, dilation: float = 0.3):
    s = _scene(scene)
    g = np.ascontiguousarray(gamma, np.float64)
    vis = np.zeros(max(1, s.n))
    lib().gor_splat_visibility(_p(g), degree, num_views, C.byref(s.c), C.byref(camera_struct(cam)),
                               C.c_double(dilation), _p(vis))
    return vis[: s.n]


def render_entropy_core(scene, cam, rc, uc, vis_by_particle, contrib: bool = False):
    s = _scene(scene)
    P = cam.width * cam.height
    H, w0, depth = np.zeros(P), np.zeros(P), np.zeros(P)
    cc = np.zeros(P, np.int32)
    v = np.ascontiguousarray(vis_by_particle, np.float64)
    if v.size == 0:
        v = np.zeros(1)
    lib().gor_render_entropy_core(C.byref(s.c), C.byref(camera_struct(cam)), C.byref(raster_struct(rc)),
                                  C.byref(unc_struct(uc)), _p(v), _p(H), _p(w0), _p(depth), _p(cc))
    return (H, w0, depth, cc) if contrib else (H, w0, depth)


def render_mixtures(scene, cam, rc, uc, vis_by_particle):
    """Per-pixel mixtures of render_entropy_core (uncertainty.hpp:185-230):
    (offsets[P+1], components[K, 8] = w, v, mean rgb, var rgb, prior w0, residual T, H)."""
    s = _scene(scene)
    P = cam.width * cam.height
    off = np.zeros(P + 1, np.int64)
    prior, resid, H = np.zeros(P), np.zeros(P), np.zeros(P)
    v = np.ascontiguousarray(vis_by_particle, np.float64)
    if v.size == 0:
        v = np.zeros(1)
    args = (C.byref(s.c), C.byref(camera_struct(cam)), C.byref(raster_struct(rc)), C.byref(unc_struct(uc)), _p(v))
    lib().gor_render_mixtures(*args, _p(off), None, _p(prior), _p(resid), _p(H))
    comps = np.zeros((max(1, int(off[-1])), 8))
    lib().gor_render_mixtures(*args, _p(off), _p(comps), None, None, None)
    return off, comps[: int(off[-1])], prior, resid, H


def render_entropy(scene, gamma, degree: int, num_views: int, cam, rc, uc, contrib: bool = False):
    s = _scene(scene)
    P = cam.width * cam.height
    H, w0, depth = np.zeros(P), np.zeros(P), np.zeros(P)
    cc = np.zeros(P, np.int32)
    g = np.ascontiguousarray(gamma, np.float64)
    if g.size == 0:
        g = np.zeros(1)
    lib().gor_render_entropy(C.byref(s.c), _p(g), degree, num_views, C.byref(camera_struct(cam)),
                             C.byref(raster_struct(rc)), C.byref(unc_struct(uc)), _p(H), _p(w0),
                             _p(depth), _p(cc))
    return (H, w0, depth, cc) if contrib else (H, w0, depth)


def image_entropy(H) -> float:
    h = np.ascontiguousarray(H, np.float64)
    return lib().gor_image_entropy(_p(h), h.size)


def select_nbv(scene, gamma, degree: int, num_views: int, cams, rc, uc, threads: int = 1,
               with_rgb: bool = False):
    s = _scene(scene)
    g = np.ascontiguousarray(gamma, np.float64)
    if g.size == 0:
        g = np.zeros(1)
    arr = cameras_array(cams)
    scores = np.zeros(max(1, len(cams)))
    best = lib().gor_select_nbv(C.byref(s.c), _p(g), degree, num_views, arr, len(cams),
                                C.byref(raster_struct(rc)), C.byref(unc_struct(uc)), threads,
                                int(with_rgb), _p(scores))
    return best, scores[: len(cams)]


def raymarch_transmittance(scene, origin, target, step: float, exclude: int = -1,
                           alpha_clamp_max: float = 0.99) -> float:
    s = _scene(scene)
    o = np.ascontiguousarray(origin, np.float64)
    t = np.ascontiguousarray(target, np.float64)
    return lib().gor_raymarch_transmittance(C.byref(s.c), _p(o), _p(t), C.c_double(step),
                                            C.c_int64(exclude), C.c_double(alpha_clamp_max))


def derive_seed(seed: int, stream: int) -> int:
    lib().gor_derive_seed.restype = C.c_uint64
    return lib().gor_derive_seed(C.c_uint64(seed), C.c_uint64(stream))


def density_control(scene, bounds_min, bounds_max, views, rho=100.0, eta=0.5, eps_v=0.95, seed=0,
                    rc=None, round_f32: bool = True):
    """density_control (vfield.hpp:157-199); returns (kept probe ids, unseen products)."""
    from paper_2605_30342_b200.model import RasterConfig
    rc = rc or RasterConfig()
    s = _scene(scene)
    bmin = np.ascontiguousarray(bounds_min, np.float64)
    bmax = np.ascontiguousarray(bounds_max, np.float64)
    ext = bmax - bmin
    n_virtual = int(np.floor(rho * (ext[0] * ext[1] * ext[2])))
    kept = np.zeros(max(1, n_virtual), np.int64)
    unseen = np.zeros(max(1, n_virtual))
    arr = cameras_array(views)
    lib().gor_density_control.restype = C.c_int64
    n = lib().gor_density_control(C.byref(s.c), _p(bmin), _p(bmax), arr, len(views), C.c_double(rho),
                                  C.c_double(eta), C.c_double(eps_v), C.c_uint64(seed),
                                  C.byref(raster_struct(rc)), 1, int(round_f32), _p(kept), _p(unseen))
    return kept[:n], unseen[:n_virtual]


class Planner(C.Structure):
    _fields_ = [("mode", C.c_int32), ("num_candidates", C.c_int32), ("se2_height", C.c_double),
                ("steps", C.c_int32), ("look_inward", C.c_int32), ("seed", C.c_uint64),
                ("clearance", C.c_double), ("cam_width", C.c_int32), ("cam_height", C.c_int32),
                ("fov_h", C.c_double), ("fov_v", C.c_double), ("cam_near", C.c_double)]


class Rect(C.Structure):
    _fields_ = [("corner", C.c_double * 3), ("edge_u", C.c_double * 3), ("edge_v", C.c_double * 3),
                ("opaque", C.c_int32), ("_pad", C.c_int32)]


def _rects(occ):
    rs = occ.rectangles if occ is not None else []
    arr = (Rect * max(1, len(rs)))()
    for i, r in enumerate(rs):
        for k in range(3):
            arr[i].corner[k], arr[i].edge_u[k], arr[i].edge_v[k] = r.corner[k], r.edge_u[k], r.edge_v[k]
        arr[i].opaque = 1 if r.opaque else 0
    return arr, len(rs)


def _camera_from(c):
    from paper_2605_30342_b200.model import CameraView
    return CameraView(rotation=np.array(list(c.rotation)).reshape(3, 3), position=np.array(list(c.position)),
                      width=c.width, height=c.height, fov_h=c.fov_h, fov_v=c.fov_v, near=c.near_plane)


def sample_candidates(bounds, occ, pc, step_seed: int):
    """sample_candidates (planner.hpp:56-107); raises ValueError where the reference throws."""
    p = Planner(int(pc.mode), int(pc.num_candidates), float(pc.se2_height), int(pc.steps),
                1 if pc.look_inward else 0, int(pc.seed), float(pc.clearance), int(pc.cam_width),
                int(pc.cam_height), float(pc.fov_h), float(pc.fov_v), float(pc.cam_near))
    bmin = np.ascontiguousarray(bounds[0], np.float64)
    bmax = np.ascontiguousarray(bounds[1], np.float64)
    rects, nr = _rects(occ)
    out = (Camera * max(1, int(pc.num_candidates)))()
    n = lib().gor_sample_candidates(_p(bmin), _p(bmax), rects, nr, C.byref(p), C.c_uint64(step_seed), out)
    if n < 0:
        raise ValueError(f"sample_candidates failed ({n})")
    return [_camera_from(out[i]) for i in range(n)]


def vis_coverage(occ, views) -> float:
    """vis_coverage (planner.hpp:155-184)"""
    lib().gor_vis_coverage.restype = C.c_double
    rects, nr = _rects(occ)
    return lib().gor_vis_coverage(rects, nr, C.c_double(occ.sample_density), cameras_array(views), len(views))
