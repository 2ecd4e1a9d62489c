"""The GAVIS reference itself on the CPU -- its unmodified hot-path headers
(/root/reference/proj/include/gavis/*.hpp) compiled against the Eigen-subset
shim (oracle/eigen_shim) into oracle/_ref/libgavis_ref.so by `make -C oracle ref`
(__graft_entry__.build() runs it when /root/reference is present; the .so then
travels with the repo snapshot). TEST INFRASTRUCTURE ONLY: it checks the CUDA
product and the oracle restatement, and is the reference arm's CPU
implementation; nothing on the product path loads it.

Same call shapes as oracle.py (scenes as OracleScene / model.Scene, cameras and
configs as model objects); every function takes `threads` (the reference's
parallel_for).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

import oracle as O

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libgavis_ref.so")
_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise ImportError(f"{LIB_PATH} missing: run `make -C oracle ref` where /root/reference exists")
        _lib = C.CDLL(LIB_PATH)
        _lib.gref_last_error.restype = C.c_char_p
    return _lib


def _check(st: int) -> None:
    if st != 0:
        raise RuntimeError(f"reference error {st}: {lib().gref_last_error().decode()}")


def single_view_visibility(scene, cam, rc, threads: int = 1) -> np.ndarray:
    s = O._scene(scene)
    v = np.zeros(max(1, s.n))
    _check(lib().gref_single_view_visibility(C.byref(s.c), C.byref(O.camera_struct(cam)),
                                             C.byref(O.raster_struct(rc)), threads, O._p(v)))
    return v[: s.n]


def construct_field(scene, views, kappa: float, degree: int, rc, threads: int = 1) -> np.ndarray:
    s = O._scene(scene)
    nb = (degree + 1) ** 2
    g = np.zeros(max(1, s.n) * nb)
    _check(lib().gref_construct_field(C.byref(s.c), O.cameras_array(views), len(views), C.c_double(kappa), degree,
                                      C.byref(O.raster_struct(rc)), threads, O._p(g)))
    return g[: s.n * nb].reshape(s.n, nb)


def rasterize(scene, cam, rc, threads: int = 1):
    s = O._scene(scene)
    P = cam.width * cam.height
    rgb, depth, T = np.zeros(3 * P), np.zeros(P), np.zeros(P)
    _check(lib().gref_rasterize(C.byref(s.c), C.byref(O.camera_struct(cam)), C.byref(O.raster_struct(rc)),
                                threads, O._p(rgb), O._p(depth), O._p(T)))
    return rgb, depth, T


def render_entropy(scene, gamma, degree: int, num_views: int, cam, rc, uc, threads: int = 1):
    s = O._scene(scene)
    P = cam.width * cam.height
    H, w0, d = np.zeros(P), np.zeros(P), np.zeros(P)
    g = np.ascontiguousarray(gamma, np.float64)
    if g.size == 0:
        g = np.zeros(1)
    _check(lib().gref_render_entropy(C.byref(s.c), O._p(g), degree, num_views, C.byref(O.camera_struct(cam)),
                                     C.byref(O.raster_struct(rc)), C.byref(O.unc_struct(uc)), threads, O._p(H),
                                     O._p(w0), O._p(d)))
    return H, w0, d


def select_nbv(scene, gamma, degree: int, num_views: int, cams, rc, uc, threads: int = 1):
    s = O._scene(scene)
    g = np.ascontiguousarray(gamma, np.float64)
    if g.size == 0:
        g = np.zeros(1)
    scores = np.zeros(max(1, len(cams)))
    best = C.c_int()
    _check(lib().gref_select_nbv(C.byref(s.c), O._p(g), degree, num_views, O.cameras_array(cams), len(cams),
                                 C.byref(O.raster_struct(rc)), C.byref(O.unc_struct(uc)), threads, O._p(scores),
                                 C.byref(best)))
    return best.value, scores[: len(cams)]


class RefScene:
    """A reference gavis::Scene built once (gref_scene_new) for timed calls."""

    def __init__(self, scene):
        self._os = O._scene(scene)  # keeps the double arrays alive while building
        lib().gref_scene_new.restype = C.c_void_p
        self.h = C.c_void_p(lib().gref_scene_new(C.byref(self._os.c)))
        if not self.h:
            raise RuntimeError(lib().gref_last_error().decode())
        self.n = self._os.n

    def close(self):
        if self.h:
            lib().gref_scene_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def construct_field_h(rs: RefScene, views, kappa: float, degree: int, rc, threads: int = 1) -> np.ndarray:
    nb = (degree + 1) ** 2
    g = np.zeros(max(1, rs.n) * nb)
    _check(lib().gref_construct_field_h(rs.h, O.cameras_array(views), len(views), C.c_double(kappa), degree,
                                        C.byref(O.raster_struct(rc)), threads, O._p(g)))
    return g[: rs.n * nb].reshape(rs.n, nb)


def select_nbv_rgb_h(rs: RefScene, gamma, degree: int, num_views: int, cams, rc, uc, threads: int = 1):
    """The bench step on the reference: select_nbv over `cams` plus the RGB
    rasterize of each, parallel over candidates (planner.hpp:125-131)."""
    g = np.ascontiguousarray(gamma, np.float64)
    if g.size == 0:
        g = np.zeros(1)
    scores = np.zeros(max(1, len(cams)))
    best = C.c_int()
    _check(lib().gref_select_nbv_rgb_h(rs.h, O._p(g), degree, num_views, O.cameras_array(cams), len(cams),
                                       C.byref(O.raster_struct(rc)), C.byref(O.unc_struct(uc)), threads,
                                       O._p(scores), C.byref(best)))
    return best.value, scores[: len(cams)]


# ---- the planner-side §8f rows: the reference's own sample_candidates,
# vis_coverage, density_control and run_active_mapping ------------------------
def _planner(pc):
    return O.Planner(int(pc.mode), int(pc.num_candidates), float(pc.se2_height), int(pc.steps),
                     1 if pc.look_inward else 0, int(pc.seed), float(pc.clearance), int(pc.cam_width),
                     int(pc.cam_height), float(pc.fov_h), float(pc.fov_v), float(pc.cam_near))


def sample_candidates(bounds, occ, pc, step_seed: int):
    """sample_candidates (planner.hpp:56-107); raises ValueError where the reference throws."""
    bmin = np.ascontiguousarray(bounds[0], np.float64)
    bmax = np.ascontiguousarray(bounds[1], np.float64)
    rects, nr = O._rects(occ)
    out = (O.Camera * max(1, int(pc.num_candidates)))()
    n = lib().gref_sample_candidates(O._p(bmin), O._p(bmax), rects, nr, C.byref(_planner(pc)),
                                     C.c_uint64(step_seed), out)
    if n < 0:
        raise ValueError(f"sample_candidates failed: {lib().gref_last_error().decode()}")
    return [O._camera_from(out[i]) for i in range(n)]


def vis_coverage(occ, views) -> float:
    """vis_coverage (planner.hpp:155-184)"""
    lib().gref_vis_coverage.restype = C.c_double
    rects, nr = O._rects(occ)
    return lib().gref_vis_coverage(rects, nr, C.c_double(occ.sample_density), O.cameras_array(views), len(views))


def density_control_positions(scene, bounds_min, bounds_max, views, rho=100.0, eta=0.5, eps_v=0.95, seed=0,
                              rc=None, threads: int = 1) -> np.ndarray:
    """density_control (vfield.hpp:157-199): positions [m, 3] of the virtual
    particles the reference appends (in probe order)."""
    from paper_2605_30342_b200.model import RasterConfig
    rc = rc or RasterConfig()
    s = O._scene(scene)
    bmin = np.ascontiguousarray(bounds_min, np.float64)
    bmax = np.ascontiguousarray(bounds_max, np.float64)
    ext = bmax - bmin
    cap = int(np.floor(rho * (ext[0] * ext[1] * ext[2])))
    pos = np.zeros(max(1, cap) * 3)
    lib().gref_density_control.restype = C.c_int64
    m = lib().gref_density_control(C.byref(s.c), O._p(bmin), O._p(bmax), O.cameras_array(views), len(views),
                                   C.c_double(rho), C.c_double(eta), C.c_double(eps_v), C.c_uint64(seed),
                                   C.byref(O.raster_struct(rc)), threads, O._p(pos), C.c_int64(cap))
    if m < 0:
        raise RuntimeError(f"reference error: {lib().gref_last_error().decode()}")
    return pos[: 3 * m].reshape(m, 3)


def active_mapping(scene, bounds, occ, init, pc, kappa: float, degree: int, rc, uc, density_enabled: bool,
                   rho=100.0, eta=0.5, eps_v=0.95, dseed=0, threads: int = 1):
    """run_active_mapping (planner.hpp:284-316) -> [(chosen index, scores, vis_coverage)] per step."""
    s = O._scene(scene)
    bmin = np.ascontiguousarray(bounds[0], np.float64)
    bmax = np.ascontiguousarray(bounds[1], np.float64)
    rects, nr = O._rects(occ)
    steps, nc = int(pc.steps), int(pc.num_candidates)
    chosen = (C.c_int * max(1, steps))()
    score = np.zeros(max(1, steps))
    cov = np.zeros(max(1, steps))
    alls = np.zeros(max(1, steps * nc))
    _check(lib().gref_active_mapping(C.byref(s.c), O._p(bmin), O._p(bmax), rects, nr,
                                     C.c_double(occ.sample_density if occ is not None else 64.0),
                                     O.cameras_array(init), len(init), C.byref(_planner(pc)), C.c_double(kappa),
                                     degree, C.byref(O.raster_struct(rc)), C.byref(O.unc_struct(uc)),
                                     1 if density_enabled else 0, C.c_double(rho), C.c_double(eta),
                                     C.c_double(eps_v), C.c_uint64(dseed), threads, chosen, O._p(score),
                                     O._p(cov), O._p(alls)))
    return [(int(chosen[k]), alls[k * nc:(k + 1) * nc].copy(), float(cov[k])) for k in range(steps)]


def render_entropy_core(scene, cam, rc, uc, vis_by_particle, coeff_var=None, var_degree: int = -1,
                        mixtures: bool = False, threads: int = 1):
    """render_entropy_core (uncertainty.hpp:124-238) with per-particle visibility;
    coeff_var [N, 3, (Lv+1)^2] selects the sh_propagation provider. Returns
    (H, w0, depth) and, with mixtures, (offsets, components [K, 8], prior, resid, H_mix)."""
    s = O._scene(scene)
    P = cam.width * cam.height
    H, w0, d = np.zeros(P), np.zeros(P), np.zeros(P)
    v = np.ascontiguousarray(vis_by_particle, np.float64)
    cv = None if coeff_var is None else np.ascontiguousarray(coeff_var, np.float64).reshape(-1)
    base = (C.byref(s.c), C.byref(O.camera_struct(cam)), C.byref(O.raster_struct(rc)), C.byref(O.unc_struct(uc)),
            O._p(v), O._p(cv) if cv is not None else None, var_degree, threads)
    off = np.zeros(P + 1, np.int64) if mixtures else None
    _check(lib().gref_render_entropy_core(*base, O._p(H), O._p(w0), O._p(d), O._p(off) if mixtures else None,
                                          None, C.c_int64(0), None, None, None))
    if not mixtures:
        return H, w0, d
    K = int(off[-1])
    comps = np.zeros((max(1, K), 8))
    prior, resid, Hm = np.zeros(P), np.zeros(P), np.zeros(P)
    _check(lib().gref_render_entropy_core(*base, None, None, None, O._p(off), O._p(comps), C.c_int64(K),
                                          O._p(prior), O._p(resid), O._p(Hm)))
    return (H, w0, d), (off, comps[:K], prior, resid, Hm)


def project_and_bin(scene, cam, dilation: float = 0.3, tile_size: int = 16):
    """project_scene (raster.hpp:114-130) + splat_binning (:145-164) of the
    reference: (splats sorted by (depth, index), tile offsets, entries)."""
    s = O._scene(scene)
    buf = (O.Splat * max(1, s.n))()
    tiles = ((cam.width + tile_size - 1) // tile_size) * ((cam.height + tile_size - 1) // tile_size)
    off = np.zeros(tiles + 1, np.int64)
    lib().gref_project_and_bin.restype = C.c_int64
    n = lib().gref_project_and_bin(C.byref(s.c), C.byref(O.camera_struct(cam)), C.c_double(dilation), tile_size,
                                   buf, O._p(off), None)
    if n < 0:
        raise RuntimeError(f"reference error: {lib().gref_last_error().decode()}")
    ent = np.zeros(max(1, int(off[-1])), np.int32)
    lib().gref_project_and_bin(C.byref(s.c), C.byref(O.camera_struct(cam)), C.c_double(dilation), tile_size,
                               buf, O._p(off), O._p(ent))
    return [buf[i] for i in range(n)], off, ent[: int(off[-1])]


def query_view(gamma, degree: int, num_views: int, scene, cam, dilation: float = 0.3):
    """query_view (vfield.hpp:121-134) -> (particle indices, visibilities)."""
    s = O._scene(scene)
    g = np.ascontiguousarray(gamma, np.float64)
    idx = np.zeros(max(1, s.n), np.int32)
    vis = np.zeros(max(1, s.n))
    lib().gref_query_view.restype = C.c_int64
    n = lib().gref_query_view(C.byref(s.c), O._p(g), degree, num_views, C.byref(O.camera_struct(cam)),
                              C.c_double(dilation), O._p(idx), O._p(vis))
    if n < 0:
        raise RuntimeError(f"reference error: {lib().gref_last_error().decode()}")
    return idx[:n], vis[:n]
