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
