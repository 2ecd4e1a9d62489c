"""Python mirror of the reference's C++ API for the two hot paths, over the C ABI.

Names, argument meaning and error behaviour follow the reference:
  construct_field          R/include/gavis/vfield.hpp:68-92
  accumulate_view          vfield.hpp:38-63
  single_view_visibility   raster.hpp:237-290
  query_visibility         vfield.hpp:96-112
  query_view               vfield.hpp:121-134
  rasterize                raster.hpp:175-231
  render_entropy(_core)    uncertainty.hpp:124-260
  image_entropy            uncertainty.hpp:264-278
  select_nbv               planner.hpp:117-137
  sample_candidates        planner.hpp:56-107
  vis_coverage             planner.hpp:155-184
  active_mapping           planner.hpp:284-316 (run_active_mapping)
ParameterError / InvariantError are raised where the reference throws them.
Everything runs on the GPU through libgavis_b200.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import weakref
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _native as N
from .model import (CameraView, EntropyMap, InvariantError, MappingLog, MappingStep, NbvResult, OccluderSet, ParameterError,
                    PlannerConfig, RasterConfig, RenderOutput, Scene, UncertaintyConfig, ViewQuery,
                    VisibilityField, VmfParams, require)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def camera_c(cam: CameraView) -> N.Camera:
    c = N.Camera()
    r = np.asarray(cam.rotation, np.float64).reshape(9)
    for i in range(9):
        c.rotation[i] = float(r[i])
    for i in range(3):
        c.position[i] = float(cam.position[i])
    c.width, c.height = int(cam.width), int(cam.height)
    c.fov_h, c.fov_v, c.near_plane = float(cam.fov_h), float(cam.fov_v), float(cam.near)
    return c


def cameras_c(cams: Sequence[CameraView]):
    arr = (N.Camera * max(1, len(cams)))()
    for i, cam in enumerate(cams):
        arr[i] = camera_c(cam)
    return arr


def raster_c(rc: RasterConfig) -> N.RasterConfigC:
    return N.RasterConfigC(int(rc.tile_size), 0, float(rc.transmittance_cutoff), float(rc.dilation),
                           float(rc.alpha_clamp_max))


def unc_c(uc: UncertaintyConfig) -> N.UncertaintyConfigC:
    u = N.UncertaintyConfigC()
    u.beta, u.prior_opacity, u.color_sigma = float(uc.beta), float(uc.prior_opacity), float(uc.color_sigma)
    q = np.asarray(uc.prior_cov, np.float64).reshape(9)
    for i in range(9):
        u.prior_cov[i] = float(q[i])
    u.variance_provider = int(uc.variance_provider)
    u.correlation = int(uc.correlation)
    u.correlation_lambda = float(uc.correlation_lambda)
    return u


class Context:
    """One device context (one process per GPU). stream: an int cudaStream_t handle or None."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        self.lib = N.load()
        h = C.c_void_p()
        N.check(self.lib.gavis_ctx_create(C.c_int32(device), C.c_void_p(stream) if stream else None,
                                          C.byref(h)))
        self.h = h
        self.device = device
        # device objects of this context, released before it (the C ABI requires
        # scenes and fields to be destroyed before their context)
        self._children = weakref.WeakSet()
        self.precision = "exact"  # the library default (gavis_ctx_set_precision)

    def close(self) -> None:
        if self.h:
            kids = list(self._children)
            for k in kids:
                if isinstance(k, DeviceField):
                    k.close()
            for k in kids:
                k.close()
            N.check(self.lib.gavis_ctx_destroy(self.h))
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self) -> None:
        N.check(self.lib.gavis_ctx_synchronize(self.h))

    def set_batch(self, n: int) -> None:
        N.check(self.lib.gavis_ctx_set_batch(self.h, C.c_int32(n)))

    def set_pair_budget(self, n: int) -> None:
        """Tile pairs one batch may hold (0 = automatic); larger batches are split."""
        N.check(self.lib.gavis_ctx_set_pair_budget(self.h, C.c_int64(n)))

    def set_precision(self, precision: str) -> None:
        """'exact' (default: the fp64 blend, the reference's arithmetic) or
        'certified' (fp32 blend, fp64 redo of uncertified pixels, fp64 argmax)."""
        modes = {"certified": N.PRECISION_CERTIFIED, "exact": N.PRECISION_EXACT}
        require(precision in modes, "precision must be 'certified' or 'exact'")
        N.check(self.lib.gavis_ctx_set_precision(self.h, C.c_int32(modes[precision])))
        self.precision = precision

    def counters(self):
        """(pixels recomputed in fp64 by the certified blend, candidates re-scored
        in fp64 to certify an argmax) since the context was created."""
        a = C.c_int64()
        b = C.c_int64()
        N.check(self.lib.gavis_ctx_get_counters(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def last_score_bounds(self) -> np.ndarray:
        """Per-candidate bounds on |certified score - fp64 score| of the last scored
        render (empty unless certified, constant provider, no correlation hook)."""
        n = C.c_int32()
        N.check(self.lib.gavis_ctx_last_score_bounds(self.h, None, C.c_int32(0), C.byref(n)))
        out = np.zeros(max(1, n.value))
        N.check(self.lib.gavis_ctx_last_score_bounds(self.h, _ptr(out), C.c_int32(out.size), C.byref(n)))
        return out[: n.value]

    def set_profiling(self, on: bool) -> None:
        N.check(self.lib.gavis_ctx_set_profiling(self.h, C.c_int32(1 if on else 0)))

    def kernel_time(self, name: str, reset: bool = False):
        ms = C.c_double()
        n = C.c_int64()
        N.check(self.lib.gavis_ctx_kernel_time(self.h, name.encode(), C.byref(ms), C.byref(n),
                                               C.c_int32(1 if reset else 0)))
        return ms.value, n.value

    def timer_start(self) -> None:
        N.check(self.lib.gavis_ctx_timer_start(self.h))

    def timer_stop(self) -> float:
        ms = C.c_double()
        N.check(self.lib.gavis_ctx_timer_stop(self.h, C.byref(ms)))
        return ms.value

    def launch_count(self) -> int:
        n = C.c_int64()
        N.check(self.lib.gavis_ctx_launch_count(self.h, C.byref(n)))
        return n.value

    def upload(self, scene: Scene) -> "DeviceScene":
        return DeviceScene(self, scene)


class DeviceScene:
    def __init__(self, ctx: Context, scene: Scene):
        s = scene.contiguous()
        self.ctx = ctx
        self.n = s.num_particles
        self.color_degree = s.color_degree
        self.bounds = (s.bounds_min, s.bounds_max)
        d = N.SceneDesc(self.n, s.color_degree, 0, _ptr(s.positions), _ptr(s.rotations),
                        _ptr(s.scales), _ptr(s.opacities), _ptr(s.colors), _ptr(s.is_virtual))
        h = C.c_void_p()
        N.check(ctx.lib.gavis_scene_upload(ctx.h, C.byref(d), C.byref(h)))
        self.h = h
        ctx._children.add(self)

    def set_coeff_variances(self, variances, degree: int) -> None:
        """UncertaintyConfig::coeff_variances for the sh_propagation provider:
        [N][3][(degree+1)^2] per-particle per-channel SH coefficient variances."""
        var = np.ascontiguousarray(variances, np.float32).reshape(-1)
        N.check(self.ctx.lib.gavis_scene_set_coeff_variances(self.ctx.h, self.h, _ptr(var) if var.size else None,
                                                             C.c_int32(degree)))

    @classmethod
    def _adopt(cls, ctx: Context, handle, n: int, color_degree: int, bounds) -> "DeviceScene":
        obj = cls.__new__(cls)
        obj.ctx, obj.h, obj.n, obj.color_degree, obj.bounds = ctx, handle, n, color_degree, bounds
        ctx._children.add(obj)
        return obj

    def close(self) -> None:
        if self.h and self.ctx.h:
            N.check(self.ctx.lib.gavis_scene_destroy(self.h))
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DensityControlConfig:
    """vfield.hpp:136-147"""

    def __init__(self, rho: float = 100.0, eta: float = 0.5, eps_v: float = 0.95, seed: int = 0):
        self.rho, self.eta, self.eps_v, self.seed = rho, eta, eps_v, seed


class DeviceField:
    def __init__(self, ctx: Context, scene: DeviceScene, handle, degree: int, vmf: VmfParams):
        self.ctx = ctx
        self.scene = scene
        self.h = handle
        self.degree = degree
        self.vmf = vmf
        ctx._children.add(self)

    @property
    def num_views(self) -> int:
        nv = C.c_int32()
        N.check(self.ctx.lib.gavis_vf_download(self.h, None, C.byref(nv), None))
        return nv.value

    def set_num_views(self, n: int) -> None:
        N.check(self.ctx.lib.gavis_vf_set_num_views(self.h, C.c_int32(n)))

    def download(self) -> VisibilityField:
        nb = (self.degree + 1) ** 2
        g = np.zeros((max(1, self.scene.n), nb), np.float64)
        nv = C.c_int32()
        N.check(self.ctx.lib.gavis_vf_download(self.h, _ptr(g), C.byref(nv), None))
        return VisibilityField(self.degree, self.vmf, nv.value, g[: self.scene.n], np.zeros(0, np.uint8))

    def device_gamma(self):
        p = C.c_void_p()
        n = C.c_int64()
        N.check(self.ctx.lib.gavis_vf_device_gamma(self.h, C.byref(p), C.byref(n)))
        return p.value, n.value

    def close(self) -> None:
        if self.h and self.ctx.h:
            N.check(self.ctx.lib.gavis_vf_destroy(self.h))
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _as_dev(ctx: Context, scene) -> DeviceScene:
    return scene if isinstance(scene, DeviceScene) else ctx.upload(scene)


def _splat_vis(vis_by_particle, n: int):
    """Per-particle visibility for render_entropy_core: one entry per particle
    (the reference checks splat_vis against its splats, uncertainty.hpp:133-134)."""
    if vis_by_particle is None:
        return None
    v = np.ascontiguousarray(vis_by_particle, np.float64).reshape(-1)
    if v.size != n:
        raise InvariantError(f"render_entropy_core: visibility has {v.size} entries, the scene {n} particles")
    return v if v.size else np.zeros(1)


# ----------------------------------------------------------------- VF CONST
def construct_field(ctx: Context, scene, views: Sequence[CameraView], vmf: VmfParams, degree: int,
                    rc: RasterConfig = RasterConfig()) -> DeviceField:
    ds = _as_dev(ctx, scene)
    arr = cameras_c(views)
    h = C.c_void_p()
    N.check(ctx.lib.gavis_vf_construct(ctx.h, ds.h, arr, C.c_int32(len(views)), C.c_double(vmf.kappa),
                                       C.c_int32(degree), C.byref(raster_c(rc)), C.byref(h)))
    return DeviceField(ctx, ds, h, degree, vmf)


def empty_field(ctx: Context, scene, vmf: VmfParams, degree: int) -> DeviceField:
    ds = _as_dev(ctx, scene)
    h = C.c_void_p()
    N.check(ctx.lib.gavis_vf_create(ctx.h, ds.h, C.c_double(vmf.kappa), C.c_int32(degree), C.byref(h)))
    return DeviceField(ctx, ds, h, degree, vmf)


def accumulate_views(ctx: Context, field: DeviceField, scene, views: Sequence[CameraView],
                     rc: RasterConfig = RasterConfig()) -> None:
    ds = _as_dev(ctx, scene)
    arr = cameras_c(views)
    N.check(ctx.lib.gavis_vf_accumulate_views(ctx.h, field.h, ds.h, arr, C.c_int32(len(views)),
                                              C.byref(raster_c(rc))))


def accumulate_view(ctx: Context, field: DeviceField, scene, view: CameraView, visibility) -> None:
    ds = _as_dev(ctx, scene)
    v = np.ascontiguousarray(visibility, np.float64).reshape(-1)
    require(v.size == ds.n, f"accumulate_view: visibility has {v.size} entries, the scene {ds.n} particles")
    if v.size == 0:
        v = np.zeros(1)
    N.check(ctx.lib.gavis_vf_accumulate_visibility(ctx.h, field.h, ds.h, C.byref(camera_c(view)), _ptr(v)))


def upload_field(ctx: Context, scene, field: VisibilityField) -> DeviceField:
    ds = _as_dev(ctx, scene)
    g = np.ascontiguousarray(field.gamma, np.float64)
    nb = (int(field.degree) + 1) ** 2
    require(g.shape == (ds.n, nb), f"upload_field: gamma has shape {g.shape}, expected ({ds.n}, {nb}) "
            f"for {ds.n} particles at degree {field.degree}")
    if g.size == 0:
        g = np.zeros((1, nb))
    h = C.c_void_p()
    N.check(ctx.lib.gavis_vf_upload(ctx.h, ds.h, C.c_double(field.vmf.kappa), C.c_int32(field.degree),
                                    C.c_int32(field.num_views), _ptr(g), C.byref(h)))
    return DeviceField(ctx, ds, h, field.degree, field.vmf)


def single_view_visibility(ctx: Context, scene, cam: CameraView, rc: RasterConfig = RasterConfig(),
                           with_counts: bool = False):
    ds = _as_dev(ctx, scene)
    n = max(1, ds.n)
    v = np.zeros(n)
    touch = np.zeros(n, np.int64)
    cc = np.zeros(cam.width * cam.height, np.int32)
    N.check(ctx.lib.gavis_single_view_visibility(ctx.h, ds.h, C.byref(camera_c(cam)), C.byref(raster_c(rc)),
                                                 _ptr(v), _ptr(touch), _ptr(cc) if with_counts else None))
    if with_counts:
        return v[: ds.n], touch[: ds.n], cc
    return v[: ds.n]


def query_visibility(ctx: Context, field: DeviceField, particle_index, d) -> np.ndarray:
    idx = np.ascontiguousarray(np.atleast_1d(particle_index), np.int64)
    dirs = np.ascontiguousarray(np.asarray(d, np.float64).reshape(-1, 3))
    require(dirs.shape[0] == idx.shape[0], "query: one direction per particle index")
    out = np.zeros(max(1, idx.size))
    N.check(ctx.lib.gavis_vf_query(ctx.h, field.h, _ptr(idx), _ptr(dirs), C.c_int64(idx.size), _ptr(out)))
    return out[: idx.size]


def query_view(ctx: Context, field: DeviceField, scene, cam: CameraView, dilation: float = 0.3) -> ViewQuery:
    ds = _as_dev(ctx, scene)
    idx = np.zeros(max(1, ds.n), np.int32)
    vis = np.zeros(max(1, ds.n))
    n = C.c_int64()
    N.check(ctx.lib.gavis_vf_query_view(ctx.h, field.h, ds.h, C.byref(camera_c(cam)), C.c_double(dilation),
                                        _ptr(idx), _ptr(vis), C.byref(n)))
    return ViewQuery(idx[: n.value], vis[: n.value])


def density_control(ctx: Context, scene, views: Sequence[CameraView], cfg: "DensityControlConfig",
                    rc: RasterConfig = RasterConfig(), bounds=None):
    """density_control (vfield.hpp:157-199) on the device. Returns the augmented device
    scene (real particles, then retained probes) and the retained probe ids."""
    ds = _as_dev(ctx, scene)
    bmin, bmax = bounds if bounds is not None else ds.bounds
    bmin = np.ascontiguousarray(bmin, np.float64)
    bmax = np.ascontiguousarray(bmax, np.float64)
    ext = bmax - bmin
    cap = max(1, int(np.floor(cfg.rho * max(0.0, ext[0] * ext[1] * ext[2]))))
    kept = np.zeros(cap, np.int64)
    n_kept = C.c_int64()
    h = C.c_void_p()
    dc = N.DensityConfigC(float(cfg.rho), float(cfg.eta), float(cfg.eps_v), int(cfg.seed))
    arr = cameras_c(views)
    N.check(ctx.lib.gavis_density_control(ctx.h, ds.h, _ptr(bmin), _ptr(bmax), arr, C.c_int32(len(views)),
                                          C.byref(dc), C.byref(raster_c(rc)), C.byref(h), C.byref(n_kept),
                                          _ptr(kept), C.c_int64(cap)))
    out = DeviceScene._adopt(ctx, h, ds.n + n_kept.value, ds.color_degree, (bmin, bmax))
    return out, kept[: n_kept.value]


# ----------------------------------------------------------------- UA render
def render(ctx: Context, scene, field: Optional[DeviceField], cams: Sequence[CameraView],
           rc: RasterConfig = RasterConfig(), uc: UncertaintyConfig = UncertaintyConfig(), *,
           rgb: bool = False, depth: bool = False, transmittance: bool = False, entropy: bool = False,
           invisible_mass: bool = False, entropy_depth: bool = False, scores: bool = False,
           contributors: bool = False, splat_visibility=None, with_rgb: bool = False) -> Dict[str, np.ndarray]:
    """Fused RGB + uncertainty render of several cameras (gavis_ua_render)."""
    ds = _as_dev(ctx, scene)
    P = sum(c.width * c.height for c in cams)
    out: Dict[str, np.ndarray] = {}

    def buf(name, flag, shape, dtype=np.float64):
        if not flag:
            return None
        out[name] = np.zeros(shape, dtype)
        return out[name]

    o = N.RenderOutputs()
    o.rgb = _ptr(buf("rgb", rgb, P * 3))
    o.depth = _ptr(buf("depth", depth, P))
    o.transmittance = _ptr(buf("transmittance", transmittance, P))
    o.entropy = _ptr(buf("entropy", entropy, P))
    o.invisible_mass = _ptr(buf("invisible_mass", invisible_mass, P))
    o.entropy_depth = _ptr(buf("entropy_depth", entropy_depth, P))
    o.scores = _ptr(buf("scores", scores, max(1, len(cams))))
    o.rgb_contributors = _ptr(buf("rgb_contributors", contributors and (rgb or with_rgb), P, np.int32))
    o.entropy_contributors = _ptr(buf("entropy_contributors", contributors and (entropy or scores), P, np.int32))
    o.with_rgb = 1 if with_rgb else 0
    o.with_entropy = 0
    vis = _splat_vis(splat_visibility, ds.n)
    arr = cameras_c(cams)
    N.check(ctx.lib.gavis_ua_render(ctx.h, ds.h, field.h if field is not None else None, _ptr(vis), arr,
                                    C.c_int32(len(cams)), C.byref(raster_c(rc)), C.byref(unc_c(uc)),
                                    C.byref(o)))
    if "scores" in out:
        out["scores"] = out["scores"][: len(cams)]
    return out


def render_mixtures(ctx: Context, scene, field: Optional[DeviceField], cam: CameraView,
                    rc: RasterConfig = RasterConfig(), uc: UncertaintyConfig = UncertaintyConfig(),
                    splat_visibility=None):
    """render_entropy's mixtures_out (uncertainty.hpp:207-230) via gavis_ua_mixtures:
    (offsets[P+1], components[K, 8] = w*, v, mean rgb, var rgb, prior w0, residual T*, H)."""
    ds = _as_dev(ctx, scene)
    P = cam.width * cam.height
    off = np.zeros(P + 1, np.int64)
    prior, resid, H = np.zeros(max(1, P)), np.zeros(max(1, P)), np.zeros(max(1, P))
    vis = _splat_vis(splat_visibility, ds.n)
    cc = camera_c(cam)
    args = (ctx.h, ds.h, field.h if field is not None else None, _ptr(vis), C.byref(cc),
            C.byref(raster_c(rc)), C.byref(unc_c(uc)))
    N.check(ctx.lib.gavis_ua_mixtures(*args, _ptr(off), None, C.c_int64(0), _ptr(prior), _ptr(resid), _ptr(H)))
    K = int(off[-1])
    comps = np.zeros((max(1, K), 8))
    if K > 0:
        N.check(ctx.lib.gavis_ua_mixtures(*args, _ptr(off), _ptr(comps), C.c_int64(K), None, None, None))
    return off, comps[:K], prior[:P], resid[:P], H[:P]


def rasterize(ctx: Context, scene, cam: CameraView, rc: RasterConfig = RasterConfig()) -> RenderOutput:
    r = render(ctx, scene, None, [cam], rc, UncertaintyConfig(), rgb=True, depth=True, transmittance=True)
    return RenderOutput(cam.width, cam.height, r["rgb"], r["depth"], r["transmittance"])


def render_entropy(ctx: Context, scene, field: DeviceField, cam: CameraView, rc: RasterConfig = RasterConfig(),
                   uc: UncertaintyConfig = UncertaintyConfig(), want_depth: bool = False):
    require(field is not None, "render_entropy needs a field")
    r = render(ctx, scene, field, [cam], rc, uc, entropy=True, invisible_mass=True, entropy_depth=want_depth)
    m = EntropyMap(cam.width, cam.height, r["entropy"], r["invisible_mass"])
    return (m, r["entropy_depth"]) if want_depth else m


def render_entropy_core(ctx: Context, scene, cam: CameraView, rc: RasterConfig, uc: UncertaintyConfig,
                        vis_by_particle, want_depth: bool = False):
    r = render(ctx, scene, None, [cam], rc, uc, entropy=True, invisible_mass=True, entropy_depth=want_depth,
               splat_visibility=vis_by_particle)
    m = EntropyMap(cam.width, cam.height, r["entropy"], r["invisible_mass"])
    return (m, r["entropy_depth"]) if want_depth else m


def image_entropy(m: EntropyMap, depth=None, uc: Optional[UncertaintyConfig] = None) -> float:
    """uncertainty.hpp:264-272 (correlation none): plain sum in pixel order."""
    if depth is not None:
        require(len(depth) == len(m.entropy), "image_entropy: depth map shape differs from the entropy map")
    s = 0.0
    for h in m.entropy:
        s += float(h)
    return s


def select_nbv(ctx: Context, scene, field: DeviceField, candidates: Sequence[CameraView],
               rc: RasterConfig = RasterConfig(), uc: UncertaintyConfig = UncertaintyConfig(),
               with_rgb: bool = False) -> NbvResult:
    require(len(candidates) > 0, "select_nbv: candidate list must be nonempty")
    ds = _as_dev(ctx, scene)
    scores = np.zeros(len(candidates))
    best = C.c_int32()
    arr = cameras_c(candidates)
    N.check(ctx.lib.gavis_select_nbv(ctx.h, ds.h, field.h, arr, C.c_int32(len(candidates)),
                                     C.byref(raster_c(rc)), C.byref(unc_c(uc)), C.c_int32(1 if with_rgb else 0),
                                     _ptr(scores), C.byref(best)))
    return NbvResult(best.value, scores)


def score_views(ctx: Context, scene, field: DeviceField, cams: Sequence[CameraView],
                rc: RasterConfig = RasterConfig(), uc: UncertaintyConfig = UncertaintyConfig(),
                with_rgb: bool = False, exact: bool = False) -> np.ndarray:
    """image_entropy(render_entropy(cam)) per camera (planner.hpp:125-131), with the
    context's precision or, with exact=True, the fp64 blend."""
    if len(cams) == 0:
        return np.zeros(0)
    prev = ctx.precision
    if exact and prev != "exact":
        ctx.set_precision("exact")
    try:
        return render(ctx, scene, field, cams, rc, uc, scores=True, with_rgb=with_rgb)["scores"]
    finally:
        if exact and prev != "exact":
            ctx.set_precision(prev)


def select_nbv_sharded(ctx: Context, scene, field: DeviceField, candidates: Sequence[CameraView],
                       rank: int, world: int, dist=None, rc: RasterConfig = RasterConfig(),
                       uc: UncertaintyConfig = UncertaintyConfig(), with_rgb: bool = False) -> NbvResult:
    """select_nbv over candidates sharded across ranks (one process per GPU): each
    rank scores its contiguous block, the scores are all-gathered, contenders of the
    certified argmax are re-scored in fp64 on their owning ranks (parallel.py)."""
    from . import parallel
    require(len(candidates) > 0, "select_nbv: candidate list must be nonempty")
    best, scores = parallel.select_nbv_sharded(
        lambda lo, hi: score_views(ctx, scene, field, candidates[lo:hi], rc, uc, with_rgb),
        len(candidates), rank, world, dist,
        rescore=None if ctx.precision == "exact" else
        (lambda idx: score_views(ctx, scene, field, [candidates[i] for i in idx], rc, uc, exact=True)))
    return NbvResult(best, scores)


def nbv_loop(ctx: Context, scene, field: DeviceField, candidates: Sequence[CameraView], steps: int,
             rc: RasterConfig = RasterConfig(), uc: UncertaintyConfig = UncertaintyConfig(),
             with_rgb: bool = False):
    """run_active_mapping (planner.hpp:284-316) over a fixed candidate pool with the
    field updated incrementally (density control off): returns (chosen, scores,
    all_scores[steps, n])."""
    ds = _as_dev(ctx, scene)
    n = len(candidates)
    chosen = np.zeros(max(1, steps), np.int32)
    best = np.zeros(max(1, steps))
    allsc = np.zeros((max(1, steps), n))
    arr = cameras_c(candidates)
    N.check(ctx.lib.gavis_nbv_loop(ctx.h, ds.h, field.h, arr, C.c_int32(n), C.c_int32(steps),
                                   C.byref(raster_c(rc)), C.byref(unc_c(uc)), C.c_int32(1 if with_rgb else 0),
                                   _ptr(chosen), _ptr(best), _ptr(allsc)))
    return chosen[:steps], best[:steps], allsc[:steps]


# ------------------------------------------------------------------ multi-GPU
class Comm:
    """A communicator of the native library (gavis_comm: NCCL, one process per GPU).
    Every rank creates it with the same unique id; `Comm.from_dist` ships rank 0's
    id over an initialised torch.distributed group (any backend)."""

    def __init__(self, ctx: Context, unique_id: bytes, nranks: int, rank: int):
        require(len(unique_id) == N.COMM_ID_BYTES, "comm: unique id must be 128 bytes")
        self.ctx, self.nranks, self.rank = ctx, int(nranks), int(rank)
        buf = (C.c_uint8 * N.COMM_ID_BYTES).from_buffer_copy(unique_id)
        h = C.c_void_p()
        N.check(ctx.lib.gavis_comm_create(ctx.h, buf, C.c_int32(nranks), C.c_int32(rank), C.byref(h)))
        self.h = h

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * N.COMM_ID_BYTES)()
        N.check(N.load().gavis_comm_unique_id(buf))
        return bytes(buf)

    @classmethod
    def from_dist(cls, ctx: Context, dist) -> "Comm":
        obj = [cls.unique_id() if dist.get_rank() == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return cls(ctx, obj[0], dist.get_world_size(), dist.get_rank())

    def close(self) -> None:
        if self.h and self.ctx.h:
            N.check(self.ctx.lib.gavis_comm_destroy(self.h))
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def vf_allreduce(comm: Comm, field: DeviceField) -> None:
    """In-place sum of a field's coefficients over the ranks (gavis_vf_allreduce)."""
    N.check(comm.ctx.lib.gavis_vf_allreduce(comm.h, field.h))


def construct_field_sharded(comm: Comm, scene, views: Sequence[CameraView], vmf: VmfParams, degree: int,
                            rc: RasterConfig = RasterConfig()) -> DeviceField:
    """construct_field with the views in static blocks over the ranks, partials
    all-reduced by the library over NCCL (gavis_vf_construct_sharded). Collective."""
    ctx = comm.ctx
    ds = _as_dev(ctx, scene)
    arr = cameras_c(views)
    h = C.c_void_p()
    N.check(ctx.lib.gavis_vf_construct_sharded(comm.h, ds.h, arr, C.c_int32(len(views)), C.c_double(vmf.kappa),
                                               C.c_int32(degree), C.byref(raster_c(rc)), C.byref(h)))
    return DeviceField(ctx, ds, h, degree, vmf)


def select_nbv_comm(comm: Comm, scene, field: DeviceField, candidates: Sequence[CameraView],
                    rc: RasterConfig = RasterConfig(), uc: UncertaintyConfig = UncertaintyConfig(),
                    with_rgb: bool = False) -> NbvResult:
    """select_nbv over the full candidate list, each rank scoring its static block,
    scores all-gathered by the library over NCCL (gavis_select_nbv_sharded). Collective."""
    require(len(candidates) > 0, "select_nbv: candidate list must be nonempty")
    ctx = comm.ctx
    ds = _as_dev(ctx, scene)
    scores = np.zeros(len(candidates))
    best = C.c_int32()
    arr = cameras_c(candidates)
    N.check(ctx.lib.gavis_select_nbv_sharded(comm.h, ds.h, field.h, arr, C.c_int32(len(candidates)),
                                             C.byref(raster_c(rc)), C.byref(unc_c(uc)),
                                             C.c_int32(1 if with_rgb else 0), _ptr(scores), C.byref(best)))
    return NbvResult(best.value, scores)


# ------------------------------------------------------------------ planner
def camera_from_c(c: N.Camera) -> CameraView:
    return CameraView(rotation=np.array(list(c.rotation), np.float64).reshape(3, 3),
                      position=np.array(list(c.position), np.float64), width=int(c.width),
                      height=int(c.height), fov_h=float(c.fov_h), fov_v=float(c.fov_v),
                      near=float(c.near_plane))


def _rects_c(occluders: Optional[OccluderSet]):
    rects = occluders.rectangles if occluders is not None else []
    arr = (N.OccluderRectC * max(1, len(rects)))()
    for i, r in enumerate(rects):
        for k in range(3):
            arr[i].corner[k] = float(r.corner[k])
            arr[i].edge_u[k] = float(r.edge_u[k])
            arr[i].edge_v[k] = float(r.edge_v[k])
        arr[i].opaque = 1 if r.opaque else 0
    return arr, len(rects)


def _planner_c(pc: PlannerConfig) -> N.PlannerConfigC:
    return N.PlannerConfigC(int(pc.mode), int(pc.num_candidates), float(pc.se2_height), int(pc.steps),
                            1 if pc.look_inward else 0, int(pc.seed), float(pc.clearance), int(pc.cam_width),
                            int(pc.cam_height), float(pc.fov_h), float(pc.fov_v), float(pc.cam_near))


def sample_candidates(bounds, occluders: Optional[OccluderSet], pc: PlannerConfig, step_seed: int) -> List[CameraView]:
    """sample_candidates (planner.hpp:56-107): host-side rejection sampling in the
    native library (no device needed). bounds = (min[3], max[3])."""
    lib = N.load()
    bmin = np.ascontiguousarray(bounds[0], np.float64)
    bmax = np.ascontiguousarray(bounds[1], np.float64)
    rects, nr = _rects_c(occluders)
    out = (N.Camera * max(1, int(pc.num_candidates)))()
    N.check(lib.gavis_sample_candidates(_ptr(bmin), _ptr(bmax), rects, C.c_int32(nr), C.byref(_planner_c(pc)),
                                        C.c_uint64(int(step_seed) & (2 ** 64 - 1)), out))
    return [camera_from_c(out[i]) for i in range(int(pc.num_candidates))]


def vis_coverage(occluders: OccluderSet, views: Sequence[CameraView]) -> float:
    """vis_coverage (planner.hpp:155-184), host-side in the native library."""
    lib = N.load()
    rects, nr = _rects_c(occluders)
    arr = cameras_c(views)
    cov = C.c_double()
    N.check(lib.gavis_vis_coverage(rects, C.c_int32(nr), C.c_double(float(occluders.sample_density)), arr,
                                   C.c_int32(len(views)), C.byref(cov)))
    return cov.value


def active_mapping(ctx: Context, scene, occluders: Optional[OccluderSet], init: Sequence[CameraView],
                   pc: PlannerConfig, vmf: VmfParams = VmfParams(1.0), field_degree: int = 2,
                   rc: RasterConfig = RasterConfig(), uc: UncertaintyConfig = UncertaintyConfig(),
                   density: Optional["DensityControlConfig"] = None, density_enabled: bool = True,
                   bounds=None) -> MappingLog:
    """run_active_mapping (planner.hpp:284-316): per step density control (reseeded
    with derive_seed(density.seed, step)), field rebuild over the trajectory,
    sample_candidates(derive_seed(pc.seed, step)), select_nbv, append. Device work
    through the C ABI; the loop itself is native (gavis_active_mapping)."""
    ds = _as_dev(ctx, scene)
    density = density or DensityControlConfig()
    bmin, bmax = bounds if bounds is not None else ds.bounds
    bmin = np.ascontiguousarray(bmin, np.float64)
    bmax = np.ascontiguousarray(bmax, np.float64)
    rects, nr = _rects_c(occluders)
    steps, nc = int(pc.steps), int(pc.num_candidates)
    mc = N.MappingConfigC(float(vmf.kappa), int(field_degree), 1 if density_enabled else 0, raster_c(rc), unc_c(uc),
                          N.DensityConfigC(float(density.rho), float(density.eta), float(density.eps_v),
                                           int(density.seed)))
    views = (N.Camera * max(1, steps))()
    idx = np.zeros(max(1, steps), np.int32)
    best = np.zeros(max(1, steps))
    allsc = np.zeros((max(1, steps), nc))
    cov = np.zeros(max(1, steps))
    ment = np.zeros(max(1, steps))
    init_arr = cameras_c(init)
    sd = occluders.sample_density if occluders is not None else 64.0
    N.check(ctx.lib.gavis_active_mapping(ctx.h, ds.h, _ptr(bmin), _ptr(bmax), rects, C.c_int32(nr), C.c_double(sd),
                                         init_arr, C.c_int32(len(init)), C.byref(_planner_c(pc)), C.byref(mc), views,
                                         _ptr(idx), _ptr(best), _ptr(allsc), _ptr(cov), _ptr(ment)))
    log = MappingLog([camera_from_c(views[i]) for i in range(steps)], [])
    for i in range(steps):
        log.steps.append(MappingStep(allsc[i].copy(), int(idx[i]), float(best[i]), float(cov[i]), float(ment[i])))
    return log


# ------------------------------------------------------------------ formats
def load_splat_ply(path: str) -> Scene:
    """load_splat_ply (io.hpp:493-637) -> fp32 SoA scene (host)."""
    lib = N.load()
    n = C.c_int64()
    deg = C.c_int32()
    N.check(lib.gavis_ply_info(path.encode(), C.byref(n), C.byref(deg)))
    nb = (deg.value + 1) ** 2
    k = max(1, n.value)
    pos, rot = np.zeros((k, 3), np.float32), np.zeros((k, 4), np.float32)
    scl, op = np.zeros((k, 3), np.float32), np.zeros(k, np.float32)
    col = np.zeros((k, 3, nb), np.float32)
    bmin, bmax = np.zeros(3), np.zeros(3)
    N.check(lib.gavis_read_splat_ply(path.encode(), C.c_int64(k), _ptr(pos), _ptr(rot), _ptr(scl), _ptr(op),
                                     _ptr(col), _ptr(bmin), _ptr(bmax)))
    m = n.value
    return Scene(pos[:m], rot[:m], scl[:m], op[:m], col[:m], np.zeros(m, np.uint8), deg.value, bmin, bmax)


def save_field_json(path: str, field: VisibilityField, is_virtual=None) -> None:
    """save_field (io.hpp:255-269)."""
    g = np.ascontiguousarray(field.gamma, np.float64)
    v = None if is_virtual is None else np.ascontiguousarray(is_virtual, np.uint8)
    N.check(N.load().gavis_field_json_write(path.encode(), C.c_int32(field.degree), C.c_double(field.vmf.kappa),
                                            C.c_int32(field.num_views), C.c_int64(g.shape[0]), _ptr(g), _ptr(v)))


def load_field_json(path: str) -> VisibilityField:
    """load_field (io.hpp:271-295)."""
    lib = N.load()
    deg, nv, n = C.c_int32(), C.c_int32(), C.c_int64()
    kappa = C.c_double()
    N.check(lib.gavis_field_json_read(path.encode(), C.c_int64(0), C.byref(deg), C.byref(kappa), C.byref(nv),
                                      C.byref(n), None, None))
    nb = (deg.value + 1) ** 2
    g = np.zeros((max(1, n.value), nb))
    v = np.zeros(max(1, n.value), np.uint8)
    N.check(lib.gavis_field_json_read(path.encode(), C.c_int64(max(1, n.value)), C.byref(deg), C.byref(kappa),
                                      C.byref(nv), C.byref(n), _ptr(g), _ptr(v)))
    return VisibilityField(deg.value, VmfParams(kappa.value), nv.value, g[: n.value], v[: n.value])


# ------------------------------------------------------------------ debug
def debug_project(ctx: Context, scene, cam: CameraView, dilation: float = 0.3, tile_size: int = 16):
    ds = _as_dev(ctx, scene)
    n = max(1, ds.n)
    culled = np.zeros(n, np.uint8)
    mean = np.zeros((n, 2))
    conic = np.zeros((n, 3))
    depth = np.zeros(n)
    cover = np.zeros((n, 4), np.int32)
    trect = np.zeros((n, 4), np.int32)
    N.check(ctx.lib.gavis_debug_project(ctx.h, ds.h, C.byref(camera_c(cam)), C.c_double(dilation),
                                        C.c_int32(tile_size), _ptr(culled), _ptr(mean), _ptr(conic),
                                        _ptr(depth), _ptr(cover), _ptr(trect)))
    k = ds.n
    return dict(culled=culled[:k], mean=mean[:k], conic=conic[:k], depth=depth[:k], cover=cover[:k],
                tile_rect=trect[:k])


def debug_binning(ctx: Context, scene, cam: CameraView, rc: RasterConfig = RasterConfig()):
    ds = _as_dev(ctx, scene)
    npairs = C.c_int64()
    N.check(ctx.lib.gavis_debug_binning(ctx.h, ds.h, C.byref(camera_c(cam)), C.byref(raster_c(rc)),
                                        None, None, None, C.byref(npairs)))
    K = npairs.value
    tiles = ((cam.width + rc.tile_size - 1) // rc.tile_size) * ((cam.height + rc.tile_size - 1) // rc.tile_size)
    keys = np.zeros(max(1, K), np.uint64)
    ids = np.zeros(max(1, K), np.int32)
    ranges = np.zeros((tiles, 2), np.int64)
    N.check(ctx.lib.gavis_debug_binning(ctx.h, ds.h, C.byref(camera_c(cam)), C.byref(raster_c(rc)),
                                        _ptr(keys), _ptr(ids), _ptr(ranges), C.byref(npairs)))
    return keys[:K], ids[:K], ranges
