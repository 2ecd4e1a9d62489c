"""ctypes binding of libgavis_b200.so (the C ABI in include/gavis_b200.h).

There is no fallback: if the library is missing or a CUDA device is absent the
calls raise. The library is built in-tree by paper_2605_30342_b200.build.
"""
from __future__ import annotations

import ctypes as C
import os

from .model import DeviceError, InvariantError, OracleError, ParameterError

_PKG = os.path.dirname(os.path.abspath(__file__))
# GAVIS_LIB_PATH: an A/B build of the same sources with other compile-time knobs
# (python -m paper_2605_30342_b200.build --variant NAME -DKNOB=V)
LIB_PATH = os.environ.get("GAVIS_LIB_PATH") or os.path.join(_PKG, "libgavis_b200.so")


class Camera(C.Structure):
    _fields_ = [("rotation", C.c_double * 9), ("position", C.c_double * 3), ("width", C.c_int32),
                ("height", C.c_int32), ("fov_h", C.c_double), ("fov_v", C.c_double),
                ("near_plane", C.c_double)]


class RasterConfigC(C.Structure):
    _fields_ = [("tile_size", C.c_int32), ("_pad", C.c_int32), ("transmittance_cutoff", C.c_double),
                ("dilation", C.c_double), ("alpha_clamp_max", C.c_double)]


class UncertaintyConfigC(C.Structure):
    _fields_ = [("beta", C.c_double), ("prior_opacity", C.c_double), ("color_sigma", C.c_double),
                ("prior_cov", C.c_double * 9), ("variance_provider", C.c_int32),
                ("correlation", C.c_int32), ("correlation_lambda", C.c_double)]


class SceneDesc(C.Structure):
    _fields_ = [("num_particles", C.c_int64), ("color_degree", C.c_int32), ("_pad", C.c_int32),
                ("positions", C.c_void_p), ("rotations", C.c_void_p), ("scales", C.c_void_p),
                ("opacities", C.c_void_p), ("colors", C.c_void_p), ("is_virtual", C.c_void_p)]


class RenderOutputs(C.Structure):
    _fields_ = [("rgb", C.c_void_p), ("depth", C.c_void_p), ("transmittance", C.c_void_p),
                ("entropy", C.c_void_p), ("invisible_mass", C.c_void_p),
                ("entropy_depth", C.c_void_p), ("scores", C.c_void_p),
                ("rgb_contributors", C.c_void_p), ("entropy_contributors", C.c_void_p),
                ("with_rgb", C.c_int32), ("with_entropy", C.c_int32)]


class DensityConfigC(C.Structure):
    _fields_ = [("rho", C.c_double), ("eta", C.c_double), ("eps_v", C.c_double), ("seed", C.c_uint64)]


class OccluderRectC(C.Structure):
    _fields_ = [("corner", C.c_double * 3), ("edge_u", C.c_double * 3), ("edge_v", C.c_double * 3),
                ("opaque", C.c_int32), ("_pad", C.c_int32)]


class PlannerConfigC(C.Structure):
    _fields_ = [("mode", C.c_int32), ("num_candidates", C.c_int32), ("se2_height", C.c_double),
                ("steps", C.c_int32), ("look_inward", C.c_int32), ("seed", C.c_uint64),
                ("clearance", C.c_double), ("cam_width", C.c_int32), ("cam_height", C.c_int32),
                ("fov_h", C.c_double), ("fov_v", C.c_double), ("cam_near", C.c_double)]


class MappingConfigC(C.Structure):
    _fields_ = [("kappa", C.c_double), ("field_degree", C.c_int32), ("density_enabled", C.c_int32),
                ("raster", RasterConfigC), ("uncertainty", UncertaintyConfigC),
                ("density", DensityConfigC)]


# Every symbol include/gavis_b200.h declares (checked by tests/test_abi_symbols.py).
EXPORTS = [
    "gavis_abi_version", "gavis_last_error", "gavis_ctx_create", "gavis_ctx_destroy",
    "gavis_ctx_synchronize", "gavis_ctx_set_batch", "gavis_ctx_set_pair_budget", "gavis_ctx_set_precision",
    "gavis_ctx_get_counters", "gavis_ctx_last_score_bounds", "gavis_ctx_set_profiling",
    "gavis_ctx_kernel_time", "gavis_ctx_timer_start", "gavis_ctx_timer_stop",
    "gavis_ctx_launch_count", "gavis_scene_upload", "gavis_scene_destroy",
    "gavis_scene_set_coeff_variances",
    "gavis_scene_num_particles", "gavis_vf_construct", "gavis_vf_create",
    "gavis_vf_accumulate_views", "gavis_vf_accumulate_visibility", "gavis_vf_upload",
    "gavis_vf_download", "gavis_vf_set_num_views", "gavis_vf_device_gamma", "gavis_vf_destroy",
    "gavis_single_view_visibility", "gavis_vf_query", "gavis_vf_query_view", "gavis_ua_render", "gavis_ua_mixtures",
    "gavis_select_nbv", "gavis_nbv_loop", "gavis_comm_unique_id", "gavis_comm_create", "gavis_comm_adopt",
    "gavis_comm_destroy", "gavis_vf_allreduce", "gavis_vf_construct_sharded", "gavis_select_nbv_sharded", "gavis_density_control", "gavis_sample_candidates",
    "gavis_vis_coverage", "gavis_active_mapping", "gavis_ply_info",
    "gavis_read_splat_ply", "gavis_field_json_write", "gavis_field_json_read", "gavis_debug_project", "gavis_debug_binning",
]

COMM_ID_BYTES = 128
PRECISION_CERTIFIED = 0
PRECISION_EXACT = 1

_lib = None


def load() -> C.CDLL:
    """Load the native library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2605_30342_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    lib.gavis_last_error.restype = C.c_char_p
    lib.gavis_abi_version.restype = C.c_int
    for name in EXPORTS:
        fn = getattr(lib, name)
        if name not in ("gavis_last_error", "gavis_abi_version"):
            fn.restype = C.c_int
    _lib = lib
    return lib


def check(status: int) -> None:
    if status == 0:
        return
    msg = load().gavis_last_error().decode("utf-8", "replace")
    if status == 2:
        raise ParameterError(msg)
    if status == 3:
        raise InvariantError(msg)
    if status == 4:
        raise OracleError(msg)
    raise DeviceError(msg)
