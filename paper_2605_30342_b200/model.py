"""Host-side data model mirroring the reference's C++ types.

Mirrors R/include/gavis/model.hpp (GaussianParticle :34-46, CameraView :66-105,
make_lookat :107-128, Scene :130-134), R/include/gavis/raster.hpp:21-35
(RasterConfig), sh.hpp:121-129 (VmfParams), uncertainty.hpp:24-52
(UncertaintyConfig) and the error taxonomy of common.hpp:25-46.

The scene is held as a structure of arrays (what the device consumes): fp32
positions/rotations/scales/opacities/colors plus a uint8 virtual mask.
Cameras stay in double like the reference's CameraView.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

K_PI = 3.14159265358979323846
K_Y00 = 0.28209479177387814  # sh.hpp:28
K_GAUSS_ENTROPY = 4.256815599614018  # uncertainty.hpp:19
K_MAX_SH_DEGREE = 20


class ParameterError(RuntimeError):
    """common.hpp:25-28 -- bad input (CLI exit code 2)."""


class InvariantError(RuntimeError):
    """common.hpp:30-33 -- broken internal invariant (exit code 3)."""


class OracleError(RuntimeError):
    """common.hpp:35-38 -- failed certification (exit code 4)."""


class DeviceError(RuntimeError):
    """CUDA / NCCL failure inside the native library (status 5)."""


def require(cond: bool, msg: str) -> None:
    if not cond:
        raise ParameterError(msg)


@dataclass
class RasterConfig:
    """raster.hpp:21-35"""
    tile_size: int = 16
    transmittance_cutoff: float = 1e-4
    dilation: float = 0.3
    alpha_clamp_max: float = 0.99

    def validate(self) -> None:
        require(self.tile_size >= 1, "tile_size must be at least 1")
        require(0.0 < self.transmittance_cutoff < 1.0, "transmittance_cutoff must lie in (0, 1)")
        require(self.dilation >= 0.0, "dilation must be non-negative")
        require(0.0 < self.alpha_clamp_max <= 1.0, "alpha_clamp_max must lie in (0, 1]")


@dataclass
class VmfParams:
    """sh.hpp:121-129: zeta = exp(-kappa)."""
    kappa: float = 1.0

    def __post_init__(self) -> None:
        require(0.0 <= self.kappa <= 50.0, "vmf kappa must lie in [0, 50]")

    @property
    def zeta(self) -> float:
        return math.exp(-self.kappa)


@dataclass
class UncertaintyConfig:
    """uncertainty.hpp:24-52. variance_provider 0 = kConstant, 1 = kShPropagation
    (coefficient variances attached to the scene); correlation 0 = kNone, 1 = kHook."""
    beta: float = 0.5
    prior_opacity: float = 0.15
    color_sigma: float = 0.1
    prior_cov: np.ndarray = field(default_factory=lambda: np.eye(3))
    variance_provider: int = 0
    correlation: int = 0
    correlation_lambda: float = 1.0


@dataclass
class CameraView:
    """model.hpp:66-105. rotation columns = camera x (right), y (down), z (forward)."""
    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    position: np.ndarray = field(default_factory=lambda: np.zeros(3))
    width: int = 128
    height: int = 128
    fov_h: float = K_PI / 2.0
    fov_v: float = K_PI / 2.0
    near: float = 0.05

    def focal_x(self) -> float:
        return 0.5 * self.width / math.tan(0.5 * self.fov_h)

    def focal_y(self) -> float:
        return 0.5 * self.height / math.tan(0.5 * self.fov_v)

    def validate(self) -> None:
        require(self.width >= 1 and self.height >= 1, "camera image size must be at least 1x1")
        require(0.0 < self.fov_h < K_PI and 0.0 < self.fov_v < K_PI, "camera fov must lie in (0, pi)")
        require(self.near > 0.0, "camera near plane must be positive")


def _cross(a: Sequence[float], b: Sequence[float]) -> List[float]:
    return [a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]]


def _norm(a: Sequence[float]) -> float:
    return math.sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2])


def make_lookat(position, target, up=(0.0, 0.0, 1.0), width: int = 128, height: int = 128,
                fov_h: float = K_PI / 2.0, fov_v: float = K_PI / 2.0) -> CameraView:
    """model.hpp:107-128 in double precision, same operation order."""
    p = [float(v) for v in position]
    t = [float(v) for v in target]
    u = [float(v) for v in up]
    forward = [t[0] - p[0], t[1] - p[1], t[2] - p[2]]
    require(_norm(forward) > 1e-12, "lookat target coincides with position")
    n = _norm(forward)
    forward = [c / n for c in forward]
    right = _cross(forward, u)
    if _norm(right) < 1e-9:
        right = _cross(forward, [1.0, 0.0, 0.0])
    n = _norm(right)
    right = [c / n for c in right]
    down = _cross(forward, right)
    rot = np.array([[right[i], down[i], forward[i]] for i in range(3)], dtype=np.float64)
    return CameraView(rotation=rot, position=np.array(p, dtype=np.float64), width=width,
                      height=height, fov_h=fov_h, fov_v=fov_v)


def fibonacci_sphere(n: int) -> np.ndarray:
    """oracle.hpp:22-34"""
    require(n >= 1, "fibonacci_sphere: need at least one direction")
    golden = K_PI * (3.0 - math.sqrt(5.0))
    out = np.zeros((n, 3))
    for i in range(n):
        z = 1.0 - 2.0 * (i + 0.5) / n
        r = math.sqrt(max(0.0, 1.0 - z * z))
        phi = golden * i
        out[i] = (r * math.cos(phi), r * math.sin(phi), z)
    return out


@dataclass
class Scene:
    """Structure-of-arrays scene (model.hpp:130-134 + GaussianParticle :34-46).

    positions (N,3), rotations (N,4) as (w,x,y,z), scales (N,3), opacities (N,),
    colors (N,3,(Lc+1)^2) channel-major per particle, is_virtual (N,) uint8.
    """
    positions: np.ndarray
    rotations: np.ndarray
    scales: np.ndarray
    opacities: np.ndarray
    colors: np.ndarray
    is_virtual: np.ndarray
    color_degree: int = 0
    bounds_min: np.ndarray = field(default_factory=lambda: np.zeros(3))
    bounds_max: np.ndarray = field(default_factory=lambda: np.zeros(3))

    @property
    def num_particles(self) -> int:
        return int(self.positions.shape[0])

    @staticmethod
    def empty(color_degree: int = 0) -> "Scene":
        nb = (color_degree + 1) ** 2
        return Scene(np.zeros((0, 3), np.float32), np.zeros((0, 4), np.float32),
                     np.zeros((0, 3), np.float32), np.zeros((0,), np.float32),
                     np.zeros((0, 3, nb), np.float32), np.zeros((0,), np.uint8), color_degree)

    @staticmethod
    def from_particles(particles: Sequence[dict], color_degree: int = 0, bounds=None,
                       dtype=np.float32) -> "Scene":
        """particles: dicts with pos, rot (w,x,y,z; default identity), scale (scalar or 3),
        opacity, color_sh (3 x nb list), virtual. dtype=float64 keeps the exact reference
        values (used to pin the CPU oracle); the device always receives fp32."""
        nb = (color_degree + 1) ** 2
        n = len(particles)
        s = Scene(np.zeros((n, 3), dtype), np.zeros((n, 4), dtype),
                  np.zeros((n, 3), dtype), np.zeros((n,), dtype),
                  np.zeros((n, 3, nb), dtype), np.zeros((n,), np.uint8), color_degree)
        for i, p in enumerate(particles):
            s.positions[i] = p["pos"]
            s.rotations[i] = p.get("rot", (1.0, 0.0, 0.0, 0.0))
            sc = p.get("scale", 1.0)
            s.scales[i] = sc if np.ndim(sc) else (sc, sc, sc)
            s.opacities[i] = p.get("opacity", 0.0)
            col = np.asarray(p.get("color_sh", np.zeros((3, nb))), dtype=np.float64)
            s.colors[i, :, : col.shape[1]] = col
            s.is_virtual[i] = 1 if p.get("virtual", False) else 0
        if bounds is not None:
            s.bounds_min = np.asarray(bounds[0], np.float64)
            s.bounds_max = np.asarray(bounds[1], np.float64)
        return s

    def subset(self, idx) -> "Scene":
        return Scene(self.positions[idx], self.rotations[idx], self.scales[idx],
                     self.opacities[idx], self.colors[idx], self.is_virtual[idx],
                     self.color_degree, self.bounds_min, self.bounds_max)

    def as_f32(self) -> "Scene":
        """The fp32 scene the device consumes (identity for an fp32 scene)."""
        return self.contiguous()

    def contiguous(self) -> "Scene":
        return Scene(np.ascontiguousarray(self.positions, np.float32),
                     np.ascontiguousarray(self.rotations, np.float32),
                     np.ascontiguousarray(self.scales, np.float32),
                     np.ascontiguousarray(self.opacities, np.float32),
                     np.ascontiguousarray(self.colors, np.float32),
                     np.ascontiguousarray(self.is_virtual, np.uint8),
                     self.color_degree, self.bounds_min, self.bounds_max)


@dataclass
class VisibilityField:
    """vfield.hpp:21-33 host copy: gamma (N, (L+1)^2) float64 row-major."""
    degree: int
    vmf: VmfParams
    num_views: int
    gamma: np.ndarray
    virtual_mask: np.ndarray

    @property
    def num_particles(self) -> int:
        return int(self.gamma.shape[0])

    def basis_size(self) -> int:
        return (self.degree + 1) ** 2


@dataclass
class EntropyMap:
    """uncertainty.hpp:85-89"""
    width: int
    height: int
    entropy: np.ndarray
    invisible_mass: np.ndarray


@dataclass
class RenderOutput:
    """raster.hpp:166-171"""
    width: int
    height: int
    color: np.ndarray
    depth: np.ndarray
    transmittance: np.ndarray


@dataclass
class ViewQuery:
    """vfield.hpp:114-117"""
    particle_indices: np.ndarray
    visibilities: np.ndarray


@dataclass
class NbvResult:
    """planner.hpp:109-112"""
    best_index: int
    scores: np.ndarray


@dataclass
class OccluderRect:
    """model.hpp:141-150: corner + u edge_u + v edge_v, u, v in [0, 1]."""
    corner: Sequence[float] = (0.0, 0.0, 0.0)
    edge_u: Sequence[float] = (1.0, 0.0, 0.0)
    edge_v: Sequence[float] = (0.0, 1.0, 0.0)
    opaque: bool = True


@dataclass
class OccluderSet:
    """model.hpp:152-155"""
    rectangles: List[OccluderRect] = field(default_factory=list)
    sample_density: float = 64.0  # surface samples per unit area


@dataclass
class PlannerConfig:
    """planner.hpp:24-42; mode 0 = kSe3, 1 = kSe2."""
    mode: int = 0
    num_candidates: int = 128
    se2_height: float = 1.5
    steps: int = 10
    seed: int = 0
    look_inward: bool = True
    clearance: float = 0.1
    cam_width: int = 128
    cam_height: int = 128
    fov_h: float = K_PI / 2.0
    fov_v: float = K_PI / 2.0
    cam_near: float = 0.05

    def validate(self) -> None:
        require(self.num_candidates >= 1, "num_candidates must be at least 1")
        require(self.steps >= 0, "steps must be non-negative")


@dataclass
class MappingStep:
    """planner.hpp:264-270"""
    scores: np.ndarray
    chosen_index: int
    score: float
    vis_coverage: float
    mean_entropy: float


@dataclass
class MappingLog:
    """planner.hpp:272-275"""
    chosen_views: List[CameraView]
    steps: List[MappingStep]
