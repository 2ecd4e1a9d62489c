"""Seeded synthetic scenes and camera sets.

The generators follow the reference's deterministic RNG (R/include/gavis/rng.hpp:
mix64 :18-23, derive_seed :26-28, SplitMix64 :30-89), vectorised with numpy:
the k-th draw of a SplitMix64 stream seeded with s is body(s + k * golden).
Values are generated in double and cast to fp32 once; the
device and the CPU oracle consume the same fp32 arrays.

Config 1-5 are BASELINE.json `configs`; the paper's datasets are not in this
container, so these seeded scenes stand in for them with the stated shapes,
sizes and value distributions.
"""
from __future__ import annotations

import math
from typing import List, Tuple

import numpy as np

from .model import K_PI, K_Y00, CameraView, Scene, fibonacci_sphere, make_lookat

_G = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)
_MASK = (1 << 64) - 1


def _body(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _C1
    z = (z ^ (z >> np.uint64(27))) * _C2
    return z ^ (z >> np.uint64(31))


def mix64(x: int) -> int:
    """rng.hpp:18-23"""
    x = (x + 0x9E3779B97F4A7C15) & _MASK
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _MASK
    return x ^ (x >> 31)


def derive_seed(seed: int, stream: int) -> int:
    """rng.hpp:26-28"""
    return mix64(seed ^ mix64((stream + 0x632BE59BD9B4E019) & _MASK))


class SplitMix64:
    """rng.hpp:30-89. Scalar draws for small fixtures; block draws for big scenes."""

    def __init__(self, seed: int):
        self.state = seed & _MASK

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        return z ^ (z >> 31)

    def next_double(self) -> float:
        return float(self.next_u64() >> 11) * (2.0 ** -53)

    def uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.next_double()

    def next_below(self, n: int) -> int:
        return self.next_u64() % n if n else 0

    def normal(self) -> float:
        u1 = self.next_double()
        u2 = self.next_double()
        r = math.sqrt(-2.0 * math.log1p(-u1))
        return r * math.cos(2.0 * K_PI * u2)

    def unit_vector(self) -> Tuple[float, float, float]:
        z = self.uniform(-1.0, 1.0)
        phi = self.uniform(0.0, 2.0 * K_PI)
        s = math.sqrt(max(0.0, 1.0 - z * z))
        return (s * math.cos(phi), s * math.sin(phi), z)

    def rotation(self) -> Tuple[float, float, float, float]:
        """Shoemake; returns (w, x, y, z) in Eigen Quaternion ctor order."""
        u1 = self.next_double()
        u2 = self.next_double()
        u3 = self.next_double()
        a = math.sqrt(1.0 - u1)
        b = math.sqrt(u1)
        return (a * math.sin(2.0 * K_PI * u2), a * math.cos(2.0 * K_PI * u2),
                b * math.sin(2.0 * K_PI * u3), b * math.cos(2.0 * K_PI * u3))

    # ---- vectorised block draws (advance the stream by `count`) ----
    def doubles(self, count: int) -> np.ndarray:
        k = np.arange(1, count + 1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            z = _body(np.uint64(self.state) + k * _G)
        self.state = (self.state + count * 0x9E3779B97F4A7C15) & _MASK
        return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)

    def uniforms(self, lo: float, hi: float, count: int) -> np.ndarray:
        return lo + (hi - lo) * self.doubles(count)

    def normals(self, count: int) -> np.ndarray:
        u = self.doubles(2 * count).reshape(count, 2)
        return np.sqrt(-2.0 * np.log1p(-u[:, 0])) * np.cos(2.0 * K_PI * u[:, 1])

    def rotations(self, count: int) -> np.ndarray:
        u = self.doubles(3 * count).reshape(count, 3)
        a = np.sqrt(1.0 - u[:, 0])
        b = np.sqrt(u[:, 0])
        return np.stack([a * np.sin(2 * K_PI * u[:, 1]), a * np.cos(2 * K_PI * u[:, 1]),
                         b * np.sin(2 * K_PI * u[:, 2]), b * np.cos(2 * K_PI * u[:, 2])], axis=1)


# --------------------------------------------------------------------------
# Reference test fixtures (R/tests/test_raster.cpp:28-43, test_uncertainty.cpp:27-41,
# acceptance_main.cpp:66-83)
# --------------------------------------------------------------------------

def random_scene(seed: int, count: int, white: bool = False, white_value: float = 1.0,
                 dtype=np.float32) -> Scene:
    """test_raster.cpp:28-43: positions U[-1.5,1.5]^2 x U[2,6], scales U[0.02,0.3],
    Shoemake rotation, opacity U[0.1,0.95], DC color U[0,1]/Y00 (or white_value/Y00)."""
    g = SplitMix64(seed)
    parts = []
    for _ in range(count):
        pos = (g.uniform(-1.5, 1.5), g.uniform(-1.5, 1.5), g.uniform(2.0, 6.0))
        scale = (g.uniform(0.02, 0.3), g.uniform(0.02, 0.3), g.uniform(0.02, 0.3))
        rot = g.rotation()
        opacity = g.uniform(0.1, 0.95)
        col = [[(white_value if white else g.uniform(0.0, 1.0)) / K_Y00] for _ in range(3)]
        parts.append(dict(pos=pos, scale=scale, rot=rot, opacity=opacity, color_sh=col))
    return Scene.from_particles(parts, 0, bounds=((-2, -2, 1), (2, 2, 7)), dtype=dtype)


def make_particle(pos, scale, opacity, color, rot=(1.0, 0.0, 0.0, 0.0)) -> dict:
    """test_raster.cpp:18-26 make_particle: DC color = color/Y00."""
    return dict(pos=pos, scale=scale, opacity=opacity, rot=rot,
                color_sh=[[color[k] / K_Y00] for k in range(3)])


def z_camera(width: int = 64, height: int = 64) -> CameraView:
    """test_raster.cpp:45-47"""
    return make_lookat((0, 0, 0), (0, 0, 1), (0, 1, 0), width, height)


def wall_scene(dtype=np.float32) -> Scene:
    """test_vfield.cpp:44-52: 5x5 wall of opaque particles in the x = 1 plane."""
    parts = []
    for i in range(5):
        for j in range(5):
            parts.append(dict(pos=(1.0, 0.3 + 0.1 * i, 0.3 + 0.1 * j), scale=0.06, opacity=0.9,
                              color_sh=[[0.62 / K_Y00]] * 3))
    return Scene.from_particles(parts, 0, bounds=((0, 0, 0), (2, 1, 1)), dtype=dtype)


# --------------------------------------------------------------------------
# BASELINE.json configs
# --------------------------------------------------------------------------

def _gaussian_cloud(seed: int, n: int, pos_lo, pos_hi, log_mu: float, log_sigma: float,
                    color_degree: int = 3) -> Scene:
    """Configs 1/2: positions uniform in a box, log-scales N(mu, sigma) per axis, uniform
    unit quaternions, opacity sigmoid(N(0,1.5)), SH colour N(0, 0.3). One derive_seed
    stream per attribute."""
    nb = (color_degree + 1) ** 2
    pos = np.empty((n, 3))
    sp = SplitMix64(derive_seed(seed, 1)).doubles(3 * n).reshape(n, 3)
    lo = np.asarray(pos_lo, np.float64)
    hi = np.asarray(pos_hi, np.float64)
    pos[:] = lo + (hi - lo) * sp
    scales = np.exp(log_mu + log_sigma * SplitMix64(derive_seed(seed, 2)).normals(3 * n)).reshape(n, 3)
    rots = SplitMix64(derive_seed(seed, 3)).rotations(n)
    op = 1.0 / (1.0 + np.exp(-1.5 * SplitMix64(derive_seed(seed, 4)).normals(n)))
    col = 0.3 * SplitMix64(derive_seed(seed, 5)).normals(3 * nb * n).reshape(n, 3, nb)
    return Scene(pos.astype(np.float32), rots.astype(np.float32), scales.astype(np.float32),
                 op.astype(np.float32), col.astype(np.float32), np.zeros(n, np.uint8),
                 color_degree, lo.copy(), hi.copy())


def _lookat_many(positions: np.ndarray, targets: np.ndarray, w: int, h: int, fov_h: float,
                 fov_v: float) -> List[CameraView]:
    return [make_lookat(p, t, (0, 0, 1), w, h, fov_h, fov_v) for p, t in zip(positions, targets)]


def _sphere_candidates(seed: int, n: int, r_lo: float, r_hi: float, w: int, h: int,
                       fov: float) -> List[CameraView]:
    g = SplitMix64(seed)
    cams = []
    for _ in range(n):
        d = g.unit_vector()
        r = g.uniform(r_lo, r_hi)
        cams.append(make_lookat((d[0] * r, d[1] * r, d[2] * r), (0, 0, 0), (0, 0, 1), w, h, fov, fov))
    return cams


def config1(seed: int = 0):
    """10k Gaussians in [-1,1]^3, log-scale N(-4,0.5); 16 Fibonacci views r=3 256^2 fov 60;
    VF degree 2; 32 candidates r in [2.5,3.5]."""
    scene = _gaussian_cloud(seed, 10_000, (-1, -1, -1), (1, 1, 1), -4.0, 0.5)
    dirs = fibonacci_sphere(16) * 3.0
    train = _lookat_many(dirs, np.zeros_like(dirs), 256, 256, K_PI / 3, K_PI / 3)
    cands = _sphere_candidates(derive_seed(seed, 6), 32, 2.5, 3.5, 256, 256, K_PI / 3)
    return dict(name="config1", scene=scene, train=train, candidates=cands, degree=2)


def config2(seed: int = 0, n: int = 500_000, n_candidates: int = 256, res: int = 800):
    """500k Gaussians in [-1.5,1.5]^3, log-scale N(-5,0.5); 100 upper-hemisphere views r=4
    800^2 fov 60; VF degree 3; 256 full-sphere candidates r=4."""
    scene = _gaussian_cloud(seed, n, (-1.5, -1.5, -1.5), (1.5, 1.5, 1.5), -5.0, 0.5)
    dirs = fibonacci_sphere(200)[:100] * 4.0  # z > 0 half
    train = _lookat_many(dirs, np.zeros_like(dirs), res, res, K_PI / 3, K_PI / 3)
    cands = _sphere_candidates(derive_seed(seed, 6), n_candidates, 4.0, 4.0, res, res, K_PI / 3)
    return dict(name="config2", scene=scene, train=train, candidates=cands, degree=3)


def _quat_from_matrix(R: np.ndarray) -> np.ndarray:
    """Rotation matrices (n,3,3) -> quaternions (w,x,y,z), Shepperd's method."""
    n = R.shape[0]
    q = np.empty((n, 4))
    tr = R[:, 0, 0] + R[:, 1, 1] + R[:, 2, 2]
    w = np.sqrt(np.maximum(0.0, 1.0 + tr)) / 2
    x = np.sqrt(np.maximum(0.0, 1.0 + R[:, 0, 0] - R[:, 1, 1] - R[:, 2, 2])) / 2
    y = np.sqrt(np.maximum(0.0, 1.0 - R[:, 0, 0] + R[:, 1, 1] - R[:, 2, 2])) / 2
    z = np.sqrt(np.maximum(0.0, 1.0 - R[:, 0, 0] - R[:, 1, 1] + R[:, 2, 2])) / 2
    q[:, 0] = w
    q[:, 1] = np.copysign(x, R[:, 2, 1] - R[:, 1, 2])
    q[:, 2] = np.copysign(y, R[:, 0, 2] - R[:, 2, 0])
    q[:, 3] = np.copysign(z, R[:, 1, 0] - R[:, 0, 1])
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def _room_poses(g: SplitMix64, n: int, x_lo: float, x_hi: float, w: int, h: int,
                fov: float) -> List[CameraView]:
    cams = []
    for _ in range(n):
        p = (g.uniform(x_lo, x_hi), g.uniform(0.5, 3.5), g.uniform(1.2, 1.8))
        yaw = g.uniform(0.0, 2.0 * K_PI)
        pitch = g.uniform(-20.0, 20.0) * K_PI / 180.0
        f = (math.cos(pitch) * math.cos(yaw), math.cos(pitch) * math.sin(yaw), math.sin(pitch))
        cams.append(make_lookat(p, (p[0] + f[0], p[1] + f[1], p[2] + f[2]), (0, 0, 1), w, h,
                                fov, fov))
    return cams


def config3(seed: int = 0, n: int = 1_000_000, n_train: int = 150, n_candidates: int = 1024,
            res: int = 800):
    """Two 6x4x3 rooms joined by a 1 m doorway; 85% flattened wall/floor/ceiling slab
    Gaussians (thin log-scale N(-7,0.3), in-plane N(-4.5,0.4)), 15% clutter inside;
    150 training views in room A (yaw U, pitch +-20 deg, height 1.2-1.8, fov 90);
    1024 candidates spanning both rooms; VF degree 2 (ref default), colour degree 3."""
    nb = 16
    sx, sy, sz = 6.0, 4.0, 3.0
    door_lo, door_hi = 0.5 * (sy - 1.0), 0.5 * (sy + 1.0)
    # faces: corner, edge_u, edge_v, normal axis
    faces = [((0, 0, 0), (2 * sx, 0, 0), (0, sy, 0)), ((0, 0, sz), (2 * sx, 0, 0), (0, sy, 0)),
             ((0, 0, 0), (0, sy, 0), (0, 0, sz)), ((2 * sx, 0, 0), (0, sy, 0), (0, 0, sz)),
             ((0, 0, 0), (2 * sx, 0, 0), (0, 0, sz)), ((0, sy, 0), (2 * sx, 0, 0), (0, 0, sz)),
             ((sx, 0, 0), (0, sy, 0), (0, 0, sz))]
    areas = np.array([np.linalg.norm(np.cross(u, v)) for _, u, v in faces])
    areas[6] *= (sy - 1.0) / sy  # doorway removed from the shared wall
    n_wall = int(n * 0.85)
    n_clut = n - n_wall
    g = SplitMix64(derive_seed(seed, 11))
    face_u = g.doubles(n_wall)
    cum = np.cumsum(areas) / areas.sum()
    face = np.searchsorted(cum, face_u, side="right").clip(0, 6)
    uv = g.doubles(2 * n_wall).reshape(n_wall, 2)
    corner = np.array([f[0] for f in faces], np.float64)
    eu = np.array([f[1] for f in faces], np.float64)
    ev = np.array([f[2] for f in faces], np.float64)
    # shared wall: remap u so it skips the doorway gap
    shared = face == 6
    u = uv[:, 0].copy()
    width_ok = (sy - 1.0) / sy
    su = u[shared] * width_ok
    u[shared] = np.where(su < door_lo / sy, su, su + 1.0 / sy)
    pos_w = corner[face] + eu[face] * u[:, None] + ev[face] * uv[:, 1:2]
    normals = np.cross(eu, ev)
    normals /= np.linalg.norm(normals, axis=1, keepdims=True)
    nrm = normals[face]
    # frame: local z -> face normal, random spin about it
    spin = g.doubles(n_wall) * 2 * K_PI
    tu = eu[face] / np.linalg.norm(eu[face], axis=1, keepdims=True)
    tv = np.cross(nrm, tu)
    c, s = np.cos(spin)[:, None], np.sin(spin)[:, None]
    ax = c * tu + s * tv
    ay = -s * tu + c * tv
    Rw = np.stack([ax, ay, nrm], axis=2)  # columns
    qw = _quat_from_matrix(Rw)
    ls = SplitMix64(derive_seed(seed, 12))
    sc_w = np.empty((n_wall, 3))
    sc_w[:, 0:2] = np.exp(-4.5 + 0.4 * ls.normals(2 * n_wall).reshape(n_wall, 2))
    sc_w[:, 2] = np.exp(-7.0 + 0.3 * ls.normals(n_wall))
    gc = SplitMix64(derive_seed(seed, 13))
    pos_c = np.stack([gc.uniforms(0.1, 2 * sx - 0.1, n_clut), gc.uniforms(0.1, sy - 0.1, n_clut),
                      gc.uniforms(0.1, sz - 0.1, n_clut)], axis=1)
    qc = gc.rotations(n_clut)
    sc_c = np.exp(-4.5 + 0.4 * gc.normals(3 * n_clut)).reshape(n_clut, 3)
    pos = np.concatenate([pos_w, pos_c]).astype(np.float32)
    rot = np.concatenate([qw, qc]).astype(np.float32)
    sc = np.concatenate([sc_w, sc_c]).astype(np.float32)
    op = (1.0 / (1.0 + np.exp(-1.5 * SplitMix64(derive_seed(seed, 4)).normals(n)))).astype(np.float32)
    col = (0.3 * SplitMix64(derive_seed(seed, 5)).normals(3 * nb * n)).astype(np.float32).reshape(n, 3, nb)
    scene = Scene(pos, rot, sc, op, col, np.zeros(n, np.uint8), 3, np.array([0.0, 0, 0]),
                  np.array([2 * sx, sy, sz]))
    gp = SplitMix64(derive_seed(seed, 14))
    train = _room_poses(gp, n_train, 0.5, sx - 0.5, res, res, K_PI / 2)
    cands = _room_poses(SplitMix64(derive_seed(seed, 15)), n_candidates, 0.5, 2 * sx - 0.5, res,
                        res, K_PI / 2)
    return dict(name="config3", scene=scene, train=train, candidates=cands, degree=2)


def _catmull_rom(pts: np.ndarray, samples: int) -> Tuple[np.ndarray, np.ndarray]:
    """Uniform Catmull-Rom through pts; returns positions and unit tangents."""
    p = np.concatenate([pts[:1], pts, pts[-1:]])
    segs = len(pts) - 1
    t = np.linspace(0, segs, samples, endpoint=False)
    i = np.floor(t).astype(int)
    u = (t - i)[:, None]
    p0, p1, p2, p3 = p[i], p[i + 1], p[i + 2], p[i + 3]
    pos = 0.5 * ((2 * p1) + (-p0 + p2) * u + (2 * p0 - 5 * p1 + 4 * p2 - p3) * u ** 2 +
                 (-p0 + 3 * p1 - 3 * p2 + p3) * u ** 3)
    tan = 0.5 * ((-p0 + p2) + 2 * (2 * p0 - 5 * p1 + 4 * p2 - p3) * u +
                 3 * (-p0 + 3 * p1 - 3 * p2 + p3) * u ** 2)
    tan /= np.maximum(np.linalg.norm(tan, axis=1, keepdims=True), 1e-12)
    return pos, tan


def config4(seed: int = 0, n: int = 3_000_000, n_train: int = 300, n_candidates: int = 512,
            width: int = 1920, height: int = 1080):
    """64 anisotropic clusters in a 40x40x10 volume, log-scale N(-4,0.6), SH degree 3;
    300 views 1920x1080 along a Catmull-Rom path through 30 waypoints (fov_h 60, fy=fx);
    VF degree 3; 512 candidates at 1080p."""
    nb = 16
    g = SplitMix64(derive_seed(seed, 21))
    centers = np.stack([g.uniforms(-20, 20, 64), g.uniforms(-20, 20, 64), g.uniforms(0, 10, 64)], 1)
    axes_sd = g.uniforms(0.5, 4.0, 3 * 64).reshape(64, 3)
    qs = g.rotations(64)
    w, x, y, z = qs.T
    R = np.stack([np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
                  np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
                  np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1)], 1)
    cl = (g.doubles(n) * 64).astype(int).clip(0, 63)
    eps = SplitMix64(derive_seed(seed, 22)).normals(3 * n).reshape(n, 3) * axes_sd[cl]
    pos = centers[cl] + np.einsum("nij,nj->ni", R[cl], eps)
    scales = np.exp(-4.0 + 0.6 * SplitMix64(derive_seed(seed, 2)).normals(3 * n)).reshape(n, 3)
    rots = SplitMix64(derive_seed(seed, 3)).rotations(n)
    op = 1.0 / (1.0 + np.exp(-1.5 * SplitMix64(derive_seed(seed, 4)).normals(n)))
    col = (0.3 * SplitMix64(derive_seed(seed, 5)).normals(3 * nb * n)).astype(np.float32).reshape(n, 3, nb)
    scene = Scene(pos.astype(np.float32), rots.astype(np.float32), scales.astype(np.float32),
                  op.astype(np.float32), col, np.zeros(n, np.uint8), 3,
                  np.array([-20.0, -20, 0]), np.array([20.0, 20, 10]))
    fov_h = K_PI / 3
    fov_v = 2.0 * math.atan(math.tan(0.5 * fov_h) * height / width)
    gw = SplitMix64(derive_seed(seed, 23))
    way = np.stack([gw.uniforms(-18, 18, 30), gw.uniforms(-18, 18, 30), gw.uniforms(2, 8, 30)], 1)
    tp, tt = _catmull_rom(way, n_train)
    train = _lookat_many(tp, tp + tt, width, height, fov_h, fov_v)
    gc = SplitMix64(derive_seed(seed, 24))
    cands = []
    for _ in range(n_candidates):
        p = (gc.uniform(-18, 18), gc.uniform(-18, 18), gc.uniform(2, 8))
        yaw = gc.uniform(0, 2 * K_PI)
        pitch = gc.uniform(-20, 20) * K_PI / 180
        f = (math.cos(pitch) * math.cos(yaw), math.cos(pitch) * math.sin(yaw), math.sin(pitch))
        cands.append(make_lookat(p, (p[0] + f[0], p[1] + f[1], p[2] + f[2]), (0, 0, 1), width,
                                 height, fov_h, fov_v))
    return dict(name="config4", scene=scene, train=train, candidates=cands, degree=3)


def config5(seed: int = 0, n_candidates: int = 4096, res: int = 400):
    """Active-mapping sweep on the config-2 scene (800^2 training views): candidates at 400^2."""
    c = config2(seed, n_candidates=0)
    c["candidates"] = _sphere_candidates(derive_seed(seed, 7), n_candidates, 4.0, 4.0, res, res,
                                         K_PI / 3)
    c["name"] = "config5"
    c["rounds"] = 20
    return c


CONFIGS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}
