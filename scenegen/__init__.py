"""Seeded synthetic scene and camera generators (shared by the oracle tests, the GPU
parity tests and bench.py).

This module holds NONE of the method's arithmetic: no projection, no covariance, no
blending, no sorting. It only draws Gaussian parameters and camera poses with numpy
`default_rng(seed)` and returns plain float32 arrays in the layout the C ABI takes
(include/rade.h):

    means      float32 [3][N]        world-space centres x_c
    scales     float32 [3][N]        activated per-axis std-devs > 0  (S)
    rotations  float32 [4][N]        raw quaternion (w, x, y, z)      (R)
    opacities  float32 [N]           activated opacity in (0, 1)
    sh         float32 [K][3][N]     SH coefficients, K = (deg+1)^2

Cameras are pinhole, world->camera rotation R (row-major) and translation t, +z forward,
+y down (SURVEY.md §8(b) rd_camera).

The recipes follow SURVEY.md §8(d): the paper gives no
Gaussian counts or distributions, so these are our choices and are printed with every
bench number.
"""
from __future__ import annotations

from dataclasses import dataclass, field
import numpy as np

SH_DEGREE = 3


@dataclass
class Camera:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    R: np.ndarray  # float32 (3,3) world->camera, row-major
    t: np.ndarray  # float32 (3,)
    znear: float = 0.2

    def as_dict(self):
        return dict(fx=self.fx, fy=self.fy, cx=self.cx, cy=self.cy, width=self.width,
                    height=self.height, R=self.R.tolist(), t=self.t.tolist(), znear=self.znear)


@dataclass
class Options:
    """Render options passed as INPUTS to both sides (values fixed by DESIGN.md readings
    S1, S5, S8, S9; SURVEY.md §8(b) rd_options defaults)."""
    tile: int = 16
    alpha_min: float = 1.0 / 255.0
    alpha_max: float = 0.99
    T_min: float = 1e-4
    median_T: float = 0.5
    dilation: float = 0.3
    bg: tuple = (0.0, 0.0, 0.0)
    sh_degree: int = 3
    guard_band: float = 0.0  # reading S6b: 0 = off (cull z <= znear only)


@dataclass
class Scene:
    means: np.ndarray
    scales: np.ndarray
    rotations: np.ndarray
    opacities: np.ndarray
    sh: np.ndarray
    sh_degree: int = SH_DEGREE
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.opacities.shape[0])

    def subset(self, idx) -> "Scene":
        idx = np.asarray(idx)
        return Scene(np.ascontiguousarray(self.means[:, idx]), np.ascontiguousarray(self.scales[:, idx]),
                     np.ascontiguousarray(self.rotations[:, idx]), np.ascontiguousarray(self.opacities[idx]),
                     np.ascontiguousarray(self.sh[:, :, idx]), self.sh_degree, dict(self.meta))

    def copy(self) -> "Scene":
        return Scene(self.means.copy(), self.scales.copy(), self.rotations.copy(), self.opacities.copy(),
                     self.sh.copy(), self.sh_degree, dict(self.meta))


def _f32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def make_scene(means, scales, rotations, opacities, sh, sh_degree=SH_DEGREE, **meta) -> Scene:
    means = _f32(means).reshape(3, -1)
    n = means.shape[1]
    return Scene(means, _f32(scales).reshape(3, n), _f32(rotations).reshape(4, n),
                 _f32(opacities).reshape(n), _f32(sh).reshape((sh_degree + 1) ** 2, 3, n), sh_degree, meta)


# ----------------------------------------------------------------------------- cameras

def look_at(eye, target, up=(0.0, 0.0, 1.0)):
    """World->camera (R, t) for a camera at `eye` looking at `target`; camera +z forward,
    +y down, +x right (OpenCV convention)."""
    eye = np.asarray(eye, np.float64)
    f = np.asarray(target, np.float64) - eye
    f /= np.linalg.norm(f)
    up = np.asarray(up, np.float64)
    r = np.cross(f, up)
    if np.linalg.norm(r) < 1e-8:
        r = np.cross(f, np.array([1.0, 0.0, 0.0]))
    r /= np.linalg.norm(r)
    d = np.cross(f, r)
    R = np.stack([r, d, f], 0)
    t = -R @ eye
    return R.astype(np.float32), t.astype(np.float32)


def camera_identity(width, height, fx, fy=None, cx=None, cy=None, znear=0.2) -> Camera:
    fy = fx if fy is None else fy
    cx = width / 2.0 if cx is None else cx
    cy = height / 2.0 if cy is None else cy
    return Camera(float(fx), float(fy), float(cx), float(cy), int(width), int(height),
                  np.eye(3, dtype=np.float32), np.zeros(3, np.float32), znear)


# ----------------------------------------------------------------------------- draws

def random_quaternions(rng, n):
    """Uniform random unit quaternions (w, x, y, z) (Shoemake)."""
    u1, u2, u3 = rng.random(n), rng.random(n), rng.random(n)
    a, b = np.sqrt(1 - u1), np.sqrt(u1)
    q = np.stack([b * np.cos(2 * np.pi * u3), a * np.sin(2 * np.pi * u2),
                  a * np.cos(2 * np.pi * u2), b * np.sin(2 * np.pi * u3)], 0)
    return q


def quaternion_with_axis3(normals, rng):
    """Quaternions (w,x,y,z) whose rotation maps the local z axis onto `normals` [3][n],
    with a random twist about it; used to lay flat Gaussians on a surface."""
    n = normals / np.linalg.norm(normals, axis=0, keepdims=True)
    nx, ny, nz = n
    # rotation taking e_z to n: axis = e_z x n, angle = acos(nz)
    ax = np.stack([-ny, nx, np.zeros_like(nx)], 0)
    s = np.linalg.norm(ax, axis=0)
    c = np.clip(nz, -1.0, 1.0)
    half = 0.5 * np.arctan2(s, c)
    axn = np.where(s > 1e-9, ax / np.maximum(s, 1e-30), np.array([[1.0], [0.0], [0.0]]))
    q1 = np.stack([np.cos(half), *(axn * np.sin(half))], 0)
    tw = rng.uniform(0, 2 * np.pi, n.shape[1]) * 0.5
    q2 = np.stack([np.cos(tw), np.zeros_like(tw), np.zeros_like(tw), np.sin(tw)], 0)  # twist about local z
    w1, x1, y1, z1 = q1
    w2, x2, y2, z2 = q2
    return np.stack([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2,
                     w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2,
                     w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2], 0)


def opacity_mixture(rng, n):
    """30% U(0.005, 0.2), 70% sigmoid(N(2.5, 1.5)) — bimodal like trained 3DGS."""
    lo = rng.uniform(0.005, 0.2, n)
    hi = 1.0 / (1.0 + np.exp(-rng.normal(2.5, 1.5, n)))
    o = np.where(rng.random(n) < 0.3, lo, hi)
    return np.clip(o, 0.005, 0.999)


def sh_coeffs(rng, n, degree=SH_DEGREE, dc_sigma=0.5, rest_sigma=0.05):
    K = (degree + 1) ** 2
    sh = rng.normal(0.0, rest_sigma, (K, 3, n))
    sh[0] = rng.normal(0.0, dc_sigma, (3, n))
    return sh


def flatness(rng, n, surfel_frac=0.2):
    """Ratio s_min / s: log-uniform in [0.05, 1], plus `surfel_frac` surfel-like at 1e-3..1e-2."""
    f = np.exp(rng.uniform(np.log(0.05), 0.0, n))
    surf = rng.random(n) < surfel_frac
    f[surf] = np.exp(rng.uniform(np.log(1e-3), np.log(1e-2), surf.sum()))
    return f


def _surface_gaussians(rng, pts, nrm, scale_med, scale_sigma=0.5, surfel_frac=0.2):
    n = pts.shape[1]
    s = scale_med * np.exp(rng.normal(0.0, scale_sigma, n))
    s_tan2 = s * np.exp(rng.normal(0.0, 0.25, n))
    s_n = s * flatness(rng, n, surfel_frac)
    scales = np.stack([s, s_tan2, s_n], 0)
    rots = quaternion_with_axis3(nrm, rng)
    return pts, scales, rots


def _volume_gaussians(rng, pts, scale_med, scale_sigma=0.5):
    n = pts.shape[1]
    s = scale_med * np.exp(rng.normal(0.0, scale_sigma, n))
    scales = np.stack([s, s * np.exp(rng.normal(0, 0.3, n)), s * flatness(rng, n, 0.1)], 0)
    return pts, scales, random_quaternions(rng, n)


def _sphere_surface(rng, n, center, radius):
    v = rng.normal(size=(3, n))
    v /= np.linalg.norm(v, axis=0, keepdims=True)
    return np.asarray(center, np.float64)[:, None] + radius * v, v


def _torus_surface(rng, n, R, r, z0=0.0):
    a = rng.uniform(0, 2 * np.pi, n)
    b = rng.uniform(0, 2 * np.pi, n)
    cx, cy = np.cos(a), np.sin(a)
    nrm = np.stack([np.cos(b) * cx, np.cos(b) * cy, np.sin(b)], 0)
    pts = np.stack([R * cx, R * cy, np.full(n, z0)], 0) + r * nrm
    return pts, nrm


def _box_surface(rng, n, center, half):
    face = rng.integers(0, 6, n)
    axis, sign = face // 2, np.where(face % 2 == 0, 1.0, -1.0)
    p = rng.uniform(-1, 1, (3, n)) * np.asarray(half)[:, None]
    nrm = np.zeros((3, n))
    for k in range(3):
        m = axis == k
        p[k, m] = sign[m] * half[k]
        nrm[k, m] = sign[m]
    return np.asarray(center, np.float64)[:, None] + p, nrm


def _disc(rng, n, radius, z, r_min=0.0):
    rr = np.sqrt(rng.uniform(r_min ** 2 / radius ** 2, 1.0, n)) * radius
    a = rng.uniform(0, 2 * np.pi, n)
    pts = np.stack([rr * np.cos(a), rr * np.sin(a), np.full(n, z)], 0)
    nrm = np.tile(np.array([[0.0], [0.0], [1.0]]), (1, n))
    return pts, nrm


def _assemble(rng, parts, sh_degree=SH_DEGREE, **meta) -> Scene:
    means = np.concatenate([p[0] for p in parts], 1)
    scales = np.concatenate([p[1] for p in parts], 1)
    rots = np.concatenate([p[2] for p in parts], 1)
    n = means.shape[1]
    # shuffle so Gaussian id order is not spatially structured (ids feed the sort tie-break)
    perm = rng.permutation(n)
    means, scales, rots = means[:, perm], scales[:, perm], rots[:, perm]
    return make_scene(means, scales, rots, opacity_mixture(rng, n), sh_coeffs(rng, n, sh_degree),
                      sh_degree, **meta)


# ----------------------------------------------------------------------------- configs

CONFIGS = {
    "C0": dict(name="single 64x64 view, 100 random Gaussians", width=64, height=64, n=100, views=1),
    "C1": dict(name="NeRF-Synthetic-shaped 800x800, 300k Gaussians, 100 views", width=800, height=800,
               n=300_000, views=100),
    "C2": dict(name="DTU-shaped 1600x1200, 400k Gaussians, 49 views", width=1600, height=1200,
               n=400_000, views=49),
    "C3": dict(name="Mip-NeRF 360-shaped outdoor 1237x822, 1.5M Gaussians, 200 views", width=1237,
               height=822, n=1_500_000, views=200),
    "C4": dict(name="Mip-NeRF 360-shaped large 1237x822, 3M Gaussians, 8-GPU", width=1237, height=822,
               n=3_000_000, views=200),
}


def scene_c0(seed=0, n=100, sh_degree=SH_DEGREE) -> Scene:
    """C0: n Gaussians uniform in the 64x64 frustum (fx = 64), z in [2, 6],
    scales log-U[0.02, 0.3], random rotations, bimodal opacity."""
    rng = np.random.default_rng(seed)
    z = rng.uniform(2.0, 6.0, n)
    x = rng.uniform(-0.5, 0.5, n) * z
    y = rng.uniform(-0.5, 0.5, n) * z
    s = np.exp(rng.uniform(np.log(0.02), np.log(0.3), (3, n)))
    return make_scene(np.stack([x, y, z]), s, random_quaternions(rng, n), opacity_mixture(rng, n),
                      sh_coeffs(rng, n, sh_degree), sh_degree, config="C0", seed=seed)


def camera_c0() -> Camera:
    return camera_identity(64, 64, 64.0)


def scene_c1(seed=1, n=300_000) -> Scene:
    """C1 NeRF-Synthetic-shaped: an object of radius <= 1.3 (sphere + torus + box
    surfaces with flat, surface-aligned Gaussians, plus 10% volumetric fuzz)."""
    rng = np.random.default_rng(seed)
    n_s, n_t, n_b = int(0.35 * n), int(0.3 * n), int(0.25 * n)
    n_v = n - n_s - n_t - n_b
    parts = [
        _surface_gaussians(rng, *_sphere_surface(rng, n_s, (0, 0, 0.15), 0.6), 0.006),
        _surface_gaussians(rng, *_torus_surface(rng, n_t, 0.95, 0.22), 0.005),
        _surface_gaussians(rng, *_box_surface(rng, n_b, (0.0, 0.0, -0.55), (0.55, 0.55, 0.2)), 0.006),
    ]
    v = rng.normal(size=(3, n_v))
    v *= (1.25 * rng.random(n_v) ** (1 / 3) / np.linalg.norm(v, axis=0))
    parts.append(_volume_gaussians(rng, v, 0.004))
    return _assemble(rng, parts, config="C1", seed=seed)


def cameras_c1(n_views=100, seed=101):
    rng = np.random.default_rng(seed)
    cams = []
    for i in range(n_views):
        az = rng.uniform(0, 2 * np.pi)
        el = np.arcsin(rng.uniform(0.05, 0.95))
        eye = 4.03 * np.array([np.cos(el) * np.cos(az), np.cos(el) * np.sin(az), np.sin(el)])
        R, t = look_at(eye, (0, 0, 0))
        cams.append(Camera(1111.1, 1111.1, 400.0, 400.0, 800, 800, R, t, 0.2))
    return cams


def scene_c2(seed=2, n=400_000) -> Scene:
    """C2 DTU-shaped: an object inside the unit sphere on a table plane."""
    rng = np.random.default_rng(seed)
    n_obj, n_tab = int(0.7 * n), int(0.2 * n)
    n_v = n - n_obj - n_tab
    n1 = n_obj // 2
    parts = [
        _surface_gaussians(rng, *_sphere_surface(rng, n1, (0, 0, 0.1), 0.55), 0.004),
        _surface_gaussians(rng, *_box_surface(rng, n_obj - n1, (0.1, -0.1, -0.35), (0.4, 0.3, 0.25)), 0.004),
        _surface_gaussians(rng, *_disc(rng, n_tab, 2.0, -0.6), 0.012),
    ]
    v = rng.normal(size=(3, n_v))
    v *= (1.0 * rng.random(n_v) ** (1 / 3) / np.linalg.norm(v, axis=0))
    parts.append(_volume_gaussians(rng, v, 0.004))
    return _assemble(rng, parts, config="C2", seed=seed)


def cameras_c2(n_views=49, seed=102):
    rng = np.random.default_rng(seed)
    cams = []
    for i in range(n_views):
        az = np.deg2rad(rng.uniform(-70, 70)) - np.pi / 2
        el = np.deg2rad(rng.uniform(20, 60))
        eye = 3.0 * np.array([np.cos(el) * np.cos(az), np.cos(el) * np.sin(az), np.sin(el)])
        R, t = look_at(eye, (0, 0, -0.1))
        cams.append(Camera(2892.0, 2892.0, 800.0, 600.0, 1600, 1200, R, t, 0.2))
    return cams


def scene_c3(seed=3, n=1_500_000) -> Scene:
    """C3 Mip-NeRF-360-shaped outdoor: 40% central region (r <= 1.5: surfaces + volume),
    20% ground disc, 40% background shell at distance 8-30 with scale proportional to
    distance."""
    rng = np.random.default_rng(seed)
    n_c, n_g = int(0.4 * n), int(0.2 * n)
    n_bg = n - n_c - n_g
    n_c1 = n_c // 2
    n_c2 = n_c // 4
    n_c3 = n_c - n_c1 - n_c2
    parts = [
        _surface_gaussians(rng, *_sphere_surface(rng, n_c1, (0, 0, 0.0), 0.8), 0.006),
        _surface_gaussians(rng, *_torus_surface(rng, n_c2, 1.1, 0.25, z0=-0.5), 0.006),
    ]
    v = rng.normal(size=(3, n_c3))
    v *= (1.5 * rng.random(n_c3) ** (1 / 3) / np.linalg.norm(v, axis=0))
    parts.append(_volume_gaussians(rng, v, 0.008))
    gp, gn = _disc(rng, n_g, 12.0, -1.0, r_min=0.0)
    gp[2] += rng.normal(0, 0.02, n_g)
    pts, sc, rq = _surface_gaussians(rng, gp, gn, 1.0)
    dist = np.linalg.norm(gp[:2], axis=0)
    sc = sc * (0.008 + 0.004 * dist)[None, :]
    parts.append((pts, sc, rq))
    # background shell: distance 8..30 from the origin, upper hemisphere-ish
    d = np.exp(rng.uniform(np.log(8.0), np.log(30.0), n_bg))
    v = rng.normal(size=(3, n_bg))
    v[2] = np.abs(v[2]) * 0.6 - 0.1
    v /= np.linalg.norm(v, axis=0, keepdims=True)
    bp = v * d
    bs = 0.004 * d * np.exp(rng.normal(0, 0.5, n_bg))
    scales = np.stack([bs, bs * np.exp(rng.normal(0, 0.3, n_bg)), bs * flatness(rng, n_bg, 0.1)], 0)
    parts.append((bp, scales, random_quaternions(rng, n_bg)))
    return _assemble(rng, parts, config="C3", seed=seed)


def cameras_c3(n_views=200, seed=103, width=1237, height=822):
    rng = np.random.default_rng(seed)
    cams = []
    for i in range(n_views):
        az = 2 * np.pi * i / n_views + rng.uniform(-0.01, 0.01)
        h = 0.3 + rng.uniform(-0.5, 0.5)
        eye = np.array([4.0 * np.cos(az), 4.0 * np.sin(az), h])
        R, t = look_at(eye, (0, 0, -0.2))
        cams.append(Camera(1160.0, 1160.0, width / 2.0, height / 2.0, width, height, R, t, 0.2))
    return cams


def scene_c4(seed=4, n=3_000_000) -> Scene:
    s = scene_c3(seed=seed, n=n)
    s.meta["config"] = "C4"
    return s


def config_scene_and_cameras(config: str, n_views=None, n_gaussians=None):
    """Returns (scene, [cameras], Options) for a named config."""
    if config == "C0":
        return scene_c0(), [camera_c0()], Options()
    if config == "C1":
        sc = scene_c1(n=n_gaussians or 300_000)
        return sc, cameras_c1(n_views or 100), Options(bg=(1.0, 1.0, 1.0))
    if config == "C2":
        return scene_c2(n=n_gaussians or 400_000), cameras_c2(n_views or 49), Options()
    # C3/C4 (outdoor orbit over a ground disc): the guard band of reading S6b
    # removes the ground splats beside and below the camera, whose centres project far off
    # screen and whose affine footprints would otherwise cover the whole image
    if config == "C3":
        return scene_c3(n=n_gaussians or 1_500_000), cameras_c3(n_views or 200), Options(guard_band=0.15)
    if config == "C4":
        return scene_c4(n=n_gaussians or 3_000_000), cameras_c3(n_views or 200), Options(guard_band=0.15)
    raise ValueError(config)


def cotangents(seed, width, height, scale=1.0):
    """Seeded per-pixel cotangents dL/d{color[3], depth, normal[3], alpha} for a scalar
    loss L = sum_px g . outputs. Planar [C][H][W] float32."""
    rng = np.random.default_rng(seed)
    g = rng.normal(0.0, scale, (8, height, width)).astype(np.float32)
    return dict(color=np.ascontiguousarray(g[0:3]), depth=np.ascontiguousarray(g[3]),
                normal=np.ascontiguousarray(g[4:7]), alpha=np.ascontiguousarray(g[7]))
