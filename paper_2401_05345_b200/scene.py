"""Synthetic Gaussian scenes and pinhole cameras (family G).

The reference has no scene data (it models traffic statistically), so the
rasterizer workloads are synthetic and seeded:

* camera: fov_x = 60 deg, fov_y from the aspect ratio, identity extrinsic for
  view 0; further views yaw on a +-15 deg arc about the scene centre;
* means: a uniform pixel (10 % margin) unprojected to depth U[2, 20];
* scales: per-axis pixel sigma LogUniform[0.5, 6] x U[0.5, 1.5] anisotropy,
  converted to world units (sigma * z / f);
* rotations: normalised N(0, 1)^4 quaternions (r, x, y, z);
* opacity U[0.05, 0.95], colour (precomputed RGB) U[0, 1];
* dL/dpixel U[-1, 1].

The high-contention scene (BASELINE configs[3]) uses pixel sigma U[100, 300]
and opacity U[0.01, 0.05] so lists stay long and T stays > 1e-4.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib

ZNEAR, ZFAR = 0.01, 100.0
SCENE_CENTER_Z = 11.0


@dataclass
class Camera:
    width: int
    height: int
    viewmatrix: np.ndarray  # 4x4 row-major math (world -> view)
    tan_fovx: float
    tan_fovy: float
    bg: tuple = (0.25, 0.5, 0.75)
    scale_modifier: float = 1.0
    projmatrix: np.ndarray = field(default=None)  # full proj @ view, row-major math

    def __post_init__(self):
        if self.projmatrix is None:
            P = np.zeros((4, 4))
            P[0, 0] = 1.0 / self.tan_fovx
            P[1, 1] = 1.0 / self.tan_fovy
            P[2, 2] = ZFAR / (ZFAR - ZNEAR)
            P[2, 3] = -(ZFAR * ZNEAR) / (ZFAR - ZNEAR)
            P[3, 2] = 1.0
            self.projmatrix = P @ self.viewmatrix

    def to_c(self) -> _lib.CameraC:
        """Column-major float32 matrices (M[col*4+row]) as the C ABI expects."""
        c = _lib.CameraC()
        c.width, c.height = self.width, self.height
        vm = np.asarray(self.viewmatrix, np.float64).T.reshape(-1).astype(np.float32)
        pm = np.asarray(self.projmatrix, np.float64).T.reshape(-1).astype(np.float32)
        c.viewmatrix[:] = vm.tolist()
        c.projmatrix[:] = pm.tolist()
        c.tan_fovx, c.tan_fovy = self.tan_fovx, self.tan_fovy
        c.bg[:] = [float(b) for b in self.bg]
        c.scale_modifier = self.scale_modifier
        return c


def make_camera(width: int, height: int, yaw_deg: float = 0.0, fov_x_deg: float = 60.0,
                bg=(0.25, 0.5, 0.75)) -> Camera:
    tx = math.tan(math.radians(fov_x_deg) / 2)
    ty = tx * height / width
    V = np.eye(4)
    if yaw_deg:
        # orbit about (0, 0, SCENE_CENTER_Z): view = T(c) R T(-c)
        a = math.radians(yaw_deg)
        R = np.eye(4)
        R[0, 0], R[0, 2], R[2, 0], R[2, 2] = math.cos(a), math.sin(a), -math.sin(a), math.cos(a)
        T1, T2 = np.eye(4), np.eye(4)
        T1[2, 3], T2[2, 3] = SCENE_CENTER_Z, -SCENE_CENTER_Z
        V = T1 @ R @ T2
    return Camera(width, height, V, tx, ty, bg)


def orbit_cameras(width: int, height: int, n: int) -> list:
    if n == 1:
        return [make_camera(width, height)]
    return [make_camera(width, height, -15.0 + 30.0 * k / (n - 1)) for k in range(n)]


def make_scene(P: int, width: int, height: int, seed: int = 0, high_contention: bool = False,
               fov_x_deg: float = 60.0) -> dict:
    """Seeded Gaussians visible from make_camera(width, height)."""
    rng = np.random.default_rng(seed)
    tx = math.tan(math.radians(fov_x_deg) / 2)
    ty = tx * height / width
    f = width / (2 * tx)
    z = rng.uniform(2.0, 20.0, P)
    u = rng.uniform(-0.9, 0.9, P)
    v = rng.uniform(-0.9, 0.9, P)
    means = np.stack([u * tx * z, v * ty * z, z], axis=1)
    if high_contention:
        sig = rng.uniform(100.0, 300.0, P)
        opac = rng.uniform(0.01, 0.05, P)
    else:
        sig = np.exp(rng.uniform(math.log(0.5), math.log(6.0), P))
        opac = rng.uniform(0.05, 0.95, P)
    aniso = rng.uniform(0.5, 1.5, (P, 3))
    scales = (sig[:, None] * aniso) * z[:, None] / f
    q = rng.normal(size=(P, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    colors = rng.uniform(0.0, 1.0, (P, 3))
    f32 = lambda a: np.ascontiguousarray(a, np.float32)  # noqa: E731
    return {"means3D": f32(means), "scales": f32(scales), "rotations": f32(q),
            "opacities": f32(opac), "colors": f32(colors)}


def make_dL_dpixels(width: int, height: int, seed: int = 1) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return np.ascontiguousarray(rng.uniform(-1.0, 1.0, (3, height, width)), np.float32)


# BASELINE.json configs: name -> (P, W, H, high_contention, views)
CONFIGS = {
    "c1_10k_256": (10_000, 256, 256, False, 1),
    "c2_100k_800": (100_000, 800, 800, False, 1),
    "c3_1m_1080p": (1_000_000, 1920, 1080, False, 1),
    "c4_200k_contention_1080p": (200_000, 1920, 1080, True, 1),
    "c5_3m_1080p_64views": (3_000_000, 1920, 1080, False, 64),
}
