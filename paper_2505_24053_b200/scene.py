"""Scene and camera types mirroring the reference's public dataclasses.

These are drop-in mirrors of ``raygauss.scene.GaussianScene``
(scene.py:35-128), ``raygauss.camera.Camera`` (camera.py:25-90) and
``raygauss.camera.BEAPImage`` (camera.py:93-104): same field names, same
stored parameter spaces (log-scale, opacity logit, raw quaternion (r,i,j,k)
renormalised on read, SH (N, B, 3)), same validation and error types.  The
renderer accepts either these or the reference's own objects (duck-typed).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

MAX_FOV_DEG = 350.0  # camera.py:22


@dataclass
class GaussianScene:
    """SoA particle store (scene.py:35-51): (N,3), (N,3), (N,4), (N,), (N,B,3)."""

    means: np.ndarray
    log_scales: np.ndarray
    quats: np.ndarray
    opacity_logits: np.ndarray
    sh: np.ndarray

    def __post_init__(self):
        self.means = np.asarray(self.means, dtype=np.float64).reshape(-1, 3)
        n = len(self.means)
        self.log_scales = np.asarray(self.log_scales, dtype=np.float64).reshape(n, 3)
        self.quats = np.asarray(self.quats, dtype=np.float64).reshape(n, 4)
        self.opacity_logits = np.asarray(self.opacity_logits, dtype=np.float64).reshape(n)
        sh = np.asarray(self.sh, dtype=np.float64)
        if n == 0:  # the reference's reshape(n, -1, 3) rejects 0-sized SH (scene.py:51); keep the band count
            self.sh = sh.reshape(0, sh.shape[1] if sh.ndim == 3 else 1, 3)
        else:
            self.sh = sh.reshape(n, -1, 3)

    def __len__(self):
        return len(self.means)

    def extent(self) -> float:
        """scene.py:82-87."""
        if len(self) == 0:
            return 1.0
        centered = self.means - self.means.mean(axis=0)
        return float(max(np.linalg.norm(centered, axis=1).max(), 1e-6))

    def copy(self) -> "GaussianScene":
        return GaussianScene(self.means.copy(), self.log_scales.copy(), self.quats.copy(),
                             self.opacity_logits.copy(), self.sh.copy())

    @classmethod
    def empty(cls, n_bands: int = 1) -> "GaussianScene":
        return cls(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 4)), np.zeros(0), np.zeros((0, n_bands, 3)))


@dataclass
class Camera:
    """camera.py:25-90: extrinsics (x_c = R_c x + t_c) plus pinhole / kb / beap."""

    width: int
    height: int
    model: str = "beap"
    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    translation: np.ndarray = field(default_factory=lambda: np.zeros(3))
    fov_x: float | None = None
    fov_y: float | None = None
    fx: float | None = None
    fy: float | None = None
    cx: float | None = None
    cy: float | None = None
    k: np.ndarray = field(default_factory=lambda: np.zeros(4))

    def __post_init__(self):
        self.rotation = np.asarray(self.rotation, dtype=np.float64).reshape(3, 3)
        self.translation = np.asarray(self.translation, dtype=np.float64).reshape(3)
        self.k = np.asarray(self.k, dtype=np.float64).reshape(4)
        validate_camera(self)

    @property
    def optical_center(self) -> np.ndarray:
        return -self.rotation.T @ self.translation


def validate_camera(cam) -> None:
    """The checks of camera.py:54-69, raising the same ValueError messages."""
    if cam.model not in ("pinhole", "kb", "beap"):
        raise ValueError(f"unknown camera model {cam.model!r}")
    rot = np.asarray(cam.rotation, dtype=np.float64).reshape(3, 3)
    err = np.abs(rot @ rot.T - np.eye(3)).max()
    if err > 1e-6 or np.linalg.det(rot) < 0:
        raise ValueError("extrinsic rotation is not in SO(3)")
    if cam.model == "beap":
        if cam.fov_x is None or cam.fov_y is None:
            raise ValueError("beap camera requires fov_x and fov_y")
    else:
        if cam.fx is None or cam.fy is None or cam.cx is None or cam.cy is None:
            raise ValueError(f"{cam.model} camera requires fx, fy, cx, cy")
        if cam.fx <= 0 or cam.fy <= 0:
            raise ValueError("focal lengths must be positive")
    for fov in (cam.fov_x, cam.fov_y):
        if fov is not None and not 0.0 < fov < np.deg2rad(MAX_FOV_DEG):
            raise ValueError("fov must lie in (0, 350) degrees")


@dataclass
class BEAPImage:
    """camera.py:93-104."""

    color: np.ndarray
    mask: np.ndarray

    def __post_init__(self):
        self.color = np.asarray(self.color, dtype=np.float64)
        self.mask = np.asarray(self.mask, dtype=bool)
        if self.color.shape[:2] != self.mask.shape:
            raise ValueError("color and mask shapes disagree")
