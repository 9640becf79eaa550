"""Camera-side data path on the GPU (raygauss/camera.py mirror for what feeds the renderer).

:func:`resample_to_beap` (camera.py:302-339) pulls a pinhole or fisheye (KB) ground-truth image onto
the equiangular grid of a BEAP target camera — the training targets of the multi-view step — with
the reference's projection (camera.py:197-246), bilinear tap (:289-299) and validity mask, computed
by ``geer_resample_to_beap`` (one thread per target pixel, fp64 geometry, fp32 image).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .scene import BEAPImage, Camera, validate_camera

__all__ = ["Camera", "BEAPImage", "resample_to_beap", "resample_to_beap_device"]


def resample_to_beap_device(source: torch.Tensor, source_camera, target_camera):
    """Device form: ``source`` (H_s,W_s,3) fp32 CUDA tensor -> (color (H,W,3) fp32, mask (H,W) bool)."""
    if source.dtype != torch.float32 or not source.is_cuda or not source.is_contiguous() or source.dim() != 3:
        raise ValueError("source must be a contiguous (H,W,3) float32 CUDA tensor")
    h, w = int(target_camera.height), int(target_camera.width)
    color = torch.empty((h, w, 3), dtype=torch.float32, device=source.device)
    mask = torch.empty((h, w), dtype=torch.uint8, device=source.device)
    src_c = _lib.camera_struct(source_camera)
    dst_c = _lib.camera_struct(target_camera)
    stream = torch.cuda.current_stream(source.device).cuda_stream
    _lib.check(_lib.load().geer_resample_to_beap(source.data_ptr(), int(source.shape[0]), int(source.shape[1]),
                                                 ctypes.byref(src_c), ctypes.byref(dst_c), color.data_ptr(),
                                                 mask.data_ptr(), stream))
    return color, mask.bool()


def resample_to_beap(source_image, source_camera, target_camera, device: int = 0) -> BEAPImage:
    """Drop-in for raygauss.camera.resample_to_beap (camera.py:302-339), same checks and errors."""
    if target_camera.model != "beap":
        raise ValueError("target camera must use the beap model")
    if not np.allclose(source_camera.rotation, target_camera.rotation) or not np.allclose(
            source_camera.translation, target_camera.translation):
        raise ValueError("source and target must share extrinsics")
    if source_camera.model not in ("pinhole", "kb"):
        raise ValueError("source camera must be pinhole or kb")
    validate_camera(source_camera)
    validate_camera(target_camera)
    src = torch.as_tensor(np.ascontiguousarray(np.asarray(source_image, dtype=np.float32)),
                          device=torch.device(f"cuda:{device}"))
    color, mask = resample_to_beap_device(src, source_camera, target_camera)
    return BEAPImage(color=color.double().cpu().numpy(), mask=mask.cpu().numpy())


# ---------------------------------------------------------------------------------- camera JSON
# camera.py:371-422: the same keys (w, h, model, R, t, fovx_deg/fovy_deg, fx/fy/cx/cy, k).


def camera_from_dict(cfg: dict) -> Camera:
    rot = np.asarray(cfg.get("R", np.eye(3).ravel()), dtype=np.float64).reshape(3, 3)
    return Camera(width=int(cfg["w"]), height=int(cfg["h"]), model=cfg.get("model", "beap"), rotation=rot,
                  translation=np.asarray(cfg.get("t", (0, 0, 0)), dtype=np.float64),
                  fov_x=np.deg2rad(cfg["fovx_deg"]) if "fovx_deg" in cfg else None,
                  fov_y=np.deg2rad(cfg["fovy_deg"]) if "fovy_deg" in cfg else None,
                  fx=cfg.get("fx"), fy=cfg.get("fy"), cx=cfg.get("cx"), cy=cfg.get("cy"),
                  k=np.asarray(cfg.get("k", (0, 0, 0, 0)), dtype=np.float64))


def camera_to_dict(camera) -> dict:
    cfg = {"model": camera.model, "w": camera.width, "h": camera.height,
           "R": [float(v) for v in np.asarray(camera.rotation).ravel()],
           "t": [float(v) for v in np.asarray(camera.translation)]}
    if camera.fov_x is not None:
        cfg["fovx_deg"] = float(np.rad2deg(camera.fov_x))
    if camera.fov_y is not None:
        cfg["fovy_deg"] = float(np.rad2deg(camera.fov_y))
    for name in ("fx", "fy", "cx", "cy"):
        val = getattr(camera, name)
        if val is not None:
            cfg[name] = float(val)
    k = np.asarray(getattr(camera, "k", np.zeros(4)), dtype=np.float64)
    if np.any(k != 0):
        cfg["k"] = [float(v) for v in k]
    return cfg


def load_cameras(path) -> list:
    """One camera or a list of cameras from a JSON file."""
    import json

    with open(path) as f:
        data = json.load(f)
    if isinstance(data, dict):
        data = [data]
    return [camera_from_dict(c) for c in data]


def save_cameras(cameras, path):
    import json

    data = [camera_to_dict(c) for c in cameras]
    with open(path, "w") as f:
        json.dump(data[0] if len(data) == 1 else data, f, indent=2)
