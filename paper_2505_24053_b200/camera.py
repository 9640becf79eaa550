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
