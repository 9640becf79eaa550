"""Tensor-level fast path: device-resident scene, no host copies.

``DeviceRenderer.forward`` / ``backward`` call ``geer_forward`` /
``geer_backward`` (include/geer.h) on torch's current CUDA stream with the
data pointers of fp32 CUDA tensors.  PyTorch only provides device memory and
streams here; all compute is the library's sm_100a kernels.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


@dataclass
class DeviceScene:
    """fp32 CUDA tensors in the reference's stored spaces (scene.py:35-51)."""

    means: torch.Tensor
    log_scales: torch.Tensor
    quats: torch.Tensor
    opacity_logits: torch.Tensor
    sh: torch.Tensor

    @classmethod
    def from_scene(cls, scene, device="cuda") -> "DeviceScene":
        t = lambda a: torch.as_tensor(np.ascontiguousarray(np.asarray(a, dtype=np.float32))).to(device)
        n = len(np.asarray(scene.means).reshape(-1, 3))
        sh = np.asarray(scene.sh, dtype=np.float32)
        return cls(t(np.asarray(scene.means).reshape(n, 3)), t(np.asarray(scene.log_scales).reshape(n, 3)),
                   t(np.asarray(scene.quats).reshape(n, 4)), t(np.asarray(scene.opacity_logits).reshape(n)),
                   t(sh.reshape(n, -1, 3)))

    def __len__(self):
        return int(self.means.shape[0])

    @property
    def n_bands(self) -> int:
        return int(self.sh.shape[1])

    def struct(self) -> _lib.GeerScene:
        for name in ("means", "log_scales", "quats", "opacity_logits", "sh"):
            v = getattr(self, name)
            if v.dtype != torch.float32 or not v.is_cuda or not v.is_contiguous():
                raise ValueError(f"{name} must be a contiguous float32 CUDA tensor")
        s = _lib.GeerScene()
        s.n = len(self)
        s.n_bands = self.n_bands
        s.means = self.means.data_ptr()
        s.log_scales = self.log_scales.data_ptr()
        s.quats = self.quats.data_ptr()
        s.opacity_logits = self.opacity_logits.data_ptr()
        s.sh = self.sh.data_ptr()
        return s

    def zeros_like_grads(self) -> "DeviceScene":
        return DeviceScene(*(torch.zeros_like(getattr(self, k)) for k in
                             ("means", "log_scales", "quats", "opacity_logits", "sh")))


class DeviceRenderer:
    """One geer context: forward a view, then (optionally) its backward."""

    def __init__(self, device: int = 0):
        self.device = device
        self.ctx = _lib.Context(device)
        self._keep = None  # tensors the last forward's state points into
        self._stream = None
        self._workspace = None

    def set_timing(self, on: bool):
        self.ctx.set_timing(on)

    def forward(self, scene: DeviceScene, camera, config, out=None, flags: int = 0, sync: bool = True):
        """Returns (color (H,W,3) f32, remaining (H,W) f32, count (H,W) i32) CUDA tensors.

        ``flags``: ``_lib.GEER_CFG_*`` debug switches (e.g. ``GEER_CFG_NO_CULL``); results do not
        depend on them.  ``sync=False`` leaves the frame in flight on the current stream (the library
        never blocks the host once the context has seen the graph's size); ``self.sync()`` then
        synchronises it and raises what the reference raises (ValueError for a non-PD view
        covariance), re-rendering a frame whose graph outgrew the context's capacity.
        """
        h, w = int(camera.height), int(camera.width)
        dev = scene.means.device
        if out is None:
            out = (torch.empty((h, w, 3), dtype=torch.float32, device=dev),
                   torch.empty((h, w), dtype=torch.float32, device=dev),
                   torch.empty((h, w), dtype=torch.int32, device=dev))
        color, remaining, count = out
        s = scene.struct()
        cam = _lib.camera_struct(camera)
        cfg = _lib.config_struct(config, flags)
        stream = torch.cuda.current_stream(dev).cuda_stream
        _lib.check(self.ctx._lib.geer_forward(self.ctx.ptr, ctypes.byref(s), ctypes.byref(cam), ctypes.byref(cfg),
                                              color.data_ptr(), remaining.data_ptr(), count.data_ptr(), stream))
        self._keep = (scene, remaining)
        self._stream = stream
        if sync:
            self.sync()
        return color, remaining, count

    def sync(self) -> bool:
        """Wait for the last forward and raise its device-side error, if any (geer_sync).

        Returns True when a frame since the previous sync outgrew the context's graph capacity: the
        capacity has grown and the last frame was rendered again (its outputs are valid), but work
        that consumed an earlier frame of this context must be redone."""
        rc = self.ctx._lib.geer_sync(self.ctx.ptr, self._stream)
        if rc == _lib.GEER_ERR_OVERFLOW:
            return True
        _lib.check(rc)
        return False

    def clear_camera_cache(self):
        _lib.check(self.ctx._lib.geer_clear_camera_cache(self.ctx.ptr))

    def workspace_bytes(self, scene: DeviceScene, camera, config, max_entries: int = 0) -> int:
        """Device bytes the forward + backward of ``scene`` through ``camera`` need (geer_workspace_bytes)."""
        cam = _lib.camera_struct(camera)
        cfg = _lib.config_struct(config, 0)
        nb = int(scene.sh.shape[1])
        b = self.ctx._lib.geer_workspace_bytes(self.ctx.ptr, int(scene.means.shape[0]), nb, ctypes.byref(cam),
                                               ctypes.byref(cfg), int(max_entries))
        if b == 0:
            raise ValueError(_lib.last_error())
        return int(b)

    def set_workspace(self, workspace: torch.Tensor | None):
        """Carve every device buffer of this renderer from ``workspace`` (a CUDA tensor owned by the caller,
        e.g. torch's caching allocator) instead of library cudaMalloc; ``None`` returns to library memory."""
        if workspace is None:
            _lib.check(self.ctx._lib.geer_set_workspace(self.ctx.ptr, None, 0))
        else:
            if not workspace.is_cuda or not workspace.is_contiguous():
                raise ValueError("workspace must be a contiguous CUDA tensor")
            _lib.check(self.ctx._lib.geer_set_workspace(self.ctx.ptr, workspace.data_ptr(),
                                                        workspace.numel() * workspace.element_size()))
        self._workspace = workspace  # (kept alive while attached)
        self._keep = None

    def workspace_used(self) -> int:
        u = ctypes.c_size_t(0)
        _lib.check(self.ctx._lib.geer_workspace_used(self.ctx.ptr, ctypes.byref(u)))
        return int(u.value)

    def backward(self, dl_dimage: torch.Tensor, grads: DeviceScene | None = None, accumulate: bool = False,
                 opacity_logit: bool = False):
        """Gradients of the last forward's scene (renderer.py:179-201 conventions).

        ``opacity_logit=True`` returns the opacity gradient in the stored logit space
        (trainer.py:208-217 ``stored_grads``) instead of w.r.t. linear opacity.
        """
        if self._keep is None:
            raise RuntimeError("backward needs a preceding forward")
        scene = self._keep[0]
        if grads is None:
            grads = scene.zeros_like_grads()
        if dl_dimage.dtype != torch.float32 or not dl_dimage.is_contiguous():
            raise ValueError("dl_dimage must be a contiguous float32 CUDA tensor")
        g = _lib.GeerGrads()
        g.dmeans = grads.means.data_ptr()
        g.dlog_scales = grads.log_scales.data_ptr()
        g.dquats = grads.quats.data_ptr()
        g.dopacities = grads.opacity_logits.data_ptr()
        g.dsh = grads.sh.data_ptr()
        stream = torch.cuda.current_stream(dl_dimage.device).cuda_stream
        _lib.check(self.ctx._lib.geer_backward(self.ctx.ptr, dl_dimage.data_ptr(), ctypes.byref(g),
                                               (1 if accumulate else 0) | (2 if opacity_logit else 0), stream))
        return grads

    def stats(self) -> dict:
        return self.ctx.stats()
