"""Drop-in ``render`` / ``render_backward`` on the B200 (raygauss/renderer.py mirror).

Same signatures, dataclasses, conventions and errors as the reference:

* :func:`render` (renderer.py:123-176) -> :class:`FrameOutput` with float64
  colour ``(H, W, 3)``, float64 ``remaining_transmittance`` and int64
  ``contributor_count`` (renderer.py:39-44).
* :func:`render_backward` (renderer.py:234-333) -> :class:`SceneGrads` in the
  stored parameter spaces: ``dopacities`` w.r.t. LINEAR opacity, ``dquats``
  including the normalisation Jacobian, ``dlog_scales`` in log space, SH view
  direction stop-gradient (renderer.py:179-201).
* ``RenderConfig.threads`` is accepted and ignored (the GPU runs every tile).

Both calls go through the host-level C ABI (``geer_render_host`` /
``geer_render_backward_host``): host float64 arrays in, host float64 arrays
out, with the copies and the fp32 device compute inside the library.  The
tensor-level fast path (device tensors, no host copies) is
:class:`paper_2505_24053_b200.device.DeviceRenderer`.
"""

from __future__ import annotations

import dataclasses

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .association import RenderGraph, export_graph
from .scene import BEAPImage, validate_camera


@dataclass
class RenderConfig:
    """renderer.py:24-37."""

    lam: float = 3.0
    tile_px: int = 16
    background: np.ndarray = field(default_factory=lambda: np.zeros(3))
    support_cutoff: bool = True
    threads: int = 1

    def __post_init__(self):
        self.background = np.asarray(self.background, dtype=np.float64).reshape(3)


@dataclass
class FrameOutput:
    """renderer.py:39-44."""

    color: BEAPImage
    remaining_transmittance: np.ndarray
    contributor_count: np.ndarray
    graph: RenderGraph | None = None


@dataclass
class SceneGrads:
    """renderer.py:179-201."""

    dmeans: np.ndarray
    dlog_scales: np.ndarray
    dquats: np.ndarray
    dopacities: np.ndarray
    dsh: np.ndarray

    @classmethod
    def zeros_like(cls, scene) -> "SceneGrads":
        return cls(np.zeros_like(scene.means), np.zeros_like(scene.log_scales), np.zeros_like(scene.quats),
                   np.zeros_like(scene.opacity_logits), np.zeros_like(scene.sh))


def resolve_threads(requested=None) -> int:
    """renderer.py:47-54 (kept for API compatibility; the GPU path ignores it)."""
    if requested is not None and requested > 0:
        return int(requested)
    env = os.environ.get("GEER_THREADS")
    if env:
        return max(1, int(env))
    return os.cpu_count() or 1


class _HostScene:
    """Contiguous float64 views of a GaussianScene (reference or mirror) + the C struct."""

    def __init__(self, scene):
        means = np.ascontiguousarray(np.asarray(scene.means, dtype=np.float64).reshape(-1, 3))
        n = len(means)
        self.n = n
        self.means = means
        self.log_scales = np.ascontiguousarray(np.asarray(scene.log_scales, dtype=np.float64).reshape(n, 3))
        self.quats = np.ascontiguousarray(np.asarray(scene.quats, dtype=np.float64).reshape(n, 4))
        self.opacity_logits = np.ascontiguousarray(np.asarray(scene.opacity_logits, dtype=np.float64).reshape(n))
        sh = np.asarray(scene.sh, dtype=np.float64)
        self.n_bands = int(sh.shape[1]) if sh.ndim == 3 else (sh.size // (3 * n) if n else 1)
        self.sh = np.ascontiguousarray(sh.reshape(n, self.n_bands, 3))
        if self.n_bands > 16:
            raise ValueError(f"unsupported SH band count {self.n_bands}; degree must be 0..3")
        s = _lib.GeerHostScene()
        s.n = n
        s.n_bands = self.n_bands
        s.means = self.means.ctypes.data
        s.log_scales = self.log_scales.ctypes.data
        s.quats = self.quats.ctypes.data
        s.opacity_logits = self.opacity_logits.ctypes.data
        s.sh = self.sh.ctypes.data
        self.struct = s


def _ctx(device: int = 0) -> _lib.Context:
    return _lib.default_context(device)


def last_h2d_bytes(device: int = 0) -> int:
    """PCIe bytes the calling thread's last ``render``/``render_backward`` sent host->device for its
    inputs (the float64 scene goes mostly as fp32 narrowed on the host cores; geer_last_h2d_bytes)."""
    ctx = _ctx(device)
    return int(ctx._lib.geer_last_h2d_bytes(ctx.ptr))


def _host_empty(shape, dtype) -> np.ndarray:
    """A fresh numpy array in page-locked memory (torch's caching host allocator).

    The device->host copies of the outputs then run at full PCIe speed instead of
    faulting in fresh pageable pages (measured 17 ms vs 1.5 ms for a 1080p frame);
    blocks are recycled once the caller drops the previous result.
    """
    import torch

    t = torch.empty(shape, dtype={np.float64: torch.float64, np.int64: torch.int64}[np.dtype(dtype).type],
                    pin_memory=True)
    return t.numpy()


def lazy_dataclass(cls, thunk):
    """An instance of dataclass ``cls`` whose fields come from ``thunk()`` on first access.

    ``FrameOutput.graph`` uses it: the reference always attaches the render graph
    (renderer.py:170-175); here it is exported from the device only if the caller reads it (the
    association is deterministic, so rebuilding it then gives the frame's own graph - as long as
    the caller has not modified the scene's arrays in place meanwhile)."""
    lazy = _LAZY_TYPES.get(cls)
    if lazy is None:
        def __getattr__(self, name):
            d = object.__getattribute__(self, "__dict__")
            if name.startswith("__") or "_thunk" not in d:
                raise AttributeError(name)
            obj = d.pop("_thunk")()
            for f in dataclasses.fields(cls):
                d[f.name] = getattr(obj, f.name)
            return object.__getattribute__(self, name)

        lazy = type("Lazy" + cls.__name__, (cls,), {"__getattr__": __getattr__})
        _LAZY_TYPES[cls] = lazy
    inst = object.__new__(lazy)
    inst.__dict__["_thunk"] = thunk
    return inst


_LAZY_TYPES: dict = {}


def render(scene, camera, config: RenderConfig | None = None, *, return_graph: bool | None = None,
           device: int = 0) -> FrameOutput:
    """Render ``scene`` through ``camera`` (renderer.py:123-176) on the GPU.

    ``FrameOutput.graph`` is the association, as in the reference: by default (``return_graph=None``)
    a lazily exported ``RenderGraph`` (nothing is copied unless it is read); ``True`` exports it
    now, ``False`` leaves ``None``.
    """
    config = config or RenderConfig()
    validate_camera(camera)
    h, w = int(camera.height), int(camera.width)
    hs = _HostScene(scene)
    color = _host_empty((h, w, 3), np.float64)
    remaining = _host_empty((h, w), np.float64)
    count = _host_empty((h, w), np.int64)
    ctx = _ctx(device)
    cam = _lib.camera_struct(camera)
    cfg = _lib.config_struct(config)
    _lib.check(ctx._lib.geer_render_host(ctx.ptr, ctypes.byref(hs.struct), ctypes.byref(cam), ctypes.byref(cfg),
                                         color.ctypes.data, remaining.ctypes.data, count.ctypes.data))
    graph = None
    if return_graph is None:
        lam, tile_px = config.lam, config.tile_px
        graph = lazy_dataclass(RenderGraph, lambda: build_graph_for(scene, camera, lam, tile_px, device=device))
    elif return_graph:
        graph = build_graph_for(scene, camera, config.lam, config.tile_px, device=device)
    return FrameOutput(color=BEAPImage(color=color, mask=np.ones((h, w), dtype=bool)),
                       remaining_transmittance=remaining, contributor_count=count, graph=graph)


def render_backward(scene, camera, dl_dimage: np.ndarray, config: RenderConfig | None = None, *,
                    device: int = 0) -> SceneGrads:
    """dLoss/dparameters from an image gradient (renderer.py:234-333) on the GPU."""
    config = config or RenderConfig()
    validate_camera(camera)
    hs = _HostScene(scene)
    if hs.n == 0:
        return SceneGrads(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 4)), np.zeros(0),
                          np.zeros((0, hs.n_bands, 3)))
    grads = SceneGrads(_host_empty((hs.n, 3), np.float64), _host_empty((hs.n, 3), np.float64),
                       _host_empty((hs.n, 4), np.float64), _host_empty((hs.n,), np.float64),
                       _host_empty((hs.n, hs.n_bands, 3), np.float64))
    h, w = int(camera.height), int(camera.width)
    dl = np.ascontiguousarray(np.asarray(dl_dimage, dtype=np.float64).reshape(h, w, 3))
    ctx = _ctx(device)
    cam = _lib.camera_struct(camera)
    cfg = _lib.config_struct(config)
    g = _lib.GeerHostGrads()
    g.dmeans = grads.dmeans.ctypes.data
    g.dlog_scales = grads.dlog_scales.ctypes.data
    g.dquats = grads.dquats.ctypes.data
    g.dopacities = grads.dopacities.ctypes.data
    g.dsh = grads.dsh.ctypes.data
    _lib.check(ctx._lib.geer_render_backward_host(ctx.ptr, ctypes.byref(hs.struct), ctypes.byref(cam),
                                                  dl.ctypes.data, ctypes.byref(cfg), ctypes.byref(g)))
    return grads


def build_graph_for(scene, camera, lam: float = 3.0, tile_px: int = 16, device: int = 0) -> RenderGraph:
    """association.build_render_graph on the GPU (see association.py)."""
    validate_camera(camera)
    hs = _HostScene(scene)
    ctx = _ctx(device)
    cam = _lib.camera_struct(camera)
    _lib.check(ctx._lib.geer_build_graph_host(ctx.ptr, ctypes.byref(hs.struct), ctypes.byref(cam), float(lam),
                                              int(tile_px)))
    return export_graph(ctx, hs.n, int(camera.width), int(camera.height))
