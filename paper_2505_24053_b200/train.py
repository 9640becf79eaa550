"""Multi-view training step (BASELINE config 4): views sharded over ranks, one NCCL allreduce.

One step:

1. every rank renders its contiguous share of the views (forward), forms the
   masked-L1 image gradient against the view's target (``geer_l1_grad``,
   trainer.py:127-132) and runs the backward, accumulating per-Gaussian
   gradients for all its views into ONE flat fp32 buffer (opacity chained to
   the stored logit, trainer.py:208-217);
2. ``torch.distributed.all_reduce(SUM)`` of that buffer (NCCL over
   NVLink/NVSwitch; gloo in CPU tests);
3. every rank applies the identical Adam update (trainer.py:181-197) with one
   ``geer_adam`` launch over the flat parameter buffer, so replicas stay
   bit-identical.

Parameters and gradients are flat buffers whose slices are the SoA tensors
the renderer reads, so the allreduce and Adam touch one contiguous buffer.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .device import DeviceRenderer, DeviceScene
from .renderer import RenderConfig

FIELDS = (("means", 3), ("log_scales", 3), ("quats", 4), ("opacity_logits", 1), ("sh", None))


def shard(n_items: int, rank: int, world: int) -> range:
    """Contiguous share of ``n_items`` views for ``rank``."""
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


SSIM_WEIGHT = 0.2  # trainer.py:114 loss(..., ssim_weight=0.2)


class LossWorkspace:
    """Device scratch of geer_loss for one image size (grow-only)."""

    def __init__(self):
        self.buf = None
        self.out = None

    def get(self, h: int, w: int, device):
        nbytes = int(_lib.load().geer_loss_workspace_bytes(h, w))
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != torch.device(device):
            self.buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
            self.out = torch.empty(3, dtype=torch.float64, device=device)
        return self.buf, self.out


def loss_device(color: torch.Tensor, target: torch.Tensor, mask: torch.Tensor | None = None,
                ssim_weight: float = SSIM_WEIGHT, grad: torch.Tensor | None = None,
                workspace: LossWorkspace | None = None):
    """trainer.loss (trainer.py:114-155) on device tensors: returns (out, grad).

    ``out`` is a float64 CUDA tensor (total, L1, 1 - SSIM); ``grad`` the (H,W,3) fp32 image gradient.
    ``mask``: (H,W) bool/uint8 CUDA tensor of valid target pixels (None = all valid).
    """
    h, w = int(color.shape[0]), int(color.shape[1])
    for t in (color, target):
        if t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous() or tuple(t.shape) != (h, w, 3):
            raise ValueError("color and target must be contiguous (H,W,3) float32 CUDA tensors")
    m = None
    if mask is not None:
        m = mask.to(torch.uint8).contiguous()
        if tuple(m.shape) != (h, w):
            raise ValueError("mask must be (H,W)")
    ws = workspace or LossWorkspace()
    buf, out = ws.get(h, w, color.device)
    if grad is None:
        grad = torch.empty_like(color)
    stream = torch.cuda.current_stream(color.device).cuda_stream
    _lib.check(_lib.load().geer_loss(color.data_ptr(), target.data_ptr(), m.data_ptr() if m is not None else None,
                                     h, w, ctypes.c_float(ssim_weight), buf.data_ptr(), out.data_ptr(),
                                     grad.data_ptr(), stream))
    return out, grad


def loss(rendered, target, ssim_weight: float = SSIM_WEIGHT, device: int = 0):
    """Drop-in for raygauss.trainer.loss (trainer.py:114-155): (total, dL/drendered) in float64 numpy.

    ``target`` is a BEAPImage-like object with ``color`` (H,W,3) and ``mask`` (H,W).  The loss and
    its gradient are computed by the CUDA kernels in fp32 with fp64 sums.
    """
    rendered = np.asarray(rendered)
    tcol = np.asarray(target.color)
    if rendered.shape != tcol.shape:
        raise ValueError("rendered and target shapes disagree")  # trainer.py:121-122
    dev = torch.device(f"cuda:{device}")
    c = torch.as_tensor(np.ascontiguousarray(rendered, dtype=np.float32), device=dev)
    t = torch.as_tensor(np.ascontiguousarray(tcol, dtype=np.float32), device=dev)
    m = torch.as_tensor(np.ascontiguousarray(np.asarray(target.mask, dtype=np.uint8)), device=dev)
    out, g = loss_device(c, t, m, ssim_weight)
    return float(out[0].item()), g.double().cpu().numpy()


def allreduce_grads(buf: torch.Tensor, world: int) -> torch.Tensor:
    """Sum the flat per-rank gradient buffer over all ranks in place (ONE collective per step).

    NCCL over NVLink/NVSwitch on the GPU box; gloo in the CPU tests.  World size 1
    is a no-op, so the 1-GPU step runs no collective at all.
    """
    if world > 1:
        import torch.distributed as dist

        dist.all_reduce(buf, op=dist.ReduceOp.SUM)
    return buf


class NaNLossError(RuntimeError):
    """trainer.py:200-205 (same message)."""

    def __init__(self, iteration, dump_path=None):
        msg = f"loss became non-finite at iteration {iteration}"
        if dump_path:
            msg += f"; scene state dumped to {dump_path}"
        super().__init__(msg)


class FlatScene:
    """A DeviceScene whose five tensors are views of one contiguous fp32 buffer."""

    def __init__(self, n: int, n_bands: int, device, buf: torch.Tensor | None = None):
        self.n, self.n_bands = n, n_bands
        widths = [w if w is not None else n_bands * 3 for _, w in FIELDS]
        self.numel = n * sum(widths)
        self.buf = buf if buf is not None else torch.zeros(self.numel, dtype=torch.float32, device=device)
        views, off = [], 0
        for (name, w), width in zip(FIELDS, widths):
            v = self.buf[off: off + n * width]
            shape = (n,) if name == "opacity_logits" else ((n, n_bands, 3) if name == "sh" else (n, width))
            views.append(v.view(shape))
            off += n * width
        self.scene = DeviceScene(*views)

    def load(self, scene):
        src = DeviceScene.from_scene(scene, device=self.buf.device)
        for name, _ in FIELDS:
            getattr(self.scene, name).copy_(getattr(src, name))

    def lr_vector(self, lrs: dict) -> torch.Tensor:
        out = torch.empty_like(self.buf)
        off = 0
        for name, _ in FIELDS:
            k = getattr(self.scene, name).numel()
            out[off: off + k] = lrs[name]
            off += k
        return out


class MultiViewTrainer:
    """C4 step: every local view rendered, lossed and back-propagated, ONE allreduce, one Adam.

    ``inflight`` views run concurrently on as many contexts/streams (each with its own gradient
    buffer; the buffers are summed before the allreduce), so one view's association overlaps
    another's raster.
    """

    def __init__(self, init_scene, cameras, targets, rank=0, world=1, device=0, config=None, lrs=None, inflight=2):
        self.rank, self.world = rank, world
        self.device = torch.device(f"cuda:{device}")
        self.config = config or RenderConfig()
        n = len(init_scene)
        nb = int(np.asarray(init_scene.sh).shape[1])
        self.params = FlatScene(n, nb, self.device)
        self.params.load(init_scene)
        self.inflight = max(1, int(inflight))
        self.grads = FlatScene(n, nb, self.device)
        self.grads_extra = [FlatScene(n, nb, self.device) for _ in range(self.inflight - 1)]
        self.m = torch.zeros_like(self.params.buf)
        self.v = torch.zeros_like(self.params.buf)
        extent = float(init_scene.extent()) if hasattr(init_scene, "extent") else 1.0
        lrs = lrs or {"means": 1.6e-4 * extent, "log_scales": 5e-3, "quats": 1e-3, "opacity_logits": 5e-2,
                      "sh": 2.5e-3}  # trainer.py:160-165,243
        self.lr = self.params.lr_vector(lrs)
        self.cameras = cameras
        self.targets = targets  # list of (H,W,3) fp32 CUDA tensors, one per local view
        self.renderers = [DeviceRenderer(device) for _ in range(self.inflight)]
        self.renderer = self.renderers[0]
        self.streams = [torch.cuda.current_stream(self.device)] + [torch.cuda.Stream(self.device)
                                                                    for _ in range(self.inflight - 1)]
        self.t = 0
        self.grad_numel = self.params.numel
        self.last_loss = None
        self._bufs = {}
        self.ssim_weight = SSIM_WEIGHT
        self.loss_ws = [LossWorkspace() for _ in range(self.inflight)]
        self.lib = _lib.load()
        # device non-finite flag of the guarded Adam (trainer.py:270-282): raised by a NaN/Inf in the
        # reduced gradients, which also skips that update; read by check_finite()
        self.nonfinite = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.dump_dir = None

    def _out(self, cam, j=0):
        key = (cam.height, cam.width, j)
        if key not in self._bufs:
            h, w, _ = key
            self._bufs[key] = (torch.empty((h, w, 3), dtype=torch.float32, device=self.device),
                               torch.empty((h, w), dtype=torch.float32, device=self.device),
                               torch.empty((h, w), dtype=torch.int32, device=self.device),
                               torch.empty((h, w, 3), dtype=torch.float32, device=self.device))
        return self._bufs[key]

    def step(self, compute_loss=False):
        loss = self.accumulate(compute_loss)
        allreduce_grads(self.grads.buf, self.world)
        self.apply()
        if compute_loss:
            self.last_loss = loss
            self.check_finite(loss)
        return loss

    def check_finite(self, loss=None):
        """Raise NaNLossError (trainer.py:270-282) if a step's loss or reduced gradients were non-finite.

        Synchronises with the device; the step loop calls it whenever it reads the loss anyway.  The
        parameters are those before the failing update (the guarded Adam skipped it); with
        ``dump_dir`` set they are saved to ``nan_dump_iter{t}.npz`` like the reference's dump."""
        bad = int(self.nonfinite.item()) != 0 or (loss is not None and not np.isfinite(loss))
        if not bad:
            return
        dump_path = None
        if self.dump_dir is not None:
            dump_path = f"{self.dump_dir}/nan_dump_iter{self.t}.npz"
            sc = self.params.scene
            np.savez(dump_path, **{name: getattr(sc, name).double().cpu().numpy() for name, _ in FIELDS})
        raise NaNLossError(self.t, dump_path)

    def apply(self):
        """One Adam update of the flat parameters from the (reduced) flat gradients (trainer.py:181-197)."""
        self.t += 1
        stream = self.streams[0].cuda_stream
        _lib.check(self.lib.geer_adam(self.params.buf.data_ptr(), self.grads.buf.data_ptr(), self.m.data_ptr(),
                                      self.v.data_ptr(), self.lr.data_ptr(), self.params.numel, ctypes.c_float(0.9),
                                      ctypes.c_float(0.999), ctypes.c_float(1e-15), self.t,
                                      self.nonfinite.data_ptr(), stream))

    def accumulate(self, compute_loss=False):
        """Sum over the local views of the stored-space gradients into ``self.grads`` (no collective)."""
        main = self.streams[0]
        gbufs = [self.grads] + self.grads_extra
        start = torch.cuda.Event()
        start.record(main)
        for j, s in enumerate(self.streams):
            if j:
                s.wait_event(start)  # the previous step's Adam update is done
            with torch.cuda.stream(s):
                gbufs[j].buf.zero_()
        outs = []
        for v, (cam, target) in enumerate(zip(self.cameras, self.targets)):
            j = v % self.inflight
            with torch.cuda.stream(self.streams[j]):
                color, rem, cnt, dl = self._out(cam, j)
                r = self.renderers[j]
                r.forward(self.params.scene, cam, self.config, out=(color, rem, cnt), sync=False)
                # trainer.py:269 loss(): (1 - w) L1 + w (1 - SSIM) and its image gradient
                out, _ = loss_device(color, target, None, self.ssim_weight, grad=dl, workspace=self.loss_ws[j])
                r.backward(dl, grads=gbufs[j].scene, accumulate=True, opacity_logit=True)
                if compute_loss:
                    outs.append(out[0].clone())
        for j, s in enumerate(self.streams[1:], start=1):
            done = torch.cuda.Event()
            done.record(s)
            main.wait_event(done)
            self.grads.buf.add_(gbufs[j].buf)
        # device-side status of every view's forward (one host sync per step): a non-PD covariance raises
        # like the reference; a graph that outgrew a context's capacity re-runs the accumulation
        if any([r.sync() for r in self.renderers if r._stream is not None]):
            return self.accumulate(compute_loss)
        return float(sum(float(o) for o in outs)) if compute_loss else 0.0
