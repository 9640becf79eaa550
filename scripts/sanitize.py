"""Small forward + backward + loss + binning run for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_24053_b200 import renderer# noqa: E402
import workloads as synth# noqa: E402
from paper_2505_24053_b200.device import DeviceRenderer, DeviceScene  # noqa: E402

for name, n, w, h in (("C2", 3000, 160, 96), ("C5", 3000, 128, 80), ("C1", 2000, 64, 64)):
    scene = synth.config_scene(name, n=n)
    cam = synth.config_camera(name, width=w, height=h)
    r = DeviceRenderer(0)
    ds = DeviceScene.from_scene(scene)
    color, rem, cnt = r.forward(ds, cam, renderer.RenderConfig())
    g = r.backward(torch.ones_like(color) / color.numel())
    # a second, asynchronous frame (capacity-sized graph buffers) and its backward
    color, rem, cnt = r.forward(ds, cam, renderer.RenderConfig(), sync=False)
    g = r.backward(torch.ones_like(color) / color.numel())
    assert r.sync() is False
    torch.cuda.synchronize()
    res = r.ctx.association_check(64)
    print(name, float(color.sum()), int(cnt.sum()), res["missing"], flush=True)
# the host-buffer entry points (float64 in/out): host narrowing with a raw device-narrowed tail,
# chunked fp32 gradient download widened on the host pool (12k Gaussians: > one 512k-element chunk)
scene = synth.config_scene("C2", n=12_000)
cam = synth.config_camera("C2", width=96, height=64)
out = renderer.render(scene, cam, renderer.RenderConfig(), return_graph=False)
grads = renderer.render_backward(scene, cam, np.full((64, 96, 3), 1e-3), renderer.RenderConfig())
print("host", float(out.color.color.sum()), float(np.abs(grads.dsh).sum()), renderer.last_h2d_bytes(0), flush=True)
print("sanitize run ok")
