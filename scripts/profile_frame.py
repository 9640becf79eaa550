"""Render C2 frames for profiling: python scripts/profile_frame.py [--frames N] [--backward] [--n N]."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_24053_b200 import renderer# noqa: E402
import workloads as synth# noqa: E402
from paper_2505_24053_b200.device import DeviceRenderer, DeviceScene  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=3)
ap.add_argument("--backward", action="store_true")
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--config", default="C2")
a = ap.parse_args()
scene = synth.config_scene(a.config, n=a.n)
cam = synth.config_camera(a.config)
ds = DeviceScene.from_scene(scene)
r = DeviceRenderer(0)
cfg = renderer.RenderConfig()
dl = torch.randn((cam.height, cam.width, 3), device="cuda") / (cam.height * cam.width)
for _ in range(a.frames):
    r.forward(ds, cam, cfg)
    if a.backward:
        r.backward(dl)
torch.cuda.synchronize()
print(r.stats())
