"""Print median stage times of C2 frames (forward + backward) with library CUDA events."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_24053_b200 import renderer# noqa: E402
import workloads as synth# noqa: E402
from paper_2505_24053_b200.device import DeviceRenderer, DeviceScene  # noqa: E402

n = int(os.environ.get("N_GAUSS", "1000000"))
scene = synth.config_scene("C2", n=n)
cam = synth.config_camera("C2")
ds = DeviceScene.from_scene(scene)
r = DeviceRenderer(0)
cfg = renderer.RenderConfig()
dl = torch.randn((cam.height, cam.width, 3), device="cuda") / (cam.height * cam.width)
for _ in range(3):
    r.forward(ds, cam, cfg)
    r.backward(dl)
r.set_timing(True)
st = []
for _ in range(7):
    r.forward(ds, cam, cfg)
    r.backward(dl)
    st.append(r.stats())
keys = ["ms_prep", "ms_dup", "ms_sort", "ms_render", "ms_total", "ms_backward", "fixup_pixels", "kappa_rechecks", "warp_entries", "evaluated_pairs", "streamed_entries"]
print(json.dumps({k: float(np.median([s[k] for s in st])) for k in keys}))
