"""Contributing pairs vs evaluated / issued pairs of one C2 forward (culling efficiency)."""
import json

import numpy as np
import torch

from paper_2505_24053_b200 import renderer
import workloads as synth
from paper_2505_24053_b200.device import DeviceRenderer, DeviceScene

scene = synth.config_scene("C2")
cam = synth.config_camera("C2")
r = DeviceRenderer(0)
ds = DeviceScene.from_scene(scene)
color, rem, cnt = r.forward(ds, cam, renderer.RenderConfig())
torch.cuda.synchronize()
st = r.stats()
npx = cam.width * cam.height
out = {"pixels": npx, "contributing_pairs": int(cnt.sum().item()), "evaluated_pairs": st["evaluated_pairs"],
       "issued_pairs": st["warp_entries"] * 32, "entries": st["n_entries"], "streamed": st["streamed_entries"],
       "opaque_fraction": float((rem < 1e-4).float().mean().item()), "mean_remaining": float(rem.mean().item())}
print(json.dumps(out))
