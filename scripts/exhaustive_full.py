"""One-off: tiled render == exhaustive render (every tile composites every kept Gaussian, the GPU
restatement of oracle.exhaustive_render) on the full C2 config.  python scripts/exhaustive_full.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_24053_b200 import _lib, renderer# noqa: E402
import workloads as synth# noqa: E402
from paper_2505_24053_b200.device import DeviceRenderer, DeviceScene  # noqa: E402

scene = synth.config_scene("C2")
cam = synth.config_camera("C2")
cfg = renderer.RenderConfig()
ds = DeviceScene.from_scene(scene)
r = DeviceRenderer(0)
tiled = [t.clone() for t in r.forward(ds, cam, cfg)]
st_t = r.stats()
torch.cuda.synchronize()
t0 = time.time()
exh = [t.clone() for t in r.forward(ds, cam, cfg, flags=_lib.GEER_CFG_EXHAUSTIVE | _lib.GEER_CFG_NO_CULL)]
torch.cuda.synchronize()
dt = time.time() - t0
st_e = r.stats()
diff = {k: int((a != b).sum().item()) for k, a, b in zip(("color", "remaining", "count"), tiled, exh)}
print(json.dumps({"config": "C2 full (1M Gaussians, 1920x1080 BEAP 180)", "differing_values": diff,
                  "evaluated_pairs_tiled": st_t["evaluated_pairs"], "evaluated_pairs_exhaustive": st_e["evaluated_pairs"],
                  "exhaustive_seconds": round(dt, 2)}))
