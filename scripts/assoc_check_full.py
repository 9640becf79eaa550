"""One-off: GPU brute-force association check (oracle.association_bruteforce on the GPU) on the full
C2 and C5 configs.  python scripts/assoc_check_full.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_24053_b200 import renderer# noqa: E402
import workloads as synth# noqa: E402
from paper_2505_24053_b200.device import DeviceRenderer, DeviceScene  # noqa: E402

for name in ("C2", "C5"):
    scene = synth.config_scene(name)
    cam = synth.config_camera(name)
    r = DeviceRenderer(0)
    ds = DeviceScene.from_scene(scene)
    r.forward(ds, cam, renderer.RenderConfig())
    torch.cuda.synchronize()
    t0 = time.time()
    res = r.ctx.association_check(64)
    dt = time.time() - t0
    print(json.dumps({"config": name, "gaussians": len(scene), "width": cam.width, "height": cam.height,
                      "rays_per_tile": 64, "seconds": round(dt, 2), **{k: v for k, v in res.items() if k != "missing_pairs"},
                      "missing_pairs": res["missing_pairs"][:5]}), flush=True)
    del r, ds
    torch.cuda.empty_cache()
