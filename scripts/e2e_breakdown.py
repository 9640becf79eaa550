"""Where the e2e (host f64 in/out) frame time goes: PCIe copies vs compute."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_24053_b200 import renderer# noqa: E402
import workloads as synth# noqa: E402


def bw(label, nbytes, fn, k=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / k
    print(f"{label}: {dt * 1e3:.2f} ms, {nbytes / dt / 1e9:.1f} GB/s")


n = 472_000_000 // 8
dev = torch.empty(n, dtype=torch.float64, device="cuda")
pin = torch.empty(n, dtype=torch.float64, pin_memory=True)
page = torch.empty(n, dtype=torch.float64)
page.numpy()[:] = 1.0
bw("H2D pinned 472MB", n * 8, lambda: dev.copy_(pin, non_blocking=True))
bw("H2D pageable 472MB", n * 8, lambda: dev.copy_(page))
m = 83_000_000 // 8
bw("D2H pinned 83MB", m * 8, lambda: pin[:m].copy_(dev[:m], non_blocking=True))
bw("D2H pageable 83MB", m * 8, lambda: page[:m].copy_(dev[:m]))
bw("np.empty+D2H pageable 83MB", m * 8, lambda: torch.from_numpy(np.empty(m)).copy_(dev[:m]))

scene = synth.config_scene("C2")
cam = synth.config_camera("C2")
cfg = renderer.RenderConfig()


def pinned(a):
    t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


hs = type(scene)(pinned(scene.means), pinned(scene.log_scales), pinned(scene.quats), pinned(scene.opacity_logits),
                 pinned(scene.sh))
bw("renderer.render (pinned scene)", 555e6, lambda: renderer.render(hs, cam, cfg))
bw("renderer.render (pageable scene)", 555e6, lambda: renderer.render(scene, cam, cfg))
