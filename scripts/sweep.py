"""Forward throughput (4 frames in flight) and single-frame stage times over scene sizes and resolutions.

    python scripts/sweep.py > profiles/r01_sweep.md
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_24053_b200 import renderer# noqa: E402
import workloads as synth# noqa: E402
from paper_2505_24053_b200.device import DeviceRenderer, DeviceScene  # noqa: E402

NF = 4
print("| scene | Gaussians | camera | entries | frame latency (ms) | throughput (FPS, 4 in flight) | Mrays/s |")
print("|---|---:|---|---:|---:|---:|---:|")
for cfg_name, n, w, h in (("C2", 100_000, 1920, 1080), ("C2", 1_000_000, 1280, 720), ("C2", 1_000_000, 1920, 1080),
                          ("C2", 1_000_000, 3840, 2160), ("C2", 3_000_000, 1920, 1080), ("C5", 6_000_000, 3840, 2160),
                          ("C1", 1_000_000, 1920, 1080)):
    scene = synth.config_scene(cfg_name, n=n)
    cam = synth.config_camera(cfg_name, width=w, height=h)
    cfg = renderer.RenderConfig()
    ds = DeviceScene.from_scene(scene)
    rs = [DeviceRenderer(0) for _ in range(NF)]
    streams = [torch.cuda.Stream() for _ in range(NF)]
    outs = [None] * NF
    for j in range(NF):
        with torch.cuda.stream(streams[j]):
            outs[j] = tuple(t.clone() for t in rs[j].forward(ds, cam, cfg))
    torch.cuda.synchronize()
    rs[0].set_timing(True)
    lat = []
    for _ in range(5):
        rs[0].forward(ds, cam, cfg, out=outs[0])
        lat.append(rs[0].stats()["ms_total"])
    st = rs[0].stats()
    rs[0].set_timing(False)
    k = 40
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for s in streams:
        s.wait_event(e0)
    for i in range(k):
        j = i % NF
        with torch.cuda.stream(streams[j]):
            rs[j].forward(ds, cam, cfg, out=outs[j])
    cur = torch.cuda.current_stream()
    for s in streams:
        ev = torch.cuda.Event()
        ev.record(s)
        cur.wait_event(ev)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / k
    lat.sort()
    model = {"C1": "pinhole 60°", "C2": "BEAP 180°", "C5": "KB fisheye 180°"}[cfg_name]
    print(f"| {cfg_name} | {n:,} | {model} {w}x{h} | {st['n_entries']:,} | {lat[len(lat) // 2]:.3f} | "
          f"{1e3 / ms:.1f} | {w * h * 1e3 / ms / 1e6:.0f} |", flush=True)
    del rs, outs, ds
    torch.cuda.empty_cache()
