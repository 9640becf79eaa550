import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2505_24053_b200 import renderer
import workloads as synth
from paper_2505_24053_b200.device import DeviceRenderer, DeviceScene
scene = synth.config_scene("C2")
cams = synth.ring_cameras(4, 2.0, 1920, 1080, fov_deg=180.0, fov_y_deg=180.0 * 1080 / 1920)
ds = DeviceScene.from_scene(scene); r = DeviceRenderer(0); cfg = renderer.RenderConfig()
for c in cams: r.forward(ds, c, cfg)
torch.cuda.synchronize()
def run(seq):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for c in seq: r.forward(ds, c, cfg)
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / len(seq)
same = run([cams[0]] * 40); alt = run([cams[i % 4] for i in range(40)])
print(f"same camera {same:.3f} ms/frame, alternating cameras {alt:.3f} ms/frame, K0 cost {alt - same:.3f} ms")
