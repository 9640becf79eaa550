"""Per-CTA timeline of one C2 forward raster (needs a build with -DGEER_CTA_TIMING).

    GEER_NVCC_DEFS=-DGEER_CTA_TIMING python -m paper_2505_24053_b200.build --force
    python scripts/cta_timing.py > gpurun_out/cta_timing.txt
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2505_24053_b200 import _lib, renderer# noqa: E402
import workloads as synth# noqa: E402
from paper_2505_24053_b200.device import DeviceRenderer, DeviceScene  # noqa: E402

scene = synth.config_scene("C2")
cam = synth.config_camera("C2")
ds = DeviceScene.from_scene(scene)
r = DeviceRenderer(0)
cfg = renderer.RenderConfig()
for _ in range(3):
    r.forward(ds, cam, cfg)
torch.cuda.synchronize()
n = 16260
t0 = np.zeros(n, np.uint64); t1 = np.zeros(n, np.uint64); sm = np.zeros(n, np.int32); went = np.zeros(n, np.int32)
lib = _lib.load()
f = lib.geer_debug_cta_times
f.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int]
f(t0.ctypes.data, t1.ctypes.data, sm.ctypes.data, went.ctypes.data, n)
st = r.stats()
ts = np.zeros(n, np.uint64); tf = np.zeros(n, np.uint64)
f2 = lib.geer_debug_cta_phases
f2.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
f2(ts.ctypes.data, tf.ctypes.data, n)
ok = t1 > 0
ph_setup = (ts[ok].astype(np.int64) - t0[ok].astype(np.int64)) / 1e3
ph_first = (tf[ok].astype(np.int64) - ts[ok].astype(np.int64)) / 1e3
print("phase us: setup (start -> pipe_init) mean %.2f p50 %.2f; first stage wait mean %.2f p50 %.2f" %
      (ph_setup.mean(), np.median(ph_setup), ph_first.mean(), np.median(ph_first)))
t0 = t0[ok].astype(np.int64); t1 = t1[ok].astype(np.int64); sm = sm[ok]; went = went[ok]
base = t0.min()
t0 -= base; t1 -= base
dur = t1 - t0
print("CTAs with work", ok.sum(), "kernel span us", (t1.max()) / 1e3)
print("CTA duration us: mean %.1f p50 %.1f p90 %.1f p99 %.1f max %.1f" % (dur.mean() / 1e3, *(np.percentile(dur, [50, 90, 99]) / 1e3), dur.max() / 1e3))
# SM busy fraction: sum of CTA durations per SM / (span * CTAs per SM capacity 3)
span = t1.max()
busy = np.bincount(sm, weights=dur, minlength=148)
print("per-SM busy (sum CTA us / span us): mean %.2f min %.2f max %.2f" % (busy.mean() / span, busy.min() / span, busy.max() / span))
# concurrency over time
edges = np.linspace(0, span, 41)
conc = [((t0 < b) & (t1 > a)).sum() for a, b in zip(edges[:-1], edges[1:])]
print("CTAs resident per 1/40 of the span:", conc)
# work vs duration
order = np.argsort(-dur)[:10]
print("longest CTAs (us, warp-entries):", [(round(dur[i] / 1e3, 1), int(went[i])) for i in order])
print("ns per warp-entry (CTAs with >1000):", float(np.median(dur[went > 1000] / went[went > 1000])))
print("stats", st)
A = np.vstack([np.ones_like(went, dtype=np.float64), went.astype(np.float64)]).T
coef, *_ = np.linalg.lstsq(A, dur.astype(np.float64), rcond=None)
print("fit: CTA ns = %.0f + %.1f * warp_entries" % (coef[0], coef[1]))
print("CTAs with 0 warp-entries:", int((went == 0).sum()), "mean dur us", float(dur[went == 0].mean() / 1e3) if (went == 0).any() else 0)
