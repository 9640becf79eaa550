"""How much of the tile-list building a depth-sliced association would keep (C2).

For a split of the depth order at rank q, a tile needs its slice-0 entries (rank < q) and, only if
some pixel streams past them (max n_eval over the tile > slice-0 length), the rest of its list.
Prints the fraction of the 7.41M entries that would be built, per q.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2505_24053_b200 import _lib, renderer  # noqa: E402
from paper_2505_24053_b200.device import DeviceRenderer, DeviceScene  # noqa: E402
import workloads as synth  # noqa: E402

scene = synth.config_scene("C2")
cam = synth.config_camera("C2")
ds = DeviceScene.from_scene(scene)
r = DeviceRenderer(0)
r.forward(ds, cam, renderer.RenderConfig())
lib = r.ctx._lib
lib.geer_debug_n_eval.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
ne = np.empty(cam.height * cam.width, np.int32)
_lib.check(lib.geer_debug_n_eval(r.ctx.ptr, ne.ctypes.data))
n_ent, n_x, n_y = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32()
_lib.check(lib.geer_graph_info(r.ctx.ptr, ctypes.byref(n_ent), ctypes.byref(n_x), ctypes.byref(n_y)))
E, nx, ny = n_ent.value, n_x.value, n_y.value
order = np.empty(E, np.int64)
ranges = np.empty(nx * ny + 1, np.int64)
_lib.check(lib.geer_graph_export(r.ctx.ptr, order.ctypes.data, None, ranges.ctypes.data, None, None, None, None, None,
                                 None, None))
depth = np.linalg.norm(scene.means @ np.asarray(cam.rotation).T + np.asarray(cam.translation), axis=1)
rank = np.empty(len(depth), np.int64)
rank[np.argsort(depth.astype(np.float32), kind="stable")] = np.arange(len(depth))
ne2 = ne.reshape(cam.height, cam.width)
tmax = np.zeros(nx * ny, np.int64)
for ty in range(ny):
    for tx in range(nx):
        blk = ne2[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16]
        tmax[ty * nx + tx] = blk.max() if blk.size else 0
lens = np.diff(ranges)
print(f"entries {E}, streamed prefix (sum of per-tile max n_eval) {tmax.sum()} = {tmax.sum() / E:.3f}")
er = rank[order]
for q in (0.05, 0.1, 0.15, 0.2, 0.3, 0.4, 0.5):
    cut = q * len(depth)
    cs = np.concatenate([[0], np.cumsum((er < cut).astype(np.int64))])
    l0 = cs[ranges[1:]] - cs[ranges[:-1]]
    need = tmax > l0
    built = l0.sum() + (lens - l0)[need].sum()
    print(f"q {q:.2f}: slice-0 entries {l0.sum() / E:.3f}, tiles needing slice 1 {need.mean():.3f}, built {built / E:.3f}")
