"""One-off: BASELINE config 5 at full size (6M Gaussians, 3840x2160 equidistant KB fisheye) through the
CUDA path and the fp64 C oracle: association bit-exact, image within the north_star tolerance.

    python scripts/parity_c5_full.py   (GPU box; ~2 minutes of oracle CPU time)
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2505_24053_b200 import association, renderer# noqa: E402
import workloads as synth# noqa: E402
from tests import parity as P  # noqa: E402

O.set_num_threads(os.cpu_count())
scene = synth.config_scene("C5")
cam = synth.config_camera("C5")
t0 = time.time()
og = O.build_render_graph(scene, cam)
t1 = time.time()
g = association.build_render_graph(scene, cam)
P.assert_graph_equal(g, og.order, og.entry_tile, og.ranges, og.keep, og.clamped)
t2 = time.time()
of = O.render(scene, cam, None, graph=og)
t3 = time.time()
fr = renderer.render(scene, cam, renderer.RenderConfig())
rep = P.assert_image_close(fr.color.color, fr.remaining_transmittance, fr.contributor_count, of.color, of.remaining,
                           of.count)
print(json.dumps({"config": "C5 full (6M Gaussians, 3840x2160 KB fisheye)", "entries": int(len(g.order)),
                  "association": "bit-exact (order, entry_tile, ranges, keep, clamped)", "image": rep,
                  "oracle_seconds": {"graph": t1 - t0, "render": t3 - t2}, "cpu_threads": os.cpu_count()},
                 default=str))
