import numpy as np, sys
sys.path.insert(0, '.')
import workloads as synth
from paper_2505_24053_b200 import renderer
for name in ("C2", "C5"):
    scene = synth.config_scene(name)
    cam = synth.config_camera(name)
    g = renderer.build_graph_for(scene, cam)
    keep = np.asarray(g.keep)
    order = np.asarray(g.order)
    emitting = np.unique(order).size
    print(name, "N", keep.size, "keep", int(keep.sum()), "emitting", emitting, "frac", emitting / keep.size)
