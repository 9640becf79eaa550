"""install() rebinds the reference's entry points (incl. the trainer's by-name imports) and restores them.

Needs the reference package importable (this build container); skipped elsewhere.
The GPU-side behaviour of the patched functions is covered by test_gpu_parity.py.
"""

import os
import sys

import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")


def test_install_patches_renderer_association_and_trainer():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import raygauss.association as ra
    import raygauss.renderer as rr
    import raygauss.trainer as rt

    import paper_2505_24053_b200 as pkg
    from paper_2505_24053_b200 import dropin

    orig = (rr.render, rr.render_backward, ra.build_render_graph, rt.render, rt.render_backward, rt.loss)
    patched = pkg.install()
    try:
        assert set(patched) == {"raygauss.renderer.render", "raygauss.renderer.render_backward",
                                "raygauss.association.build_render_graph", "raygauss.trainer.render",
                                "raygauss.trainer.render_backward", "raygauss.trainer.loss"}
        assert rr.render is rt.render and rr.render is not orig[0]
        assert rr.render_backward is dropin.render_backward is rt.render_backward
        assert ra.build_render_graph is dropin.build_render_graph
    finally:
        pkg.uninstall()
    assert (rr.render, rr.render_backward, ra.build_render_graph, rt.render, rt.render_backward, rt.loss) == orig


def test_frame_output_graph_is_lazy_render_graph():
    """renderer.py:170-175: the reference always attaches the graph; here it is a lazily exported
    RenderGraph (materialised on first access, nothing copied otherwise)."""
    from paper_2505_24053_b200 import renderer
    from paper_2505_24053_b200.association import RenderGraph

    calls = []

    def thunk():
        calls.append(1)
        import numpy as np
        from paper_2505_24053_b200.association import CSFGrid

        grid = CSFGrid(n_x=1, n_y=1, mirror_edges_x=np.zeros(2), mirror_edges_y=np.zeros(2), pixel_tile=np.zeros((1, 1)))
        return RenderGraph(grid=grid, order=np.arange(3), entry_tile=np.zeros(3, int), ranges=np.array([0, 3]),
                           mu_c=np.zeros((3, 3)), depth=np.ones(3), keep=np.ones(3, bool), clamped=np.zeros(3, bool))

    g = renderer.lazy_dataclass(RenderGraph, thunk)
    assert isinstance(g, RenderGraph) and not calls
    assert list(g.order) == [0, 1, 2] and g.grid.n_x == 1 and len(calls) == 1
    _ = g.ranges
    assert len(calls) == 1
