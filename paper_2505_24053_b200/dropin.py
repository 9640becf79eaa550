"""Patch a live ``raygauss`` (the reference package) so its callers render on the B200.

    import raygauss.trainer
    from paper_2505_24053_b200 import dropin
    dropin.install()          # raygauss.renderer / association / trainer now call libgeer_b200.so
    ...
    dropin.uninstall()

The trainer imports ``render`` / ``render_backward`` by name (trainer.py:23),
so both ``raygauss.renderer`` and ``raygauss.trainer`` are patched (SURVEY
§3.3); ``raygauss.trainer.loss`` (L1 + SSIM, trainer.py:114-155) runs on the GPU too.  Results come back as the reference's OWN dataclasses
(``raygauss.renderer.FrameOutput`` with a ``raygauss.camera.BEAPImage``,
``raygauss.renderer.SceneGrads``, ``raygauss.association.RenderGraph``), so
code that type-checks or pattern-matches on them keeps working.
"""

from __future__ import annotations

import importlib
import sys

_saved: dict = {}


def _ref(name: str):
    return importlib.import_module(f"raygauss.{name}")


def _to_ref_graph(g, ra):
    if g is None:
        return None
    grid = ra.CSFGrid(n_x=g.grid.n_x, n_y=g.grid.n_y, mirror_edges_x=g.grid.mirror_edges_x,
                      mirror_edges_y=g.grid.mirror_edges_y, pixel_tile=g.grid.pixel_tile)
    return ra.RenderGraph(order=g.order, entry_tile=g.entry_tile, ranges=g.ranges, mu_c=g.mu_c, depth=g.depth,
                          keep=g.keep, clamped=g.clamped, grid=grid)


def make_render(with_graph: bool | None = None):
    """``raygauss.renderer.render`` replacement (renderer.py:123-176): ``FrameOutput.graph`` is the
    reference's ``RenderGraph`` (lazily exported by default, see ``renderer.lazy_dataclass``)."""
    from . import renderer

    def render(scene, camera, config=None):
        rr, rc, ra = _ref("renderer"), _ref("camera"), _ref("association")
        out = renderer.render(scene, camera, config, return_graph=False if with_graph is None else with_graph)
        if with_graph is None:
            cfg = config or renderer.RenderConfig()
            graph = renderer.lazy_dataclass(
                ra.RenderGraph, lambda: _to_ref_graph(renderer.build_graph_for(scene, camera, cfg.lam, cfg.tile_px), ra))
        else:
            graph = _to_ref_graph(out.graph, ra)
        return rr.FrameOutput(color=rc.BEAPImage(color=out.color.color, mask=out.color.mask),
                              remaining_transmittance=out.remaining_transmittance,
                              contributor_count=out.contributor_count, graph=graph)

    render.__doc__ = "B200 drop-in for raygauss.renderer.render (libgeer_b200.so)"
    return render


def render_backward(scene, camera, dl_dimage, config=None):
    """``raygauss.renderer.render_backward`` replacement (renderer.py:234-333)."""
    from . import renderer

    rr = _ref("renderer")
    g = renderer.render_backward(scene, camera, dl_dimage, config)
    return rr.SceneGrads(dmeans=g.dmeans, dlog_scales=g.dlog_scales, dquats=g.dquats, dopacities=g.dopacities,
                         dsh=g.dsh)


def build_render_graph(scene, camera, lam: float = 3.0, tile_px: int = 16, grid=None):
    """``raygauss.association.build_render_graph`` replacement (association.py:391-476).

    ``grid`` is accepted for signature compatibility; the grid is rebuilt on the
    device from the camera (it is a pure function of camera and tile size).
    """
    from . import association

    return _to_ref_graph(association.build_render_graph(scene, camera, lam, tile_px), _ref("association"))


def loss(rendered, target, ssim_weight: float = 0.2):
    """``raygauss.trainer.loss`` replacement (trainer.py:114-155): masked L1 + SSIM on the GPU."""
    from . import train

    return train.loss(rendered, target, ssim_weight)


# (module, attribute) pairs that install() rebinds
TARGETS = (("renderer", "render"), ("renderer", "render_backward"), ("association", "build_render_graph"),
           ("trainer", "render"), ("trainer", "render_backward"), ("trainer", "loss"))


def install(with_graph: bool | None = None) -> list[str]:
    """Rebind the reference's render entry points to the B200 path; returns what was patched.

    Modules of ``raygauss`` that are not importable (or do not bind a name) are
    skipped.  The CUDA library is loaded eagerly so a missing build fails here,
    not on the first frame.
    """
    from . import _lib

    _lib.load()
    repl = {"render": make_render(with_graph), "render_backward": render_backward,
            "build_render_graph": build_render_graph, "loss": loss}
    patched = []
    for mod_name, attr in TARGETS:
        try:
            mod = _ref(mod_name)
        except ImportError:
            continue
        if not hasattr(mod, attr):
            continue
        key = (mod.__name__, attr)
        if key not in _saved:
            _saved[key] = getattr(mod, attr)
        setattr(mod, attr, repl[attr])
        patched.append(f"{mod.__name__}.{attr}")
    return patched


def uninstall() -> None:
    """Restore every attribute install() replaced."""
    for (mod_name, attr), fn in list(_saved.items()):
        mod = sys.modules.get(mod_name)
        if mod is not None:
            setattr(mod, attr, fn)
        del _saved[(mod_name, attr)]
