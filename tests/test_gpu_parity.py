"""GPU parity: the CUDA path (through the C ABI) against the reference fixtures and the oracle.

Small fixtures and BASELINE config 1 are compared with the outputs of the
unmodified reference (tests/golden, made by make_golden.py); bigger scenes up
to the full 1M-Gaussian 1080p config are compared with the fp64 C oracle,
which is itself pinned to the reference by tests/test_oracle_golden.py.
"""

import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2505_24053_b200 import association, renderer
import workloads as synth
from tests import golden_cases as G
from tests import parity as P

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", G.SMALL_CASES)
def test_fixture_association_forward_backward(name):
    c = G.case(name)
    d = c.data
    if "error" in d:
        with pytest.raises(ValueError, match=str(d["error"])):
            renderer.render(c.scene, c.camera, c.config)
        with pytest.raises(ValueError, match=str(d["error"])):
            association.build_render_graph(c.scene, c.camera, c.config.lam, c.config.tile_px)
        return
    fr = renderer.render(c.scene, c.camera, c.config)
    assert fr.color.color.dtype == np.float64 and fr.contributor_count.dtype == np.int64
    if len(c.scene) == 0:  # background through the fp32 output buffer
        np.testing.assert_allclose(fr.color.color, d["color"], rtol=0, atol=1e-7)
        np.testing.assert_array_equal(fr.remaining_transmittance, d["remaining"])
        np.testing.assert_array_equal(fr.contributor_count, d["count"])
        return
    g = association.build_render_graph(c.scene, c.camera, c.config.lam, c.config.tile_px)
    P.assert_graph_equal(g, d["order"], d["entry_tile"], d["ranges"], d["keep"], d["clamped"])
    np.testing.assert_array_equal(g.grid.pixel_tile, d["grid_pixel_tile"])
    np.testing.assert_allclose(g.grid.mirror_edges_x, d["grid_ex"], rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(g.grid.mirror_edges_y, d["grid_ey"], rtol=1e-14, atol=1e-15)
    # contributor_count is not comparable fp32-vs-fp64 without the support cutoff
    P.assert_image_close(fr.color.color, fr.remaining_transmittance, fr.contributor_count, d["color"],
                         d["remaining"], d["count"], check_count=bool(c.config.support_cutoff))
    gr = renderer.render_backward(c.scene, c.camera, d["dl_dimage"], c.config)
    P.assert_grads_close(gr, d)


def test_c1_against_reference():
    """BASELINE config 1: 10k Gaussians, 256x256 pinhole, vs the reference's own outputs."""
    d = G.load("C1")
    scene = synth.config_scene("C1")
    cam = synth.config_camera("C1")
    g = association.build_render_graph(scene, cam)
    P.assert_graph_equal(g, d["order"], None, d["ranges"], d["keep"], d["clamped"])
    fr = renderer.render(scene, cam, renderer.RenderConfig())
    P.assert_image_close(fr.color.color, fr.remaining_transmittance, fr.contributor_count, d["color"],
                         d["remaining"], d["count"])
    dl = np.random.default_rng(1).standard_normal((256, 256, 3)) / (256 * 256)
    gr = renderer.render_backward(scene, cam, dl, renderer.RenderConfig())
    P.assert_grads_close(gr, d, idx=d["grad_sample"])


@pytest.mark.parametrize("n,w,h", [(100_000, 480, 270)])
def test_c2_distribution_reduced_vs_oracle(n, w, h):
    """C2 scene distribution at reduced size: association, image and gradients vs the oracle."""
    scene = synth.config_scene("C2", n=n)
    cam = synth.config_camera("C2", width=w, height=h)
    og = O.build_render_graph(scene, cam)
    g = association.build_render_graph(scene, cam)
    P.assert_graph_equal(g, og.order, og.entry_tile, og.ranges, og.keep, og.clamped)
    cfg = renderer.RenderConfig(background=np.array([0.1, 0.0, 0.3]))
    of = O.render(scene, cam, cfg, graph=og)
    fr = renderer.render(scene, cam, cfg)
    P.assert_image_close(fr.color.color, fr.remaining_transmittance, fr.contributor_count, of.color, of.remaining,
                         of.count)
    dl = np.random.default_rng(1).standard_normal((h, w, 3)) / (h * w)
    ob = O.render_backward(scene, cam, dl, cfg, graph=og)
    gr = renderer.render_backward(scene, cam, dl, cfg)
    P.assert_grads_close(gr, vars(ob))


def test_kb_wide_vs_oracle():
    """Equidistant KB fisheye (C5 camera model, reduced): non-separable grid, empty and oversized tiles."""
    scene = synth.config_scene("C5", n=60_000)
    cam = synth.config_camera("C5", width=640, height=360)
    og = O.build_render_graph(scene, cam)
    g = association.build_render_graph(scene, cam)
    np.testing.assert_array_equal(g.grid.pixel_tile, og.grid.pixel_tile)
    P.assert_graph_equal(g, og.order, og.entry_tile, og.ranges, og.keep, og.clamped)
    cfg = renderer.RenderConfig()
    of = O.render(scene, cam, cfg, graph=og)
    fr = renderer.render(scene, cam, cfg)
    P.assert_image_close(fr.color.color, fr.remaining_transmittance, fr.contributor_count, of.color, of.remaining,
                         of.count)
    dl = np.random.default_rng(2).standard_normal((360, 640, 3)) / (360 * 640)
    ob = O.render_backward(scene, cam, dl, cfg, graph=og)
    gr = renderer.render_backward(scene, cam, dl, cfg)
    P.assert_grads_close(gr, vars(ob))


def test_full_c2_association_and_forward_vs_oracle():
    """BASELINE config 2 at full size (1M Gaussians, 1920x1080 BEAP 180 deg): bit-exact graph, image."""
    scene = synth.config_scene("C2")
    cam = synth.config_camera("C2")
    og = O.build_render_graph(scene, cam)
    g = association.build_render_graph(scene, cam)
    P.assert_graph_equal(g, og.order, og.entry_tile, og.ranges, og.keep, og.clamped)
    of = O.render(scene, cam, None, graph=og)
    fr = renderer.render(scene, cam, renderer.RenderConfig())
    rep = P.assert_image_close(fr.color.color, fr.remaining_transmittance, fr.contributor_count, of.color,
                               of.remaining, of.count)
    print("C2 image parity", rep, "entries", len(g.order))


def test_full_c5_association_and_forward_vs_oracle():
    """BASELINE config 5 at full size (6M Gaussians, 3840x2160 equidistant KB fisheye): bit-exact graph
    (23.7M entries), image within tolerance, exact contributor counts."""
    O.set_num_threads(os.cpu_count())
    scene = synth.config_scene("C5")
    cam = synth.config_camera("C5")
    og = O.build_render_graph(scene, cam)
    g = association.build_render_graph(scene, cam)
    P.assert_graph_equal(g, og.order, og.entry_tile, og.ranges, og.keep, og.clamped)
    of = O.render(scene, cam, None, graph=og)
    fr = renderer.render(scene, cam, renderer.RenderConfig())
    rep = P.assert_image_close(fr.color.color, fr.remaining_transmittance, fr.contributor_count, of.color,
                               of.remaining, of.count)
    print("C5 image parity", rep, "entries", len(g.order))


def test_full_c3_backward_vs_oracle():
    """BASELINE config 3 at full size: 1M-Gaussian gradients (means/scales/rotations/opacity/SH) vs the oracle."""
    scene = synth.config_scene("C2")
    cam = synth.config_camera("C2")
    cfg = renderer.RenderConfig()
    dl = np.random.default_rng(1).standard_normal((1080, 1920, 3)) / (1080 * 1920)
    og = O.build_render_graph(scene, cam)
    ob = O.render_backward(scene, cam, dl, cfg, graph=og)
    gr = renderer.render_backward(scene, cam, dl, cfg)
    rep = P.assert_grads_close(gr, vars(ob))
    print("C3 gradient parity", rep)


def _mixed_scene(n_small, n_big, seed):
    """Many small Gaussians plus large ones (x/y tile ranges far beyond 32 tiles) and a few huge,
    very transparent ones around the camera (clamped, routed to every tile)."""
    rng = np.random.default_rng(seed)
    parts = [synth.config_scene("C2", n=n_small),
             synth.random_scene(n_big, rng, spread=1.5, scale_range=(0.2, 0.9), sh_bands=16, anisotropy=4.0),
             synth.random_scene(6, rng, spread=0.3, scale_range=(2.5, 4.0), sh_bands=16, opacity_range=(0.3, 0.5))]
    cat = lambda k: np.concatenate([getattr(p, k) for p in parts])
    from paper_2505_24053_b200.scene import GaussianScene

    return synth.to_f32_values(GaussianScene(cat("means"), cat("log_scales"), cat("quats"), cat("opacity_logits"),
                                             cat("sh")))


@pytest.mark.parametrize("camera", ["c2_1080p", "beap300_inside", "kb_720p_tile8"])
def test_binning_edge_cases_vs_oracle(camera):
    """Tile lists (two-level bucketing) bit-exact against the oracle where ranges are long (> 32 tiles),
    split in several pieces (300 deg camera inside the cloud) or cover every tile (clamped)."""
    from paper_2505_24053_b200.scene import Camera

    scene = _mixed_scene(30_000, 300, 5)
    tile_px = 16
    if camera == "c2_1080p":
        cam = synth.config_camera("C2")
    elif camera == "beap300_inside":
        rot, t = synth.look_at((0.1, -0.05, 0.2), target=(1.0, 0.2, 0.4))
        cam = Camera(width=960, height=512, model="beap", rotation=rot, translation=t, fov_x=np.deg2rad(300.0),
                     fov_y=np.deg2rad(160.0))
    else:
        cam = synth.config_camera("C5", width=1280, height=720)
        tile_px = 8
    og = O.build_render_graph(scene, cam, tile_px=tile_px)
    assert og.clamped.any()
    g = association.build_render_graph(scene, cam, tile_px=tile_px)
    P.assert_graph_equal(g, og.order, og.entry_tile, og.ranges, og.keep, og.clamped)
    cfg = renderer.RenderConfig(tile_px=tile_px)
    of = O.render(scene, cam, cfg, graph=og)
    fr = renderer.render(scene, cam, cfg)
    P.assert_image_close(fr.color.color, fr.remaining_transmittance, fr.contributor_count, of.color, of.remaining,
                         of.count)


def test_binning_many_rows_vs_oracle():
    """More than 1024 tile rows (the row-segment scan loops) and a wide 480-tile row (lane-owned
    counters up to 15 per lane): association bit-exact against the oracle."""
    from paper_2505_24053_b200.scene import Camera

    scene = synth.config_scene("C2", n=20_000)
    for w, h in ((48, 8400), (3840, 40)):
        rot, t = synth.look_at((0.0, 0.0, -2.0))
        cam = Camera(width=w, height=h, model="beap", rotation=rot, translation=t,
                     fov_x=np.deg2rad(180.0 * w / max(w, h)), fov_y=np.deg2rad(180.0 * h / max(w, h)))
        og = O.build_render_graph(scene, cam, tile_px=8)
        g = association.build_render_graph(scene, cam, tile_px=8)
        assert og.grid.n_y > 1024 or og.grid.n_x > 400
        P.assert_graph_equal(g, og.order, og.entry_tile, og.ranges, og.keep, og.clamped)
