"""Randomised GPU-vs-oracle parity: many small scenes and cameras drawn at random.

Each case draws a scene (size, spread, scales, anisotropy, opacity, SH bands), a camera (BEAP with
fields of view up to 300 x 160 degrees, KB fisheye with random distortion, or pinhole; placed
outside or inside the cloud) and a render config (lambda, tile size, support cutoff, background),
then checks the CUDA path against the fp64 C oracle: the association bit for bit, the image
within the north_star tolerance, contributor counts exactly (when the cutoff is on),
and the backward within the gradient tolerance.
"""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2505_24053_b200 import association, renderer
import workloads as synth
from paper_2505_24053_b200.scene import Camera
from tests import parity as P

pytestmark = pytest.mark.gpu

N_CASES = 150
N_LARGE = 20  # 5k-40k Gaussians at up to 480 x 320


def draw_case(seed, large=False):
    rng = np.random.default_rng(1000 + seed + (100_000 if large else 0))
    n = int(rng.integers(5_000, 40_000)) if large else int(rng.integers(50, 3000))
    bands = int(rng.choice([1, 4, 9, 16]))
    scene = synth.to_f32_values(synth.random_scene(
        n, rng, spread=float(rng.uniform(0.5, 2.0)),
        scale_range=(float(rng.uniform(0.01, 0.05)), float(rng.uniform(0.06, 0.4))),
        opacity_range=(float(rng.uniform(0.05, 0.5)), float(rng.uniform(0.6, 0.99))), sh_bands=bands,
        anisotropy=float(rng.uniform(1.0, 6.0))))
    inside = rng.random() < 0.3
    pos = rng.normal(size=3)
    pos *= (0.2 if inside else float(rng.uniform(2.0, 4.0))) / np.linalg.norm(pos)
    target = rng.normal(size=3) * 0.5
    rot, t = synth.look_at(pos, target=tuple(target))
    w, h = (int(rng.integers(200, 480)), int(rng.integers(120, 320))) if large else \
        (int(rng.integers(24, 200)), int(rng.integers(16, 140)))
    model = rng.choice(["beap", "beap", "kb", "pinhole"])
    if model == "beap":
        fx_deg = float(rng.uniform(60.0, 300.0))
        cam = Camera(width=w, height=h, model="beap", rotation=rot, translation=t, fov_x=np.deg2rad(fx_deg),
                     fov_y=np.deg2rad(min(160.0, fx_deg * h / w)))
    elif model == "kb":
        f = (w / 2) / float(rng.uniform(0.8, 1.6))
        k = rng.uniform(-0.02, 0.02, 4)
        cam = Camera(width=w, height=h, model="kb", rotation=rot, translation=t, fx=f, fy=f * float(rng.uniform(0.9, 1.1)),
                     cx=(w - 1) / 2 + float(rng.uniform(-3, 3)), cy=(h - 1) / 2 + float(rng.uniform(-3, 3)), k=k)
    else:
        f = (w / 2) / np.tan(np.deg2rad(float(rng.uniform(20.0, 60.0))))
        cam = Camera(width=w, height=h, model="pinhole", rotation=rot, translation=t, fx=f, fy=f, cx=w / 2,
                     cy=h / 2)
    cfg = renderer.RenderConfig(lam=float(rng.uniform(2.0, 4.0)), tile_px=int(rng.choice([8, 16, 32])),
                                support_cutoff=bool(rng.random() < 0.8), background=rng.uniform(0, 1, 3))
    return scene, cam, cfg


CASES = [(s, False) for s in range(N_CASES)] + [(s, True) for s in range(N_LARGE)]


@pytest.mark.parametrize("seed,large", CASES, ids=[f"{'large' if l else 'small'}{s}" for s, l in CASES])
def test_random_case_vs_oracle(seed, large):
    scene, cam, cfg = draw_case(seed, large)
    try:
        og = O.build_render_graph(scene, cam, cfg.lam, cfg.tile_px)
    except O.OracleValueError as exc:  # (e.g. a degenerate covariance): the CUDA path must refuse too
        with pytest.raises(ValueError):
            renderer.render(scene, cam, cfg)
        return
    g = association.build_render_graph(scene, cam, cfg.lam, cfg.tile_px)
    P.assert_graph_equal(g, og.order, og.entry_tile, og.ranges, og.keep, og.clamped)
    of = O.render(scene, cam, cfg, graph=og)
    fr = renderer.render(scene, cam, cfg)
    P.assert_image_close(fr.color.color, fr.remaining_transmittance, fr.contributor_count, of.color, of.remaining,
                         of.count, check_count=cfg.support_cutoff)
    dl = np.random.default_rng(seed).standard_normal((cam.height, cam.width, 3)) / (cam.height * cam.width)
    ob = O.render_backward(scene, cam, dl, cfg, graph=og)
    gr = renderer.render_backward(scene, cam, dl, cfg)
    P.assert_grads_close(gr, vars(ob))


@pytest.mark.parametrize("w,h,model,tile", [(1, 1, "beap", 16), (1, 7, "beap", 8), (7, 1, "kb", 16),
                                            (3, 2, "pinhole", 32), (33, 1, "beap", 32), (1, 65, "pinhole", 16)])
def test_degenerate_images_vs_oracle(w, h, model, tile):
    """1-pixel rows / columns and single-pixel images through the whole path."""
    rng = np.random.default_rng(w * 100 + h)
    scene = synth.to_f32_values(synth.random_scene(400, rng, spread=1.0, sh_bands=4))
    rot, t = synth.look_at((0.3, -0.2, -2.5))
    if model == "beap":
        cam = Camera(width=w, height=h, model="beap", rotation=rot, translation=t, fov_x=np.deg2rad(90.0),
                     fov_y=np.deg2rad(60.0))
    elif model == "kb":
        cam = Camera(width=w, height=h, model="kb", rotation=rot, translation=t, fx=4.0, fy=4.0, cx=(w - 1) / 2,
                     cy=(h - 1) / 2, k=np.zeros(4))
    else:
        cam = Camera(width=w, height=h, model="pinhole", rotation=rot, translation=t, fx=30.0, fy=30.0, cx=w / 2,
                     cy=h / 2)
    cfg = renderer.RenderConfig(tile_px=tile)
    og = O.build_render_graph(scene, cam, cfg.lam, cfg.tile_px)
    g = association.build_render_graph(scene, cam, cfg.lam, cfg.tile_px)
    P.assert_graph_equal(g, og.order, og.entry_tile, og.ranges, og.keep, og.clamped)
    of = O.render(scene, cam, cfg, graph=og)
    fr = renderer.render(scene, cam, cfg)
    P.assert_image_close(fr.color.color, fr.remaining_transmittance, fr.contributor_count, of.color, of.remaining,
                         of.count)
    dl = rng.standard_normal((h, w, 3))
    ob = O.render_backward(scene, cam, dl, cfg, graph=og)
    gr = renderer.render_backward(scene, cam, dl, cfg)
    P.assert_grads_close(gr, vars(ob))
