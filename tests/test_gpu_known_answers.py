"""Closed-form known answers through the CUDA path (SPEC.md examples restated as scenes).

Each case is small enough to evaluate by hand from the reference semantics
(renderer.py:96-118, core.py:27-31, 289-313), independently of the oracle:

* kappa of a line at whitened distance 2 is 4 and T = sigma e^{-2};
* a Gaussian straight BEHIND the camera renders at the image centre with full
  weight: the integral is over the whole line;
* two Gaussians on one ray composite front to back;
* the support cutoff kappa <= lam^2 is a hard edge (renderer.py:103-105);
* early stop: remaining < 1e-4 ends a pixel, t is clamped to 0.999 (core.py:30-31);
* dC/dsigma and dC/dsh_dc of one contribution (renderer.py:284-292, 332).
"""

import numpy as np
import pytest

from paper_2505_24053_b200 import renderer
from paper_2505_24053_b200.scene import Camera, GaussianScene

pytestmark = pytest.mark.gpu

C0 = 0.28209479177387814  # core.py:34


def f32(x):
    return np.asarray(x, np.float32).astype(np.float64)


def scene_of(means, opac, dc, log_scale=0.0):
    means = f32(np.atleast_2d(means))
    n = len(means)
    logit = f32(np.log(np.asarray(opac, np.float64) / (1 - np.asarray(opac, np.float64))) * np.ones(n))
    sh = np.zeros((n, 1, 3))
    sh[:, 0, :] = f32(dc)
    return GaussianScene(means, f32(np.full((n, 3), log_scale)), f32(np.tile([1.0, 0, 0, 0], (n, 1))), logit, sh)


def sigma_of(scene):
    return 1.0 / (1.0 + np.exp(-scene.opacity_logits))


def pinhole_1px():
    # camera.py:213-219: pixel x has u = (x - cx) / fx, so cx = cy = 0 puts pixel (0, 0) on the optical axis
    return Camera(width=1, height=1, model="pinhole", rotation=np.eye(3), translation=np.zeros(3), fx=100.0, fy=100.0,
                  cx=0.0, cy=0.0)


def test_kappa_4_single_contribution():
    sc = scene_of([[2.0, 0.0, 5.0]], 0.8, [0.3, -0.2, 0.9])
    bg = np.array([0.1, 0.2, 0.3])
    out = renderer.render(sc, pinhole_1px(), renderer.RenderConfig(background=bg))
    t = sigma_of(sc)[0] * np.exp(-2.0)  # kappa = |o x d|^2 = 4
    c = np.maximum(0.5 + C0 * sc.sh[0, 0], 0.0)
    np.testing.assert_allclose(out.color.color[0, 0], t * c + (1 - t) * bg, rtol=0, atol=2e-6)
    np.testing.assert_allclose(out.remaining_transmittance[0, 0], 1 - t, rtol=0, atol=2e-7)
    assert out.contributor_count[0, 0] == 1


def test_behind_camera_renders_at_centre_with_full_weight():
    sc = scene_of([[0.0, 0.0, -5.0]], 0.6, [0.4, 0.1, -0.3])
    cam = Camera(width=64, height=64, model="beap", rotation=np.eye(3), translation=np.zeros(3),
                 fov_x=np.deg2rad(120.0), fov_y=np.deg2rad(120.0))
    out = renderer.render(sc, cam, renderer.RenderConfig())
    # camera.py:126: pixel w/2 has angle exactly 0 -> the optical axis, kappa = 0 along the full line
    c = np.maximum(0.5 + C0 * sc.sh[0, 0], 0.0)
    np.testing.assert_allclose(out.color.color[32, 32], sigma_of(sc)[0] * c, rtol=0, atol=2e-6)
    assert out.contributor_count[32, 32] == 1


def test_front_to_back_composite_of_two():
    sc = scene_of([[0.0, 0.0, 4.0], [0.0, 0.0, 6.0]], [0.5, 0.7], [[0.2, 0.3, 0.4], [-0.5, 0.6, 0.1]])
    bg = np.array([0.05, 0.0, 0.2])
    out = renderer.render(sc, pinhole_1px(), renderer.RenderConfig(background=bg))
    s = sigma_of(sc)
    c = np.maximum(0.5 + C0 * sc.sh[:, 0], 0.0)
    exp = s[0] * c[0] + (1 - s[0]) * s[1] * c[1] + (1 - s[0]) * (1 - s[1]) * bg
    np.testing.assert_allclose(out.color.color[0, 0], exp, rtol=0, atol=2e-6)
    assert out.contributor_count[0, 0] == 2


@pytest.mark.parametrize("dist,inside", [(2.999, True), (3.001, False)])
def test_support_cutoff_is_a_hard_edge(dist, inside):
    sc = scene_of([[dist, 0.0, 5.0]], 0.9, [0.5, 0.5, 0.5])
    out = renderer.render(sc, pinhole_1px(), renderer.RenderConfig())
    assert out.contributor_count[0, 0] == (1 if inside else 0)
    t = sigma_of(sc)[0] * np.exp(-0.5 * f32(dist) ** 2) if inside else 0.0
    np.testing.assert_allclose(out.remaining_transmittance[0, 0], 1 - t, rtol=0, atol=2e-7)


def test_early_stop_and_clamp():
    # 12 nearly opaque Gaussians on the axis: t = min(sigma, 0.999); rem 1 -> 1e-3 -> 1e-6 < 1e-4 stops
    n = 12
    sc = scene_of(np.c_[np.zeros(n), np.zeros(n), 3.0 + np.arange(n)], 0.9999, np.zeros((n, 3)))
    out = renderer.render(sc, pinhole_1px(), renderer.RenderConfig())
    assert out.contributor_count[0, 0] == 2  # the third entry is not alive (remaining 1e-6 < 1e-4)
    np.testing.assert_allclose(out.remaining_transmittance[0, 0], 0.001 ** 2, rtol=0, atol=1e-9)


def test_gradient_of_one_contribution():
    sc = scene_of([[2.0, 0.0, 5.0]], 0.8, [0.3, -0.2, 0.9])
    bg = np.array([0.1, 0.2, 0.3])
    g_img = np.array([[[1.0, -2.0, 0.5]]])
    gr = renderer.render_backward(sc, pinhole_1px(), g_img, renderer.RenderConfig(background=bg))
    e = np.exp(-2.0)
    c = np.maximum(0.5 + C0 * sc.sh[0, 0], 0.0)
    # C = sigma e^-2 c + (1 - sigma e^-2) bg  ->  dL/dsigma (linear opacity, renderer.py:292) and dL/dsh_dc
    np.testing.assert_allclose(gr.dopacities[0], e * np.dot(c - bg, g_img[0, 0]), rtol=1e-4)
    np.testing.assert_allclose(gr.dsh[0, 0], sigma_of(sc)[0] * e * C0 * g_img[0, 0], rtol=1e-4)


def test_forward_is_deterministic():
    from paper_2505_24053_b200 import association
    import workloads as synth

    scene = synth.config_scene("C2", n=30_000)
    cam = synth.config_camera("C2", width=320, height=180)
    a = renderer.render(scene, cam, renderer.RenderConfig())
    b = renderer.render(scene, cam, renderer.RenderConfig())
    np.testing.assert_array_equal(a.color.color, b.color.color)
    np.testing.assert_array_equal(a.contributor_count, b.contributor_count)
    g1 = association.build_render_graph(scene, cam)
    g2 = association.build_render_graph(scene, cam)
    np.testing.assert_array_equal(g1.order, g2.order)
    np.testing.assert_array_equal(g1.ranges, g2.ranges)
