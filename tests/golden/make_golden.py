"""Generate the golden fixtures by running the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Each case stores the fp32-rounded scene, the camera, the config, the
reference ``build_render_graph`` output (order / entry_tile / ranges / keep /
clamped), the reference ``render`` output (colour, remaining, count) and the
reference ``render_backward`` gradients for a seeded ``dl_dimage``.  The C1
case (BASELINE config 1: 10k Gaussians, 256x256 pinhole) stores the full
association and forward plus the gradients of a 2,000-Gaussian sample; its
scene is rebuilt from the seed by ``paper_2505_24053_b200.synth`` and checked
against the stored checksum.

The GPU box never runs this script: the fixtures travel as files.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from raygauss import association as ras  # noqa: E402
from raygauss import camera as rcam  # noqa: E402
from raygauss import renderer as rr  # noqa: E402
from raygauss import synth as rsynth  # noqa: E402
from raygauss.scene import GaussianScene  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def f32(scene):
    c = lambda a: np.asarray(a, np.float32).astype(np.float64)
    return GaussianScene(c(scene.means), c(scene.log_scales), c(scene.quats), c(scene.opacity_logits), c(scene.sh))


def scene_digest(scene) -> str:
    h = hashlib.sha256()
    for a in (scene.means, scene.log_scales, scene.quats, scene.opacity_logits, scene.sh):
        h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    return h.hexdigest()


def cam_fields(cam):
    nan = np.nan
    return dict(
        cam_width=cam.width, cam_height=cam.height, cam_model=cam.model, cam_rotation=cam.rotation,
        cam_translation=cam.translation, cam_fov=np.array([cam.fov_x if cam.fov_x is not None else nan,
                                                           cam.fov_y if cam.fov_y is not None else nan]),
        cam_intr=np.array([v if v is not None else nan for v in (cam.fx, cam.fy, cam.cx, cam.cy)]), cam_k=cam.k,
    )


def beap(w, h, fovx, fovy, pos, target=(0, 0, 0)):
    R, t = rsynth.look_at(pos, target)
    return rcam.Camera(width=w, height=h, model="beap", rotation=R, translation=t, fov_x=np.deg2rad(fovx),
                       fov_y=np.deg2rad(fovy))


def cases():
    rng = np.random.default_rng
    # 1. random scene, BEAP 120x90, SH degree 2, coloured background
    yield "beap_small", f32(rsynth.random_scene(200, rng(0), sh_bands=9)), beap(64, 48, 120, 90, (0, 0, -4)), \
        rr.RenderConfig(background=np.array([0.1, 0.2, 0.3])), 1
    # 2. pinhole, SH degree 3
    R, t = rsynth.look_at((0, 0, -4))
    yield "pinhole_small", f32(rsynth.random_scene(200, rng(1), sh_bands=16)), \
        rcam.Camera(width=64, height=48, model="pinhole", rotation=R, translation=t, fx=50, fy=50, cx=32, cy=24), \
        rr.RenderConfig(), 2
    # 3. KB equidistant 180 deg, camera inside a cloud (clamped + behind-camera Gaussians)
    R, t = rsynth.look_at((0.3, 0.2, 0.1), (2, 0.5, 1))
    f = 48 / (np.pi / 2)
    yield "kb_inside", f32(rsynth.random_scene(150, rng(2), spread=3.0, sh_bands=4)), \
        rcam.Camera(width=96, height=54, model="kb", rotation=R, translation=t, fx=f, fy=f, cx=47.5, cy=26.5), \
        rr.RenderConfig(background=np.array([0.5, 0.5, 0.5])), 3
    # 4. BEAP 300x160 (wide FoV mirror arcs), camera inside the cloud
    yield "beap_wide300", f32(rsynth.random_scene(150, rng(3), spread=3.0, sh_bands=9)), \
        beap(96, 52, 300, 160, (0.2, -0.1, 0.3), (1, 0, 2)), rr.RenderConfig(), 4
    # 5. one Gaussian straight behind the camera (full-line integral) + a few in front
    sc = rsynth.random_scene(6, rng(5), sh_bands=1)
    sc.means[0] = [0.0, 0.0, -9.0]
    sc.log_scales[0] = np.log([0.5, 0.5, 0.5])
    yield "behind_camera", f32(sc), beap(48, 32, 120, 80, (0, 0, -4)), rr.RenderConfig(), 5
    # 6. support_cutoff=False, SH degree 0, anisotropic Gaussians
    yield "nocutoff_aniso", f32(rsynth.random_scene(80, rng(6), sh_bands=1, anisotropy=20.0)), \
        beap(40, 40, 90, 90, (0, 0, -4)), rr.RenderConfig(support_cutoff=False, background=np.array([1.0, 0, 0])), 6
    # 7. tile_px=8, lam=2.5, ragged tiles (width not a multiple)
    yield "tile8_lam25", f32(rsynth.random_scene(120, rng(7), sh_bands=4)), beap(37, 29, 100, 80, (0.5, 0, -4)), \
        rr.RenderConfig(tile_px=8, lam=2.5), 7
    # 8. dense small scene, many early stops
    yield "dense_early_stop", f32(rsynth.random_scene(400, rng(8), spread=0.6, scale_range=(0.1, 0.3),
                                                      opacity_range=(0.8, 0.99), sh_bands=4)), \
        beap(48, 48, 90, 90, (0, 0, -3)), rr.RenderConfig(), 8
    # 9. empty scene
    # (the reference's GaussianScene.empty() cannot reshape a 0-sized SH array, scene.py:51, so build it raw)
    empty = object.__new__(GaussianScene)
    empty.means, empty.log_scales, empty.quats = np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 4))
    empty.opacity_logits, empty.sh = np.zeros(0), np.zeros((0, 4, 3))
    yield "empty", empty, beap(32, 16, 90, 45, (0, 0, -4)), \
        rr.RenderConfig(background=np.array([0.2, 0.4, 0.6])), 9
    # 10. degenerate scale -> ValueError("view covariance must be positive definite")
    sc = f32(rsynth.random_scene(30, rng(10), sh_bands=1))
    sc.log_scales[7] = np.log([0.2, 0.1, 1e-12])
    sc.quats[7] = [0.3, 0.5, -0.7, 0.4]
    yield "not_pd", f32(sc), beap(32, 32, 90, 90, (0, 0, -4)), rr.RenderConfig(), 10


def run_case(name, scene, cam, cfg, seed):
    out = dict(name=name, scene_means=scene.means, scene_log_scales=scene.log_scales, scene_quats=scene.quats,
               scene_opacity_logits=scene.opacity_logits, scene_sh=scene.sh, cfg_lam=cfg.lam, cfg_tile_px=cfg.tile_px,
               cfg_background=cfg.background, cfg_support_cutoff=int(cfg.support_cutoff), numpy_version=np.__version__,
               **cam_fields(cam))
    dl = np.random.default_rng(100 + seed).standard_normal((cam.height, cam.width, 3))
    out["dl_dimage"] = dl
    try:
        g = ras.build_render_graph(scene, cam, lam=cfg.lam, tile_px=cfg.tile_px)
    except ValueError as e:
        out["error"] = str(e)
        return out
    out.update(order=g.order.astype(np.int64), entry_tile=g.entry_tile.astype(np.int64), ranges=g.ranges.astype(np.int64),
               keep=g.keep, clamped=g.clamped, grid_pixel_tile=g.grid.pixel_tile, grid_ex=g.grid.mirror_edges_x,
               grid_ey=g.grid.mirror_edges_y)
    fr = rr.render(scene, cam, cfg)
    out.update(color=fr.color.color, remaining=fr.remaining_transmittance, count=fr.contributor_count)
    gr = rr.render_backward(scene, cam, dl, cfg)
    out.update(dmeans=gr.dmeans, dlog_scales=gr.dlog_scales, dquats=gr.dquats, dopacities=gr.dopacities, dsh=gr.dsh)
    return out


def make_c1():
    t0 = time.time()
    scene = f32(rsynth.random_scene(10_000, np.random.default_rng(0), sh_bands=16))
    R, t = rsynth.look_at((0.0, 0.0, -4.0))
    f = 128 / np.tan(np.deg2rad(30.0))
    cam = rcam.Camera(width=256, height=256, model="pinhole", rotation=R, translation=t, fx=f, fy=f, cx=128, cy=128)
    cfg = rr.RenderConfig(threads=8)
    g = ras.build_render_graph(scene, cam)
    fr = rr.render(scene, cam, cfg)
    dl = np.random.default_rng(1).standard_normal((256, 256, 3)) / (256 * 256)
    gr = rr.render_backward(scene, cam, dl, cfg)
    sample = np.sort(np.random.default_rng(7).choice(10_000, 2_000, replace=False))
    out = dict(name="C1", scene_sha256=scene_digest(scene), numpy_version=np.__version__,
               order=g.order.astype(np.int32), ranges=g.ranges.astype(np.int64), keep=g.keep, clamped=g.clamped,
               color=fr.color.color, remaining=fr.remaining_transmittance, count=fr.contributor_count.astype(np.int32),
               grad_sample=sample, dmeans=gr.dmeans[sample], dlog_scales=gr.dlog_scales[sample],
               dquats=gr.dquats[sample], dopacities=gr.dopacities[sample], dsh=gr.dsh[sample], **cam_fields(cam))
    np.savez_compressed(os.path.join(HERE, "C1.npz"), **out)
    print(f"C1: {len(g.order)} entries, {time.time() - t0:.1f}s")


def main():
    for name, scene, cam, cfg, seed in cases():
        out = run_case(name, scene, cam, cfg, seed)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(name, "error" if "error" in out else len(out["order"]))
    if "--skip-c1" not in sys.argv:
        make_c1()


if __name__ == "__main__":
    main()
