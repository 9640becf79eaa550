"""Benchmark and test workloads: synthetic scenes and camera rigs (restated from synth.py:12-100).

Fixture generators, not part of the product package: bench.py, smoke() and the tests use them.

The BASELINE configurations are defined on these generators, so
bench.py and the tests rebuild bit-identical inputs from a seed without the
reference installed.  ``random_scene`` consumes the numpy Generator in the
same call order as the reference, so ``random_scene(n, default_rng(0), ...)``
equals the reference's output exactly (pinned by tests/test_oracle_golden.py::test_synth_scene_regenerates_c1_fixture).
"""

from __future__ import annotations

import numpy as np

from paper_2505_24053_b200.scene import Camera, GaussianScene


def logit(p):
    """core.py:70-72."""
    p = np.asarray(p, dtype=np.float64)
    return np.log(p) - np.log1p(-p)


def random_scene(n, rng, center=(0.0, 0.0, 0.0), spread=1.2, scale_range=(0.06, 0.25),
                 opacity_range=(0.3, 0.95), sh_bands=1, anisotropy=1.0) -> GaussianScene:
    """synth.py:12-43."""
    means = np.asarray(center)[None, :] + rng.uniform(-spread, spread, (n, 3))
    log_s = rng.uniform(np.log(scale_range[0]), np.log(scale_range[1]), (n, 3))
    if anisotropy > 1.0:
        log_s[:, 0] += rng.uniform(0.0, np.log(anisotropy), n)
    quats = rng.normal(size=(n, 4))
    quats /= np.linalg.norm(quats, axis=1, keepdims=True)
    sh = np.zeros((n, sh_bands, 3))
    sh[:, 0, :] = rng.uniform(-0.8, 1.8, (n, 3))
    if sh_bands > 1:
        sh[:, 1:, :] = rng.uniform(-0.25, 0.25, (n, sh_bands - 1, 3))
    return GaussianScene(means=means, log_scales=log_s, quats=quats,
                         opacity_logits=logit(rng.uniform(*opacity_range, n)), sh=sh)


def look_at(position, target=(0.0, 0.0, 0.0), up=(0.0, 1.0, 0.0)):
    """synth.py:46-57: extrinsics (R_c, t_c) of a camera at ``position``."""
    position = np.asarray(position, dtype=np.float64)
    forward = np.asarray(target, dtype=np.float64) - position
    forward /= np.linalg.norm(forward)
    right = np.cross(forward, np.asarray(up, dtype=np.float64))
    if np.linalg.norm(right) < 1e-9:
        right = np.cross(forward, np.array([1.0, 0.0, 0.0]))
    right /= np.linalg.norm(right)
    down = np.cross(forward, right)
    rot = np.stack([right, down, forward])
    return rot, -rot @ position


def ring_positions(n_views, radius, elevation=0.35):
    """Camera centres of synth.py:72-76."""
    out = []
    for i in range(n_views):
        ang = 2.0 * np.pi * i / n_views
        out.append(np.array([radius * np.cos(ang), elevation * radius * np.sin(2 * ang), radius * np.sin(ang)]))
    return out


def ring_cameras(n_views, radius, width, height, fov_deg=100.0, target=(0.0, 0.0, 0.0), elevation=0.35,
                 fov_y_deg=None):
    """synth.py:60-88 (``fov_y_deg`` extends it for non-square angular images)."""
    cams = []
    for pos in ring_positions(n_views, radius, elevation):
        rot, t = look_at(pos, target)
        cams.append(Camera(width=width, height=height, model="beap", rotation=rot, translation=t,
                           fov_x=np.deg2rad(fov_deg), fov_y=np.deg2rad(fov_y_deg if fov_y_deg else fov_deg)))
    return cams


def perturbed(scene: GaussianScene, rng, strength: float = 1.0) -> GaussianScene:
    """synth.py:91-100."""
    out = scene.copy()
    extent = scene.extent()
    out.means = out.means + rng.normal(0.0, 0.02 * extent * strength, out.means.shape)
    out.log_scales = out.log_scales + rng.normal(0.0, 0.15 * strength, out.log_scales.shape)
    out.quats = out.quats + rng.normal(0.0, 0.05 * strength, out.quats.shape)
    out.opacity_logits = out.opacity_logits + rng.normal(0.0, 0.3 * strength, out.opacity_logits.shape)
    out.sh = out.sh + rng.normal(0.0, 0.08 * strength, out.sh.shape)
    return out


def to_f32_values(scene: GaussianScene) -> GaussianScene:
    """Round every parameter to fp32 (kept as f64) so CPU and GPU see identical inputs."""
    c = lambda a: np.asarray(a, dtype=np.float32).astype(np.float64)
    return GaussianScene(c(scene.means), c(scene.log_scales), c(scene.quats), c(scene.opacity_logits), c(scene.sh))


# --------------------------------------------------------------------------- BASELINE configs

def config_scene(name: str, n: int | None = None) -> GaussianScene:
    """Scenes of BASELINE configs C1..C5 (seed 0, sh_bands=16, fp32-rounded)."""
    if name == "C1":
        n = n or 10_000
        return to_f32_values(random_scene(n, np.random.default_rng(0), sh_bands=16))
    if name in ("C2", "C3", "C4"):
        n = n or 1_000_000
        k = (1e4 / n) ** 0.5
        return to_f32_values(random_scene(n, np.random.default_rng(0), sh_bands=16,
                                          scale_range=(0.06 * k, 0.25 * k)))
    if name == "C5":
        n = n or 6_000_000
        k = (1e4 / n) ** 0.5
        return to_f32_values(random_scene(n, np.random.default_rng(0), sh_bands=16,
                                          scale_range=(0.06 * k, 0.25 * k)))
    raise KeyError(name)


def config_camera(name: str, width: int | None = None, height: int | None = None) -> Camera:
    if name == "C1":
        rot, t = look_at((0.0, 0.0, -4.0))
        w = width or 256
        h = height or 256
        f = (w / 2) / np.tan(np.deg2rad(30.0))
        return Camera(width=w, height=h, model="pinhole", rotation=rot, translation=t, fx=f, fy=f, cx=w / 2, cy=h / 2)
    if name in ("C2", "C3", "C4"):
        rot, t = look_at((0.0, 0.0, -2.0))
        w = width or 1920
        h = height or 1080
        return Camera(width=w, height=h, model="beap", rotation=rot, translation=t,
                      fov_x=np.deg2rad(180.0), fov_y=np.deg2rad(180.0 * h / w))
    if name == "C5":
        rot, t = look_at((0.0, 0.0, -2.0))
        w = width or 3840
        h = height or 2160
        f = (w / 2) / (np.pi / 2)
        return Camera(width=w, height=h, model="kb", rotation=rot, translation=t, fx=f, fy=f,
                      cx=(w - 1) / 2, cy=(h - 1) / 2, k=np.zeros(4))
    raise KeyError(name)


def c4_trainer(target_scene, n_views=64, rank=0, world=1, device=0, width=1920, height=1080, inflight=2):
    """BASELINE config 4 step: target = C2 scene, init = perturbed(C2, default_rng(1)), a ring of BEAP
    180 x 101.25 deg views sharded over ranks; the targets are rendered by the GPU renderer."""
    from paper_2505_24053_b200.device import DeviceRenderer, DeviceScene
    from paper_2505_24053_b200.renderer import RenderConfig
    from paper_2505_24053_b200.train import MultiViewTrainer, shard

    cams_all = ring_cameras(n_views, 2.0, width, height, fov_deg=180.0, fov_y_deg=180.0 * height / width)
    mine = [cams_all[i] for i in shard(n_views, rank, world)]
    init = to_f32_values(perturbed(target_scene, np.random.default_rng(1)))
    r = DeviceRenderer(device)
    tscene = DeviceScene.from_scene(target_scene, device=f"cuda:{device}")
    cfg = RenderConfig()
    targets = []
    for cam in mine:
        color, _, _ = r.forward(tscene, cam, cfg)
        targets.append(color.clone())
    del r, tscene
    return MultiViewTrainer(init, mine, targets, rank, world, device, cfg, inflight=inflight)
