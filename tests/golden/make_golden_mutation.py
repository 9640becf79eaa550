"""Single-ray gradient golden vectors with and without the reference's mutation hook.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_mutation.py

SURVEY §4 tier 1: the backward tests must be shown to catch a wrong cross-product operand order.
The reference's hook ``gradients._debug_negate_dir_cross_term`` (gradients.py:20-22,114-115) flips
the o_u-cross term of dL/dd_u in ``backward_ray``.  For each case (one Gaussian seen by a 1x1 BEAP
camera whose single ray passes through the Gaussian's support) this script stores:

* the reference ``render_backward`` gradients of that one-pixel scene (the GPU's target);
* ``backward_ray`` with the hook off — checked here to equal ``render_backward`` (same chain:
  dL/dT = <c, dL/dC> with a black background, the quaternion gradient projected with the normalisation Jacobian);
* ``backward_ray`` with the hook ON — the mutant the GPU result must be far from.

The GPU box never runs this script: the vectors travel as a file.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from raygauss import camera as rcam  # noqa: E402
from raygauss import gradients as rgrad  # noqa: E402
from raygauss import renderer as rr  # noqa: E402
from raygauss import synth as rsynth  # noqa: E402
from raygauss.core import Gaussian3D, Ray  # noqa: E402
from raygauss.scene import GaussianScene  # noqa: E402

from make_golden import HERE  # noqa: E402

N_CASES = 24


def one_case(rng):
    mean = rng.uniform(-0.3, 0.3, 3)
    log_s = np.log(rng.uniform(0.1, 0.4, 3))
    q = rng.normal(size=4)
    logit = float(rng.uniform(-1.0, 1.5))
    sh = np.zeros((1, 3))
    sh[0] = rng.uniform(-0.5, 1.5, 3)
    # camera 3-4 units away looking at a point near the Gaussian so the one ray crosses its support
    pos = rng.normal(size=3)
    pos = pos / np.linalg.norm(pos) * rng.uniform(3.0, 4.0)
    target = mean + rng.uniform(-0.15, 0.15, 3)
    R, t = rsynth.look_at(pos, target)
    cam = rcam.Camera(width=1, height=1, model="beap", rotation=R, translation=t, fov_x=np.deg2rad(0.5),
                      fov_y=np.deg2rad(0.5))
    f = lambda a: np.asarray(a, np.float32).astype(np.float64)
    scene = GaussianScene(f(mean[None]), f(log_s[None]), f(q[None]), f(np.array([logit])), f(sh[None]))
    return scene, cam


def main():
    rng = np.random.default_rng(77)
    rows = []
    while len(rows) < N_CASES:
        scene, cam = one_case(rng)
        cfg = rr.RenderConfig()
        fr = rr.render(scene, cam, cfg)
        t_eff = 1.0 - fr.remaining_transmittance[0, 0]
        if not (0.02 < t_eff < 0.9):  # the ray must cross the support, below the 0.999 clamp
            continue
        dl = rng.normal(size=(1, 1, 3))
        ref = rr.render_backward(scene, cam, dl, cfg)
        g = Gaussian3D(scene.means[0], scene.log_scales[0], scene.quats[0], float(scene.opacity_logits[0]),
                       scene.sh[0])
        d = rcam.pixel_ray_grid(cam).reshape(3) @ cam.rotation
        ray = Ray(cam.optical_center, d)
        color = fr.color.color[0, 0] / t_eff  # one contributor, black background: C = t c
        dl_dt = float(color @ dl[0, 0])
        out = {}
        for hook in (False, True):
            rgrad._debug_negate_dir_cross_term = hook
            gg = rgrad.backward_ray(g, ray, dl_dt)
            out[hook] = (gg.dmean, gg.dlog_scale, rgrad.project_quat_grad(g.quat, gg.dquat), gg.dopacity)
        rgrad._debug_negate_dir_cross_term = False
        for a, b in zip(out[False], (ref.dmeans[0], ref.dlog_scales[0], ref.dquats[0], ref.dopacities[0])):
            assert np.allclose(a, b, rtol=1e-9, atol=1e-12), (a, b)  # the hook-off chain is render_backward's
        rows.append(dict(scene=scene, cam=cam, dl=dl, ref=ref, mut=out[True]))
    cat = lambda f: np.stack([f(r) for r in rows])
    np.savez_compressed(
        os.path.join(HERE, "mutation_cases.npz"),
        scene_means=cat(lambda r: r["scene"].means), scene_log_scales=cat(lambda r: r["scene"].log_scales),
        scene_quats=cat(lambda r: r["scene"].quats), scene_opacity_logits=cat(lambda r: r["scene"].opacity_logits),
        scene_sh=cat(lambda r: r["scene"].sh), dl_dimage=cat(lambda r: r["dl"]),
        cam_rotation=cat(lambda r: r["cam"].rotation), cam_translation=cat(lambda r: r["cam"].translation),
        cam_fov=np.array([np.deg2rad(0.5), np.deg2rad(0.5)]),
        dmeans=cat(lambda r: r["ref"].dmeans[0]), dlog_scales=cat(lambda r: r["ref"].dlog_scales[0]),
        dquats=cat(lambda r: r["ref"].dquats[0]), dopacities=cat(lambda r: r["ref"].dopacities[0]),
        mut_dmeans=cat(lambda r: r["mut"][0]), mut_dlog_scales=cat(lambda r: r["mut"][1]),
        mut_dquats=cat(lambda r: r["mut"][2]), mut_dopacities=cat(lambda r: np.array(r["mut"][3])),
        numpy_version=np.__version__)
    mut = np.abs(cat(lambda r: r["mut"][1]) - cat(lambda r: r["ref"].dlog_scales[0])).max()
    print(f"{len(rows)} cases; max |dlog_scales(mutant) - dlog_scales(ref)| = {mut:.3g}")


if __name__ == "__main__":
    main()
