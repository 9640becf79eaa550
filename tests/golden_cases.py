"""Load the golden fixtures (tests/golden/*.npz, made by make_golden.py from the reference)."""

from __future__ import annotations

import glob
import os
from types import SimpleNamespace

import numpy as np

from paper_2505_24053_b200.scene import Camera, GaussianScene

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

SMALL_CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                     if os.path.basename(p) not in ("C1.npz", "loss_cases.npz", "resample_cases.npz", "assoc_brute.npz",
                                                                 "pd_boundary.npz", "mutation_cases.npz",
                                                                 "train_spec8.npz"))


def load(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def camera_of(d: dict) -> Camera:
    fov = d["cam_fov"]
    intr = d["cam_intr"]
    opt = lambda v: None if np.isnan(v) else float(v)
    return Camera(width=int(d["cam_width"]), height=int(d["cam_height"]), model=str(d["cam_model"]),
                  rotation=d["cam_rotation"], translation=d["cam_translation"], fov_x=opt(fov[0]), fov_y=opt(fov[1]),
                  fx=opt(intr[0]), fy=opt(intr[1]), cx=opt(intr[2]), cy=opt(intr[3]), k=d["cam_k"])


def scene_of(d: dict) -> GaussianScene:
    return GaussianScene(d["scene_means"], d["scene_log_scales"], d["scene_quats"], d["scene_opacity_logits"],
                         d["scene_sh"])


def config_of(d: dict):
    from paper_2505_24053_b200.renderer import RenderConfig

    return RenderConfig(lam=float(d["cfg_lam"]), tile_px=int(d["cfg_tile_px"]), background=d["cfg_background"],
                        support_cutoff=bool(int(d["cfg_support_cutoff"])))


def case(name: str):
    d = load(name)
    return SimpleNamespace(data=d, scene=scene_of(d), camera=camera_of(d), config=config_of(d))


PD_TIE_ULPS = 64


def pd_boundary():
    """The PD-boundary sweep (make_golden_extreme.py): list of (s_min, seed, raised, tie, scene, order,
    ranges) and the shared camera.  ``tie``: the reference's own last Cholesky pivot lies within
    PD_TIE_ULPS * eps * max|cov_c| of zero, i.e. its raise/no-raise decision is decided by rounding
    noise (numpy's SIMD exp alone differs from a correctly rounded exp in ~5 % of inputs)."""
    d = load("pd_boundary")
    cam = camera_of(d)
    out = []
    for i in range(len(d["s_min"])):
        scene = GaussianScene(d["scene_means"][i], d["scene_log_scales"][i], d["scene_quats"][i],
                              d["scene_opacity_logits"][i], d["scene_sh"][i])
        o0, o1 = d["order_off"][i], d["order_off"][i + 1]
        r0, r1 = d["ranges_off"][i], d["ranges_off"][i + 1]
        tie = abs(float(d["pivot_ref"][i])) <= PD_TIE_ULPS * 2.0 ** -52 * float(d["cov_scale"][i])
        out.append((float(d["s_min"][i]), int(d["seed"][i]), int(d["raised"][i]), tie, scene, d["order"][o0:o1],
                    d["ranges"][r0:r1]))
    return out, cam


def mutation_cases():
    """Single-ray cases of make_golden_mutation.py: (scene, camera, dl_dimage, ref grads, mutant grads)."""
    d = load("mutation_cases")
    out = []
    for i in range(len(d["dmeans"])):
        scene = GaussianScene(d["scene_means"][i], d["scene_log_scales"][i], d["scene_quats"][i],
                              d["scene_opacity_logits"][i], d["scene_sh"][i])
        cam = Camera(width=1, height=1, model="beap", rotation=d["cam_rotation"][i],
                     translation=d["cam_translation"][i], fov_x=float(d["cam_fov"][0]), fov_y=float(d["cam_fov"][1]))
        ref = {k: d[k][i][None] for k in ("dmeans", "dlog_scales", "dquats", "dopacities")}
        mut = {k: d["mut_" + k][i][None] for k in ("dmeans", "dlog_scales", "dquats", "dopacities")}
        out.append((scene, cam, d["dl_dimage"][i], ref, mut))
    return out
