"""Load the golden fixtures (tests/golden/*.npz, made by make_golden.py from the reference)."""

from __future__ import annotations

import glob
import os
from types import SimpleNamespace

import numpy as np

from paper_2505_24053_b200.scene import Camera, GaussianScene

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

SMALL_CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                     if os.path.basename(p) not in ("C1.npz", "loss_cases.npz", "resample_cases.npz", "assoc_brute.npz"))


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
