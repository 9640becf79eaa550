"""Golden vectors of camera.resample_to_beap, produced by the UNMODIFIED reference.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_resample.py

Pinhole and equidistant/distorted KB sources resampled onto BEAP targets (camera.py:302-339).
Source images are stored as float32 (what the GPU reads).  The GPU box never runs this script.
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from raygauss import camera as rc  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def cam_dict(c, prefix):
    nan = float("nan")
    opt = lambda v: nan if v is None else float(v)
    return {f"{prefix}_wh": np.array([c.width, c.height]), f"{prefix}_model": np.array(c.model),
            f"{prefix}_R": c.rotation, f"{prefix}_t": c.translation,
            f"{prefix}_fov": np.array([opt(c.fov_x), opt(c.fov_y)]),
            f"{prefix}_intr": np.array([opt(c.fx), opt(c.fy), opt(c.cx), opt(c.cy)]), f"{prefix}_k": c.k}


def main():
    rng = np.random.default_rng(11)
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w_, x_, y_, z_ = q
    R = np.array([[1 - 2 * (y_ * y_ + z_ * z_), 2 * (x_ * y_ - w_ * z_), 2 * (x_ * z_ + w_ * y_)],
                  [2 * (x_ * y_ + w_ * z_), 1 - 2 * (x_ * x_ + z_ * z_), 2 * (y_ * z_ - w_ * x_)],
                  [2 * (x_ * z_ - w_ * y_), 2 * (y_ * z_ + w_ * x_), 1 - 2 * (x_ * x_ + y_ * y_)]])
    t = rng.normal(size=3)
    cases = {}
    src_pin = rc.Camera(width=96, height=72, model="pinhole", rotation=R, translation=t, fx=60.0, fy=58.0, cx=47.3,
                        cy=36.1)
    src_kb = rc.Camera(width=128, height=96, model="kb", rotation=R, translation=t, fx=40.0, fy=40.5, cx=63.5,
                       cy=47.5, k=np.array([0.05, -0.01, 0.002, -0.0005]))
    src_eq = rc.Camera(width=128, height=72, model="kb", rotation=R, translation=t, fx=64.0 / (np.pi / 2), fy=64.0 / (np.pi / 2),
                       cx=63.5, cy=35.5, k=np.zeros(4))
    for name, src, fov in (("pinhole", src_pin, (100.0, 80.0)), ("kb", src_kb, (200.0, 160.0)),
                           ("equidistant", src_eq, (180.0, 101.25))):
        tgt = rc.Camera(width=80, height=60, model="beap", rotation=R, translation=t, fov_x=np.deg2rad(fov[0]),
                        fov_y=np.deg2rad(fov[1]))
        img = rng.uniform(0, 1, (src.height, src.width, 3)).astype(np.float32)
        out = rc.resample_to_beap(img.astype(np.float64), src, tgt)
        d = {"image": img, "color": out.color, "mask": out.mask}
        d.update(cam_dict(src, "src"))
        d.update(cam_dict(tgt, "tgt"))
        cases[name] = d
    out = {f"{k}__{f}": v for k, d in cases.items() for f, v in d.items()}
    np.savez_compressed(os.path.join(HERE, "resample_cases.npz"), **out)
    print({k: int(d["mask"].sum()) for k, d in cases.items()})


if __name__ == "__main__":
    main()
