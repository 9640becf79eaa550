"""GPU ground-truth resampling (geer_resample_to_beap) against reference golden vectors.

tests/golden/resample_cases.npz: camera.resample_to_beap of the unmodified reference (pinhole,
distorted KB and equidistant fisheye sources onto BEAP targets).  The mask is compared exactly, the
bilinear colour to fp32 rounding of the source image.
"""

import os

import numpy as np
import pytest

from paper_2505_24053_b200 import camera
from paper_2505_24053_b200.scene import Camera

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "resample_cases.npz")


def load():
    with np.load(GOLD) as z:
        names = sorted({k.split("__")[0] for k in z.files})
        return {n: {k.split("__")[1]: z[k] for k in z.files if k.startswith(n + "__")} for n in names}


def cam(d, p):
    opt = lambda v: None if np.isnan(v) else float(v)
    w, h = (int(v) for v in d[f"{p}_wh"])
    fov, intr = d[f"{p}_fov"], d[f"{p}_intr"]
    return Camera(width=w, height=h, model=str(d[f"{p}_model"]), rotation=d[f"{p}_R"], translation=d[f"{p}_t"],
                  fov_x=opt(fov[0]), fov_y=opt(fov[1]), fx=opt(intr[0]), fy=opt(intr[1]), cx=opt(intr[2]),
                  cy=opt(intr[3]), k=d[f"{p}_k"])


@pytest.mark.parametrize("name", sorted(load()))
def test_resample_matches_reference(name):
    d = load()[name]
    out = camera.resample_to_beap(d["image"], cam(d, "src"), cam(d, "tgt"))
    np.testing.assert_array_equal(out.mask, d["mask"])
    np.testing.assert_allclose(out.color, d["color"], rtol=0, atol=2e-6)


def test_resample_validation_errors():
    d = load()["pinhole"]
    src, tgt = cam(d, "src"), cam(d, "tgt")
    with pytest.raises(ValueError, match="target camera must use the beap model"):
        camera.resample_to_beap(d["image"], src, src)
    moved = Camera(width=tgt.width, height=tgt.height, model="beap", rotation=tgt.rotation,
                   translation=tgt.translation + 1.0, fov_x=tgt.fov_x, fov_y=tgt.fov_y)
    with pytest.raises(ValueError, match="share extrinsics"):
        camera.resample_to_beap(d["image"], src, moved)
