"""GPU training loss (geer_loss) against the reference trainer.loss golden vectors.

tests/golden/loss_cases.npz was produced by the unmodified reference (make_golden_loss.py):
masked (1 - w) L1 + w (1 - SSIM) and its analytic image gradient (trainer.py:114-155).
The GPU computes in fp32 with fp64 sums; the L1 sign term is exact for these inputs (the same fp32
images on both sides), the SSIM terms carry fp32 blur rounding.
"""

import os

import numpy as np
import pytest
import torch

from paper_2505_24053_b200 import train
from paper_2505_24053_b200.scene import BEAPImage

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "loss_cases.npz")


def cases():
    with np.load(GOLD) as z:
        names = sorted({k.split("__")[0] for k in z.files})
        return {n: {k.split("__")[1]: z[k] for k in z.files if k.startswith(n + "__")} for n in names}


@pytest.mark.parametrize("name", sorted(cases()))
def test_loss_matches_reference(name):
    d = cases()[name]
    total, grad = train.loss(d["rendered"], BEAPImage(color=d["target"].astype(np.float64), mask=d["mask"]),
                             float(d["weight"]))
    assert abs(total - float(d["total"])) <= 1e-6 * max(1.0, abs(float(d["total"])))
    ref = d["grad"]
    scale = np.abs(ref).max()
    err = np.abs(grad - ref)
    assert (err <= 1e-3 * np.abs(ref) + 1e-4 * scale).all(), float(err.max() / scale)


def test_loss_device_full_hd_runs_and_is_finite():
    h, w = 1080, 1920
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.rand((h, w, 3), device="cuda", generator=g)
    b = (a + 0.05 * torch.randn((h, w, 3), device="cuda", generator=g)).clamp(0, 1)
    out, grad = train.loss_device(a, b)
    torch.cuda.synchronize()
    assert torch.isfinite(grad).all() and 0.0 < float(out[0]) < 1.0
    same, _ = train.loss_device(a, a.clone())
    assert abs(float(same[0])) < 1e-6  # identical images: L1 = 0, SSIM = 1
