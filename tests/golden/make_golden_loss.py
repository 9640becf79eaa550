"""Golden vectors of the training loss, produced by the UNMODIFIED reference trainer.loss.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_loss.py

trainer.loss (trainer.py:114-155) = masked (1 - w) L1 + w (1 - SSIM) with its analytic image
gradient.  Inputs are stored as float32 (what the GPU renders); the reference consumes them as
float64.  The GPU box never runs this script.
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from raygauss import trainer as rt  # noqa: E402
from raygauss.camera import BEAPImage  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def case(rng, h, w, mask_frac, weight, smooth=True):
    base = rng.uniform(0, 1, (h, w, 3))
    if smooth:  # image-like content so SSIM is not degenerate
        from scipy.ndimage import gaussian_filter

        base = gaussian_filter(base, sigma=(2, 2, 0))
    rendered = np.clip(base + rng.normal(0, 0.05, base.shape), 0, 1).astype(np.float32)
    target = np.clip(base + rng.normal(0, 0.05, base.shape), 0, 1).astype(np.float32)
    mask = rng.uniform(0, 1, (h, w)) >= mask_frac
    total, grad = rt.loss(rendered.astype(np.float64), BEAPImage(target.astype(np.float64), mask), weight)
    return dict(rendered=rendered, target=target, mask=mask, weight=np.float64(weight), total=np.float64(total),
                grad=grad)


def main():
    rng = np.random.default_rng(7)
    cases = {
        "full_120x160": case(rng, 120, 160, 0.0, 0.2),
        "masked_96x128": case(rng, 96, 128, 0.3, 0.2),
        "w05_64x80": case(rng, 64, 80, 0.1, 0.5),
        "w0_40x48": case(rng, 40, 48, 0.0, 0.0),
        "tiny_8x9": case(rng, 8, 9, 0.0, 0.2),  # no SSIM region (trainer.py:72-76)
    }
    out = {f"{k}__{f}": v for k, d in cases.items() for f, v in d.items()}
    np.savez_compressed(os.path.join(HERE, "loss_cases.npz"), **out)
    print({k: float(d["total"]) for k, d in cases.items()})


if __name__ == "__main__":
    main()
