"""Golden run of the reference's own training loop on SPEC acceptance criterion 8.

Run in the build container (where /root/reference exists; ~5 min of CPU):

    python tests/golden/make_golden_train.py

Setup: a synthetic 50-Gaussian scene, 8 BEAP views at 64x64 on a ring, the targets rendered by the
reference, a perturbed initialisation, ``trainer.train`` with the default TrainConfig (2,000
iterations, seed 42).  Stored: the scene, the init, the target images, the per-iteration losses of the
first 20 iterations (a separate 20-iteration run with eval_interval=1) and the metric rows of the full
run (PSNR > 30 dB is the criterion).  tests/test_gpu_dropin_train.py replays it with the B200
renderer installed into the same, unmodified ``raygauss.trainer``.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from raygauss import renderer as rr  # noqa: E402
from raygauss import synth as rsynth  # noqa: E402
from raygauss import trainer as rt  # noqa: E402

from make_golden import HERE, f32  # noqa: E402

N_GAUSSIANS, N_VIEWS, SIZE, FOV = 50, 8, 64, 100.0


def setup():
    target = f32(rsynth.random_scene(N_GAUSSIANS, np.random.default_rng(0), sh_bands=4))
    cams = rsynth.ring_cameras(N_VIEWS, 3.0, SIZE, SIZE, fov_deg=FOV)
    views = rsynth.render_targets(target, cams, rr.render, rr.RenderConfig())
    init = f32(rsynth.perturbed(target, np.random.default_rng(1)))
    return target, init, views


def main():
    target, init, views = setup()
    t0 = time.time()
    _, head, _ = rt.train(init, views, rt.TrainConfig(iterations=20, eval_interval=1))
    t1 = time.time()
    _, rows, _ = rt.train(init, views, rt.TrainConfig())
    t2 = time.time()
    np.savez_compressed(
        os.path.join(HERE, "train_spec8.npz"),
        init_means=init.means, init_log_scales=init.log_scales, init_quats=init.quats,
        init_opacity_logits=init.opacity_logits, init_sh=init.sh,
        targets=np.stack([v[1].color for v in views]),
        head_loss=np.array([r["loss"] for r in head]), head_psnr=np.array([r["psnr"] for r in head]),
        rows_iter=np.array([r["iter"] for r in rows]), rows_loss=np.array([r["loss"] for r in rows]),
        rows_psnr=np.array([r["psnr"] for r in rows]), rows_ssim=np.array([r["ssim"] for r in rows]),
        cpu_seconds=np.array([t1 - t0, t2 - t1]), numpy_version=np.__version__)
    print(f"first losses {[round(r['loss'], 6) for r in head[:5]]}; final PSNR {rows[-1]['psnr']:.2f} dB; "
          f"{t2 - t1:.0f}s for {rows[-1]['iter']} iterations")


if __name__ == "__main__":
    main()
