"""Golden fixtures for the degenerate regime, made by running the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_extreme.py

Two kinds of fixture (VERDICT r1 "next" #1):

* ``pd_boundary.npz`` — the PD check of ``solve_pbf`` (association.py:154-160) swept across its
  boundary: 8-Gaussian scenes whose Gaussian 0 has scales (0.2, 0.1, s_min) and a random
  orientation, s_min in {1e-8, 3e-9, 1e-9, 3e-10} x 50 seeds.  Per scene: whether
  ``build_render_graph`` raised ``ValueError("view covariance must be positive definite")`` and,
  when it did not, the association (order, ranges).
* ``aniso_1e2/1e3/1e4.npz`` and ``smin_1e8.npz`` — flat Gaussians (anisotropy up to 1e4, and thin
  axes of 1e-8) rendered and back-propagated by the reference; the same case layout as
  make_golden.py, so the oracle and GPU parity tests pick them up with the other small cases.

The GPU box never runs this script: the fixtures travel as files.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from raygauss import association as ras  # noqa: E402
from raygauss import renderer as rr  # noqa: E402
from raygauss import synth as rsynth  # noqa: E402

from make_golden import HERE, beap, cam_fields, f32, run_case  # noqa: E402

PD_SMIN = (1e-8, 3e-9, 1e-9, 3e-10)
PD_SEEDS = 50


def random_quat(rng):
    q = rng.normal(size=4)
    return q / np.linalg.norm(q)


def pd_scene(s_min, seed):
    rng = np.random.default_rng(1000 + seed)
    sc = rsynth.random_scene(8, rng, sh_bands=1)
    sc.log_scales[0] = np.log([0.2, 0.1, s_min])
    sc.quats[0] = random_quat(rng)
    sc.means[0] = rng.uniform(-0.5, 0.5, 3)
    return f32(sc)


def last_pivot(cov):
    """The last Cholesky pivot a22 - l20^2 - l21^2 of LAPACK potf2 (lower; column scaled by the
    reciprocal pivot, the dot product as one fma) on the reference's own view covariance: the quantity
    whose sign np.linalg.cholesky decides on (reproduces its decision on all 200 scenes here)."""
    from fractions import Fraction

    def fma(a, b, c):
        return float(Fraction(a) * Fraction(b) + Fraction(c))

    l00 = np.sqrt(cov[0, 0])
    r0 = 1.0 / l00
    l10, l20 = cov[1, 0] * r0, cov[2, 0] * r0
    a11 = cov[1, 1] - l10 * l10
    l21 = (cov[2, 1] - l20 * l10) * (1.0 / np.sqrt(a11)) if a11 > 0 else 0.0
    return float(cov[2, 2] - fma(l21, l21, l20 * l20)) if a11 > 0 else float(a11)


def pd_camera():
    return beap(32, 32, 90, 90, (0, 0, -4))


def make_pd_boundary():
    cam = pd_camera()
    smins, seeds, raised, orders, ranges, scenes, pivots, scales = [], [], [], [], [], [], [], []
    for s_min in PD_SMIN:
        for seed in range(PD_SEEDS):
            scene = pd_scene(s_min, seed)
            scenes.append(scene)
            _, cov_c, _ = ras.view_scene(scene, cam)
            pivots.append(last_pivot(cov_c[0]))
            scales.append(float(np.abs(cov_c[0]).max()))
            smins.append(s_min)
            seeds.append(seed)
            try:
                g = ras.build_render_graph(scene, cam)
            except ValueError as e:
                assert "positive definite" in str(e) or "symmetric" in str(e), e
                raised.append(1 if "positive definite" in str(e) else 2)
                orders.append(np.zeros(0, np.int64))
                ranges.append(np.zeros(0, np.int64))
                continue
            raised.append(0)
            orders.append(g.order.astype(np.int64))
            ranges.append(g.ranges.astype(np.int64))
    off = np.concatenate([[0], np.cumsum([len(o) for o in orders])])
    roff = np.concatenate([[0], np.cumsum([len(r) for r in ranges])])
    np.savez_compressed(os.path.join(HERE, "pd_boundary.npz"), s_min=np.array(smins), seed=np.array(seeds),
                        raised=np.array(raised, np.int8), pivot_ref=np.array(pivots),
                        cov_scale=np.array(scales), order=np.concatenate(orders), order_off=off,
                        ranges=np.concatenate(ranges), ranges_off=roff, numpy_version=np.__version__,
                        scene_means=np.stack([s.means for s in scenes]),
                        scene_log_scales=np.stack([s.log_scales for s in scenes]),
                        scene_quats=np.stack([s.quats for s in scenes]),
                        scene_opacity_logits=np.stack([s.opacity_logits for s in scenes]),
                        scene_sh=np.stack([s.sh for s in scenes]), **cam_fields(cam))
    r = np.array(raised)
    for s in PD_SMIN:
        sel = np.array(smins) == s
        print(f"pd_boundary s_min={s:g}: {int((r[sel] == 1).sum())}/{int(sel.sum())} raised")


def flat_scene(n, seed, anisotropy=None, s_min=None, n_flat=None):
    """random_scene (C1 distribution) whose first n_flat Gaussians are flattened discs: the thin axis is
    s_big / anisotropy (log-uniform over the upper half of the range), or exactly s_min."""
    rng = np.random.default_rng(seed)
    sc = rsynth.random_scene(n, rng, sh_bands=4, scale_range=(0.05, 0.2))
    k = n if n_flat is None else n_flat
    if anisotropy is not None:
        sc.log_scales[:k, 2] = sc.log_scales[:k, 0] - np.log(anisotropy) * rng.uniform(0.5, 1.0, k)
    if s_min is not None:
        sc.log_scales[:k, 2] = np.log(s_min)
    return f32(sc)


def extreme_cases():
    cfg = rr.RenderConfig(background=np.array([0.1, 0.1, 0.2]))
    for i, a in enumerate((1e2, 1e3, 1e4)):
        yield f"aniso_{a:.0e}".replace("+0", ""), flat_scene(120, 20 + i, anisotropy=a), \
            beap(64, 48, 120, 90, (0.3, -0.2, -3.5)), cfg, 20 + i
    # s_min = 1e-8 (SPEC #3): half the Gaussians are discs 1e-8 thick, the rest the usual spread
    yield "smin_1e8", flat_scene(120, 30, s_min=1e-8, n_flat=60), beap(64, 48, 120, 90, (0.2, 0.3, -3.5)), cfg, 30


def main():
    t0 = time.time()
    make_pd_boundary()
    print(f"pd_boundary: {time.time() - t0:.1f}s")
    for name, scene, cam, cfg, seed in extreme_cases():
        t0 = time.time()
        out = run_case(name, scene, cam, cfg, seed)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(name, "error " + str(out["error"]) if "error" in out else len(out["order"]), f"{time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
