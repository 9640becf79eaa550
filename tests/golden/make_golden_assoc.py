"""Golden vectors of oracle.association_bruteforce, produced by the UNMODIFIED reference.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_assoc.py

For the small fixture cases (make_golden.py) and one 2000-Gaussian fisheye scene, the reference's
brute-force per-tile sets (oracle.py:235-281) are stored as (n_tiles, ceil(n/32)) uint32 bitmaps,
next to the (tile, Gaussian) pairs whose minimum kappa is within 1e-9 (relative) of lam^2
(recomputed here the same way): rounding may decide those either way.  The GPU box never runs this.
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from raygauss import oracle as ro  # noqa: E402
from raygauss.association import build_grid  # noqa: E402
from raygauss.camera import Camera as RCamera, angles_to_dir  # noqa: E402
from raygauss.scene import GaussianScene as RScene  # noqa: E402

import workloads as synth# noqa: E402
from tests import golden_cases as G  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def kappa_min(scene, camera, grid, side):
    whit = RScene(scene.means, scene.log_scales, scene.quats, scene.opacity_logits, scene.sh).whitening_matrices()
    o_u = np.einsum("nij,nj->ni", whit, camera.optical_center[None, :] - scene.means)
    frac = (np.arange(side) + 0.5) / side
    out = np.empty((grid.n_tiles, len(scene)))
    for tile in range(grid.n_tiles):
        iy, ix = divmod(tile, grid.n_x)
        t0, t1 = 2.0 * np.arctan(grid.mirror_edges_x[ix]), 2.0 * np.arctan(grid.mirror_edges_x[ix + 1])
        p0, p1 = 2.0 * np.arctan(grid.mirror_edges_y[iy]), 2.0 * np.arctan(grid.mirror_edges_y[iy + 1])
        tt, pp = np.meshgrid(t0 + (t1 - t0) * frac, p0 + (p1 - p0) * frac)
        dirs = angles_to_dir(tt, pp).reshape(-1, 3) @ camera.rotation
        d_u = np.einsum("nij,rj->nri", whit, dirs)
        m = np.cross(o_u[:, None, :], d_u)
        out[tile] = ((m * m).sum(-1) / (d_u * d_u).sum(-1)).min(axis=1)
    return out


def ref_types(scene, cam):
    rs = RScene(means=scene.means, log_scales=scene.log_scales, quats=scene.quats,
                opacity_logits=scene.opacity_logits, sh=scene.sh)
    rc = RCamera(width=cam.width, height=cam.height, model=cam.model, rotation=cam.rotation,
                 translation=cam.translation, fov_x=cam.fov_x, fov_y=cam.fov_y, fx=cam.fx, fy=cam.fy, cx=cam.cx,
                 cy=cam.cy, k=cam.k)
    return rs, rc


def bitmap(sets, n_tiles, n):
    words = (n + 31) // 32
    bits = np.zeros((n_tiles, words), np.uint32)
    for t, s in enumerate(sets):
        for g in s:
            bits[t, g >> 5] |= np.uint32(1 << (g & 31))
    return bits


def main():
    cases = [(name, G.case(name).scene, G.case(name).camera, G.case(name).config.lam, G.case(name).config.tile_px, 64)
             for name in G.SMALL_CASES if name not in ("empty", "not_pd")]
    scene = synth.config_scene("C2", n=2000)
    cases.append(("c2_2k", scene, synth.config_camera("C2", width=256, height=144), 3.0, 16, 64))
    c = G.case("beap_small")
    cases.append(("beap_small_r100", c.scene, c.camera, 3.0, 16, 100))
    out = {}
    for name, scene0, cam0, lam, tile_px, rays in cases:
        scene, cam = ref_types(scene0, cam0)
        grid = build_grid(cam, tile_px)
        sets = ro.association_bruteforce(scene, cam, lam=lam, rays_per_tile=rays, grid=grid)
        side = max(8, int(np.ceil(np.sqrt(rays))))
        out[f"{name}__bits"] = bitmap(sets, grid.n_tiles, len(scene))
        km = kappa_min(scene, cam, grid, side)
        out[f"{name}__border"] = np.argwhere(np.abs(km / (lam * lam) - 1.0) < 1e-9).astype(np.int32)
        out[f"{name}__params"] = np.array([lam, tile_px, rays], np.float64)
        if name == "c2_2k":
            for k, v in (("means", scene.means), ("log_scales", scene.log_scales), ("quats", scene.quats),
                         ("opacity_logits", scene.opacity_logits), ("sh", scene.sh)):
                out[f"{name}__scene_{k}"] = v
        print(name, len(scene), grid.n_tiles, sum(len(s) for s in sets), flush=True)
    np.savez_compressed(os.path.join(HERE, "assoc_brute.npz"), **out)


if __name__ == "__main__":
    main()
