"""The numpy restatement of oracle.association_bruteforce against the reference's own sets.

tests/golden/assoc_brute.npz holds the unmodified reference's brute-force tile sets
(make_golden_assoc.py); pairs whose minimum kappa lies within 1e-9 of lam^2 may round either way.
The same fixture pins the GPU version (tests/test_gpu_assoc_check.py).
"""

import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2505_24053_b200.scene import GaussianScene
import workloads as synth
from tests import golden_cases as G

FIX = os.path.join(G.GOLDEN, "assoc_brute.npz")


def brute_cases():
    with np.load(FIX) as z:
        return sorted({k.split("__")[0] for k in z.files})


def brute_case(name):
    """(scene, camera, lam, tile_px, rays, golden bits, borderline pairs)."""
    with np.load(FIX) as z:
        d = {k.split("__", 1)[1]: z[k] for k in z.files if k.split("__")[0] == name}
    lam, tile_px, rays = d["params"]
    if name == "c2_2k":
        scene = GaussianScene(d["scene_means"], d["scene_log_scales"], d["scene_quats"], d["scene_opacity_logits"],
                              d["scene_sh"])
        cam = synth.config_camera("C2", width=256, height=144)
    else:
        c = G.case(name.replace("_r100", ""))
        scene, cam = c.scene, c.camera
    return scene, cam, float(lam), int(tile_px), int(rays), d["bits"], d["border"]


def unpack(bits, n):
    return np.unpackbits(bits.view(np.uint8).reshape(bits.shape[0], -1), axis=1, bitorder="little")[:, :n].astype(bool)


def assert_sets_equal(got, want, border, n):
    a, b = unpack(got, n), unpack(want, n)
    diff = np.argwhere(a != b)
    bset = {tuple(p) for p in border.tolist()}
    bad = [tuple(p) for p in diff.tolist() if tuple(p) not in bset]
    assert not bad, f"{len(bad)} (tile, gid) pairs differ, e.g. {bad[:5]}"


@pytest.mark.parametrize("name", brute_cases())
def test_numpy_bruteforce_matches_reference(name):
    scene, cam, lam, tile_px, rays, want, border = brute_case(name)
    got = O.association_bruteforce(scene, cam, lam, rays, tile_px)
    assert_sets_equal(got, want, border, len(scene))


@pytest.mark.parametrize("name", ["beap_small", "kb_inside", "pinhole_small", "tile8_lam25", "c2_2k"])
def test_oracle_graph_is_a_superset_of_bruteforce(name):
    """Soundness of the C oracle's association: every brute-force pair is in the tile lists."""
    scene, cam, lam, tile_px, rays, want, _ = brute_case(name)
    g = O.build_render_graph(scene, cam, lam, tile_px)
    n = len(scene)
    have = np.zeros((g.grid.n_tiles, n), bool)
    have[g.entry_tile, g.order] = True
    assert not (unpack(want, n) & ~have).any()
