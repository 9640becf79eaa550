"""GPU oracle at scale: brute-force association (geer_association_check).

The GPU restatement of oracle.association_bruteforce (oracle.py:235-281) is pinned to the
reference's own brute-force sets (tests/golden/assoc_brute.npz), then used on the 100k-1M
Gaussian configs, where the Python oracle cannot go, to show that every (tile, Gaussian) pair
the dense ray sampling finds is in the render graph's tile lists.
"""

import numpy as np
import pytest
import torch

from paper_2505_24053_b200 import renderer
import workloads as synth
from paper_2505_24053_b200.device import DeviceRenderer, DeviceScene
from paper_2505_24053_b200.scene import Camera
from tests.test_oracle_bruteforce import assert_sets_equal, brute_case, brute_cases

pytestmark = pytest.mark.gpu


def _graph(scene, cam, cfg):
    r = DeviceRenderer(0)
    ds = DeviceScene.from_scene(scene)
    r.forward(ds, cam, cfg)
    torch.cuda.synchronize()
    return r, ds


@pytest.mark.parametrize("name", brute_cases())
def test_gpu_bruteforce_matches_reference(name):
    scene, cam, lam, tile_px, rays, want, border = brute_case(name)
    r, ds = _graph(scene, cam, renderer.RenderConfig(lam=lam, tile_px=tile_px))
    n_tiles = want.shape[0]
    hits = torch.zeros(want.size, dtype=torch.int32, device="cuda")
    res = r.ctx.association_check(rays, hit_bits_ptr=hits.data_ptr())
    got = hits.cpu().numpy().view(np.uint32).reshape(n_tiles, -1)
    assert_sets_equal(got, want, border, len(scene))
    assert res["missing"] == 0, res["missing_pairs"]
    assert res["brute_pairs"] == int(np.unpackbits(want.view(np.uint8)).sum())


SCALE = {
    # name: (config, n, width, height, RenderConfig kwargs, rays per tile)
    "c2_1m_1080p": ("C2", 1_000_000, 1920, 1080, {}, 64),
    "c2_200k_lam2_tile8": ("C2", 200_000, 960, 540, {"lam": 2.0, "tile_px": 8}, 64),
    "c2_100k_r256": ("C2", 100_000, 480, 270, {}, 256),
    "kb_1m_1080p": ("C5", 1_000_000, 1920, 1080, {}, 64),
    "pinhole_200k": ("C1", 200_000, 640, 480, {}, 64),
}


@pytest.mark.parametrize("name", list(SCALE))
def test_association_is_sound_at_scale(name):
    cfgname, n, w, h, kw, rays = SCALE[name]
    scene = synth.config_scene(cfgname, n=n)
    cam = synth.config_camera(cfgname, width=w, height=h)
    r, _ = _graph(scene, cam, renderer.RenderConfig(**kw))
    res = r.ctx.association_check(rays)
    assert res["missing"] == 0, f"{res['missing']} brute-force pairs not in the tile lists: {res['missing_pairs']}"
    assert 0 < res["brute_pairs"] <= res["graph_entries"]
    print(name, res)


def test_behind_camera_wide_fov_sound():
    """Camera inside the cloud, 300 x 160 degree BEAP: antipodal arcs and behind-camera Gaussians."""
    scene = synth.config_scene("C2", n=100_000)
    rot, t = synth.look_at((0.05, 0.02, 0.0), target=(1.0, 0.0, 0.3))
    cam = Camera(width=600, height=320, model="beap", rotation=rot, translation=t, fov_x=np.deg2rad(300.0),
                 fov_y=np.deg2rad(160.0))
    r, _ = _graph(scene, cam, renderer.RenderConfig())
    res = r.ctx.association_check(64)
    assert res["missing"] == 0, res["missing_pairs"]
