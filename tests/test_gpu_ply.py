"""PLY straight to the device SoA (geer_ply_to_soa) equals the host loader's values."""

import numpy as np
import pytest
import torch

from paper_2505_24053_b200 import ply
import workloads as synth
from paper_2505_24053_b200.device import DeviceScene

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("bands", [1, 9, 16])
def test_load_scene_device_matches_host(tmp_path, bands):
    scene = synth.to_f32_values(synth.random_scene(5000, np.random.default_rng(bands), sh_bands=bands))
    path = tmp_path / "s.ply"
    ply.save_scene(scene, path)
    dev = ply.load_scene_device(path)
    ref = DeviceScene.from_scene(ply.load_scene(path))
    torch.cuda.synchronize()
    for k in ("means", "log_scales", "quats", "opacity_logits", "sh"):
        assert torch.equal(getattr(dev, k), getattr(ref, k)), k
