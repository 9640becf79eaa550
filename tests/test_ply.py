"""PLY scene I/O (ply.py mirror): layout-compatible with the reference in both directions, same errors."""

import os
import sys

import numpy as np
import pytest

from paper_2505_24053_b200 import ply
import workloads as synth

REF = "/root/reference/pkg/src"


@pytest.mark.parametrize("bands", [1, 4, 16])
def test_round_trip(tmp_path, bands):
    scene = synth.to_f32_values(synth.random_scene(300, np.random.default_rng(bands), sh_bands=bands))
    path = tmp_path / "s.ply"
    ply.save_scene(scene, path)
    back = ply.load_scene(path)
    for k in ("means", "log_scales", "quats", "opacity_logits", "sh"):
        np.testing.assert_array_equal(getattr(back, k), getattr(scene, k))


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")
def test_files_interchange_with_the_reference(tmp_path):
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from raygauss import ply as rply
    from raygauss.scene import GaussianScene as RScene

    scene = synth.to_f32_values(synth.random_scene(257, np.random.default_rng(3), sh_bands=9))
    ours, theirs = tmp_path / "ours.ply", tmp_path / "theirs.ply"
    ply.save_scene(scene, ours)
    rply.save_scene(RScene(scene.means, scene.log_scales, scene.quats, scene.opacity_logits, scene.sh), theirs)
    assert ours.read_bytes() == theirs.read_bytes()  # byte-identical files
    a, b = ply.load_scene(theirs), rply.load_scene(ours)
    for k in ("means", "log_scales", "quats", "opacity_logits", "sh"):
        np.testing.assert_array_equal(getattr(a, k), getattr(b, k))


def test_errors(tmp_path):
    p = tmp_path / "bad.ply"
    p.write_bytes(b"nope\n")
    with pytest.raises(ply.PLYFormatError, match="missing 'ply' magic"):
        ply.load_scene(p)
    p.write_bytes(b"ply\nformat ascii 1.0\nelement vertex 1\nproperty float x\nend_header\n")
    with pytest.raises(ply.PLYFormatError, match="unsupported format"):
        ply.load_scene(p)
    p.write_bytes(b"ply\nformat binary_little_endian 1.0\nelement vertex 1\nproperty float x\nend_header\n" + b"\0" * 4)
    with pytest.raises(ply.PLYFormatError, match="missing required properties"):
        ply.load_scene(p)
    names = ["x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2", "f_rest_0", "opacity", "scale_0", "scale_1", "scale_2",
             "rot_0", "rot_1", "rot_2", "rot_3"]
    hdr = "ply\nformat binary_little_endian 1.0\nelement vertex 1\n" + "".join(f"property float {n}\n" for n in names)
    p.write_bytes((hdr + "end_header\n").encode() + b"\0" * 4 * len(names))
    with pytest.raises(ply.PLYFormatError, match="not divisible by 3"):
        ply.load_scene(p)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")
def test_camera_json_interchanges_with_the_reference(tmp_path):
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from raygauss import camera as rcam

    from paper_2505_24053_b200 import camera

    cams = [synth.config_camera("C1"), synth.config_camera("C2"), synth.config_camera("C5", 320, 180)]
    ours = tmp_path / "ours.json"
    camera.save_cameras(cams, ours)
    back = rcam.load_cameras(ours)
    theirs = tmp_path / "theirs.json"
    rcam.save_cameras(back, theirs)
    assert ours.read_text() == theirs.read_text()
    for a, b in zip(camera.load_cameras(theirs), cams):
        assert (a.width, a.height, a.model) == (b.width, b.height, b.model)
        np.testing.assert_array_equal(a.rotation, b.rotation)
