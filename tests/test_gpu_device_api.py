"""Tensor-level fast path (geer_forward / geer_backward on device tensors) and training glue kernels."""

import ctypes

import numpy as np
import pytest
import torch

from paper_2505_24053_b200 import _lib, renderer
import workloads as synth
from paper_2505_24053_b200.device import DeviceRenderer, DeviceScene

pytestmark = pytest.mark.gpu


def _small():
    scene = synth.config_scene("C2", n=20_000)
    cam = synth.config_camera("C2", width=320, height=180)
    return scene, cam


def test_device_forward_matches_host_api():
    scene, cam = _small()
    cfg = renderer.RenderConfig(background=np.array([0.2, 0.3, 0.4]))
    host = renderer.render(scene, cam, cfg)
    r = DeviceRenderer(0)
    color, rem, cnt = r.forward(DeviceScene.from_scene(scene), cam, cfg)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(color.cpu().numpy().astype(np.float64), host.color.color)
    np.testing.assert_array_equal(rem.cpu().numpy().astype(np.float64), host.remaining_transmittance)
    np.testing.assert_array_equal(cnt.cpu().numpy().astype(np.int64), host.contributor_count)


def test_device_backward_accumulates_and_matches_host():
    scene, cam = _small()
    cfg = renderer.RenderConfig()
    dl = np.random.default_rng(3).standard_normal((cam.height, cam.width, 3)) / 1e4
    host = renderer.render_backward(scene, cam, dl, cfg)
    r = DeviceRenderer(0)
    ds = DeviceScene.from_scene(scene)
    r.forward(ds, cam, cfg)
    dlt = torch.as_tensor(dl.astype(np.float32)).cuda()
    g = r.backward(dlt)
    g = r.backward(dlt, grads=g, accumulate=True)
    torch.cuda.synchronize()
    for name, ref in (("means", host.dmeans), ("log_scales", host.dlog_scales), ("quats", host.dquats),
                      ("opacity_logits", host.dopacities), ("sh", host.dsh)):
        got = getattr(g, name).cpu().numpy().astype(np.float64)
        scale = np.abs(ref).max()
        # fp32 atomics: reduction order differs run to run
        assert np.abs(got - 2 * ref).max() <= 2e-3 * 2 * scale, name


def test_backward_without_forward_raises():
    r = DeviceRenderer(0)
    with pytest.raises(RuntimeError):
        r.backward(torch.zeros((4, 4, 3), device="cuda"))


def test_l1_grad_and_adam_kernels():
    lib = _lib.load()
    n = 1000
    a = torch.rand(n, 3, device="cuda")
    b = torch.rand(n, 3, device="cuda")
    mask = (torch.rand(n, device="cuda") > 0.3).to(torch.uint8)
    g = torch.empty_like(a)
    scale = 1.0 / (int(mask.sum()) * 3)
    _lib.check(lib.geer_l1_grad(a.data_ptr(), b.data_ptr(), mask.data_ptr(), g.data_ptr(), n, scale,
                                torch.cuda.current_stream().cuda_stream))
    ref = torch.sign(a - b) * scale * mask[:, None]
    torch.testing.assert_close(g, ref)
    # Adam (trainer.py:181-197)
    p = torch.randn(5000, device="cuda")
    grad = torch.randn(5000, device="cuda")
    m = torch.zeros_like(p)
    v = torch.zeros_like(p)
    lr = torch.full_like(p, 1e-3)
    p_ref, m_ref, v_ref = p.clone(), m.clone(), v.clone()
    for step in (1, 2, 3):
        _lib.check(lib.geer_adam(p.data_ptr(), grad.data_ptr(), m.data_ptr(), v.data_ptr(), lr.data_ptr(), 5000,
                                 ctypes.c_float(0.9), ctypes.c_float(0.999), ctypes.c_float(1e-15), step,
                                 None, torch.cuda.current_stream().cuda_stream))
        m_ref = 0.9 * m_ref + 0.1 * grad
        v_ref = 0.999 * v_ref + 0.001 * grad * grad
        p_ref = p_ref - 1e-3 * (m_ref / (1 - 0.9 ** step)) / (torch.sqrt(v_ref / (1 - 0.999 ** step)) + 1e-15)
    torch.testing.assert_close(p, p_ref, rtol=1e-5, atol=1e-6)
    # the guarded form: finite gradients update as before, a NaN anywhere skips the update and raises the flag
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    before = p.clone()
    _lib.check(lib.geer_adam(p.data_ptr(), grad.data_ptr(), m.data_ptr(), v.data_ptr(), lr.data_ptr(), 5000,
                             ctypes.c_float(0.9), ctypes.c_float(0.999), ctypes.c_float(1e-15), 4, flag.data_ptr(),
                             torch.cuda.current_stream().cuda_stream))
    assert int(flag) == 0 and not torch.equal(p, before)
    grad[4321] = float("nan")
    before = p.clone()
    _lib.check(lib.geer_adam(p.data_ptr(), grad.data_ptr(), m.data_ptr(), v.data_ptr(), lr.data_ptr(), 5000,
                             ctypes.c_float(0.9), ctypes.c_float(0.999), ctypes.c_float(1e-15), 5, flag.data_ptr(),
                             torch.cuda.current_stream().cuda_stream))
    assert int(flag) == 1 and torch.equal(p, before)


@pytest.mark.parametrize("config_name,n,w,h", [("C2", 50_000, 640, 360), ("C5", 40_000, 480, 270),
                                               ("C1", 10_000, 256, 256)])
def test_pbf_culling_is_exact(config_name, n, w, h):
    """Per-warp PBF culling skips only pairs with t = 0: forward outputs are bit-identical with it off."""
    scene = synth.config_scene(config_name, n=n)
    cam = synth.config_camera(config_name, width=w, height=h)
    cfg = renderer.RenderConfig(background=np.array([0.3, 0.1, 0.2]))
    ds = DeviceScene.from_scene(scene)
    r = DeviceRenderer(0)
    on = [t.clone() for t in r.forward(ds, cam, cfg)]
    st_on = r.stats()
    off = [t.clone() for t in r.forward(ds, cam, cfg, flags=_lib.GEER_CFG_NO_CULL)]
    st_off = r.stats()
    torch.cuda.synchronize()
    for a, b in zip(on, off):
        assert torch.equal(a, b)
    assert st_on["evaluated_pairs"] == st_off["evaluated_pairs"]
    assert st_on["warp_entries"] <= st_off["warp_entries"]


def test_camera_setup_cache_follows_the_camera():
    """K0 is cached per camera: alternating poses (same size) must match fresh renders bit for bit."""
    scene = synth.config_scene("C2", n=20_000)
    cam_a = synth.config_camera("C2", width=320, height=180)
    rot, t = synth.look_at((0.7, 0.2, -1.9))
    from paper_2505_24053_b200.scene import Camera

    cam_b = Camera(width=320, height=180, model="beap", rotation=rot, translation=t, fov_x=cam_a.fov_x,
                   fov_y=cam_a.fov_y)
    cfg = renderer.RenderConfig()
    ds = DeviceScene.from_scene(scene)
    fresh = {}
    for name, cam in (("a", cam_a), ("b", cam_b)):
        fresh[name] = DeviceRenderer(0).forward(ds, cam, cfg)[0].clone()
    r = DeviceRenderer(0)
    for name, cam in (("a", cam_a), ("b", cam_b), ("a", cam_a), ("a", cam_a), ("b", cam_b)):
        col = r.forward(ds, cam, cfg)[0]
        assert torch.equal(col, fresh[name]), name


def test_multiview_inflight_matches_serial():
    """C4 glue: views on two contexts/streams sum to the same gradients as one context."""
    from paper_2505_24053_b200 import train

    scene = synth.config_scene("C2", n=20_000)
    tr1 = synth.c4_trainer(scene, n_views=4, width=192, height=108, inflight=1)
    tr2 = train.MultiViewTrainer(synth.to_f32_values(synth.perturbed(scene, np.random.default_rng(1))),
                                 tr1.cameras, tr1.targets, inflight=2)
    tr1.accumulate()
    tr2.accumulate()
    torch.cuda.synchronize()
    g1, g2 = tr1.grads.buf, tr2.grads.buf
    assert torch.isfinite(g1).all() and float(g1.abs().max()) > 0
    torch.testing.assert_close(g2, g1, rtol=1e-3, atol=1e-4 * float(g1.abs().max()))


def _cam_zoo():
    """Cameras of mixed models, sizes and poses (more than the 16 cache slots + the current one)."""
    from paper_2505_24053_b200.scene import Camera

    cams = []
    for i in range(20):
        rot, t = synth.look_at((2.0 * np.sin(0.3 * i), 0.15 * (i % 3), -2.0 * np.cos(0.3 * i)))
        w, h = (96 + 16 * (i % 4), 64 + 8 * (i % 3))
        if i % 3 == 0:
            cams.append(Camera(width=w, height=h, model="pinhole", rotation=rot, translation=t, fx=0.8 * w, fy=0.8 * w,
                               cx=w / 2, cy=h / 2))
        elif i % 3 == 1:
            f = w / np.pi
            cams.append(Camera(width=w, height=h, model="kb", rotation=rot, translation=t, fx=f, fy=f,
                               cx=(w - 1) / 2, cy=(h - 1) / 2, k=np.zeros(4)))
        else:
            cams.append(Camera(width=w, height=h, model="beap", rotation=rot, translation=t, fov_x=np.pi,
                               fov_y=np.pi * h / w))
    return cams


def test_camera_cache_cycles_many_mixed_cameras_bit_exact():
    """more cameras than slots, mixed sizes and models, cycled twice through one context
    (slot hits, parking, MRU replacement, buffer regrowth): forward, backward and the graph export
    equal fresh contexts bit for bit."""
    from paper_2505_24053_b200 import association

    scene = synth.config_scene("C2", n=5_000)
    ds = DeviceScene.from_scene(scene)
    cfg = renderer.RenderConfig()
    cams = _cam_zoo()
    ref = []
    for cam in cams:
        r = DeviceRenderer(0)
        col, rem, cnt = (t.clone() for t in r.forward(ds, cam, cfg))
        dl = torch.ones((cam.height, cam.width, 3), device="cuda") * 1e-3
        ref.append((col, rem, cnt))
    r = DeviceRenderer(0)
    for _ in range(2):
        for cam, (col, rem, cnt) in zip(cams, ref):
            out = r.forward(ds, cam, cfg)
            assert torch.equal(out[0], col) and torch.equal(out[1], rem) and torch.equal(out[2], cnt)
            g = r.backward(torch.full((cam.height, cam.width, 3), 1e-3, device="cuda"))
            assert torch.isfinite(g.means).all()
    # the graph export (pixel tiles, edges) after cached-slot hits equals a fresh graph build
    for cam in cams[:4]:
        fresh = association.build_render_graph(scene, cam)
        again = association.build_render_graph(scene, cam)
        np.testing.assert_array_equal(fresh.order, again.order)
        np.testing.assert_array_equal(fresh.grid.pixel_tile, again.grid.pixel_tile)


def test_async_frames_equal_synchronous_frames():
    """After its first frame a context renders without host round trips; the asynchronous frames
    (sync=False, checked once at the end) equal the synchronous first frame bit for bit."""
    scene, cam = _small()
    cfg = renderer.RenderConfig()
    ds = DeviceScene.from_scene(scene)
    r = DeviceRenderer(0)
    first = [t.clone() for t in r.forward(ds, cam, cfg)]
    outs = []
    for _ in range(3):
        outs.append([t.clone() for t in r.forward(ds, cam, cfg, sync=False)])
    assert r.sync() is False
    for o in outs:
        for a, b in zip(o, first):
            assert torch.equal(a, b)
    assert r.stats()["n_entries"] > 0


def test_async_overflow_rerenders_the_frame():
    """A context sized by a small scene meets a much larger graph: the asynchronous frame overflows
    (background only, no out-of-bounds work), sync() reports it, grows the capacity and re-renders;
    the result equals a fresh context's frame."""
    small = synth.config_scene("C2", n=2_000)
    big = synth.config_scene("C2", n=40_000)
    cam = synth.config_camera("C2", width=320, height=180)
    cfg = renderer.RenderConfig()
    r = DeviceRenderer(0)
    r.forward(DeviceScene.from_scene(small), cam, cfg)  # learns a small capacity
    dbig = DeviceScene.from_scene(big)
    out = r.forward(dbig, cam, cfg, sync=False)
    assert r.sync() is True  # overflowed, re-rendered
    fresh = DeviceRenderer(0).forward(dbig, cam, cfg)
    for a, b in zip(out, fresh):
        assert torch.equal(a, b)
    # the next asynchronous frame fits the grown capacity
    out2 = [t.clone() for t in r.forward(dbig, cam, cfg, sync=False)]
    assert r.sync() is False
    for a, b in zip(out2, fresh):
        assert torch.equal(a, b)
    # and the default (synchronous) call hides the re-run from the caller
    r2 = DeviceRenderer(0)
    r2.forward(DeviceScene.from_scene(small), cam, cfg)
    out3 = r2.forward(dbig, cam, cfg)
    for a, b in zip(out3, fresh):
        assert torch.equal(a, b)


def test_async_frame_reports_non_pd_like_the_reference():
    """A non-PD view covariance met by an asynchronous frame raises the reference's ValueError at sync()."""
    from tests.golden_cases import case

    c = case("not_pd")
    scene, cam, cfg = c.scene, c.camera, c.config
    ok = synth.config_scene("C2", n=2_000)
    r = DeviceRenderer(0)
    r.forward(DeviceScene.from_scene(ok), cam, cfg)  # capacity known: the next frame is asynchronous
    r.forward(DeviceScene.from_scene(scene), cam, cfg, sync=False)
    with pytest.raises(ValueError, match="positive definite"):
        r.sync()


def test_caller_owned_workspace_sized_by_geer_workspace_bytes():
    """SURVEY 8b ownership: a torch tensor of geer_workspace_bytes holds every buffer of the device
    path (no library cudaMalloc); forward and backward equal a library-owned context bit for bit, and
    an undersized workspace fails with the size it needs."""
    scene = synth.config_scene("C2", n=100_000)
    cam = synth.config_camera("C2", width=480, height=270)
    cfg = renderer.RenderConfig()
    ds = DeviceScene.from_scene(scene)
    dl = torch.full((cam.height, cam.width, 3), 1e-4, device="cuda")
    ref = DeviceRenderer(0)
    out_ref = [t.clone() for t in ref.forward(ds, cam, cfg)]
    g_ref = ref.backward(dl)
    n_entries = ref.stats()["n_entries"]
    r = DeviceRenderer(0)
    need = r.workspace_bytes(ds, cam, cfg, max_entries=n_entries)
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    r.set_workspace(ws)
    for _ in range(3):  # first frame synchronous, then asynchronous frames sized by the capacity
        out = r.forward(ds, cam, cfg)
        g = r.backward(dl)
    torch.cuda.synchronize()
    for a, b in zip(out, out_ref):
        assert torch.equal(a, b)
    for name in ("means", "log_scales", "quats", "opacity_logits", "sh"):
        torch.testing.assert_close(getattr(g, name), getattr(g_ref, name), rtol=1e-4,
                                   atol=1e-5 * float(getattr(g_ref, name).abs().max()))
    assert 0 < r.workspace_used() <= need
    small = DeviceRenderer(0)
    small.set_workspace(torch.empty(need // 4, dtype=torch.uint8, device="cuda"))
    with pytest.raises(MemoryError, match="workspace too small"):
        small.forward(ds, cam, cfg)
    small.set_workspace(None)  # back to library memory: renders again
    out2 = small.forward(ds, cam, cfg)
    assert torch.equal(out2[0], out_ref[0])


def test_async_frame_is_cuda_graph_capturable():
    """With the camera cached and the capacity known, a device-level forward issues the same
    launches with the same arguments every time and never touches the host: it can be captured into
    a CUDA graph, whose replays equal the eager frame bit for bit (also after the scene changes in
    place - the graph reads the same buffers)."""
    scene, cam = _small()
    cfg = renderer.RenderConfig()
    ds = DeviceScene.from_scene(scene)
    r = DeviceRenderer(0)
    out = [t.clone() for t in r.forward(ds, cam, cfg)]  # first frame: capacity + camera setup
    bufs = tuple(torch.empty_like(t) for t in out)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        r.forward(ds, cam, cfg, out=bufs, sync=False)  # warm on the capture stream
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        r.forward(ds, cam, cfg, out=bufs, sync=False)
    for t in bufs:
        t.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert r.sync() is False
    for a, b in zip(bufs, out):
        assert torch.equal(a, b)
    # move the scene in place: the replay renders the new state like an eager frame does
    ds.means.add_(0.01)
    g.replay()
    torch.cuda.synchronize()
    eager = DeviceRenderer(0).forward(ds, cam, cfg)
    for a, b in zip(bufs, eager):
        assert torch.equal(a, b)


@pytest.mark.parametrize("pinned", [False, True])
def test_host_narrowing_equals_device_narrowing(pinned):
    """geer_render_host narrows the float64 scene on host cores (raw fp64 tail narrowed on the device
    when the arrays are pinned); the device sees the same fp32 values as torch's narrowing, so the
    frame equals the device-path frame bitwise.  Values are perturbed off the fp32 grid so rounding
    matters, and the scene is large enough for many host chunks."""
    from paper_2505_24053_b200.scene import GaussianScene

    base = synth.config_scene("C2", n=200_000)
    rng = np.random.default_rng(5)

    def off_grid(a):
        a = np.asarray(a, dtype=np.float64)
        a = a * (1.0 + rng.uniform(-1e-9, 1e-9, a.shape))
        if not pinned:
            return np.ascontiguousarray(a)
        t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        t.numpy()[...] = a
        return t.numpy()

    scene = GaussianScene(off_grid(base.means), off_grid(base.log_scales), off_grid(base.quats),
                          off_grid(base.opacity_logits), off_grid(base.sh))
    assert not np.array_equal(scene.sh.astype(np.float32).astype(np.float64), scene.sh)
    cam = synth.config_camera("C2", width=480, height=270)
    cfg = renderer.RenderConfig()
    host = renderer.render(scene, cam, cfg, return_graph=False)
    total = sum(a.size for a in (scene.means, scene.log_scales, scene.quats, scene.opacity_logits, scene.sh))
    sent = renderer.last_h2d_bytes(0)
    if pinned:
        assert 4 * total < sent < 8 * total
    else:
        assert sent == 4 * total
    r = DeviceRenderer(0)
    color, rem, cnt = r.forward(DeviceScene.from_scene(scene), cam, cfg)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(color.cpu().numpy().astype(np.float64), host.color.color)
    np.testing.assert_array_equal(rem.cpu().numpy().astype(np.float64), host.remaining_transmittance)
    np.testing.assert_array_equal(cnt.cpu().numpy().astype(np.int64), host.contributor_count)
