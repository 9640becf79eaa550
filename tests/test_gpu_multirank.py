"""The C4 training step across real ranks with real CUDA gradients (trainer.py:181-197,230-296).

Two ranks each run the CUDA forward + loss + backward over their contiguous share of 4 views, sum the
flat gradient buffer with one all_reduce (NCCL when two GPUs are visible, else gloo with both ranks on
one GPU — ``GEER_DIST_BACKEND`` overrides), and apply the guarded Adam.  Checked against one rank
rendering all 4 views:

* the reduced buffer equals the 1-rank sum to per-element 1e-5 |g| + 1e-6 max|g| (the per-view
  backward accumulates with fp32 atomics, so the summation order differs run to run);
* after Adam the two ranks' parameter replicas are bit-identical.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N_GAUSSIANS, VIEWS, W, H = 20_000, 4, 192, 108


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, outdir):
    import torch.distributed as dist

    import workloads
    from paper_2505_24053_b200.train import allreduce_grads

    n_dev = torch.cuda.device_count()
    dev = rank % n_dev
    torch.cuda.set_device(dev)
    if world > 1:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        backend = os.environ.get("GEER_DIST_BACKEND") or ("nccl" if n_dev >= world else "gloo")
        dist.init_process_group(backend, rank=rank, world_size=world)
    try:
        scene = workloads.config_scene("C2", n=N_GAUSSIANS)
        tr = workloads.c4_trainer(scene, n_views=VIEWS, rank=rank, world=world, device=dev, width=W, height=H,
                                  inflight=1)
        tr.accumulate()
        allreduce_grads(tr.grads.buf, world)
        reduced = tr.grads.buf.cpu().numpy().copy()
        tr.apply()
        tr.check_finite()
        torch.cuda.synchronize()
        np.savez(os.path.join(outdir, f"w{world}_r{rank}.npz"), reduced=reduced,
                 params=tr.params.buf.cpu().numpy(), views=np.array(list(range(len(tr.cameras)))))
    finally:
        if world > 1:
            dist.destroy_process_group()


def _run(world, outdir):
    mp.start_processes(_worker, args=(world, _free_port(), outdir), nprocs=world, join=True, start_method="spawn")


def test_two_ranks_equal_one_rank(tmp_path):
    _run(1, str(tmp_path))
    _run(2, str(tmp_path))
    one = np.load(tmp_path / "w1_r0.npz")
    r0, r1 = np.load(tmp_path / "w2_r0.npz"), np.load(tmp_path / "w2_r1.npz")
    g1, g2 = one["reduced"].astype(np.float64), r0["reduced"].astype(np.float64)
    assert np.isfinite(g2).all()
    scale = np.abs(g1).max()
    err = np.abs(g2 - g1)
    bad = err > 1e-5 * np.abs(g1) + 1e-6 * scale
    assert not bad.any(), (int(bad.sum()), float(err.max()), float(scale))
    # both ranks hold the same reduced buffer and, after the identical Adam update, identical replicas
    np.testing.assert_array_equal(r0["reduced"], r1["reduced"])
    np.testing.assert_array_equal(r0["params"], r1["params"])


def test_nonfinite_step_raises_and_keeps_parameters():
    """trainer.py:270-282: a non-finite loss raises NaNLossError; the guarded Adam skipped the update."""
    import workloads
    from paper_2505_24053_b200.train import NaNLossError

    scene = workloads.config_scene("C2", n=5_000)
    tr = workloads.c4_trainer(scene, n_views=2, width=96, height=54, inflight=1)
    tr.targets[0][10, 10, 0] = float("nan")
    before = tr.params.buf.clone()
    with pytest.raises(NaNLossError, match="loss became non-finite at iteration 1"):
        tr.step(compute_loss=True)
    if int(tr.nonfinite.item()):
        assert torch.equal(tr.params.buf, before)
