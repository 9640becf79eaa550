"""Host-side logic of the multi-view training step on CPU (gloo, world size 2).

The C4 step shards views contiguously over ranks, accumulates each rank's
per-Gaussian gradients into one flat fp32 buffer whose slices are the SoA
parameter groups, and sums it with ONE all_reduce.  Here the
per-view gradients are synthetic (the CUDA backward is covered by the GPU
tests); what is checked is sharding, the flat layout and the reduction.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_24053_b200.train import FIELDS, FlatScene, allreduce_grads, shard

N, NB, VIEWS = 37, 9, 11


def view_grad(flat: FlatScene, v: int):
    """Deterministic synthetic gradient of view v, written through the SoA views."""
    for k, (name, _) in enumerate(FIELDS):
        t = getattr(flat.scene, name)
        g = torch.Generator().manual_seed(1000 * v + k)
        t.add_(torch.randn(t.shape, generator=g))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        grads = FlatScene(N, NB, "cpu")
        for v in shard(VIEWS, rank, world):
            view_grad(grads, v)
        allreduce_grads(grads.buf, world)
        out[rank] = grads.buf.clone()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_covers_every_view_once(world):
    seen = [v for r in range(world) for v in shard(VIEWS, r, world)]
    assert seen == list(range(VIEWS))
    sizes = [len(shard(VIEWS, r, world)) for r in range(world)]
    assert max(sizes) - min(sizes) <= 1


def test_flat_buffer_slices_are_the_soa_groups():
    f = FlatScene(N, NB, "cpu")
    assert f.numel == N * (3 + 3 + 4 + 1 + NB * 3)
    f.scene.sh.fill_(2.0)
    f.scene.means.fill_(1.0)
    assert float(f.buf.sum()) == pytest.approx(N * 3 * 1.0 + N * NB * 3 * 2.0)
    assert f.scene.sh.shape == (N, NB, 3) and f.scene.opacity_logits.shape == (N,)


def test_two_rank_allreduce_equals_single_rank_sum():
    world = 2
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        bufs = [out[r] for r in range(world)]
    ref = FlatScene(N, NB, "cpu")
    for v in range(VIEWS):
        view_grad(ref, v)
    assert torch.equal(bufs[0], bufs[1]), "replicas must hold identical reduced gradients"
    torch.testing.assert_close(bufs[0], ref.buf, rtol=1e-6, atol=1e-6)
