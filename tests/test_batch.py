"""BASELINE config C5: batches of independent images sharing the operator (SpMM solve).
The batched kernel keeps the per-image arithmetic order of the single-image kernel, so a
batch must reproduce single-image deblurs BITWISE; the sharding of a batch across ranks
(bench.py --gpus N) is host logic, covered on CPU with gloo."""
import os

import numpy as np
import pytest

from paper_1512_08401_b200 import synthetic as S
from paper_1512_08401_b200 import waveblur as W
from paper_1512_08401_b200.sharding import shard


def test_shard_partition_covers_each_image_once():
    for n in (1, 7, 64):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                lo, hi = shard(n, world, r)
                seen.extend(range(lo, hi))
            assert seen == list(range(n))


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard(64, world, rank)
    t = torch.tensor([float(hi - lo)])
    dist.all_reduce(t)
    mx = torch.tensor([float(rank + 1)])
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    q.put((rank, lo, hi, float(t.item()), float(mx.item())))
    dist.destroy_process_group()


def test_batch_sharding_world2_gloo():
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert out[0][1:3] == (0, 32) and out[1][1:3] == (32, 64)
    assert all(o[3] == 64.0 and o[4] == 2.0 for o in out)  # all images counted; max over ranks


@pytest.mark.gpu
@pytest.mark.parametrize("batch", [4, 8])
def test_batched_deblur_bitwise_equals_single(golden, batch, monkeypatch):
    # the fp32 single-image window engine is the batch kernel's per-image arithmetic (the default
    # single-image engine for this invariant operator is the fp64 spectral one)
    monkeypatch.setenv("WBX_ENGINE", "window")
    g = golden("c1_db4_256")
    op = g.operator()
    basis = W.make_basis(W.FilterFamily.Daubechies, 4, (256, 256), 4)
    P = W.spai(op)
    w = g.weights()
    cfg = W.SolverConfig(max_iters=50, track_energy=False)
    imgs = np.stack([S.degrade((256, 256), 5.0, 5e-3, seed)[1] for seed in range(batch)])
    single = W.Deblurrer(op, basis, P, w, 1e-4, cfg)
    ref = np.stack([single.deblur(im, clamp=True)[0] for im in imgs])
    many = W.Deblurrer(op, basis, P, w, 1e-4, cfg, batch=batch)
    out, rep = many.deblur(imgs, clamp=True)
    assert out.shape == (batch, 256, 256)
    assert np.array_equal(out, ref)
    assert abs(rep.tau - g.meta["tau"]) <= 1e-6 * g.meta["tau"]


@pytest.mark.gpu
def test_batch_rejects_tracking():
    n = 64
    eye = W.SparseOperator(n, np.arange(n + 1, dtype=np.uint64), np.arange(n, dtype=np.uint32), np.ones(n))
    basis = W.make_basis(W.FilterFamily.Haar, 1, (8, 8), 2)
    with pytest.raises(W.BadSpec):
        W.Deblurrer(eye, basis, W.identity_precond(n), np.ones(n), 1e-4, W.SolverConfig(max_iters=5), batch=4)
    with pytest.raises(W.BadSpec):
        W.Deblurrer(eye, basis, W.identity_precond(n), np.ones(n), 1e-4,
                    W.SolverConfig(max_iters=5, track_energy=False), batch=3)
