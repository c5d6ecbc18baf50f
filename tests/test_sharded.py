"""BASELINE config C4: one image row-sharded across ranks.

CPU: the partition plan (wbx_shard_plan, host-only) covers every nonempty row/column once and
balances nonzeros; the exchange protocol (padded slices all-gathered, scalars all-reduced)
runs at world size 2 over gloo. GPU: the shards of worlds 1-3 emulated on ONE GPU (all
shards bind the same padded buffers; the partition code runs exactly as on N GPUs) must give
a restored image BITWISE equal to the single-GPU solver's, given the same tau."""
import os
import socket
from pathlib import Path

import numpy as np
import pytest

from paper_1512_08401_b200 import waveblur as W
from paper_1512_08401_b200.sharded import shard_plan

GOLDEN = Path(__file__).resolve().parent / "golden"


def c1_operator():
    z = np.load(GOLDEN / "c1_db4_256.npz")
    gl = W.GeneratorList((256, 256), 4, W.FilterFamily.Daubechies, 4, z["gen_block"].astype(np.uint32),
                         z["gen_index"].astype(np.uint32), z["gen_count"].astype(np.uint64), z["gen_value"])
    return W.theta_from_generators(gl), z


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_plan_covers_and_balances(world):
    op, _ = c1_operator()
    rb, cb = shard_plan(op, world)
    rowlen = np.diff(op.row_offsets.astype(np.int64))
    collen = np.bincount(op.col_indices, minlength=op.n)
    nR, nC = np.count_nonzero(rowlen), np.count_nonzero(collen)
    assert rb[0] == 0 and rb[-1] == nR and np.all(np.diff(rb) >= 0)
    assert cb[0] == 0 and cb[-1] == nC and np.all(np.diff(cb) >= 0)
    # nnz balance: rows are sorted by descending length, so each range's nnz is within one
    # (longest) row of the ideal share
    order = np.argsort(-rowlen[rowlen > 0], kind="stable")
    lens = rowlen[rowlen > 0][order]
    per = [lens[rb[q]:rb[q + 1]].sum() for q in range(world)]
    assert max(per) - op.nnz() / world <= lens.max() + 1


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_1512_08401_b200.sharded import TorchExchange
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    op, _ = c1_operator()
    rb, cb = shard_plan(op, world)
    maxC = int(np.max(np.diff(cb)))
    buf = torch.full((world * maxC,), -1.0, dtype=torch.float32)
    own = torch.arange(cb[rank], cb[rank + 1], dtype=torch.float32)   # this rank's owned C positions
    buf[rank * maxC: rank * maxC + own.numel()] = own
    ex = TorchExchange(torch, dist, None)
    ex.gather(buf, None)
    # power-iteration sums: each rank fills its [2] slot, the all-gather gives every rank the
    # same [world][2] buffer, which the device then sums in rank order
    sums = torch.zeros(2 * world, dtype=torch.float64)
    sums[2 * rank:2 * rank + 2] = torch.tensor([float(rank + 1), 2.0 * rank], dtype=torch.float64)
    ex.gather(sums, None)
    q.put((rank, buf.numpy().tolist(), sums.numpy().tolist(), maxC, cb.tolist()))
    dist.destroy_process_group()


def test_exchange_protocol_world2_gloo():
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
    out = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    (_, b0, s0, maxC, cb), (_, b1, s1, _, _) = out
    assert b0 == b1  # every rank holds the same assembled vector
    for q_ in range(2):
        seg = b0[q_ * maxC: q_ * maxC + (cb[q_ + 1] - cb[q_])]
        assert seg == list(map(float, range(cb[q_], cb[q_ + 1])))
    assert s0 == s1 == [1.0, 0.0, 2.0, 2.0]


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_bitwise_equals_single_gpu(world, monkeypatch):
    import torch

    from paper_1512_08401_b200.sharded import LocalExchange, ShardedDeblurrer
    op, z = c1_operator()
    basis = W.make_basis(W.FilterFamily.Daubechies, 4, (256, 256), 4)
    ctx = W.Context(0)
    P = W.spai(op, ctx)
    w = W.scale_weights(basis.layout)
    tau = float(__import__("json").loads(bytes(z["meta_json"]).decode())["tau"])
    single = W.Deblurrer(op, basis, P, w, 1e-4, W.SolverConfig(max_iters=50, track_energy=False, tau=tau), ctx)
    ref, _ = single.deblur(z["u0"], clamp=True)
    sh = ShardedDeblurrer(torch, ctx, op, basis, P, w, 1e-4, 50, world, list(range(world)), LocalExchange())
    dev = torch.device("cuda", 0)
    u0 = torch.from_numpy(z["u0"].copy()).to(dev)
    out = torch.empty_like(u0)
    torch.cuda.synchronize()
    sh.deblur_dev(u0.data_ptr(), out.data_ptr(), tau=tau, clamp=True)
    ctx.synchronize()
    assert np.array_equal(out.cpu().numpy().reshape(256, 256), ref)
    # estimate_step through the sharded Lanczos estimate (default) and the sharded power
    # iteration (WBX_TAU=power): the reference's stopping iteration and tau
    t1, it1 = W.estimate_step(W.SparseThetaOp(op, ctx), P, 1.01, ctx=ctx, return_iters=True)
    t2 = sh.estimate_step(1.01)
    assert abs(t2 - tau) <= 1e-6 * tau
    assert sh.tau_iters == it1 and sh.tau_steps < it1
    monkeypatch.setenv("WBX_TAU", "power")
    t3 = sh.estimate_step(1.01)
    assert abs(t3 - tau) <= 1e-6 * tau and sh.tau_iters == it1
    del sh, single
