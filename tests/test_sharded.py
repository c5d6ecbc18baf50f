"""BASELINE config C4: one image row-sharded across ranks.

CPU: the partition plan (wbx_shard_plan, host-only) covers every nonempty row/column once and
balances nonzeros; the communicator setup (rank 0's NCCL unique id broadcast to every rank)
runs at world size 2 over gloo. GPU: the shards of worlds 1-8 emulated on ONE GPU (all shards
bind the same padded buffers; the partition code runs exactly as on N GPUs) give BITWISE the
same restored image for every world size, given tau, within 1e-5 of the reference's; the NCCL
path of the library through a one-rank communicator gives the same bits."""
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

    from paper_1512_08401_b200.sharded import broadcast_unique_id
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # the communicator setup of a multi-GPU run: rank 0 draws the NCCL unique id through libwbx
    # (wbx_comm_get_unique_id), the process group broadcasts it (wbx_comm_create then takes it)
    uid = broadcast_unique_id(torch, dist)
    op, _ = c1_operator()
    rb, cb = shard_plan(op, world)
    q.put((rank, uid, rb.tolist(), cb.tolist()))
    dist.destroy_process_group()


def test_communicator_setup_world2_gloo():
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
    (_, u0, rb0, cb0), (_, u1, rb1, cb1) = out
    assert len(u0) == 128 and u0 == u1 and any(u0)   # every rank holds rank 0's NCCL id
    assert rb0 == rb1 and cb0 == cb1                   # and plans the same partition


def _solve(op, basis, ctx, P, w, tau, world, z, comm=None, ranks=None):
    import torch

    from paper_1512_08401_b200.sharded import ShardedDeblurrer
    sh = ShardedDeblurrer(ctx, op, basis, P, w, 1e-4, 50, world, ranks if ranks is not None else list(range(world)),
                          comm=comm, tau=tau)
    dev = torch.device("cuda", 0)
    u0 = torch.from_numpy(z["u0"].copy()).to(dev)
    out = torch.empty_like(u0)
    torch.cuda.synchronize()
    sh.deblur_dev(u0.data_ptr(), out.data_ptr(), clamp=True)
    ctx.synchronize()
    return sh, out.cpu().numpy().reshape(256, 256)


@pytest.mark.gpu
def test_sharded_worlds_bitwise_and_vs_reference(monkeypatch):
    """Worlds 1, 2, 3, 8 emulated on one GPU give the same bits (given tau), within the 1e-5
    bar of the reference's restored image; the sharded Lanczos estimate reproduces the
    reference's iteration count and tau (and WBX_TAU=power the literal power iteration)."""
    op, z = c1_operator()
    basis = W.make_basis(W.FilterFamily.Daubechies, 4, (256, 256), 4)
    ctx = W.Context(0)
    P = W.spai(op, ctx)
    w = W.scale_weights(basis.layout)
    meta = __import__("json").loads(bytes(z["meta_json"]).decode())
    tau = float(meta["tau"])
    _, ref = _solve(op, basis, ctx, P, w, tau, 1, z)
    rest = z["restored"].reshape(256, 256)
    assert np.linalg.norm(np.clip(rest, 0, 1) - ref) <= 1e-5 * np.linalg.norm(np.clip(rest, 0, 1))
    for world in (2, 3, 8):
        sh, out = _solve(op, basis, ctx, P, w, tau, world, z)
        assert np.array_equal(out, ref), world
    t1, it1 = W.estimate_step(W.SparseThetaOp(op, ctx), P, 1.01, ctx=ctx, return_iters=True)
    t2 = sh.estimate_step(1.01)
    assert abs(t2 - tau) <= 1e-6 * tau
    assert sh.tau_iters == it1 and sh.tau_steps < it1
    monkeypatch.setenv("WBX_TAU", "power")
    sh2, _ = _solve(op, basis, ctx, P, w, tau, 2, z)
    t3 = sh2.estimate_step(1.01)
    assert abs(t3 - tau) <= 1e-6 * tau and sh2.tau_iters == it1


@pytest.mark.gpu
def test_sharded_through_a_real_nccl_communicator():
    """World 1 through an actual NCCL communicator (one rank on this GPU): the library's NCCL
    path (all-gathers and the all-reduce captured in the iteration graph) gives the bits of the
    communicator-free run."""
    from paper_1512_08401_b200.sharded import Comm, unique_id
    op, z = c1_operator()
    basis = W.make_basis(W.FilterFamily.Daubechies, 4, (256, 256), 4)
    ctx = W.Context(0)
    P = W.spai(op, ctx)
    w = W.scale_weights(basis.layout)
    tau = float(__import__("json").loads(bytes(z["meta_json"]).decode())["tau"])
    _, ref = _solve(op, basis, ctx, P, w, tau, 1, z)
    comm = Comm(ctx, 1, 0, unique_id())
    sh, out = _solve(op, basis, ctx, P, w, tau, 1, z, comm=comm, ranks=[0])
    assert np.array_equal(out, ref)
    _, again = _solve(op, basis, ctx, P, w, tau, 1, z, comm=comm, ranks=[0])  # graph replay
    assert np.array_equal(again, ref)
