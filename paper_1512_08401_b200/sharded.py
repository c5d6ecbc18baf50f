"""Row-sharded deblur of ONE image across GPUs (BASELINE config C4).

The whole sharded solve lives behind the C ABI (include/wbx.h `wbx_sharded_*`, csrc/shard.cu):
the partition, the per-rank phase kernels, the exchange (NCCL all-gathers over NVLink inside
libwbx, captured with the phase kernels in one CUDA graph of the FISTA iterations) and the
device-resident step estimate. This module only
  * plans partitions on the host (`shard_plan`, no GPU needed),
  * sets up the NCCL communicator: rank 0 draws the 128-byte unique id (wbx_comm_get_unique_id),
    the caller's process group broadcasts it, every rank creates its communicator
    (`nccl_comm`),
  * wraps a prepared solve (`ShardedDeblurrer`): either one rank of a real multi-GPU run
    (comm given, ranks = [rank]) or every rank of `world` in this process on one GPU sharing
    the padded buffers (comm None: the partition code runs exactly as on `world` GPUs).
The restored image is bitwise the same for every world size (given tau).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional

import numpy as np

from . import _native as N
from . import waveblur as W

lib = N.lib
_check = W._check


def shard_plan(op: W.SparseOperator, world: int):
    """Row / column range bounds of each rank (host-only; wbx_shard_plan)."""
    rb = np.zeros(world + 1, dtype=np.uint64)
    cb = np.zeros(world + 1, dtype=np.uint64)
    _check(lib.wbx_shard_plan(op.n, W._u64ptr(op.row_offsets), W._u32ptr(op.col_indices), world, W._u64ptr(rb),
                              W._u64ptr(cb)))
    return rb.astype(np.int64), cb.astype(np.int64)


def unique_id() -> bytes:
    """ncclGetUniqueId through libwbx (rank 0 of a run)."""
    buf = C.create_string_buffer(128)
    _check(lib.wbx_comm_get_unique_id(buf))
    return buf.raw


def broadcast_unique_id(torch, dist, device=None) -> bytes:
    """Rank 0's unique id on every rank of the torch.distributed group (any backend)."""
    t = torch.zeros(128, dtype=torch.uint8, device=device)
    if dist.get_rank() == 0:
        t.copy_(torch.frombuffer(bytearray(unique_id()), dtype=torch.uint8))
    dist.broadcast(t, src=0)
    return bytes(t.cpu().numpy().tobytes())


class Comm:
    """An NCCL communicator owned by libwbx (wbx_comm)."""

    def __init__(self, ctx: W.Context, world: int, rank: int, uid: bytes):
        if len(uid) != 128:
            raise W.BadSpec("NCCL unique id must be 128 bytes")
        h = C.c_void_p()
        _check(lib.wbx_comm_create(ctx.handle, world, rank, uid, C.byref(h)))
        self.h, self.ctx, self.world, self.rank = h, ctx, world, rank

    def __del__(self):
        if lib is None or N is None or not N.alive():  # interpreter exit: leave it to the process
            return
        if getattr(self, "h", None):
            lib.wbx_comm_destroy(self.h)
            self.h = None


def nccl_comm(torch, dist, ctx: W.Context) -> Comm:
    """The libwbx NCCL communicator of this torch.distributed rank (one GPU per rank)."""
    dev = torch.device("cuda", ctx.device) if dist.get_backend() == "nccl" else None
    return Comm(ctx, dist.get_world_size(), dist.get_rank(), broadcast_unique_id(torch, dist, dev))


class ShardedDeblurrer:
    """C4 deblur (wbx_sharded): `ranks` are the shard ranks held by THIS process (all of range(world)
    when emulating on one GPU, [rank] with an NCCL `comm` in a real multi-GPU run)."""

    def __init__(self, ctx: W.Context, op: W.SparseOperator, basis: W.WaveletBasis, P: W.DiagonalPreconditioner,
                 weights, lambda_: float, iters: int, world: int, ranks: List[int], comm: Optional[Comm] = None,
                 tau: Optional[float] = None, step_safety: float = 1.01):
        self.ctx, self.basis, self.op, self.comm, self.world = ctx, basis, op, comm, world
        self.n = op.n
        p = W._f64(P.p, op.n, "preconditioner")
        w = W._f64(weights, op.n, "weights")
        cfg = W.SolverConfig(max_iters=iters, track_energy=False, precision=32, tau=tau or 0.0,
                             step_safety=step_safety).to_c()
        rk = np.array(ranks, dtype=np.uint32)
        h = C.c_void_p()
        _check(lib.wbx_sharded_create(ctx.handle, op.n, W._u64ptr(op.row_offsets), W._u32ptr(op.col_indices),
                                      W._dptr(op.values), basis.device(ctx), W._dptr(p), W._dptr(w),
                                      float(lambda_), C.byref(cfg), world, W._u32ptr(rk), rk.size,
                                      comm.h if comm is not None else None, C.byref(h)))
        self.h = h
        self.tau_iters = 0
        self.tau_steps = 0

    def estimate_step(self, step_safety: float = 1.01) -> float:
        """tau as the single-GPU fp32 solver computes it (the reference's power-iteration
        estimate, solver.cpp:69-99, by Lanczos; WBX_TAU=power: the literal power iteration)."""
        tau, it, st = C.c_double(), C.c_uint32(), C.c_uint32()
        _check(lib.wbx_sharded_estimate_step(self.h, float(step_safety), C.byref(tau), C.byref(it), C.byref(st)))
        self.tau_iters, self.tau_steps = int(it.value), int(st.value)
        return float(tau.value)

    def deblur_dev(self, u0_ptr: int, u_ptr: int, clamp: bool = True) -> None:
        """u0 (every rank: the whole image) -> restored image (device pointers, async)."""
        _check(lib.wbx_sharded_deblur_dev(self.h, C.c_void_p(u0_ptr), C.c_void_p(u_ptr), int(clamp)))

    def stats(self) -> dict:
        """tau, its iteration counts, device ms and launches of the last deblur (synchronises)."""
        self.ctx.synchronize()
        tau, it, st = C.c_double(), C.c_uint32(), C.c_uint32()
        t0, t1 = C.c_float(), C.c_float()
        ln = C.c_uint64()
        _check(lib.wbx_sharded_stats(self.h, C.byref(tau), C.byref(it), C.byref(st), C.byref(t0), C.byref(t1),
                                     C.byref(ln)))
        if it.value:
            self.tau_iters, self.tau_steps = int(it.value), int(st.value)
        return {"tau": float(tau.value), "tau_iters": int(it.value), "tau_steps": int(st.value),
                "tau_ms": float(t0.value), "iters_ms": float(t1.value), "launches": int(ln.value)}

    def __del__(self):
        if lib is None or N is None or not N.alive():  # interpreter exit: leave it to the process
            return
        if getattr(self, "h", None):
            lib.wbx_sharded_destroy(self.h)
            self.h = None
