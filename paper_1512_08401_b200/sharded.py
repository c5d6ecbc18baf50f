"""Row-sharded deblur of ONE image across GPUs (BASELINE config C4).

The device work per rank is the libwbx shard API (include/wbx.h, csrc/shard.cu). This
module is the host-side orchestration:
  * `Exchange`: how the owned slices of the padded cross-rank vectors reach every rank:
    - `LocalExchange`: all shards live in this process on one GPU and bind the SAME padded
      buffers, so the exchange is implicit (used to test the partition code on one GPU);
    - `TorchExchange`: one rank per GPU, NCCL `all_gather_into_tensor` over NVLink on the
      solver's stream (gloo list form on CPU for the tests).
  * `ShardedDeblurrer`: analyze -> estimate_step (device-resident power iteration: per-rank
    sums all-gathered and reduced in rank order on every rank, no host round trip) ->
    FISTA (phase A, all-gather res, phase T, all-gather y) -> assemble x -> synthesize.
A sharded solve is bitwise equal to the single-GPU fp32 solve given the same tau.
"""
from __future__ import annotations

import ctypes as C
import os
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


class _Shard:
    def __init__(self, ctx: W.Context, op: W.SparseOperator, world: int, rank: int):
        h = C.c_void_p()
        _check(lib.wbx_shard_create(ctx.handle, op.n, W._u64ptr(op.row_offsets), W._u32ptr(op.col_indices),
                                    W._dptr(op.values), world, rank, C.byref(h)))
        self.h = h
        self.ctx = ctx  # the context (stream) must outlive the shard
        info = np.zeros(8, dtype=np.uint64)
        _check(lib.wbx_shard_get_info(h, W._u64ptr(info)))
        self.world, self.rank, self.rlo, self.rhi, self.clo, self.chi, self.maxR, self.maxC = (int(v) for v in info)

    def __del__(self):
        if lib is None or N is None or not N.alive():  # interpreter exit: leave it to the process
            return
        if getattr(self, "h", None):
            lib.wbx_shard_destroy(self.h)
            self.h = None


class LocalExchange:
    """All shards in one process share the padded buffers: nothing to move."""

    def gather(self, buf, rank_slices):
        return None

    def allreduce_sum_(self, t):
        return None


class TorchExchange:
    """One shard per process; NCCL collectives on the solver's CUDA stream."""

    def __init__(self, torch, dist, stream=None):
        self.torch, self.dist, self.stream = torch, dist, stream

    def _ctx(self):
        import contextlib
        return self.torch.cuda.stream(self.stream) if self.stream is not None else contextlib.nullcontext()

    def gather(self, buf, rank_slices):
        """All-gather of each rank's equal-size slice of the padded buffer, in place."""
        rank, world = self.dist.get_rank(), self.dist.get_world_size()
        m = buf.numel() // world
        with self._ctx():
            if buf.is_cuda:
                self.dist.all_gather_into_tensor(buf, buf[rank * m:(rank + 1) * m])
            else:  # gloo (CPU tests): list form
                parts = [self.torch.empty_like(buf[:m]) for _ in range(world)]
                self.dist.all_gather(parts, buf[rank * m:(rank + 1) * m].clone())
                for q in range(world):
                    buf[q * m:(q + 1) * m] = parts[q]

    def allreduce_sum_(self, t):
        with self._ctx():
            self.dist.all_reduce(t)


class ShardedDeblurrer:
    """C4 deblur. ranks: the shard ranks held by THIS process (all of them when emulating
    on one GPU, [dist.get_rank()] in a real multi-GPU run)."""

    def __init__(self, torch, ctx: W.Context, op: W.SparseOperator, basis: W.WaveletBasis,
                 P: W.DiagonalPreconditioner, weights, lambda_: float, iters: int, world: int,
                 ranks: List[int], exchange, accelerate: bool = True):
        self.torch, self.ctx, self.basis, self.iters, self.world = torch, ctx, basis, int(iters), world
        self.n = op.n
        self.exchange = exchange
        self.stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", ctx.device))
        self.dev = torch.device("cuda", ctx.device)
        self.shards = [_Shard(ctx, op, world, r) for r in ranks]
        s0 = self.shards[0]
        with torch.cuda.stream(self.stream):
            self.y = torch.zeros(world * s0.maxC, dtype=torch.float32, device=self.dev)
            self.res = torch.zeros(world * s0.maxR, dtype=torch.float32, device=self.dev)
            self.u = torch.zeros(world * s0.maxC, dtype=torch.float64, device=self.dev)
            self.t = torch.zeros(world * s0.maxR, dtype=torch.float64, device=self.dev)
            self.sums = torch.zeros(world * 2, dtype=torch.float64, device=self.dev)
            self.x0 = torch.empty(self.n, dtype=torch.float64, device=self.dev)
            self.x = torch.empty(self.n, dtype=torch.float64, device=self.dev)
        p = W._f64(P.p, op.n, "preconditioner")
        w = W._f64(weights, op.n, "weights")
        for s in self.shards:
            _check(lib.wbx_shard_bind(s.h, C.c_void_p(self.y.data_ptr()), C.c_void_p(self.res.data_ptr()),
                                      C.c_void_p(self.u.data_ptr()), C.c_void_p(self.t.data_ptr())))
            _check(lib.wbx_shard_setup(s.h, W._dptr(p), W._dptr(w), float(lambda_), self.iters, int(accelerate)))
            _check(lib.wbx_shard_bind_power(s.h, C.c_void_p(self.sums.data_ptr())))
        self.basis_h = basis.device(ctx)
        self.tau_iters = 0

    # ---- estimate_step (solver.cpp:69-99): device-resident power iteration. Each step is
    # enqueued blindly; the device applies the stopping rule and turns the remaining steps
    # into no-ops, so the host waits only once, for the result.
    def estimate_step(self, step_safety: float = 1.01) -> float:
        """tau as the single-GPU fp32 solver computes it: the reference's power-iteration
        estimate (solver.cpp:69-99) by Lanczos (WBX_TAU=power: the literal power iteration)."""
        if os.environ.get("WBX_TAU") == "power":
            return self._estimate_step_power(step_safety)
        first = int(os.environ.get("WBX_LZ_FIRST", 60))
        every = int(os.environ.get("WBX_LZ_EVERY", 4))
        gap = int(os.environ.get("WBX_LZ_GAP", 4))
        for s in self.shards:
            _check(lib.wbx_shard_lz_begin(s.h))
        self.exchange.gather(self.sums, None)
        for s in self.shards:
            _check(lib.wbx_shard_lz_update(s.h, 0, first, every, gap))
        self.exchange.gather(self.u, None)
        done = C.c_int(0)
        for j in range(1, 201):
            for s in self.shards:
                _check(lib.wbx_shard_lz_step_a(s.h))
            self.exchange.gather(self.t, None)
            self.exchange.gather(self.sums, None)
            for s in self.shards:
                _check(lib.wbx_shard_lz_update(s.h, 1, first, every, gap))
            for s in self.shards:
                _check(lib.wbx_shard_lz_step_t(s.h))
            self.exchange.gather(self.sums, None)
            self.exchange.gather(self.u, None)
            for s in self.shards:
                _check(lib.wbx_shard_lz_update(s.h, 2, first, every, gap))
            if j == 200 or (j >= first and (j - first) % every == 0) or j == 1:
                _check(lib.wbx_shard_lz_done(self.shards[0].h, C.byref(done)))  # a check ran (or breakdown)
                if done.value:
                    break
        tau, iters, steps = C.c_double(), C.c_uint32(), C.c_uint32()
        _check(lib.wbx_shard_lz_result(self.shards[0].h, float(step_safety), C.byref(tau), C.byref(iters),
                                       C.byref(steps)))
        self.tau_iters = int(iters.value)
        self.tau_steps = int(steps.value)
        return float(tau.value)

    def _estimate_step_power(self, step_safety: float) -> float:
        for s in self.shards:
            _check(lib.wbx_shard_power_begin(s.h))
        self.exchange.gather(self.sums, None)
        for s in self.shards:
            _check(lib.wbx_shard_power_update(s.h, 1))
        self.exchange.gather(self.u, None)
        for _ in range(200):
            for s in self.shards:
                _check(lib.wbx_shard_power_step_a(s.h))
            self.exchange.gather(self.t, None)
            for s in self.shards:
                _check(lib.wbx_shard_power_step_t(s.h))
            self.exchange.gather(self.sums, None)
            for s in self.shards:
                _check(lib.wbx_shard_power_update(s.h, 0))
            self.exchange.gather(self.u, None)
        tau, iters = C.c_double(), C.c_uint32()
        _check(lib.wbx_shard_power_result(self.shards[0].h, float(step_safety), C.byref(tau), C.byref(iters)))
        self.tau_iters = int(iters.value)
        return float(tau.value)

    def deblur_dev(self, u0_ptr: int, u_ptr: int, tau: Optional[float] = None, clamp: bool = True) -> float:
        torch = self.torch
        _check(lib.wbx_analyze_dev(self.ctx.handle, self.basis_h, C.c_void_p(u0_ptr), C.c_void_p(self.x0.data_ptr())))
        if tau is None:
            tau = self.estimate_step()
        with torch.cuda.stream(self.stream):
            self.x.zero_()
        for s in self.shards:
            _check(lib.wbx_shard_init(s.h, float(tau), C.c_void_p(self.x0.data_ptr()), C.c_void_p(self.x.data_ptr())))
        self.exchange.gather(self.y, None)
        for k in range(1, self.iters + 1):
            for s in self.shards:
                _check(lib.wbx_shard_phase_a(s.h))
            self.exchange.gather(self.res, None)
            for s in self.shards:
                _check(lib.wbx_shard_phase_t(s.h, k))
            self.exchange.gather(self.y, None)
        for s in self.shards:
            _check(lib.wbx_shard_finalize(s.h, C.c_void_p(self.x.data_ptr())))
        self.exchange.allreduce_sum_(self.x)  # disjoint pieces: exact (a + 0 == a)
        _check(lib.wbx_synthesize_dev(self.ctx.handle, self.basis_h, C.c_void_p(self.x.data_ptr()), C.c_void_p(u_ptr)))
        if clamp:
            with torch.cuda.stream(self.stream):
                out = torch.as_tensor(_DevArray(u_ptr, self.n), device=self.dev)
                out.clamp_(0.0, 1.0)
        return tau


class _DevArray:
    """Zero-copy view of a device fp64 buffer for torch (CUDA array interface)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                         "strides": None}
