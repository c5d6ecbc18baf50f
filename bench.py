#!/usr/bin/env python3
"""bench.py — ms per 1024^2 deblur (100 preconditioned FISTA iterations) on B200.

Workload (BASELINE.json configs[1], "C2"): 1024x1024 synthetic scene, stationary
Gaussian blur sigma=5, noise 5e-3 (seed 2024), Daubechies-4 wavelets J=4, Theta_K with
K = 3N by the reference's dyadic-weighted global top-K (operator = the reference's own
threshold output, tests/golden/c2_db4_1024.npz, expanded to CSR), SPAI preconditioner,
lambda = 1e-4, 100 FISTA iterations. One step = one deblur: u0 -> analyze -> tau
(estimate_step, inside the step as in the reference's fista()) -> 100 FISTA iterations ->
synthesize -> clamp. fp32 hot path (fp64 DWT and tau).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--gpus N > 1 without torchrun re-executes itself under torch.distributed.run (one rank per
GPU, NCCL). Each rank deblurs its own image every step (weak scaling, no collective on the
data path); value = max-over-ranks device time / images. The C5 batch (64 images split over
the N ranks, batches of 8 per SpMM launch) is reported beside it at every N.

--impl reference: the reference's own CPU implementation (oracle/_ref/oracle_driver linked
against the unmodified reference library built from /root/reference; all host threads) on the
same workload and config. It imports nothing from this repository's package.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "ms per 1024² deblur (100 precond. FISTA iters); Θx SpMV HBM GB/s vs peak"
DIMS = (1024, 1024)
ITERS = 100
GOLDEN = ROOT / "tests" / "golden" / "c2_db4_1024.npz"
L2_FLUSH_BYTES = 512 << 20   # > 126 MB L2: written between timed steps
C5_IMAGES = 64


def bench_config(world: int) -> dict:
    """The `config` object of BOTH arms (identical dicts: the driver compares them)."""
    z = np.load(GOLDEN)
    return {"workload": "C2: 1024x1024 stationary Gaussian sigma=5 deblur, db4 J=4, K=3N dyadic top-K, SPAI, "
                        "lambda=1e-4, 100 FISTA iters incl. tau (estimate_step)",
            "image": list(DIMS), "iters": ITERS, "K_over_N": 3, "nnz": int(np.sum(z["gen_count"])),
            "images_per_step": world, "parallelism": f"dp{world}: independent images, one per rank",
            "l2": "flushed (512 MiB write) between timed steps"}


def load_traffic():
    """DRAM bytes per launch of the solver kernels from the committed ncu --set full capture
    (profiles/traffic.json, written by tools/ncu_traffic.py), or None."""
    p = ROOT / "profiles" / "traffic.json"
    try:
        return json.loads(p.read_text())
    except (OSError, ValueError):
        return None


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region (NVML, else nvidia-smi)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._ready = threading.Event()   # set after the first sample (NVML init is slow)
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        try:  # NVML: millisecond sampling, enough samples even for a ~100 ms timed region
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            bits = (0x8, 0x40, 0x20, 0x4)  # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
            while True:  # at least one sample, and one more after the timed region ends
                stop = self._stop.is_set()
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = get_reasons(h)
                self.samples.append([str(self.device), str(sm), str(mx), ""] +
                                    ["Active" if r & b else "Not Active" for b in bits])
                self._ready.set()
                if stop:
                    return
                self._stop.wait(0.002)
        except Exception:
            pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._ready.set()
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        self._ready.wait(timeout=30)  # sampling is live before the timed region starts
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[4 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------------------------- reference arm
def reference_deblur_times(reps: int, warmup: int, threads=None) -> dict:
    """The reference's own deblur unit (analyze + fista incl. estimate_step + synthesize) timed
    by oracle/_ref/oracle_driver, which links the UNMODIFIED reference library built from
    /root/reference (oracle/Makefile). The operator is the reference's C2 threshold output
    (generator groups from the golden fixture, expanded by the reference's walk); the observed
    image is the reference's own degrade(). Imports nothing from the repo's package."""
    drv = ROOT / "oracle" / "_ref" / "oracle_driver"
    if not drv.exists():
        raise RuntimeError("oracle/_ref/oracle_driver missing (build() compiles it where /root/reference exists)")
    z = np.load(GOLDEN)
    rec = np.zeros(z["gen_block"].size, dtype=[("b", "<u4"), ("i", "<u4"), ("c", "<u8"), ("v", "<f8")])
    rec["b"], rec["i"], rec["c"], rec["v"] = z["gen_block"], z["gen_index"], z["gen_count"], z["gen_value"]
    env = dict(os.environ)
    if threads:
        env["OMP_NUM_THREADS"] = str(threads)
    with tempfile.TemporaryDirectory() as td:
        rec.tofile(Path(td) / "gens.bin")
        r = subprocess.run([str(drv), "--out", td, "--dims", str(DIMS[0]), str(DIMS[1]), "--iters", str(ITERS),
                            "--gens", str(Path(td) / "gens.bin"), "--bench-reps", str(reps),
                            "--bench-warmup", str(warmup)], capture_output=True, text=True, env=env)
        if r.returncode != 0:
            raise RuntimeError(r.stderr[-2000:])
        meta = json.loads((Path(td) / "meta.json").read_text())
    times = meta["bench_deblur_s"]
    return {"ms": 1e3 * float(np.mean(times)), "per_rep_s": times, "threads": int(meta.get("omp_threads", 1)),
            "tau": meta.get("tau"), "psnr_restored_db": meta.get("psnr_restored_db"),
            "fista_wall_time_s": meta.get("fista_wall_time_s")}


def cpu_baseline_obj(multi: dict, single=None) -> dict:
    cb = {"value": round(multi["ms"], 1), "unit": "ms", "cores": multi["threads"], "kind": "reference",
          "sample": f"{len(multi['per_rep_s'])} full deblur(s) of the workload: analyze + fista (incl. "
                    f"estimate_step) + synthesize, 1024^2, {ITERS} iters, the unmodified reference built from "
                    f"/root/reference (oracle/_ref), OpenMP over {multi['threads']} threads",
          "cpu_model": cpu_model(), "nproc": os.cpu_count()}
    if single is not None:
        cb["value_1_thread"] = round(single["ms"], 1)
    return cb


def run_reference(args, world: int) -> dict:
    reps = max(1, min(args.steps, 20))
    multi = reference_deblur_times(reps, min(args.warmup, 3))
    single = None
    if not args.no_single_thread:
        try:
            single = reference_deblur_times(1, 0, threads=1)
        except Exception:
            pass
    cb = cpu_baseline_obj(multi, single)
    return {"metric": METRIC, "value": cb["value"], "unit": "ms", "n_gpus": world, "steps": reps,
            "warmup": args.warmup, "ms_per_step": cb["value"], "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": bench_config(world), "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ----------------------------------------------------------------------------- our arm
def make_inputs():
    from paper_1512_08401_b200 import synthetic as S
    from paper_1512_08401_b200 import waveblur as W
    z = np.load(GOLDEN)
    gl = W.GeneratorList(DIMS, 4, W.FilterFamily.Daubechies, 4, z["gen_block"].astype(np.uint32),
                         z["gen_index"].astype(np.uint32), z["gen_count"].astype(np.uint64), z["gen_value"])
    op = W.theta_from_generators(gl)
    basis = W.make_basis(W.FilterFamily.Daubechies, 4, DIMS, 4)
    _, u0 = S.degrade(DIMS, 5.0, 5e-3, 2024)
    return op, basis, u0


def _max_over_ranks(v: float, world: int, dev) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_ours(args, rank, world, local_rank):
    import torch
    from paper_1512_08401_b200 import waveblur as W

    torch.cuda.set_device(local_rank)
    op, basis, u0 = make_inputs()
    ctx = W.Context(local_rank)
    P = W.spai(op, ctx)
    w = W.scale_weights(basis.layout)
    cfg = W.SolverConfig(max_iters=ITERS, track_energy=False, precision=32)
    deb = W.Deblurrer(op, basis, P, w, 1e-4, cfg, ctx)
    info = op.info(ctx)
    n = op.n
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    with torch.cuda.stream(stream):
        u0_dev = torch.from_numpy(u0.ravel().copy()).to(dev)
        out_dev = torch.empty(n, dtype=torch.float64, device=dev)
        flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    torch.cuda.synchronize(dev)

    def step():
        deb.deblur_dev(u0_dev.data_ptr(), out_dev.data_ptr(), clamp=True)

    for _ in range(args.warmup):
        with torch.cuda.stream(stream):
            flush.zero_()
        step()
    torch.cuda.synchronize(dev)

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    solve_ms, phase_ms = [], []
    launches0 = ctx.launches
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local_rank) as clk:
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()   # L2 flush between timed steps (outside the events)
                starts[i].record(stream)
            step()
            with torch.cuda.stream(stream):
                ends[i].record(stream)
            ends[i].synchronize()
            solve_ms.append(deb.last_stats()[1])
            phase_ms.append(deb.phase_ms())
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    launches = (ctx.launches - launches0) // args.steps
    per_step = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = _max_over_ranks(float(sum(per_step)), world, dev)
    ms_per_step = total_ms / args.steps
    value = ms_per_step / world   # whole job: `world` images per step

    # e2e through the public API with HOST buffers (H2D of u0 and D2H of the restored image
    # inside the timed region), pinned memory
    u0_pin = torch.from_numpy(u0.ravel().copy()).pin_memory()
    out_pin = torch.empty(n, dtype=torch.float64).pin_memory()
    u0_np, out_np = u0_pin.numpy(), out_pin.numpy()
    for _ in range(max(1, args.warmup)):
        deb.deblur(u0_np, clamp=True, out=out_np)
    e2e = []
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        _, rep = deb.deblur(u0_np, clamp=True, out=out_np)
        e2e.append((time.perf_counter() - t0) * 1e3)
    e2e_ms = _max_over_ranks(float(np.mean(e2e)), world, dev)

    tau_kernel, it_kernel = deb.kernels()
    tau_iters = int(rep.tau_iters)
    _, _, tau_pairs = deb.tau_stats()  # operator product pairs actually spent (Lanczos steps)
    s_ms = float(np.median(solve_ms))
    tau_ms = float(np.mean([p[0] for p in phase_ms]))
    it_ms = float(np.mean([p[1] for p in phase_ms]))
    peak, peak_src = load_peaks()
    nnz, nR, nC = int(info.nnz), int(info.nonempty_rows), int(info.nonempty_cols)
    # Algorithmic bytes per unit, two models:
    #  * SURVEY 8(d) dense model: fp32 values + u32 indices, dense n-vectors read/written once
    #  * compacted model: what the kernel must move in the compacted spaces (coordinates with an
    #    empty Theta column are iterated in registers by the decoupled pass, outside these bytes)
    b_iter = 16 * nnz + 36 * n
    b_iter_c = 16 * nnz + 12 * nR + 28 * nC
    b_pair = 2 * (8 * nnz + 16 * n)             # one operator product pair, fp64 dense vectors
    b_pair_c = 16 * nnz + 12 * nR + 16 * nC     # fp32 compacted: Θ, Θᵀ, u/t windows, own state
    if tau_kernel.startswith("circ_"):  # block-Fourier estimate: no full-operator products
        tau_entry = {"kernel": "circ_* (estimate_step, block-Fourier: 7 launches)", "launch_ms": round(tau_ms, 4),
                     "units": f"the reference's {tau_iters} power iterations as 2050 independent 12x12 Fourier-block "
                              "iterations (Lanczos to tridiagonal + power steps, fp64)",
                     "bound": "latency (fp64 dependent chains, <1 wave); reads the 38 representative rows of "
                              "Theta, not the operator",
                     "algorithmic_bytes": 0, "dense_model_bytes": 0,
                     "reference_equivalent_bytes": tau_iters * b_pair}
    else:
        tau_entry = {"kernel": f"{tau_kernel} (estimate_step, persistent)", "launch_ms": round(tau_ms, 4),
                     "units": f"{tau_pairs} operator product pairs (Lanczos steps standing in for the reference's "
                              f"{tau_iters} power iterations)",
                     "algorithmic_bytes": tau_pairs * b_pair_c, "dense_model_bytes": tau_pairs * b_pair}
    kernels = [
        tau_entry,
        {"kernel": f"{it_kernel} ({ITERS} FISTA iterations, persistent)", "launch_ms": round(it_ms, 4),
         "units": f"{ITERS} iterations", "algorithmic_bytes": ITERS * b_iter_c, "dense_model_bytes": ITERS * b_iter},
    ]
    spectral = it_kernel == "circ_fista_kernel"
    if spectral:
        # the spectral engine moves no operator stream: per iteration two exchanges of the row /
        # column transforms (T1, T2: written once, read once, nCo x NG complex fp64 each), plus the
        # decoupled coordinates (x0, w, p read, x written: fp64) and the G_f blocks once per launch
        n_co, ng = 12, (1024 >> 4) ** 2
        own = ITERS * 4 * n_co * ng * 16 + 32 * n + 2050 * n_co * n_co * 16
        kernels[1]["algorithmic_bytes"] = ITERS * b_iter  # SURVEY 8(d) per-iteration figure (work-equivalent)
        kernels[1]["kernel_bytes"] = own
        kernels[1]["kernel_bytes_model"] = ("per iteration 4 x nCo x NG x 16 B (T1/T2 written + read), + 32 n "
                                            "(decoupled coordinates) + the G_f blocks once")
    for k in kernels:
        if "kernel_bytes" in k:
            k["kernel_bytes_achieved"] = round(k["kernel_bytes"] / (k["launch_ms"] * 1e-3) / 1e9, 1)
            k["kernel_bytes_frac"] = round(k["kernel_bytes_achieved"] / peak, 4)
        k["achieved"] = round(k["algorithmic_bytes"] / (k["launch_ms"] * 1e-3) / 1e9, 1)
        k["frac"] = round(k["achieved"] / peak, 4)
        k["dense_model_achieved"] = round(k["dense_model_bytes"] / (k["launch_ms"] * 1e-3) / 1e9, 1)
        k["dense_model_frac"] = round(k["dense_model_achieved"] / peak, 4)
    dom = max(kernels, key=lambda k: k["launch_ms"])
    traffic = load_traffic()
    result = {
        "metric": METRIC, "value": round(value, 4), "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64" if spectral else "f32 (fp64 DWT/tau)", "data": "synthetic",
        "config": bench_config(world),
        "e2e": {"value": round(e2e_ms / world, 4), "unit": "ms",
                "median_ms": round(float(np.median(e2e)) / world, 4), "min_ms": round(float(np.min(e2e)) / world, 4),
                "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": 8 * n, "api": "wbx_deblur (host fp64 image in/out, pinned)"},
        "gpu_launches": int(launches),
        "roofline": roofline_of(dom, kernels, peak, peak_src, traffic, spectral),
        "breakdown": {"solve_ms": round(s_ms, 4), "tau_ms": round(tau_ms, 4), "iterations_ms": round(it_ms, 4),
                      "tau_iters": tau_iters, "tau_product_pairs": tau_pairs, "tau": rep.tau,
                      "dwt_and_idwt_ms": round(ms_per_step - s_ms, 4), "kernels": [tau_kernel, it_kernel]},
        "clocks": clk.summary(),
    }
    result["c5_batch"] = run_c5(W, torch, ctx, stream, dev, op, basis, P, w, flush, rank, world)
    if not args.no_extra and world == 1:
        result["extra_workloads"] = extra_workloads(W, torch, ctx, stream, dev, op, basis, P, w, u0, rep.tau, flush)
        # second half of the metric: the Theta x SpMV alone against the HBM roofline, on the C2
        # operator carried to 4096^2 (403 MB operator stream > L2; profiles/r02_spmv_roofline.md)
        import importlib.util
        spec = importlib.util.spec_from_file_location("spmv_roofline", ROOT / "tools" / "spmv_roofline.py")
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        result["spmv_roofline"] = mod.measure(4096, 10)
    return result


def roofline_of(dom, kernels, peak, peak_src, traffic, spectral):
    """The bench line's `roofline` object for the dominant kernel."""
    r = {"bound": "hbm", "kernel": dom["kernel"], "achieved": dom["achieved"], "peak": peak, "unit": "GB/s",
         "frac": dom["frac"], "traffic": traffic.get(dom["kernel"].split()[0]) if traffic else None,
         "traffic_source": traffic.get("source") if traffic else None, "peak_source": peak_src,
         "algorithmic_bytes_per_launch": dom["algorithmic_bytes"], "launch_ms": dom["launch_ms"], "kernels": kernels}
    if spectral and "kernel_bytes" in dom:  # (under a profiler the estimate can time as the dominant kernel)
        r["bytes_model"] = ("SURVEY 8(d): per iteration 16*nnz + 36*n -- work-equivalent: the spectral engine "
                            "applies Theta^T Theta as Fourier blocks and streams no operator, so frac > 1 is the "
                            "algorithm beating the SpMV formulation's HBM bound, not a measured bandwidth")
        r["kernel_bytes"] = {"bytes_per_launch": dom["kernel_bytes"], "achieved": dom["kernel_bytes_achieved"],
                             "frac": dom["kernel_bytes_frac"], "model": dom["kernel_bytes_model"]}
        r["limiter"] = ("latency: two grid-wide exchanges per iteration (row transforms -> column spectra -> row "
                        "transforms) through L2, each a barrier plus an L2 round trip, and fp64 warp FFTs; the "
                        "HBM-streamed Theta x SpMV is measured separately (`spmv_roofline`)")
    else:
        r["bytes_model"] = ("compacted: per iteration 16*nnz + 12*|R| + 28*|C| (Θ and Θᵀ streams, x0/res on R, "
                            "y gather + y/x_prev/τ/p/threshold state on C)")
        r["dense_model"] = {"bytes_per_launch": dom["dense_model_bytes"], "achieved": dom["dense_model_achieved"],
                            "frac": dom["dense_model_frac"], "model": "SURVEY 8(d): per iteration 16*nnz + 36*n"}
        r["limiter"] = ("grid-barrier and gather latency: the operator (dictionary-coded, ~2.7 B/nonzero) and "
                        "vectors stay L2-resident across iterations; HBM sees one cold read (`traffic`). The "
                        "HBM-streamed SpMV is measured separately (`spmv_roofline`).")
    return r


def _time_dev(deb, torch, stream, flush, u0_dev, out_dev, reps=5):
    for _ in range(2):
        deb.deblur_dev(u0_dev.data_ptr(), out_dev.data_ptr(), clamp=True)
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            flush.zero_()
            a.record(stream)
        deb.deblur_dev(u0_dev.data_ptr(), out_dev.data_ptr(), clamp=True)
        with torch.cuda.stream(stream):
            b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def run_c5(W, torch, ctx, stream, dev, op, basis, P, w, flush, rank, world):
    """BASELINE config C5: 64 independent 1024^2 deblurs split over the `world` ranks (64/world
    per rank, one batched solve per 8 images: for this translation-invariant operator the
    spectral engine, 8 images per launch at 4 per CTA, G_f and tau shared; otherwise the SpMM
    kernel that streams the operator once per 8 right-hand sides), no collective on the data
    path; images/s of the whole job from the max over ranks of the device time (strong scaling
    of the fixed 64-image job)."""
    from paper_1512_08401_b200 import synthetic as S
    B = 8
    per_rank = C5_IMAGES // world
    nb = max(1, per_rank // B)
    n = op.n
    seeds = [rank * per_rank + j for j in range(B)]
    imgs = np.stack([S.degrade(DIMS, 5.0, 5e-3, s)[1] for s in seeds])
    with torch.cuda.stream(stream):
        ub = torch.from_numpy(imgs.reshape(-1).copy()).to(dev)
        ob = torch.empty(B * n, dtype=torch.float64, device=dev)
    db = W.Deblurrer(op, basis, P, w, 1e-4, W.SolverConfig(max_iters=ITERS, track_energy=False), ctx, batch=B)
    for _ in range(2):
        db.deblur_dev(ub.data_ptr(), ob.data_ptr(), clamp=True)
    torch.cuda.synchronize(dev)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        flush.zero_()
        a.record(stream)
    for _ in range(nb):   # the rank's share: nb batches of 8 (inputs resident, L2 flushed once)
        db.deblur_dev(ub.data_ptr(), ob.data_ptr(), clamp=True)
    with torch.cuda.stream(stream):
        b.record(stream)
    b.synchronize()
    ms = _max_over_ranks(a.elapsed_time(b), world, dev)
    kernels = db.kernels()
    del db
    return {"images": nb * B * world, "images_per_rank": nb * B, "batch": B, "ms_job": round(ms, 3),
            "images_per_s": round(1e3 * nb * B * world / ms, 1), "ms_per_image": round(ms / (nb * B * world), 4),
            "tau": "estimated once per batch (inside the timed region)", "scaling": "strong (64-image job)",
            "kernels": list(kernels)}


def extra_workloads(W, torch, ctx, stream, dev, op, basis, P, w, u0, tau, flush):
    """The other BASELINE configs on this GPU (reported beside the headline, same run):
    C2 with tau cached per operator, C2 in the bitwise fp64 reference mode, C3 spatially
    varying, the per-operator setup kernels."""
    out = {}
    n = op.n
    with torch.cuda.stream(stream):
        u0_dev = torch.from_numpy(u0.ravel().copy()).to(dev)
        out_dev = torch.empty(n, dtype=torch.float64, device=dev)
    # C2, tau cached (a deployment estimates tau once per operator, like P)
    d = W.Deblurrer(op, basis, P, w, 1e-4, W.SolverConfig(max_iters=ITERS, track_energy=False, tau=tau), ctx)
    out["c2_tau_cached"] = {"ms_per_deblur": round(_time_dev(d, torch, stream, flush, u0_dev, out_dev), 4)}
    # C2 in the fp64 reference mode (iterates bitwise equal to the reference's, literal power
    # iteration for tau)
    d64 = W.Deblurrer(op, basis, P, w, 1e-4, W.SolverConfig(max_iters=ITERS, track_energy=False, precision=64), ctx)
    out["c2_fp64_bitwise"] = {"ms_per_deblur": round(_time_dev(d64, torch, stream, flush, u0_dev, out_dev, reps=3), 3),
                              "kernels": list(d64.kernels())}
    del d64
    # the reference's own API call fista(problem, P, cfg) with its per-iteration energies (what
    # the drop-in binding forwards: wbx_pgd with track_energy, host fp64 vectors in and out,
    # tau inside), wall time; its iteration kernel
    x0 = W.analyze(u0, basis, ctx).values
    prob = W.DeblurProblem(W.SparseThetaOp(op, ctx), x0, w, 1e-4)
    fcfg = W.SolverConfig(max_iters=ITERS, precision=32, track_energy=True)
    W.fista(prob, P, fcfg, ctx)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        rep = W.fista(prob, P, fcfg, ctx)
        ts.append(1e3 * (time.perf_counter() - t0))
    dt = W.Deblurrer(op, basis, P, w, 1e-4, W.SolverConfig(max_iters=ITERS, track_energy=True), ctx)
    out["c2_fista_api_tracked"] = {"ms_wall": round(float(np.median(ts)), 3), "iters_used": int(rep.iters_used),
                                   "energies": len(rep.energies), "kernels": list(dt.kernels()),
                                   "ms_deblur_dev_tracked": round(_time_dev(dt, torch, stream, flush, u0_dev,
                                                                            out_dev, reps=3), 4),
                                   "api": "waveblur.fista -> wbx_pgd (host fp64 x0/x_final, energies every "
                                          "iteration, tau inside)"}
    del dt
    # C3: 1024^2 spatially varying blur (sigma 2.5 -> 7.5 px down the image)
    lad = W.SigmaLadder.from_npz(np.load(ROOT / "tests" / "golden" / "c3_ladder_1024.npz"))
    opv = W.theta_varying(lad, 2.5, 7.5)
    Pv = W.spai(opv, ctx)
    dv = W.Deblurrer(opv, basis, Pv, w, 1e-4, W.SolverConfig(max_iters=ITERS, track_energy=False), ctx)
    out["c3_varying"] = {"ms_per_deblur": round(_time_dev(dv, torch, stream, flush, u0_dev, out_dev), 4),
                         "nnz": int(opv.nnz()), "kernels": list(dv.kernels()),
                         "note": "u0 = the C2 observation (timing only)"}
    # per-operator setup on the device (outside the timed unit): Theta_K construction
    # (build_theta_conv + weighted top-K, bitwise the reference's) and SPAI
    psf = W.gaussian_psf_kernel(DIMS, 5.0)
    bw = W.dyadic_band_weights(basis.layout)
    W.theta_conv_topk(basis, psf, 3 * n, bw, ctx)
    t0 = time.perf_counter()
    gl = W.theta_conv_topk(basis, psf, 3 * n, bw, ctx)
    t1 = time.perf_counter()
    W.spai(op, ctx)
    t2 = time.perf_counter()
    out["setup_c2"] = {"theta_build_ms": round(1e3 * (t1 - t0), 1), "theta_groups": int(gl.blocks.size),
                       "spai_ms": round(1e3 * (t2 - t1), 1),
                       "note": "wall time incl. host transfers; reference CPU: ~30 s build+threshold, ~0.2 s SPAI"}
    return out


def run_c4(args, rank, world, local_rank):
    """BASELINE config C4: one size^2 spatially varying deblur (sigma 2.5 -> 7.5 px), Theta_K
    row-sharded over `world` GPUs by the library's sharded solver (wbx_sharded: per-rank phase
    kernels, NCCL all-gathers of the padded y / res slices over NVLink inside libwbx, the FISTA
    iterations as one CUDA graph); strong scaling (total work fixed). At one GPU the same
    engine runs world 1; the single-GPU persistent solver (Deblurrer) is reported beside it."""
    import torch
    from paper_1512_08401_b200 import synthetic as S
    from paper_1512_08401_b200 import waveblur as W
    from paper_1512_08401_b200.sharded import ShardedDeblurrer, nccl_comm
    size = args.size
    dims = (size, size)
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(local_rank)
    t_setup = time.perf_counter()
    lad = W.SigmaLadder.from_npz(np.load(ROOT / "tests" / "golden" / "c3_ladder_1024.npz"))
    if size != 1024:
        lad = W.SigmaLadder(lad.sigmas, [W.rescale_generators(g, dims) for g in lad.levels])
    op = W.theta_varying(lad, 2.5, 7.5)
    ctx = W.Context(local_rank)
    basis = W.make_basis(W.FilterFamily.Daubechies, 4, dims, 4)
    clean = S.synthetic_scene(dims)
    x = W.analyze(clean, basis, ctx).values
    u0 = S.add_noise(W.synthesize(W.spmv(op, x, ctx), basis, ctx), 5e-3, 2024)
    P = W.spai(op, ctx)
    w = W.scale_weights(basis.layout)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    comm = None
    if world > 1:
        import torch.distributed as dist
        comm = nccl_comm(torch, dist, ctx)
    sh = ShardedDeblurrer(ctx, op, basis, P, w, 1e-4, ITERS, world, [rank], comm=comm)
    with torch.cuda.stream(stream):
        u0_dev = torch.from_numpy(u0.ravel().copy()).to(dev)
        out = torch.empty_like(u0_dev)
    setup_s = time.perf_counter() - t_setup

    def timed(fn, steps):
        for _ in range(max(1, args.warmup)):
            fn()
        ctx.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a.record(stream)
        for _ in range(steps):
            fn()
        with torch.cuda.stream(stream):
            b.record(stream)
        b.synchronize()
        return _max_over_ranks(a.elapsed_time(b) / steps, world, dev)

    steps = max(1, min(args.steps, 5))
    ms = timed(lambda: sh.deblur_dev(u0_dev.data_ptr(), out.data_ptr(), clamp=True), steps)
    st = sh.stats()
    restored = out.cpu().numpy().reshape(dims)
    line = {"metric": f"ms per {size}x{size} spatially varying deblur (C4)", "value": round(ms, 3),
            "unit": "ms", "n_gpus": world, "steps": steps, "higher_is_better": False, "scaling": "strong",
            "impl": "ours", "config": {"workload": f"C4: {size}^2 varying Gaussian 2.5->7.5 px, db4 J=4, K~3.4N, "
                                                   f"SPAI, 100 FISTA iters incl. tau", "nnz": int(op.nnz()),
                                       "parallelism": f"Theta row-sharded x{world} (wbx_sharded, NCCL inside libwbx)"},
            "breakdown": st, "setup_s": round(setup_s, 1),
            "psnr_observed_db": round(S.psnr(u0, clean), 3), "psnr_restored_db": round(S.psnr(restored, clean), 3)}
    if world == 1:  # the single-GPU persistent solver on the same operator, for comparison
        d = W.Deblurrer(op, basis, P, w, 1e-4, W.SolverConfig(max_iters=ITERS, track_energy=False), ctx)
        line["single_gpu_persistent"] = {
            "ms": round(timed(lambda: d.deblur_dev(u0_dev.data_ptr(), out.data_ptr(), clamp=True), steps), 3),
            "kernels": list(d.kernels())}
    return line


def relaunch_under_torchrun(gpus: int) -> int:
    """`bench.py --gpus N` outside torchrun: re-execute under torch.distributed.run with one
    rank per GPU (the driver's own launch line), rendezvous on 127.0.0.1."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-single-thread", action="store_true", help="reference arm: skip the 1-thread deblur")
    ap.add_argument("--no-extra", action="store_true", help="skip the C3/fp64/setup/SpMV side measurements")
    ap.add_argument("--workload", choices=["c2", "c4"], default="c2",
                    help="c4: one 4096^2 spatially varying deblur row-sharded over the --gpus ranks")
    ap.add_argument("--size", type=int, default=4096, help="image side for --workload c4")
    ap.add_argument("--backend", default="nccl", help="torch.distributed backend (gloo: CPU tests of the launch)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, world)), flush=True)
        return

    if world > 1:
        import torch
        import torch.distributed as dist
        if args.backend == "nccl":
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(args.backend)
    if args.workload == "c4":
        line = run_c4(args, rank, world, local_rank)
        if rank == 0:
            print(json.dumps(line), flush=True)
    else:
        result = run_ours(args, rank, world, local_rank)
        if rank == 0:
            if not args.no_cpu_baseline:
                try:
                    result["cpu_baseline"] = cpu_baseline_obj(reference_deblur_times(1, 0))
                except Exception as e:  # reported, never fatal
                    result["cpu_baseline"] = {"value": None, "unit": "ms", "cores": None, "kind": None,
                                              "sample": f"failed: {e}"}
            print(json.dumps(result), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
