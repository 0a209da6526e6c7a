#!/usr/bin/env python
"""Benchmark of the 3D-FSR reconstruction hot path on B200.

Headline workload (BASELINE.json configs[1]): closed-form Tikhonov SR, fp64,
HR 256^3 ellipsoid+texture phantom, Gaussian PSF sigma 1.5 / 13^3, decimation
2x2x2 -> LR 128^3, 30 dB BSNR, tau (TikhonovConfig::lambda) = 1e-3.
One step = one TikhonovOperator::solve (reference src/solvers.cpp:48-67).

  value : HR voxels/s, inputs resident in HBM (device-pointer C ABI).
  e2e   : same metric through the public host-buffer C ABI
          (vsr_tikhonov_solve: pinned y H2D + solve + x D2H + checks).
  tv    : ADMM-TV iteration throughput on configs[2] (256^3, d = 64), extra.

Run: python bench.py [--gpus N --steps K --warmup W] [--impl reference]
For N > 1 (torchrun) every rank solves its own config-1 volume (replicas,
weak scaling) for the headline; the `sharded` / `sharded_config4` blocks time
configs 3 and 4 slab-sharded over all N GPUs (strong scaling).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "HR voxels/s per ADMM-TV iteration and per Tikhonov solve; % of HBM roofline"
UNIT = "HR voxels/s"


def load_peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, phys_index: int):
        self.idx = phys_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.idx)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sms, maxs, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sms.append(float(f[1]))
                maxs.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sms)) if sms else None,
                "sm_max_mhz": max(maxs) if maxs else None,
                "reasons": sorted(reasons), "samples": len(sms)}


def phys_gpu_index(local: int) -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        try:
            return int(vis.split(",")[local])
        except Exception:
            return local
    return local


# ---------------------------------------------------------------- CPU baseline
def host_threads() -> int:
    """Host threads the CPU legs use: every core this process may run on.  The
    reference itself is single-threaded (FFTW without threads, no OpenMP); what
    is threaded is the FFTW-API shim's transforms (VSR_SHIM_THREADS), the
    part a real FFTW build would also run faster."""
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except Exception:
        return max(1, os.cpu_count() or 1)


def cpu_baseline(cfg, inp, budget_s: float = 25.0):
    """Reference CPU path on a bounded sample of the same workload: the
    reference compiled from its sources (oracle/_ref, FFTW-API shim) when
    built, else the numpy oracle port.  The reference is single-threaded (FFTW
    without threads, no OpenMP); the shim's FFTs use every host thread
    (host_threads())."""
    sys.path.insert(0, str(ROOT / "oracle"))
    ref = None
    try:
        import ref_binding  # noqa
        if ref_binding.available():
            ref = ref_binding
    except Exception:
        ref = None
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    N = cfg.voxels
    threads = host_threads()
    if ref is not None:
        os.environ["VSR_SHIM_THREADS"] = str(threads)
        op = ref.TikhonovOperator(inp.psf, cfg.hr, cfg.rates, cfg.reg, inp.xbar)
        times = []
        t_start = time.perf_counter()
        while not times or (time.perf_counter() - t_start < budget_s and len(times) < 3):
            t0 = time.perf_counter()
            op.solve(inp.y)
            times.append(time.perf_counter() - t0)
        kind, sample = "reference", (f"reference volsr TikhonovOperator::solve (oracle/_ref, FFTW3-API shim), "
                                     f"config1 256^3, {len(times)} solves, best; the shim's FFTs (a radix-2 "
                                     f"row-column transform, slower per core than real FFTW) run on {threads} "
                                     f"threads, every other pass single-threaded as in the reference")
    else:
        threads = 1
        import volsr_oracle as O
        spec = O.DecimationSpec(cfg.hr, cfg.rates)
        op = O.TikhonovOperator(O.psf_to_spectrum(inp.psf), spec, cfg.reg, inp.xbar)
        times = []
        t_start = time.perf_counter()
        while not times or (time.perf_counter() - t_start < budget_s and len(times) < 3):
            t0 = time.perf_counter()
            op.solve(inp.y)
            times.append(time.perf_counter() - t0)
        kind, sample = "port", (f"numpy oracle TikhonovOperator.solve, config1 256^3, {len(times)} solves, best")
    best = min(times)
    return {"value": N / best, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample,
            "seconds_per_solve": best}


# ---------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return 0
    from paper_2010_15491_b200 import synth
    cfg = synth.CONFIGS[1]
    inp = synth.make_inputs(cfg, with_truth=False)
    sys.path.insert(0, str(ROOT / "oracle"))
    ref = None
    try:
        import ref_binding
        if ref_binding.available():
            ref = ref_binding
    except Exception:
        ref = None
    threads = host_threads()
    if ref is not None:
        os.environ["VSR_SHIM_THREADS"] = str(threads)
        op = ref.TikhonovOperator(inp.psf, cfg.hr, cfg.rates, cfg.reg, inp.xbar)
        kind = "reference"
        sample = (f"reference volsr TikhonovOperator::solve (oracle/_ref, FFTW3-API shim), config1; the shim's "
                  f"FFTs (radix-2 row-column, slower per core than real FFTW) on {threads} threads, every other "
                  f"pass single-threaded as in the reference")
    else:
        threads = 1
        import volsr_oracle as O
        spec = O.DecimationSpec(cfg.hr, cfg.rates)
        op = O.TikhonovOperator(O.psf_to_spectrum(inp.psf), spec, cfg.reg, inp.xbar)
        kind = "port"
        sample = "numpy oracle TikhonovOperator.solve, config1, 1 thread"
    for _ in range(args.warmup):
        op.solve(inp.y)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        op.solve(inp.y)
    dt = (time.perf_counter() - t0) / args.steps
    val = cfg.voxels / dt
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded ellipsoid+texture phantom, BSNR 30 dB)",
            "config": config_block(cfg),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def config_block(cfg):
    return {"workload": f"config{cfg.idx}: closed-form Tikhonov SR fp64, HR {cfg.hr[0]}x{cfg.hr[1]}x{cfg.hr[2]}"
                        f" -> LR {cfg.lr[0]}x{cfg.lr[1]}x{cfg.lr[2]} (d={cfg.d}), PSF sigma {cfg.psf_sigma[0]}"
                        f" {cfg.psf_size[0]}^3, BSNR {cfg.bsnr:g} dB, tau={cfg.reg:g}",
            "hr": list(cfg.hr), "rates": list(cfg.rates), "step": "TikhonovOperator::solve",
            "l2": "L2 flushed between timed solves (256 MB write, outside the per-solve CUDA events)"}


# ---------------------------------------------------------------- B200 arm
STAGE_BYTES = {
    # algorithmic bytes per launch as multiples of (N, Nl): read + write of the stage
    "fft_inv_axis3": (32, 0), "fft_inv_axis2": (32, 0), "fft_inv_axis1_c2r": (24, 0),
    "fft_fwd_axis1_r2c": (24, 0), "fft_fwd_axis2": (32, 0), "fft_fwd_axis3": (32, 0),
    "tik_fold": (48, 16), "tv_fold": (48, 16), "tv_stencil": (64, 0),
    # fused kernels: Lambda (+ X̄ or W) in, spectrum out (+ LR spectrum of y)
    "tik_fold_ifft_axis3": (48, 16), "tv_fft3_fold_ifft3": (48, 16),
    "tik_fold_ifft_axis1": (48, 16), "tv_fft1_fold_ifft1": (48, 16),
    "fft_inv_axis3_c2r": (24, 0), "fft_fwd_axis3_r2c": (24, 0),
    # TV on the Hermitian half spectrum along axis 3 (planes 0..s/2)
    "fft_fwd_axis3_r2c_half": (16, 0), "fft_fwd_axis2_half": (16, 0), "tv_fft1_fold_ifft1_half": (32, 16),
    "fft_inv_axis2_half": (16, 0), "fft_inv_axis3_c2r_half": (16, 0),
    # spatial-expansion Tikhonov: LR transforms (r2c 24 + 2 x 32), LR pointwise
    # U (Yl, Zl in, U out), expansion (x out, u and decimate(xbar) in)
    "lr_fft3": (0, 88), "lr_ifft3": (0, 88), "spatial_u": (0, 48), "spatial_expand": (8, 16),
    # fused LR stage: r2c + axis 2 forward, axis-3 sandwich (Y, Zl in, Y out), inverse axis 2, c2r
    "lr_fft12": (0, 56), "lr_sandwich_axis3": (0, 48), "lr_ifft_axis2": (0, 32), "lr_ifft_axis1_c2r": (0, 24),
    # half-spectrum LR stage (pitch ~ ml/2 + 8 complex per row: ~9 bytes per LR point per complex pass)
    "lr_r2c_axis1": (0, 17), "lr_fft_axis2_half": (0, 18), "lr_filter_axis3_half": (0, 18),
    "lr_ifft_axis2_half": (0, 18), "lr_c2r_axis1": (0, 25),
}


# fused fold stages that read the 16N-byte HR Lambda unless it is separable
SEP_STAGES = {"tik_fold_ifft_axis3", "tv_fft3_fold_ifft3", "tik_fold_ifft_axis1", "tv_fft1_fold_ifft1",
              "tv_fft1_fold_ifft1_half"}


def _guarded(fn):
    """A side block that fails reports its error instead of losing the headline line."""
    try:
        return fn()
    except Exception as e:  # noqa: BLE001
        return {"error": f"{type(e).__name__}: {e}"[:400]}


def run_b200(args, rank, world, local):
    import torch
    from paper_2010_15491_b200 import synth
    from paper_2010_15491_b200 import volsr as V

    dist = world > 1
    if dist:
        import torch.distributed as tdist
    torch.cuda.set_device(local)
    cfg = synth.CONFIGS[1]
    inp = synth.make_inputs(cfg, with_truth=False)
    N, Nl = cfg.voxels, cfg.voxels // cfg.d
    ctx = V.Context(local)
    spec = V.DecimationSpec(cfg.hr, cfg.rates)
    lam = V.psf_to_spectrum(inp.psf, ctx)
    lam_d = V.DeviceBuffer(ctx, lam.nbytes)
    lam_d.upload(lam)
    xbar_d = V.DeviceBuffer(ctx, inp.xbar.nbytes)
    xbar_d.upload(inp.xbar)
    y_d = V.DeviceBuffer(ctx, inp.y.nbytes)
    y_d.upload(inp.y)
    x_d = V.DeviceBuffer(ctx, N * 8)
    op = V.TikhonovDevice(ctx, spec, lam_d, cfg.reg, xbar_d)
    stream = torch.cuda.ExternalStream(ctx.stream(), device=local)

    def barrier():
        if dist:
            tdist.barrier()

    for _ in range(max(args.warmup, 3)):
        op.solve_d(y_d, x_d)
    op.check()

    clocks = ClockSampler(phys_gpu_index(local))
    clocks.start()
    # keep the GPU under load long enough for the sampler (untimed)
    t_burn = time.perf_counter()
    while time.perf_counter() - t_burn < 1.5:
        for _ in range(20):
            op.solve_d(y_d, x_d)
        ctx.synchronize()

    # ---- timed region (device-resident).  Each solve is bracketed by its own
    # CUDA events on the library stream; a 256 MB write between solves (outside
    # the events) evicts L2 so no solve reads the previous one's data from L2.
    flush = torch.empty(32 << 20, dtype=torch.float64, device=f"cuda:{local}")
    def timed_solves(profile):
        barrier()
        torch.cuda.synchronize()
        ctx.synchronize()
        V.profile_enable(ctx, profile)
        l0 = V.launch_count()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(float(i))
            evs[i][0].record(stream)
            op.solve_d(y_d, x_d)
            evs[i][1].record(stream)
        evs[-1][1].synchronize()
        n_launch = V.launch_count() - l0
        st_ = V.profile_read(ctx) if profile else {}
        V.profile_enable(ctx, False)
        op.check()
        ctx.synchronize()
        torch.cuda.synchronize()
        barrier()
        return sum(a.elapsed_time(b) for a, b in evs) / args.steps, n_launch, st_

    # headline: the user path (CUDA-graph replay of the solve, no profiler)
    ms, launches, _ = timed_solves(False)
    clk = clocks.stop()
    # stage breakdown: a second pass with the library's per-stage event profiler
    ms_prof, _, stages = timed_solves(True)
    if dist:
        t = torch.tensor([ms], device=f"cuda:{local}", dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        ms = float(t.item())
    value = N * world / (ms * 1e-3)

    # ---- end to end through the host-buffer C ABI (pinned buffers)
    yp = V.PinnedBuffer(inp.y.shape)
    yp.array[...] = inp.y
    xp = V.PinnedBuffer(V.shape_of(cfg.hr))
    for _ in range(2):
        op.solve_host(yp.array, xp.array)
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        op.solve_host(yp.array, xp.array)
    e2e_s = (time.perf_counter() - t0) / args.steps
    if dist:
        t = torch.tensor([e2e_s], device=f"cuda:{local}", dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": N * world / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(inp.y.nbytes),
           "d2h_bytes_per_step": int(N * 8), "ms_per_step": e2e_s * 1e3,
           "api": "vsr_tikhonov_solve (pinned host y, x)"}

    # ---- roofline from the live per-stage events
    peaks = load_peaks()
    hbm = peaks.get("hbm_gbs")
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    if not hbm:
        hbm, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    st_rows = {}
    sep = op.separable()
    lat = op.lattice_prior()
    spatial = op.spatial()
    for name, (tot_ms, cnt) in stages.items():
        avg = tot_ms / max(cnt, 1)
        row = {"avg_us": avg * 1e3, "launches": cnt, "share": tot_ms / (ms_prof * args.steps)}
        if name in STAGE_BYTES:
            a, b = STAGE_BYTES[name]
            if sep and name in SEP_STAGES:
                a -= 16  # Lambda rebuilt from 1-D tables, not streamed
            if lat and name in ("tik_fold_ifft_axis3", "tik_fold_ifft_axis1"):
                a, b = a - 16, b + 16  # LR prior spectrum instead of the HR fft3(xbar)
            byts = a * N + b * Nl
            row["alg_bytes"] = byts
            row["gbs"] = byts / (avg * 1e-3) / 1e9
            row["frac"] = row["gbs"] / hbm
        st_rows[name] = row
    timed = {k: v for k, v in st_rows.items() if "alg_bytes" in v}
    dom = max(timed, key=lambda k: timed[k]["avg_us"] * timed[k]["launches"])
    d = timed[dom]
    path_bytes = V.tikhonov_algorithmic_bytes(cfg.hr, cfg.rates)
    own_bytes = sum(r.get("alg_bytes", 0) * r["launches"] for r in st_rows.values()) / args.steps
    roofline = {"bound": "hbm", "kernel": dom, "achieved": d["gbs"], "peak": hbm, "unit": "GB/s",
                "frac": d["frac"], "traffic": None, "peak_source": peak_src,
                "alg_bytes_per_launch": d["alg_bytes"],
                "path": {"alg_bytes_per_step": own_bytes, "achieved": own_bytes / (ms * 1e-3) / 1e9,
                         "frac": own_bytes / (ms * 1e-3) / 1e9 / hbm,
                         "lambda_separable": sep, "prior_on_lattice": lat, "spatial_expansion": spatial,
                         "reference_algorithm_bytes": path_bytes,
                         "reference_algorithm_model": "(72 + 40/d) N bytes per solve (SURVEY 8(d): HR "
                                                      "Lambda, fft3(xbar), x_hat and three HR passes)",
                         "reference_algorithm_equiv_frac": path_bytes / (ms * 1e-3) / 1e9 / hbm,
                         "note": "alg_bytes_per_step sums the stages this path runs; with a separable compact "
                                 "PSF and the CLI-default lattice prior the solve is x = xbar + sqrt(d) H^T D^H "
                                 "F_l^-1(U) with the LR stage on the Hermitian half spectrum: 8 N + 112 N_l bytes"}}
    if spatial and not args.no_fft_path:
        roofline["path"]["fft_path_ms"] = tik_fft_path_ms(args, ctx, V, spec, lam_d, cfg, xbar_d, y_d, x_d,
                                                           stream, torch, flush)
    try:
        prof = json.loads((ROOT / "profiles" / "traffic.json").read_text())
        if dom in prof:
            roofline["traffic"] = prof[dom]["bytes"] if isinstance(prof[dom], dict) else prof[dom]
            roofline["traffic_source"] = (prof.get("_source") or "committed ncu capture") + \
                " -- dram__bytes_read.sum + dram__bytes_write.sum of this kernel from the capture, not this run"
    except Exception:
        pass
    # the spatial path's own compulsory bytes: read y, write x
    comp = 8 * N + 8 * Nl
    roofline["path_compulsory"] = {"bytes": comp, "achieved": comp / (ms * 1e-3) / 1e9,
                                   "frac": comp / (ms * 1e-3) / 1e9 / hbm,
                                   "model": "(8 N + 8 N/d) bytes per solve: y in, x out"}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded ellipsoid+texture phantom, BSNR 30 dB; paper volumes proprietary)",
            "config": config_block(cfg), "roofline": roofline, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk, "stages": st_rows, "stages_ms_per_step": ms_prof,
            "timing": "per-solve CUDA events on the library stream, L2 flushed between solves; headline pass "
                      "runs the user path (CUDA-graph replay), stage table from a second profiled pass"}

    line["config0"] = bench_tik_config(args, ctx, V, synth, torch, stream, local, hbm, 0)
    if not args.no_fp32:
        line["fp32"] = bench_tik_fp32(args, ctx, V, op, inp, cfg, torch, stream, flush, hbm)
    if not args.no_tv:
        line["tv"] = bench_tv(args, ctx, V, synth, torch, stream, local, hbm, 2)
        line["config3"] = bench_tv(args, ctx, V, synth, torch, stream, local, hbm, 3)
        if not args.no_fp32:
            line["fp32"]["tv_config2"] = bench_tv(args, ctx, V, synth, torch, stream, local, hbm, 2, "f32")
            line["fp32"]["tv_config3"] = bench_tv(args, ctx, V, synth, torch, stream, local, hbm, 3, "f32")
        if rank == 0 and world == 1 and not args.no_cpu:
            line["tv"]["cpu_baseline"] = cpu_baseline_tv(synth.CONFIGS[2], synth.make_inputs(synth.CONFIGS[2],
                                                                                          with_truth=False))
    if not args.no_fft_path:
        line["fft3_vs_cufft"] = bench_fft_compare(args, ctx, V, torch, stream, local, hbm)
    if not args.no_sharded:
        line["sharded"] = _guarded(lambda: bench_sharded(args, ctx, V, synth, torch, rank, world, local, 3))
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(cfg, inp)
    op.close()
    if world == 1 and not args.no_config4:
        line["config4"] = bench_config4(args, ctx, V, synth, torch, stream, local, hbm)
    if not args.no_sharded and not args.no_config4:
        line["sharded_config4"] = _guarded(lambda: bench_sharded(args, ctx, V, synth, torch, rank, world, local, 4,
                                                                 iters=3))
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def tik_fft_path_ms(args, ctx, V, spec, lam_d, cfg, xbar_d, y_d, x_d, stream, torch, flush):
    """Same solve through the general FFT path (VSR_NO_SPATIAL=1 for this
    operator): fused fold + inverse axis-3, then axes 2 and 1."""
    os.environ["VSR_NO_SPATIAL"] = "1"
    try:
        op = V.TikhonovDevice(ctx, spec, lam_d, cfg.reg, xbar_d)
    finally:
        del os.environ["VSR_NO_SPATIAL"]
    for _ in range(3):
        op.solve_d(y_d, x_d)
    tot = 0.0
    for i in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        op.solve_d(y_d, x_d)
        b.record(stream)
        b.synchronize()
        tot += a.elapsed_time(b)
    op.check()
    op.close()
    return tot / args.steps


def bench_fft_compare(args, ctx, V, torch, stream, local, hbm, edge=256):
    """The hand-written fp64 3D FFT engine (vsr_fft3_d: unitary C2C, three
    axis passes) next to cuFFT (torch.fft.fftn, norm="ortho") on the same
    256^3 complex128 buffer; cuFFT is timed only as a comparison (BASELINE
    north_star).  Inputs exceed L2 (268 MB), so no flush is needed."""
    import ctypes as C
    dev = torch.device("cuda", local)
    n = edge ** 3
    g = torch.Generator(device=dev).manual_seed(5)
    x = torch.complex(torch.rand(n, generator=g, device=dev, dtype=torch.float64),
                      torch.rand(n, generator=g, device=dev, dtype=torch.float64))
    ours = torch.empty_like(x)
    dims = (C.c_size_t * 3)(edge, edge, edge)
    scale = 1.0 / math.sqrt(n)

    def run_ours():
        V.check(V._lib.vsr_fft3_d(ctx.handle, dims, C.c_void_p(x.data_ptr()), 0, C.c_void_p(ours.data_ptr()),
                                  scale))

    def run_cufft():
        return torch.fft.fftn(x.view(edge, edge, edge), norm="ortho")

    def timed(fn, st):
        for _ in range(3):
            with torch.cuda.stream(st):
                fn()
        torch.cuda.synchronize()
        tot = 0.0
        reps = max(5, args.steps)
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st):
                a.record(st)
                fn()
                b.record(st)
            b.synchronize()
            tot += a.elapsed_time(b)
        return tot / reps

    ms_ours = timed(run_ours, stream)
    ms_cufft = timed(run_cufft, torch.cuda.current_stream(dev))
    ref = run_cufft().reshape(-1)
    torch.cuda.synchronize()
    err = float(torch.linalg.vector_norm(ours - ref) / torch.linalg.vector_norm(ref))
    alg = 32.0 * n  # read + write 16 B per point, once (SURVEY 8(d) compulsory model)
    return {"workload": f"unitary forward 3D C2C FFT, complex128 {edge}^3 (out of place)",
            "ms_ours": ms_ours, "ms_cufft": ms_cufft, "speedup_vs_cufft": ms_cufft / ms_ours,
            "ours_gbs_compulsory": alg / (ms_ours * 1e-3) / 1e9, "ours_frac": alg / (ms_ours * 1e-3) / 1e9 / hbm,
            "rel_l2_vs_cufft": err, "cufft": "torch.fft.fftn (cuFFT, library) -- comparison only"}


class _Dev:
    """A torch device tensor seen through the C ABI's device-pointer entry points."""

    def __init__(self, t):
        import ctypes as C
        self.t = t
        self.ptr = C.c_void_p(t.data_ptr())


def bench_config4(args, ctx, V, synth, torch, stream, local, hbm):
    """configs[4] on ONE GPU (the P = 1 point of its slab-sharded run): HR
    1024^3 -> LR 512^3 (d = 8), sigma 1.5 13^3 PSF; one Tikhonov solve
    (tau 1e-3, CLI-default lattice prior) then 20 ADMM-TV iterations (lambda
    2e-3, mu 0.05).  Timing only: y is a seeded uniform LR volume generated on
    the device (the kernels' work is value-independent; parity at this size is
    tests/test_full_configs.py).  Needs ~135 GB of device memory."""
    import ctypes as C
    cfg = synth.CONFIGS[4]
    dev = torch.device("cuda", local)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info(dev)
    if free < 150e9:
        return {"skipped": f"needs ~150 GB free device memory, {free / 1e9:.0f} GB free"}
    m, n, s = cfg.hr
    N = m * n * s
    d = int(np.prod(cfg.rates))
    r1, r2, r3 = cfg.rates
    spec = V.DecimationSpec(cfg.hr, cfg.rates)
    g = torch.Generator(device=dev).manual_seed(cfg.seeds[-1])
    y = torch.rand(s // r3, n // r2, m // r1, generator=g, device=dev, dtype=torch.float64)
    kern = torch.from_numpy(np.ascontiguousarray(V.make_gaussian_psf(cfg.psf_size, cfg.psf_sigma,
                                                                     cfg.psf_size))).to(dev)
    psf = torch.zeros(s, n, m, device=dev, dtype=torch.float64)
    idx = []
    for k, L in zip(kern.shape, (s, n, m)):
        i = torch.arange(k, device=dev)
        idx.append(torch.where(i <= k // 2, i, i - k) % L)
    psf[idx[0][:, None, None], idx[1][None, :, None], idx[2][None, None, :]] = kern
    out = {"workload": "config4 on 1 GPU: HR 1024^3 -> LR 512^3 (d=8), PSF sigma 1.5 13^3, Tikhonov tau 1e-3 "
                       "then 20 ADMM-TV iterations (lambda 2e-3, mu 0.05, tau 1e-3*mu)",
           "data": "seeded uniform LR y generated on the device (timing only)"}

    def ev_time(fn, reps):
        tot = 0.0
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            tot += a.elapsed_time(b)
        return tot / reps

    # Tikhonov: Lambda on the device (unnormalised DFT of the PSF), lattice prior d D^H y
    lam = torch.empty(N, device=dev, dtype=torch.complex128)
    dims = (C.c_size_t * 3)(m, n, s)
    torch.cuda.synchronize()
    V.check(V._lib.vsr_fft3_d(ctx.handle, dims, C.c_void_p(psf.data_ptr()), 1, C.c_void_p(lam.data_ptr()), 1.0))
    ctx.synchronize()
    xbar = torch.zeros(s, n, m, device=dev, dtype=torch.float64)
    xbar[::r3, ::r2, ::r1] = d * y
    x = torch.empty(s, n, m, device=dev, dtype=torch.float64)
    torch.cuda.synchronize()
    op = V.TikhonovDevice(ctx, spec, _Dev(lam), cfg.reg, _Dev(xbar))
    for _ in range(3):
        op.solve_d(_Dev(y), _Dev(x))
    ms_tik = ev_time(lambda: op.solve_d(_Dev(y), _Dev(x)), max(3, min(args.steps, 10)))
    op.check()
    out["tikhonov_ms"] = ms_tik
    out["tikhonov_value"] = N / (ms_tik * 1e-3)
    out["tikhonov_spatial_path"] = op.spatial()
    op.close()
    del lam, xbar, x
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    # ADMM-TV: construction timed separately (setup: Lambda, tables, init)
    iters = 20
    tcfg = V.TvAdmmConfig(lambda_=cfg.tv_lambda, mu=cfg.tv_mu, max_iters=iters + 6, rel_tol=0.0,
                          tau=1e-3 * cfg.tv_mu, init=V.INIT_UPSAMPLED)
    t0 = time.perf_counter()
    tv = V.TvDevice(ctx, spec, _Dev(y), _Dev(psf), tcfg)
    ctx.synchronize()
    out["tv_setup_s"] = time.perf_counter() - t0
    tv.iterate(2)
    k = 4
    ms_it = ev_time(lambda: tv.iterate(k), 1) / k
    # per-stage table from a second, profiled pass (as the config-2/3 blocks)
    V.profile_enable(ctx, True)
    tv.iterate(2)
    ctx.synchronize()
    st4 = V.profile_read(ctx)
    V.profile_enable(ctx, False)
    out["tv_stages_us"] = {name: tot / max(cnt, 1) * 1e3 for name, (tot, cnt) in st4.items()}
    rep = tv.report()
    tv.close()
    out["tv_ms_per_iter"] = ms_it
    out["tv_value"] = N / (ms_it * 1e-3)
    out["tv_iters_timed"] = k
    out["objective_last"] = rep.objective[-1]
    out["job_ms"] = ms_tik + iters * ms_it
    out["job_note"] = "one Tikhonov solve + 20 ADMM-TV iterations, device-resident inputs, setup excluded"
    out["tik_frac_general_model"] = V.tikhonov_algorithmic_bytes(cfg.hr, cfg.rates) / (ms_tik * 1e-3) / 1e9 / hbm
    out["tv_frac_model"] = V.tv_algorithmic_bytes(cfg.hr, cfg.rates) / (ms_it * 1e-3) / 1e9 / hbm
    del psf, y
    torch.cuda.empty_cache()
    return out


def bench_tik_fp32(args, ctx, V, op, inp, cfg, torch, stream, flush, hbm):
    """fp32 mode on the headline workload (config 1): TikhonovOperator solve_f32
    (fp64 LR stage, fp32 expansion and x), device-resident and end to end with
    pinned fp32 host buffers; timed like the headline (per-solve events, L2
    flushed between solves).  Not the headline: the reference precision is fp64."""
    N = cfg.voxels
    y32 = inp.y.astype(np.float32)
    yd = V.DeviceBuffer(ctx, y32.nbytes)
    yd.upload(y32)
    xd = V.DeviceBuffer(ctx, N * 4)
    for _ in range(max(args.warmup, 3)):
        op.solve_f32_d(yd, xd)
    op.check()
    ctx.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(float(i))
        evs[i][0].record(stream)
        op.solve_f32_d(yd, xd)
        evs[i][1].record(stream)
    evs[-1][1].synchronize()
    op.check()
    ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    yp = V.PinnedBuffer(y32.shape, np.float32)
    yp.array[...] = y32
    xp = V.PinnedBuffer(V.shape_of(cfg.hr), np.float32)
    for _ in range(2):
        op.solve_f32_host(yp.array, xp.array)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        op.solve_f32_host(yp.array, xp.array)
    e2e_s = (time.perf_counter() - t0) / args.steps
    comp = 4 * N + 4 * (N // cfg.d)
    return {"workload": "config1 Tikhonov solve in fp32 mode (y, x fp32; LR stage fp64; expansion fp32)",
            "value": N / (ms * 1e-3), "unit": UNIT, "ms_per_solve": ms,
            "path_compulsory": {"bytes": comp, "frac": comp / (ms * 1e-3) / 1e9 / hbm,
                                "model": "(4 N + 4 N/d) bytes: fp32 y in, fp32 x out"},
            "e2e": {"value": N / e2e_s, "unit": UNIT, "ms_per_step": e2e_s * 1e3,
                    "h2d_bytes_per_step": int(y32.nbytes), "d2h_bytes_per_step": int(N * 4),
                    "api": "vsr_tikhonov_solve_f32 (pinned fp32 host y, x)"},
            "accuracy": "rel L2 vs the fp64 solve ~5e-8 (tests/test_fp32.py)"}


def bench_tv(args, ctx, V, synth, torch, stream, local, hbm, idx=2, precision="f64"):
    """ADMM-TV iteration throughput on configs[2] (256^3, d = 64) or configs[3]
    (512x512x256, d = (2,2,4)) through the single-GPU path (precision "f32":
    the fp32 mode)."""
    cfg = synth.CONFIGS[idx]
    inp = synth.make_inputs(cfg, with_truth=False)
    N = cfg.voxels
    spec = V.DecimationSpec(cfg.hr, cfg.rates)
    y_d = V.DeviceBuffer(ctx, inp.y.nbytes)
    y_d.upload(inp.y)
    p_d = V.DeviceBuffer(ctx, inp.psf.nbytes)
    p_d.upload(inp.psf)
    x0_d = None
    if inp.x0 is not None:
        x0_d = V.DeviceBuffer(ctx, inp.x0.nbytes)
        x0_d.upload(inp.x0)
    k = max(args.steps, 10)
    iters = 2 * k + max(args.warmup, 3)
    tcfg = V.TvAdmmConfig(lambda_=cfg.tv_lambda, mu=cfg.tv_mu, max_iters=iters, rel_tol=0.0,
                          tau=1e-3 * cfg.tv_mu, init=V.INIT_PROVIDED if x0_d is not None else V.INIT_UPSAMPLED,
                          precision=precision)
    tv = V.TvDevice(ctx, spec, y_d, p_d, tcfg, x0_d)
    tv.iterate(max(args.warmup, 3))
    ctx.synchronize()

    def timed(profile):
        V.profile_enable(ctx, profile)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        tv.iterate(k)
        e1.record(stream)
        e1.synchronize()
        st_ = V.profile_read(ctx) if profile else {}
        V.profile_enable(ctx, False)
        return e0.elapsed_time(e1) / k, st_

    # the iteration's working set (W 268 MB, duals 805 MB, x, theta) exceeds L2
    ms, _ = timed(False)
    ms_prof, stages = timed(True)
    rep = tv.report()
    tv_sep = tv.separable()
    tv.close()
    f32 = precision == "f32"
    # fp32 mode: every HR volume / spectrum term halves; the LR tables stay fp64
    path = V.tv_algorithmic_bytes(cfg.hr, cfg.rates)
    if f32:
        path = 80 * N + 16 * (N // cfg.d)
    rows = {}
    sep = tv_sep
    for name, (tot, cnt) in stages.items():
        avg = tot / max(cnt, 1)
        r = {"avg_us": avg * 1e3, "launches": cnt, "share": tot / (ms_prof * k)}
        if name in STAGE_BYTES:
            a, b = STAGE_BYTES[name]
            if sep and name in SEP_STAGES:
                a -= 16
            if f32:
                a = a / 2
            byts = a * N + b * (N // cfg.d)
            r["gbs"] = byts / (avg * 1e-3) / 1e9
            r["frac"] = r["gbs"] / hbm
        rows[name] = r
    hr, lr = cfg.hr, cfg.lr
    return {"workload": f"config{idx}: ADMM-TV {'fp32 mode' if f32 else 'fp64'} {hr[0]}x{hr[1]}x{hr[2]} -> "
                        f"{lr[0]}x{lr[1]}x{lr[2]} (d={cfg.d}), lambda {cfg.tv_lambda:g}, mu {cfg.tv_mu:g}, "
                        f"tau 1e-3*mu, single GPU",
            "value": N / (ms * 1e-3), "unit": "HR voxels/s per ADMM-TV iteration", "ms_per_iter": ms,
            "iters_timed": k, "path_frac": path / (ms * 1e-3) / 1e9 / hbm, "lambda_separable": tv_sep,
            "path_model": "(80 + 16/d) N bytes per iteration (fp32 state)" if f32
                          else "(160 + 16/d) N bytes per iteration", "objective_last": rep.objective[-1],
            "stages": rows, "stages_ms_per_iter": ms_prof}


def bench_tik_config(args, ctx, V, synth, torch, stream, local, hbm, idx=0):
    """configs[0] (64^3 -> 32^3, d = 8): the same device Tikhonov solve at the
    reference's CPU-runnable size.  L2-resident and launch-bound (SURVEY
    8(d)): reported, but its roofline fraction is not meaningful."""
    cfg = synth.CONFIGS[idx]
    inp = synth.make_inputs(cfg, with_truth=False)
    spec = V.DecimationSpec(cfg.hr, cfg.rates)
    lam = V.psf_to_spectrum(inp.psf, ctx)
    lam_d = V.DeviceBuffer(ctx, lam.nbytes)
    lam_d.upload(lam)
    xbar_d = V.DeviceBuffer(ctx, inp.xbar.nbytes)
    xbar_d.upload(inp.xbar)
    y_d = V.DeviceBuffer(ctx, inp.y.nbytes)
    y_d.upload(inp.y)
    x_d = V.DeviceBuffer(ctx, cfg.voxels * 8)
    op = V.TikhonovDevice(ctx, spec, lam_d, cfg.reg, xbar_d)
    for _ in range(max(args.warmup, 3)):
        op.solve_d(y_d, x_d)
    op.check()
    ctx.synchronize()
    k = max(args.steps, 20)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(k):
        op.solve_d(y_d, x_d)
    e1.record(stream)
    e1.synchronize()
    op.check()
    ms = e0.elapsed_time(e1) / k
    path = {"spatial": op.spatial(), "separable": op.separable(), "lattice_prior": op.lattice_prior()}
    op.close()
    return {"workload": f"config{idx}: closed-form Tikhonov SR fp64 64^3 -> 32^3 (d=8), back-to-back solves "
                        "(graph replay; inputs L2-resident: launch-bound)",
            "value": cfg.voxels / (ms * 1e-3), "unit": UNIT, "ms_per_solve": ms, "solves_timed": k,
            "path": path}


def cpu_baseline_tv(cfg, inp, iters=2):
    """The reference admm_tv (oracle/_ref, shim FFTs on every host thread) on configs[2] at
    rel_tol = 0: report.seconds / iterations (solvers.cpp:409), which includes
    its precompute and the 2 objective FFTs per iteration; bounded to `iters`
    iterations."""
    sys.path.insert(0, str(ROOT / "oracle"))
    try:
        import ref_binding
        if not ref_binding.available():
            return None
    except Exception:
        return None
    threads = host_threads()
    os.environ["VSR_SHIM_THREADS"] = str(threads)
    x, rep = ref_binding.admm_tv(inp.y, inp.psf, cfg.hr, cfg.rates, cfg.tv_lambda, cfg.tv_mu, iters, 0.0,
                                 tau=1e-3 * cfg.tv_mu, init=2 if inp.x0 is not None else 1, init_volume=inp.x0)
    per = rep["seconds"] / rep["iterations"]
    return {"value": cfg.voxels / per, "unit": "HR voxels/s per ADMM-TV iteration", "cores": threads,
            "kind": "reference", "seconds_per_iteration": per,
            "sample": f"reference volsr admm_tv (oracle/_ref) config{cfg.idx}, {rep['iterations']} iterations at "
                      "rel_tol 0, report.seconds / iterations (includes its precompute); the FFTW3-API shim's FFTs "
                      f"(radix-2 row-column, slower per core than real FFTW) on {threads} threads, every other pass "
                      "single-threaded as in the reference"}


def bench_sharded(args, ctx, V, synth, torch, rank, world, local, idx=3, iters=None):
    """configs[3] (512x512x256, d = (2,2,4)) or configs[4] (1024^3, d = 8)
    ADMM-TV, slab-sharded over all ranks (csrc/slab.cu through the C ABI):
    y-slabs, the axis-3 half spectrum split by plane over conjugate LR class
    pairs, the exchanges as the kernels' own NVLink peer stores / loads
    between stream-ordered NCCL barriers (N > 1), P = 1 on one GPU.  Strong
    scaling: the whole volume is split over the N ranks."""
    import torch.distributed as tdist
    from paper_2010_15491_b200 import dist as D
    cfg = synth.CONFIGS[idx]
    hr, rates = cfg.hr, cfg.rates
    m, n, s = hr
    N = m * n * s
    free = torch.cuda.mem_get_info(local)[0]
    need = 110.0 * N / world + 24.0 * N  # per rank: slab state ~96 N / P + the setup's full Lambda
    if free < need:
        return {"skipped": f"needs ~{need / 1e9:.0f} GB of free device memory per GPU ({free / 1e9:.0f} GB free)"}
    dist_on = world > 1 and tdist.is_available() and tdist.is_initialized()
    comm = D.SlabComm.nccl(ctx) if dist_on else D.SlabComm.local(1, ctx)
    psf = synth.make_gaussian_psf(cfg.psf_size, cfg.psf_sigma, hr)
    rng = np.random.default_rng(99)
    y = rng.uniform(0.0, 1.0, V.shape_of(cfg.lr))  # the work is value-independent; parity: tests/test_dist.py
    k = iters or max(3, min(args.steps, 10))
    spec = V.DecimationSpec(hr, rates)
    tcfg = V.TvAdmmConfig(lambda_=cfg.tv_lambda, mu=cfg.tv_mu, max_iters=k + 2, rel_tol=0.0,
                          tau=1e-3 * cfg.tv_mu, init=V.INIT_UPSAMPLED)
    tv = D.SlabADMMTV(comm, y, psf, spec, tcfg)
    del psf
    tv.iterate(2)
    dev = torch.device("cuda", local)
    lib = torch.cuda.ExternalStream(ctx.stream(), device=dev)  # the stream the slab stages run on
    if dist_on:
        tdist.barrier()
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = V.launch_count()
    e0.record(lib)
    tv.iterate(k)
    e1.record(lib)
    e1.synchronize()
    launches = V.launch_count() - l0
    ms = e0.elapsed_time(e1) / k
    _, rep = tv.finish()
    tv.close()
    comm.close()
    if dist_on:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        ms = float(t.item())
    # peer traffic per rank per iteration: its rows of the half planes it does
    # not own, out (r2c stores) and back (c2r loads), plus 5 halo rows per plane
    half_bytes = 16.0 * m * (n // world) * (s // 2 + 1)
    peer = 2 * half_bytes * (world - 1) / world + 5 * 8.0 * m * s * (world > 1)
    hbm = load_peaks().get("hbm_gbs") or 6650.0
    path = V.tv_algorithmic_bytes(hr, rates)
    return {"workload": f"config{idx}: ADMM-TV fp64 {m}x{n}x{s} -> {cfg.lr[0]}x{cfg.lr[1]}x{cfg.lr[2]} "
                        f"(d={cfg.d}), slab-sharded over {world} GPU(s)",
            "value": N / (ms * 1e-3), "unit": "HR voxels/s per ADMM-TV iteration", "ms_per_iter": ms,
            "iters_timed": k, "scaling": "strong", "gpu_launches_per_iter": launches / k,
            "per_gpu_hbm_frac_of_model": path / world / (ms * 1e-3) / 1e9 / hbm,
            "peer_bytes_per_rank_per_iter": peer,
            "peer_gbs_per_rank": peer / (ms * 1e-3) / 1e9 if world > 1 else 0.0,
            "peer_frac_of_nvlink_900": peer / (ms * 1e-3) / 1e9 / 900.0 if world > 1 else 0.0,
            "objective_last": rep.objective[-1],
            "design": "exchange = r2c peer stores / c2r peer loads over NVLink (CUDA IPC), 3 stream-ordered "
                      "barriers per iteration; no pack/unpack passes; half-spectrum planes only"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-tv", action="store_true")
    ap.add_argument("--no-config4", action="store_true", help="skip the 1024^3 single-GPU config-4 timing")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-fp32", action="store_true", help="skip the fp32-mode blocks")
    ap.add_argument("--no-fft-path", action="store_true", help="skip timing the general FFT-path solve")
    ap.add_argument("--no-sharded", action="store_true", help="skip the slab-sharded config-3/4 timings")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(local)
        tdist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    try:
        return run_b200(args, rank, world, local)
    finally:
        if world > 1:
            import torch.distributed as tdist
            tdist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
