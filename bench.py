#!/usr/bin/env python
"""Benchmark of the B200 tiled fast-convolution forward pass (BASELINE.json metric:
"ms/layer & effective TFLOP/s (direct-conv FLOPs) + roofline fraction, 1/2/4/8 B200").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fastconv|reference]
                    [--workload vgg3_2|vgg1_2|k5|deep|tiny] [--scaling strong|weak]
                    [--flush-l2 auto|on|off] [--method M --m m] [--gemm auto|f16x3|tcgen05|ffma]

A *step* is one full pass of the hot path: NK1 kernel transform,
NK2 input transform, NK3 contraction, NK4 output transform + crop, over one batch
of the workload (the paper times the kernel transform as part of the layer,
P:455-460; reading R13).  Workload: BASELINE.json configs[1], the
VGG-3.2-shaped layer (B=64, C=C'=256, 58x58, r=3).  The (method, m) is chosen
per the paper's comparison rule (each method at its fastest m): every
(method, m) the config lists is timed briefly, the fastest is the headline and
all are reported under "sweep".

Multi-GPU: ``--gpus N`` without torchrun re-launches this script
under ``torch.distributed.run`` with N ranks (one per GPU); under torchrun,
WORLD_SIZE must equal N.  Strong scaling (default): ONE global seeded draw of the
config's B images; rank k owns images parallel.shard_range(B, k, N) and runs
conv_plan(B_k, ...), transforming the kernels locally -- no collective on the data
path.  ``--scaling weak`` draws B*N images once and gives every rank B of them.

Timing: inputs resident in HBM; W untimed warm-up steps; K steps bracketed by a
barrier + cuda synchronize on both sides, timed with CUDA events on the launching
stream, max over ranks.  L2: when a rank's inputs + outputs are smaller than 2x
the 126 MB L2 (``--flush-l2 auto``), a 2x-L2 buffer is written between timed
steps and only the steps themselves are timed (per-step events); otherwise the
inputs are larger than L2 and no flush is needed.  nvidia-smi and NVML sample SM
clocks and throttle reasons during the run.

``--impl reference`` times the fp64 CPU oracle (oracle/, the only other place this
script runs it) on bounded samples of the same workload: the paper has no GPU
implementation to compare against.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "ms/layer & effective TFLOP/s (direct-conv FLOPs) + roofline fraction, 1/2/4/8 B200"
UNIT = "TFLOP/s"
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
TF32_OVER_BF16 = 0.5  # nominal dense ratio (1.1 vs 2.25 PFLOP/s, B200_PROFILING.md)
F16_OVER_BF16 = 1.0   # kind::f16 (fp16 in, fp32 accumulate) runs at the bf16 dense rate


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return d, "measured"
    except Exception:
        return dict(FALLBACK_PEAKS), "fallback"


# ------------------------------------------------------------------ clocks ---
class ClockSampler:
    """nvidia-smi sampler running while the GPU works (B200_PROFILING.md clocks line)."""
    Q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.samples = []
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=" + self.Q, "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.samples.append((time.time(), parts))

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0: float, t1: float) -> dict:
        inside = [p for (t, p) in self.samples if t0 <= t <= t1]
        used = inside if inside else [p for (t, p) in self.samples if t >= t0 - 2.0]
        if not used:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(p[1]) for p in used if num(p[1]) is not None]
        mx = [num(p[2]) for p in used if num(p[2]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for p in used for i in range(4) if p[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(used), "samples_in_timed_region": len(inside),
                "power_w_max": max((num(p[3]) or 0.0) for p in used)}


class NvmlProbe:
    """Direct NVML reads (milliseconds each) taken while the queued timed steps execute, so
    even a timed region shorter than nvidia-smi's 100 ms period carries clock samples."""
    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4))

    def __init__(self, index: int):
        self.samples = []
        self.h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_sm = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self.h = None

    def sample(self):
        if self.h is None:
            return
        try:
            nv = self.nv
            sm = float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
            try:
                mask = int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                mask = int(nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h))
            pw = nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0
            self.samples.append((sm, mask, pw))
        except Exception:
            pass

    def merge(self, clk: dict) -> dict:
        """Fold the NVML samples into ClockSampler.summary()'s dict."""
        if not self.samples:
            return clk
        sm = [x[0] for x in self.samples]
        reasons = set(clk.get("reasons") or [])
        reasons |= {n for (n, bit) in self.REASONS for (_, mask, _) in self.samples if mask & bit}
        out = dict(clk)
        smi = clk.get("samples_in_timed_region", 0) or 0
        if not smi:  # no nvidia-smi sample fell inside the region: the NVML reads are the evidence
            out["sm_mhz"] = statistics.median(sm)
        out["sm_max_mhz"] = clk.get("sm_max_mhz") or self.max_sm
        out["reasons"] = sorted(reasons)
        out["nvml_samples_in_timed_region"] = len(sm)
        out["nvml_sm_mhz_median"] = statistics.median(sm)
        out["power_w_max"] = max(clk.get("power_w_max") or 0.0, max(x[2] for x in self.samples))
        return out


# --------------------------------------------------------------- reference ---
def run_reference(args, rank, world):
    """The oracle as the reference arm: bounded samples of the workload on host cores."""
    if rank != 0:
        return
    import numpy as np
    import oracle
    import synth
    cfg = synth.CONFIGS[args.workload]
    I, W = synth.make_inputs(cfg.with_batch(1))
    # calibrate: one image x 2 output channels, then size a step to the budget
    co = 2
    t = time.perf_counter()
    oracle.conv_fp64(I, W[:co].contiguous())
    per_co = max((time.perf_counter() - t) / co, 1e-4)
    budget = max(0.5, args.reference_budget_s / max(1, args.steps + args.warmup))
    co = int(max(1, min(cfg.Cout, budget / per_co)))
    Ws = W[:co].contiguous()
    flops = 2.0 * cfg.C * co * cfg.Ho * cfg.Wo * cfg.r * cfg.r
    for _ in range(args.warmup):
        oracle.conv_fp64(I, Ws)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.conv_fp64(I, Ws)
    dt = (time.perf_counter() - t0) / max(1, args.steps)
    value = flops / dt / 1e12
    sample = "1 image x %d of %d output channels of %s per step (%.3g of the layer's direct FLOPs)" % (
        co, cfg.Cout, cfg.name, flops / cfg.direct_flops)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "B": cfg.B, "C": cfg.C, "Cout": cfg.Cout, "H": cfg.H, "W": cfg.W,
                       "r": cfg.r, "impl": "fp64 CPU direct-convolution oracle (oracle/conv_oracle.c)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg, seconds: float):
    """Oracle (as it stands) on a bounded sample: the first n images x a slice of output channels."""
    import oracle
    import synth
    I, W = synth.make_inputs(cfg)
    oracle.conv_fp64(I[:1].contiguous(), W[:2].contiguous())  # warm the OpenMP pool
    t = time.perf_counter()
    oracle.conv_fp64(I[:1].contiguous(), W[:8].contiguous())
    per_img_co = max((time.perf_counter() - t) / 8, 1e-5)
    work = seconds / per_img_co  # image x output-channel units that fit the budget
    co = int(max(1, min(cfg.Cout, work)))
    nb = int(max(1, min(cfg.B, work / co)))
    Is, Ws = I[:nb].contiguous(), W[:co].contiguous()
    t = time.perf_counter()
    oracle.conv_fp64(Is, Ws)
    dt = time.perf_counter() - t
    flops = 2.0 * nb * cfg.C * co * cfg.Ho * cfg.Wo * cfg.r * cfg.r
    return {"value": flops / dt / 1e12, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
            "sample": "%d of %d images x %d of %d output channels of %s (%.3g of the layer's direct FLOPs), %.1f s"
                      % (nb, cfg.B, co, cfg.Cout, cfg.name, flops / cfg.direct_flops, dt)}


def cpu_direct_baseline(cfg, seconds: float):
    """The straightforward multithreaded fp32 CPU direct convolution (cpu_baseline/) on a
    bounded sample of the workload: the first n images, all output channels."""
    import cpu_baseline
    import synth
    I, W = synth.make_inputs(cfg)
    cpu_baseline.conv_fp32(I[:1].contiguous(), W[:8].contiguous())  # warm the OpenMP pool
    t = time.perf_counter()
    cpu_baseline.conv_fp32(I[:1].contiguous(), W)
    per_img = max(time.perf_counter() - t, 1e-5)
    nb = int(max(1, min(cfg.B, seconds / per_img)))
    Is = I[:nb].contiguous()
    t = time.perf_counter()
    cpu_baseline.conv_fp32(Is, W)
    dt = time.perf_counter() - t
    flops = 2.0 * nb * cfg.C * cfg.Cout * cfg.Ho * cfg.Wo * cfg.r * cfg.r
    return {"value": flops / dt / 1e12, "unit": UNIT, "cores": cpu_baseline.num_threads(),
            "kind": "direct_fp32 (OpenMP over (b, c'), -O3 -mavx2 -mfma, no blocking)",
            "sample": "%d of %d images x all %d output channels of %s (%.3g of the layer's direct FLOPs), %.1f s"
                      % (nb, cfg.B, cfg.Cout, cfg.name, flops / cfg.direct_flops, dt)}


# ------------------------------------------------------------------- main ---
L2_BYTES = 126 * 1024 * 1024


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch_under_torchrun(n: int) -> int:
    """--gpus N without a torchrun environment: run this script as N ranks (one per GPU)."""
    # "--m" is an ambiguous prefix of torchrun's own options: pass it on as "--tile"
    argv = ["--tile" if a == "--m" else ("--tile=" + a[4:] if a.startswith("--m=") else a) for a in sys.argv[1:]]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=%d" % n,
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + argv
    return subprocess.call(cmd)


def measure_matmul_peaks(dev, sustained_s: float = 1.5) -> dict:
    """Dense tensor-core peaks measured like MEASURED_PEAKS.json's bf16 figure:
    torch.matmul at 8192^3, best of 10 (burst) and back to back for `sustained_s` (sustained),
    for fp32 inputs with TF32 allowed (the 3xTF32 contraction's pipe) and for fp16 (F16X3's)."""
    import torch
    out = {}
    n = 8192
    prev = torch.backends.cuda.matmul.allow_tf32
    try:
        torch.backends.cuda.matmul.allow_tf32 = True
        for name, dt in (("tf32", torch.float32), ("fp16", torch.float16)):
            a = torch.randn(n, n, device=dev, dtype=dt)
            b = torch.randn(n, n, device=dev, dtype=dt)
            for _ in range(3):
                torch.matmul(a, b)
            best = 1e30
            for _ in range(10):
                s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s0.record()
                torch.matmul(a, b)
                s1.record()
                s1.synchronize()
                best = min(best, s0.elapsed_time(s1))
            burst = 2.0 * n ** 3 / (best * 1e-3) / 1e12
            reps = max(5, int(sustained_s * 1e3 / best))
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            for _ in range(reps):
                torch.matmul(a, b)
            s1.record()
            s1.synchronize()
            sus = 2.0 * n ** 3 * reps / (s0.elapsed_time(s1) * 1e-3) / 1e12
            out[name] = {"burst_tflops": burst, "sustained_tflops": sus}
            del a, b
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    torch.cuda.empty_cache()
    out["how"] = ("torch.matmul 8192^3 (cuBLAS), 2 n^3 FLOPs: best of 10 (burst), back to back for %.1f s "
                  "(sustained); tf32 = fp32 inputs with allow_tf32" % sustained_s)
    return out


class StepTimer:
    """The timed region: K steps on `stream`, bracketed by barrier + synchronize.  Without a
    flush one event pair spans the K back-to-back steps; with a flush (2x L2 written between
    steps) each step has its own pair and ms/step is the mean of the steps alone."""

    def __init__(self, dev, stream, flush: bool):
        import torch
        self.torch = torch
        self.stream = stream
        self.flush = flush
        self.buf = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev) if flush else None

    def run(self, steps: int, fn, on_step=None):
        torch = self.torch
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record(self.stream)
        for k in range(steps):
            if self.flush:
                self.buf.fill_(float(k))
            ev[k][0].record(self.stream)
            fn()
            ev[k][1].record(self.stream)
            if on_step:
                on_step(k)
        end.record(self.stream)
        end.synchronize()
        per = [a.elapsed_time(b) for a, b in ev]
        if self.flush:
            total = sum(per)
        else:  # back to back: the span from the first step's start to the last step's end
            total = ev[0][0].elapsed_time(ev[-1][1])
        return total, per


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="fastconv", choices=["fastconv", "reference"])
    ap.add_argument("--workload", default="vgg3_2")
    ap.add_argument("--seed", type=int, default=None, help="override the config's input seed (synth)")
    ap.add_argument("--method", default="auto", help="auto (sweep) or winograd|regular_fft|gauss_fft|direct")
    ap.add_argument("--m", "--tile", dest="m", type=int, default=0)
    ap.add_argument("--gemm", default="auto", choices=["auto", "tcgen05", "ffma", "f16x3"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--flush-l2", default="auto", choices=["auto", "on", "off"])
    ap.add_argument("--sweep-steps", type=int, default=10)
    ap.add_argument("--stage-every", type=int, default=4,
                    help="per-stage CUDA events on every k-th timed step (1 = every step)")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-baseline-s", type=float, default=12.0)
    ap.add_argument("--reference-budget-s", type=float, default=120.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the 3xTF32 arm, cached/graph runs, peaks")
    ap.add_argument("--mode", default="batch", choices=["batch", "eshard"],
                    help="batch-sharded ranks (no data-path collective) or element-sharded ranks "
                         "(all-to-alls of U and X, SURVEY 8(f)3); eshard needs --method and --m")
    ap.add_argument("--exchange", default="collective", choices=["collective", "p2p"],
                    help="eshard: U / X through all_to_all, or copied straight into the peers' "
                         "IPC-mapped receive buffers (conv_eshard_forward_*_peer)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    from paper_1809_07851_b200 import parallel
    rank, world, local = parallel.env_rank_world()
    if args.impl == "reference":
        if world > 1:
            parallel.init("gloo")
        run_reference(args, rank, world)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args.gpus))
    if world != args.gpus:
        print("bench.py: --gpus %d but WORLD_SIZE=%d" % (args.gpus, world), file=sys.stderr)
        sys.exit(2)

    import torch
    import synth
    import paper_1809_07851_b200 as fc
    ndev = torch.cuda.device_count()
    if ndev < 1:
        print("bench.py: no CUDA device", file=sys.stderr)
        sys.exit(1)
    # one rank per GPU; with fewer GPUs than ranks (a dry multi-rank run on one box) ranks share
    # devices, the data path still has no collective, and the line says "oversubscribed"
    oversub = world > ndev
    dev_index = local % ndev
    rank, world, local = parallel.init("gloo" if oversub else None)
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    fc.load()
    base = synth.CONFIGS[args.workload]
    peaks, peaks_src = load_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", FALLBACK_PEAKS["hbm_gbs"]))
    bf16_burst = float(peaks.get("bf16_tflops", FALLBACK_PEAKS["bf16_tflops"]))

    # one global seeded draw; rank k slices its images (strong: B/N each, weak: B each)
    gcfg = base if args.scaling == "strong" else base.with_batch(base.B * world)
    I_all, W = synth.make_inputs(gcfg, seed=args.seed)
    lo, hi = parallel.shard_range(gcfg.B, rank, world)
    I = I_all[lo:hi].contiguous()
    del I_all
    cfg = base.with_batch(hi - lo)  # this rank's layer
    job_flops = gcfg.direct_flops  # whole-job direct-conv FLOPs per step
    x, w = I.to(dev), W.to(dev)
    out = torch.empty((cfg.B, cfg.Cout, cfg.Ho, cfg.Wo), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    io_bytes = (I.numel() + W.numel() + out.numel()) * 4
    flush = args.flush_l2 == "on" or (args.flush_l2 == "auto" and io_bytes < 2 * L2_BYTES)
    timer_fn = StepTimer(dev, stream, flush)

    clocks = ClockSampler(dev_index)  # started before the sweep so it is streaming by the timed region
    nvml = NvmlProbe(dev_index)

    def time_plan(plan, ws, steps):
        for _ in range(2):
            plan.forward(x, w, out, ws)
        torch.cuda.synchronize()
        total, _ = timer_fn.run(steps, lambda: plan.forward(x, w, out, ws))
        return total / steps

    if args.mode == "eshard":
        run_eshard(args, fc, parallel, base, gcfg, cfg, I_all_shape=None, x=x, w=w, dev=dev, stream=stream,
                   timer_fn=timer_fn, job_flops=job_flops, rank=rank, world=world, oversub=oversub, clocks=clocks,
                   nvml=nvml, flush=flush, io_bytes=io_bytes)
        return

    # ---- sweep (the paper's rule: each method at its fastest m) -----------------
    runs = list(cfg.runs) if args.method == "auto" else [(args.method, args.m)]
    sweep = {}
    for method, m in runs:
        plan = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m, args.gemm)
        ws = plan.alloc_workspace(dev)
        ms = parallel.max_over_ranks(time_plan(plan, ws, args.sweep_steps), dev if not oversub else None)
        prof = [plan.forward_profiled(x, w, out, ws) for _ in range(3)]
        stage_ms_sweep = [round(min(p[s] for p in prof), 4) for s in range(4)]
        sweep["%s/m=%d" % (method, plan.info["m"])] = {
            "method": method, "m": plan.info["m"], "t": plan.info["t"], "ms": ms,
            "tflops": job_flops / (ms * 1e-3) / 1e12, "stage_ms": stage_ms_sweep}
        del ws, plan
        torch.cuda.empty_cache()
    best = min(sweep.values(), key=lambda d: d["ms"])
    method, m = best["method"], best["m"]
    # the paper's model (stage-sum roofline) against the measured sweep
    from paper_1809_07851_b200 import planner
    plan = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m, args.gemm)
    ws = plan.alloc_workspace(dev)
    info = plan.info
    gemm_name = fc.GEMM_NAMES.get(info["gemm"], args.gemm)
    # the tensor-pipe peaks are measured after the timed region (cuBLAS at full power heats the
    # part and would push the timed steps into the power cap); until then: nominal ratios
    PK = {"fp16": bf16_burst * F16_OVER_BF16, "tf32": bf16_burst * TF32_OVER_BF16, "measured": None}

    def contraction_peak_of(gname):
        mm = PK["measured"]
        if gname == "tcgen05_f16x3":
            return PK["fp16"] / 3.0, ("measured fp16 matmul burst / 3 (F16X3 split)" if mm else
                                      "bf16 burst x 1.0 (FP16/BF16 nominal) / 3 (F16X3 split)")
        if gname == "ffma":
            return None, "FFMA (no tensor peak)"
        return PK["tf32"] / 3.0, ("measured tf32 matmul burst / 3 (3xTF32 split)" if mm else
                                  "bf16 burst x 0.5 (TF32/BF16 nominal) / 3 (3xTF32 split)")

    c_peak, c_peak_src = contraction_peak_of(gemm_name)
    plan_report = planner.report(
        {(d["method"], d["m"]): fc.plan_query(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, d["method"], d["m"],
                                              args.gemm)
         for d in sweep.values() if d["method"] != "direct"},
        {(d["method"], d["m"]): d["ms"] for d in sweep.values()},
        hbm_peak, c_peak or PK["tf32"] / 3.0)
    if method != "direct":
        mb, mb_ms, _ = fc.best_m(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, args.gemm)
        plan_report["conv_plan_best_m"] = {"method": method, "m": mb, "model_ms": mb_ms}
    nst = 4 if method != "direct" else 1

    # ---- timed region -------------------------------------------------------------
    for _ in range(args.warmup):
        plan.forward(x, w, out, ws)
    torch.cuda.synchronize()
    # per-launch CUDA events recorded by the library itself (conv_forward_timed): the
    # timed loop runs exactly the launches of conv_forward, with no host sync inside
    timer = fc.StageTimer((plan.launches + 2) * args.steps + 8)  # + 2 start markers per call (NK1 || NK2)

    def on_step(k):
        if args.steps >= 200 and k == args.steps // 2:
            nvml.sample()  # host-side read; hundreds of launches stay queued meanwhile

    parallel.barrier()
    torch.cuda.synchronize()
    t_wall0 = time.time()
    # every stage_every-th step runs conv_forward_timed (CUDA events around each of its kernels,
    # on the stream it runs on); the others plain conv_forward -- the events between kernels add
    # a few us of gaps per step, which matters for the 0.1 ms layers
    every = max(1, args.stage_every)
    n_inst = len(range(0, args.steps, every))
    step_k = [0]

    def one_step():
        if step_k[0] % every == 0:
            timer.forward(plan, x, w, out, ws)
        else:
            plan.forward(x, w, out, ws)
        step_k[0] += 1

    total_ms, per_step = timer_fn.run(args.steps, one_step, on_step)
    nvml.sample()
    torch.cuda.synchronize()
    parallel.barrier()
    t_wall1 = time.time()
    per_step = sorted(per_step)
    step_stats = {"median": statistics.median(per_step), "min": per_step[0], "max": per_step[-1]}
    rank_ms = total_ms / args.steps
    ms_step = parallel.max_over_ranks(rank_ms, dev if not oversub else None)
    rank_ms_all = parallel.all_gather_scalar(rank_ms, dev if not oversub else None)
    clk = nvml.merge(clocks.summary(t_wall0, t_wall1))
    clocks.stop()
    stage_sum, nl = timer.read()
    # per step: each stage's launches (NK2-4 run once per chunk) summed
    stage_ms = [stage_sum[s] / n_inst for s in range(4)] if nst == 4 else [stage_sum[2] / n_inst]
    value = job_flops / (ms_step * 1e-3) / 1e12

    extras = {}
    if not args.no_extras and nst == 4:
        extras = run_extras(args, fc, cfg, plan, x, w, out, ws, stream, timer_fn, job_flops, world, dev, oversub,
                            hbm_peak, contraction_peak_of, method, m, parallel)

    # ---- end to end through the public API (host buffers, copies in the region) ---
    hi_, hw_ = I.pin_memory(), W.pin_memory()
    ho_ = torch.empty(out.shape, dtype=torch.float32).pin_memory()
    for _ in range(2):
        plan.forward_host(hi_, hw_, ho_, x, w, out, ws)
    torch.cuda.synchronize()
    parallel.barrier()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for _ in range(args.e2e_steps):
        plan.forward_host(hi_, hw_, ho_, x, w, out, ws)
    s1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = parallel.max_over_ranks(s0.elapsed_time(s1) / args.e2e_steps, dev if not oversub else None)
    h2d_job = parallel.sum_over_ranks(float(I.numel() * 4 + W.numel() * 4), dev if not oversub else None)
    d2h_job = parallel.sum_over_ranks(float(out.numel() * 4), dev if not oversub else None)
    e2e = {"value": job_flops / (e2e_ms * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": e2e_ms,
           "h2d_bytes_per_step": int(h2d_job), "d2h_bytes_per_step": int(d2h_job),
           "api": "conv_forward_host (pinned host in/w/out; H2D, kernels and D2H pipelined over 8 image chunks)"}

    # ---- tensor-pipe peaks (after every timed GPU measurement), then the rooflines ---
    mm_peaks = None
    if rank == 0 and not args.no_extras:
        mm_peaks = measure_matmul_peaks(dev)
        PK.update(fp16=mm_peaks["fp16"]["burst_tflops"], tf32=mm_peaks["tf32"]["burst_tflops"], measured=True)
        c_peak, c_peak_src = contraction_peak_of(gemm_name)
        if "stage_ms" in extras.get("arm_3xtf32", {}):
            a3 = extras["arm_3xtf32"]
            pk3, pk3_src = contraction_peak_of("tcgen05_3xtf32")
            a3["contraction"] = dict(stage_rooflines(a3.pop("_info"), a3["stage_ms"], 4, hbm_peak, pk3, cfg)[2],
                                     peak_source=pk3_src)
            a3["layer_roofline_frac"] = layer_roofline_frac(a3["contraction_info"], hbm_peak, pk3, a3["ms_rank"])
    for a3 in (extras.get("arm_3xtf32", {}),):
        a3.pop("_info", None)
        a3.pop("contraction_info", None)
        a3.pop("ms_rank", None)
    # ---- roofline of the dominant kernel ------------------------------------------
    stages = stage_rooflines(info, stage_ms, nst, hbm_peak, c_peak, cfg)
    if nst == 4:  # NK1 runs on the plan's auxiliary stream concurrently with NK2 (NK3 joins both):
        # its event span overlaps NK2's, so it is reported but not a candidate for the dominant kernel
        stages[0]["concurrent_with"] = "NK2 input transform (auxiliary stream; event span overlaps NK2)"
    dom = max((d for d in stages if "concurrent_with" not in d), key=lambda d: d["ms"])
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            key = "%s/%s/m=%d" % (cfg.name, method, m)
            ent = tj.get("%s/B=%d/%s" % (key, cfg.B, gemm_name)) or (tj.get(key) if cfg.B == base.B else None)
            traffic = (ent or {}).get(dom["kernel"])
        except Exception:
            traffic = None
    roofline = {"bound": dom["bound"], "achieved": dom["achieved"], "peak": dom["peak"], "unit": dom["unit"],
                "frac": dom["frac"], "traffic": traffic, "kernel": dom["kernel"],
                "peak_source": ("%s: %s" % (peaks_src,
                                            "HBM copy GB/s" if dom["bound"] == "hbm" else c_peak_src))}
    layer_frac = layer_roofline_frac(info, hbm_peak, c_peak, ms_step if world == 1 else rank_ms) if nst == 4 else None

    cpu = cpu_fp32 = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(base, args.cpu_baseline_s)
        cpu_fp32 = cpu_direct_baseline(base, args.cpu_baseline_s)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": args.scaling,
            "stage_timing": "CUDA events around every kernel of %d of the %d timed steps (every %d-th; "
                            "conv_forward_timed), on the stream each kernel runs on" % (n_inst, args.steps, every),
            "ms_per_step_stats": {"rank0_median": step_stats["median"], "rank0_min": step_stats["min"],
                                  "rank0_max": step_stats["max"], "per_rank_ms": rank_ms_all,
                                  "how": "CUDA events around each step of the timed region (rank 0)"},
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": base.name, "global_batch": gcfg.B, "B_per_gpu": cfg.B, "C": cfg.C,
                       "Cout": cfg.Cout, "H": cfg.H, "W": cfg.W, "r": cfg.r, "method": method, "m": m,
                       "t": info["t"], "gemm": gemm_name,
                       "l2": ("flushed: 2x126 MB written between timed steps, steps timed alone "
                              "(inputs+outputs %.0f MB/GPU < 2x L2)" % (io_bytes / 1e6)) if flush else
                             ("no flush: inputs+outputs %.0f MB/GPU > 2x 126 MB L2" % (io_bytes / 1e6)),
                       "parallelism": "dp%d (batch-sharded ranks of one global draw, no collective on the data "
                                      "path, kernels transformed locally)" % world,
                       "oversubscribed": oversub,
                       "arith": ("fp32 storage; contraction %s with fp32 TMEM accumulation" % (
                           "F16X3 (scaled fp16 hi/lo split, 3 products, kind::f16) on tcgen05"
                           if gemm_name == "tcgen05_f16x3" else "3xTF32 on tcgen05"
                           if gemm_name == "tcgen05_3xtf32" else "FFMA"))},
            "roofline": roofline,
            "layer_roofline_frac": layer_frac,
            "stages": stages,
            "sweep": sweep,
            "planner": plan_report,
            "matmul_peaks": mm_peaks,
            "cpu_baseline": cpu,
            "cpu_direct_fp32": cpu_fp32,
            "clocks": clk,
            "e2e": e2e,
            "gpu_launches": plan.launches * args.steps * world,
            "gpu_launches_per_rank": plan.launches * args.steps,
        }
        line.update(extras)
        print(json.dumps(line), flush=True)
    parallel.barrier()


def run_eshard(args, fc, parallel, base, gcfg, cfg, I_all_shape, x, w, dev, stream, timer_fn, job_flops, rank, world,
               oversub, clocks, nvml, flush, io_bytes):
    """Element-sharded mode: rank k owns the transformed elements
    parallel.shard_range(E, k, N) of every image and the transforms of its own images; one
    step = forward_a (NK1 on own elements, NK2, U pack) -> all-to-all U + all-gather of the
    per-image maxima -> forward_b (NK3) -> all-to-all X -> forward_c (NK4), timed with CUDA
    events around the whole step (collectives included), max over ranks."""
    import torch
    if args.method == "auto" or args.method == "direct":
        raise SystemExit("--mode eshard needs --method winograd|regular_fft|gauss_fft and --m")
    batch = [hi - lo for lo, hi in (parallel.shard_range(gcfg.B, k, world) for k in range(world))]
    es = fc.EShard(world, rank, batch, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, args.method, args.m, args.gemm)
    ws = es.alloc_workspace(dev)
    out = torch.empty(es.out_shape, device=dev)
    host = oversub or not torch.distributed.is_initialized() or torch.distributed.get_backend() != "nccl"
    fwd = parallel.eshard_forward_p2p if args.exchange == "p2p" else parallel.eshard_forward
    bufs = fwd(es, x, w, out, ws, host_staging=host and world > 1)
    for _ in range(args.warmup):
        fwd(es, x, w, out, ws, bufs, host_staging=host and world > 1)
    torch.cuda.synchronize()
    parallel.barrier()
    t0 = time.time()
    total, per = timer_fn.run(args.steps, lambda: fwd(es, x, w, out, ws, bufs, host_staging=host and world > 1))
    torch.cuda.synchronize()
    parallel.barrier()
    t1 = time.time()
    rank_ms = total / args.steps
    ms = parallel.max_over_ranks(rank_ms, dev if not oversub else None)
    per_rank = parallel.all_gather_scalar(rank_ms, dev if not oversub else None)
    clk = nvml.merge(clocks.summary(t0, t1))
    clocks.stop()
    if rank == 0:
        line = {"metric": METRIC, "value": job_flops / (ms * 1e-3) / 1e12, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "ms_per_step_stats": {"per_rank_ms": per_rank},
                "config": {"workload": base.name, "global_batch": gcfg.B, "B_per_gpu": cfg.B, "C": cfg.C,
                           "Cout": cfg.Cout, "H": cfg.H, "W": cfg.W, "r": cfg.r, "method": args.method, "m": args.m,
                           "gemm": fc.GEMM_NAMES.get(es.info["gemm"], args.gemm),
                           "parallelism": "es%d (element-sharded: elements [e0, e1) of every image per rank; %s)" % (
                               world, ("U and X copied into the peers' IPC-mapped receive buffers, all-gather of "
                                       "per-image maxima" if args.exchange == "p2p" else
                                       "all-to-all of U and X, all-gather of per-image maxima" +
                                       (", staged through the host (gloo)" if host and world > 1 else
                                        ", NCCL" if world > 1 else ""))),
                           "exchange": args.exchange,
                           "elements_per_rank": es.e_count, "E": es.info["E"],
                           "bytes_exchanged_per_rank": {"u_send": sum(es.u_send), "x_send": sum(es.x_send)},
                           "l2": "flushed between steps" if flush else "no flush (%.0f MB/GPU)" % (io_bytes / 1e6),
                           "oversubscribed": oversub},
                "clocks": clk, "e2e": None, "gpu_launches": None}
        print(json.dumps(line), flush=True)
    parallel.barrier()


def stage_rooflines(info, stage_ms, nst, hbm_peak, c_peak, cfg):
    names = ["NK1 kernel transform", "NK2 input transform", "NK3 contraction", "NK4 output transform"]
    stages = []
    for s in range(nst):
        tsec = stage_ms[s] * 1e-3
        if nst == 4 and s == 2 and c_peak:
            # the binding roofline of the contraction: max(FLOPs / tensor ceiling, bytes / HBM)
            flops, byts = info["alg_flops"][2], info["alg_bytes"][2]
            t_tc, t_hbm = flops / (c_peak * 1e12), byts / (hbm_peak * 1e9)
            tens = {"tensor_tflops": flops / tsec / 1e12, "tensor_peak": c_peak,
                    "tensor_frac": flops / tsec / 1e12 / c_peak, "hbm_gbs": byts / tsec / 1e9,
                    "hbm_frac": byts / tsec / 1e9 / hbm_peak}
            if t_tc >= t_hbm:
                stages.append(dict({"kernel": names[s], "ms": stage_ms[s], "bound": "tensor",
                                    "achieved": flops / tsec / 1e12, "peak": c_peak, "unit": "TFLOP/s",
                                    "frac": flops / tsec / 1e12 / c_peak}, **tens))
            else:
                stages.append(dict({"kernel": names[s], "ms": stage_ms[s], "bound": "hbm",
                                    "achieved": byts / tsec / 1e9, "peak": hbm_peak, "unit": "GB/s",
                                    "frac": byts / tsec / 1e9 / hbm_peak}, **tens))
        elif nst == 4:
            ach = info["alg_bytes"][s] / tsec / 1e9
            stages.append({"kernel": names[s], "ms": stage_ms[s], "bound": "hbm", "achieved": ach,
                           "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak})
        else:
            ach = cfg.direct_flops / tsec / 1e12
            stages.append({"kernel": "NK5 direct", "ms": stage_ms[s], "bound": "alu", "achieved": ach,
                           "peak": None, "unit": "TFLOP/s", "frac": None})
    return stages


def layer_roofline_frac(info, hbm_peak, c_peak, ms):
    """Whole-layer stage-sum roofline (paper Eq. running-time) / measured time."""
    t_roof = 0.0
    for s in range(4):
        tb = info["alg_bytes"][s] / (hbm_peak * 1e9)
        tc = info["alg_flops"][s] / (c_peak * 1e12) if (s == 2 and c_peak) else 0.0
        t_roof += max(tb, tc)
    return (t_roof * 1e3) / ms


def run_extras(args, fc, cfg, plan, x, w, out, ws, stream, timer_fn, job_flops, world, dev, oversub, hbm_peak,
               contraction_peak_of, method, m, parallel):
    """Secondary measurements on the same rank-local layer and protocol: the 3xTF32 arm (the
    north_star's arithmetic), inference with cached weight transforms, a CUDA-graph replay."""
    import torch
    red = dev if not oversub else None
    res = {}
    # ---- 3xTF32 contraction arm (same config, method, m and protocol) ------------------
    try:
        p3 = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m, "tcgen05")
        ws3 = p3.alloc_workspace(dev)
        for _ in range(args.warmup):
            p3.forward(x, w, out, ws3)
        torch.cuda.synchronize()
        parallel.barrier()
        n3 = max(20, args.steps // 5)
        t3, _ = timer_fn.run(n3, lambda: p3.forward(x, w, out, ws3))
        ms3 = parallel.max_over_ranks(t3 / n3, red)
        prof = [p3.forward_profiled(x, w, out, ws3) for _ in range(3)]
        st3 = [min(p_[s] for p_ in prof) for s in range(4)]
        # the contraction's roofline is filled in once the tensor peaks are measured (main())
        res["arm_3xtf32"] = {"ms_per_step": ms3, "value": job_flops / (ms3 * 1e-3) / 1e12, "unit": UNIT,
                             "method": method, "m": m, "stage_ms": [round(v, 4) for v in st3],
                             "_info": p3.info, "contraction_info": p3.info, "ms_rank": t3 / n3}
        del ws3, p3
        torch.cuda.empty_cache()
    except Exception as exc:  # reported, never fatal to the bench line
        res["arm_3xtf32"] = {"error": str(exc)[:200]}
    # ---- inference with cached weight transforms (NK1 once, NK2-4 per call) -------
    ws_c = plan.alloc_workspace(dev)
    plan.transform_weights(w, ws_c)
    for _ in range(3):
        plan.forward_cached(x, ws_c, out)
    torch.cuda.synchronize()
    nc = max(10, args.steps // 5)
    tc_, _ = timer_fn.run(nc, lambda: plan.forward_cached(x, ws_c, out))
    cms = parallel.max_over_ranks(tc_ / nc, red)
    res["inference_cached_weights"] = {"ms_per_step": cms, "value": job_flops / (cms * 1e-3) / 1e12, "unit": UNIT,
                                       "api": "conv_transform_weights once + conv_forward_cached (NK2-NK4) per step"}
    del ws_c
    # ---- the same forward replayed as a CUDA graph of 10 steps (conv_graph_*) --------
    try:
        gr = plan.capture(x, w, out, ws, steps=10)
        for _ in range(2):
            gr.launch(stream)
        torch.cuda.synchronize()
        ng = max(5, args.steps // 10)
        tg, _ = timer_fn.run(ng, lambda: gr.launch(stream))
        gms = parallel.max_over_ranks(tg / (10 * ng), red)
        res["cuda_graph"] = {"ms_per_step": gms, "value": job_flops / (gms * 1e-3) / 1e12, "unit": UNIT,
                             "api": "conv_graph_create(steps=10) once + conv_graph_launch per 10 steps"}
        del gr
    except Exception as exc:
        res["cuda_graph"] = {"error": str(exc)[:200]}
    return res


if __name__ == "__main__":
    main()
