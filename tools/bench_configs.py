#!/usr/bin/env python
"""Every BASELINE.json config on one B200 (not the bench contract line; bench.py is).

For each (method, m) -- the config's listed runs, or with ``--all-m`` every output tile
whose transforms are compiled (Winograd t <= 8, FFT t <= 32: the tile-size autotuner of
SURVEY.md 8(f) row 1) -- ms/layer (CUDA events on the launching stream, inputs resident
in HBM, warm-up first; ``--flush-l2`` writes 2x the 126 MB L2 between steps and times the
steps alone), effective direct-conv TFLOP/s, per-stage ms, and the paper's stage-sum model
(planner.py with the measured peaks; conv_plan_best_m with B200 kernel efficiencies)
against the measurement: each method's measured-best and model-best m, the speedups,
rRMSE and fitness.  Writes profiles/<tag>_configs.json.

    python tools/bench_configs.py [--steps 20] [--tag r02] [--all-m] [--flush-l2]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_1809_07851_b200 as fc  # noqa: E402
from paper_1809_07851_b200 import planner  # noqa: E402

L2_BYTES = 126 * 1024 * 1024
FFT_T = [4, 5, 6, 7, 8, 9, 10, 12, 13, 14, 15, 16, 18, 20, 21, 24, 25, 27, 28, 30, 31, 32]
# the paper's CPU-measured optimal FFT tile t per layer for the comparison
PAPER_BEST_T = {"vgg1_2": 27, "vgg3_2": 21, "deep": 9, "k5": 31}


def all_runs(cfg):
    runs = []
    if cfg.r >= 2:
        _, _, cw = fc.best_m(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, "winograd")
        runs += [("winograd", m) for m in sorted(cw)]
    for t in FFT_T:
        m = t - cfg.r + 1
        if 1 <= m <= max(cfg.Ho, cfg.Wo):
            runs += [("regular_fft", m), ("gauss_fft", m)]
    return runs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--tag", default="r02")
    ap.add_argument("--configs", default="tiny,vgg3_2,vgg1_2,k5,deep")
    ap.add_argument("--gemm", default="auto", choices=["auto", "f16x3", "tcgen05", "ffma"])
    ap.add_argument("--all-m", action="store_true", help="sweep every compiled tile size (autotuner)")
    ap.add_argument("--flush-l2", action="store_true", help="write 2x L2 between timed steps")
    ap.add_argument("--no-direct", action="store_true")
    ap.add_argument("--no-fused", action="store_true", help="skip the fused F(2,3) kernel (conv_plan_options.fused)")
    args = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
    hbm = float(peaks["hbm_gbs"])
    # contraction ceiling of the plans' default (AUTO = F16X3): fp16 dense = bf16 dense, / 3 products
    tc = float(peaks["bf16_tflops"]) / 3.0 if args.gemm in ("auto", "f16x3") else float(peaks["bf16_tflops"]) * 0.5 / 3.0
    fc.load()
    stream = torch.cuda.current_stream()
    flush_buf = torch.empty(2 * L2_BYTES // 4, device="cuda") if args.flush_l2 else None
    result = {"device": torch.cuda.get_device_name(0), "steps": args.steps, "gemm": args.gemm,
              "l2": "flushed between steps (2x126 MB), steps timed alone" if args.flush_l2 else "hot (back to back)",
              "configs": {}}
    for name in args.configs.split(","):
        cfg = synth.CONFIGS[name]
        I, W = synth.make_inputs(cfg)
        x, w = I.cuda(), W.cuda()
        out = torch.empty((cfg.B, cfg.Cout, cfg.Ho, cfg.Wo), device="cuda")
        rows, infos, meas = {}, {}, {}
        runs = all_runs(cfg) if args.all_m else list(cfg.runs)
        if not args.no_direct:
            runs.append(("direct", 0))
        if cfg.r == 3 and not args.no_fused:  # the fused F(2,3) kernel beside the rest
            runs.append(("winograd", 2, {"fused": 1}))
        for run in runs:
            method, m = run[0], run[1]
            opts = run[2] if len(run) > 2 else {}
            try:
                p = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m,
                            (args.gemm if method != "direct" else "auto") if not opts else "auto", **opts)
                ws = p.alloc_workspace()
            except (fc.ConvError, RuntimeError) as exc:  # e.g. a workspace beyond HBM
                rows["%s/m=%d%s" % (method, m, "+fused" if opts else "")] = {"error": str(exc)[:160]}
                torch.cuda.empty_cache()
                continue
            for _ in range(3):
                p.forward(x, w, out, ws)
            steps = args.steps if method != "direct" else max(2, args.steps // 10)
            torch.cuda.synchronize()
            if args.flush_l2:
                evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                       for _ in range(steps)]
                for k in range(steps):
                    flush_buf.fill_(float(k))
                    evs[k][0].record(stream)
                    p.forward(x, w, out, ws)
                    evs[k][1].record(stream)
                torch.cuda.synchronize()
                ms = sum(a.elapsed_time(b) for a, b in evs) / steps
            else:
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                for _ in range(steps):
                    p.forward(x, w, out, ws)
                b.record(stream)
                torch.cuda.synchronize()
                ms = a.elapsed_time(b) / steps
            st = [round(v, 4) for v in p.forward_profiled(x, w, out, ws)]
            key = "%s/m=%d%s" % (method, m, "+fused" if opts else "")
            rows[key] = {"ms": round(ms, 4), "tflops": round(cfg.direct_flops / (ms * 1e-3) / 1e12, 2),
                         "stage_ms": st, "t": p.info["t"]}
            if opts:
                rows[key]["options"] = opts
            if method != "direct" and not opts:
                infos[(method, m)] = p.info
                meas[(method, m)] = ms
                rows[key]["stage_hbm_frac"] = [round(p.info["alg_bytes"][s] / (st[s] * 1e-3) / (hbm * 1e9), 3)
                                               if st[s] > 0 else None for s in range(4)]
            del ws, p
            torch.cuda.empty_cache()
        rep = planner.report(infos, meas, hbm, tc)
        timed = [(v["ms"], k) for k, v in rows.items() if "ms" in v and not k.startswith("direct")]
        best = min(timed)
        entry = {"shape": dict(B=cfg.B, C=cfg.C, Cout=cfg.Cout, H=cfg.H, W=cfg.W, r=cfg.r),
                 "direct_gflop": cfg.direct_flops / 1e9, "runs": rows, "best": best[1], "planner": rep}
        # conv_plan_best_m (the library's model with B200 kernel efficiencies) per method
        entry["conv_plan_best_m"] = {}
        for method in ("winograd", "regular_fft", "gauss_fft"):
            try:
                mb, mms, cand = fc.best_m(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, args.gemm)
                mm = {m: v for (me, m), v in meas.items() if me == method}
                entry["conv_plan_best_m"][method] = {
                    "model_m": mb, "model_ms": round(mms, 4),
                    "measured_best_m": min(mm, key=mm.get) if mm else None,
                    "measured_ms_at_model_m": round(mm[mb], 4) if mb in mm else None,
                    "measured_best_ms": round(min(mm.values()), 4) if mm else None}
            except fc.ConvError:
                pass
        if name in PAPER_BEST_T:
            t = PAPER_BEST_T[name]
            mp = t - cfg.r + 1
            entry["paper_cpu_best_t"] = {"t": t, "m": mp, "cite": "P:655-660",
                                         "measured_ms_regular": rows.get("regular_fft/m=%d" % mp, {}).get("ms"),
                                         "measured_ms_gauss": rows.get("gauss_fft/m=%d" % mp, {}).get("ms")}
        result["configs"][name] = entry
        print(name, "best", best, flush=True)
        del x, w, out
        torch.cuda.empty_cache()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    path = os.path.join(ROOT, "profiles", "%s_configs.json" % args.tag)
    json.dump(result, open(path, "w"), indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
