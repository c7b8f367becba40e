#!/usr/bin/env python
"""Every BASELINE.json config on one B200: for each (method, m) the config lists,
ms/layer (CUDA events, inputs resident in HBM, warm-up first), effective direct-conv
TFLOP/s, per-stage ms, and the paper's model (planner.py) against the measurement.
Not the bench contract line (bench.py is); this writes profiles/<tag>_configs.json.

    python tools/bench_configs.py [--steps 20] [--tag r01]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--configs", default="tiny,vgg3_2,vgg1_2,k5,deep")
    ap.add_argument("--gemm", default="auto", choices=["auto", "f16x3", "tcgen05", "ffma"])
    args = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
    hbm = float(peaks["hbm_gbs"])
    # contraction ceiling of the plans' default (AUTO = F16X3): fp16 dense = bf16 dense, / 3 products
    tc = float(peaks["bf16_tflops"]) / 3.0 if args.gemm in ("auto", "f16x3") else float(peaks["bf16_tflops"]) * 0.5 / 3.0
    fc.load()
    stream = torch.cuda.current_stream()
    result = {"device": torch.cuda.get_device_name(0), "steps": args.steps, "gemm": args.gemm, "configs": {}}
    for name in args.configs.split(","):
        cfg = synth.CONFIGS[name]
        I, W = synth.make_inputs(cfg)
        x, w = I.cuda(), W.cuda()
        out = torch.empty((cfg.B, cfg.Cout, cfg.Ho, cfg.Wo), device="cuda")
        rows, infos, meas = {}, {}, {}
        for method, m in list(cfg.runs) + [("direct", 0)]:
            p = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m, args.gemm if method != "direct" else "auto")
            ws = p.alloc_workspace()
            for _ in range(3):
                p.forward(x, w, out, ws)
            steps = args.steps if method != "direct" else max(2, args.steps // 10)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(stream)
            for _ in range(steps):
                p.forward(x, w, out, ws)
            b.record(stream)
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / steps
            st = [round(v, 4) for v in p.forward_profiled(x, w, out, ws)]
            rows["%s/m=%d" % (method, m)] = {"ms": round(ms, 4), "tflops": round(cfg.direct_flops / (ms * 1e-3) / 1e12, 2),
                                            "stage_ms": st, "t": p.info["t"]}
            if method != "direct":
                infos[(method, m)] = p.info
                meas[(method, m)] = ms
            del ws, p
            torch.cuda.empty_cache()
        rep = planner.report(infos, meas, hbm, tc)
        best = min((v["ms"], k) for k, v in rows.items() if not k.startswith("direct"))
        result["configs"][name] = {"shape": dict(B=cfg.B, C=cfg.C, Cout=cfg.Cout, H=cfg.H, W=cfg.W, r=cfg.r),
                                   "direct_gflop": cfg.direct_flops / 1e9, "runs": rows, "best": best[1],
                                   "planner": rep}
        print(name, "best", best, flush=True)
        del x, w, out
        torch.cuda.empty_cache()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    path = os.path.join(ROOT, "profiles", "%s_configs.json" % args.tag)
    json.dump(result, open(path, "w"), indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
