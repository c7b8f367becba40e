#!/usr/bin/env python
"""Run one (config, method, m, gemm) forward a few times -- a short command for ncu
captures and quick per-stage timings (not the bench contract line; bench.py is).

    python tools/run_layer.py --config vgg1_2 --method regular_fft --m 25 [--iters 3] [--time]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="vgg3_2")
    ap.add_argument("--method", default="winograd")
    ap.add_argument("--m", type=int, default=4)
    ap.add_argument("--gemm", default="auto")
    ap.add_argument("--B", type=int, default=0)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--time", action="store_true", help="print per-stage ms (best of --iters profiled runs)")
    ap.add_argument("--opt", action="append", default=[], help="plan option name=value (conv_plan_options)")
    ap.add_argument("--lib", default=None, help="experiment build of the library (A/B variants)")
    args = ap.parse_args()
    if args.lib:
        from paper_1809_07851_b200 import _build
        _build.LIB = os.path.abspath(args.lib)
    cfg = synth.CONFIGS[args.config]
    if args.B:
        cfg = cfg.with_batch(args.B)
    I, W = synth.make_inputs(cfg)
    x, w = I.cuda(), W.cuda()
    opts = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in args.opt}
    p = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, args.method, args.m, args.gemm, **opts)
    ws = p.alloc_workspace()
    out = torch.empty(p.out_shape, device="cuda")
    for _ in range(args.iters):
        p.forward(x, w, out, ws)
    torch.cuda.synchronize()
    if args.time:
        prof = [p.forward_profiled(x, w, out, ws) for _ in range(max(3, args.iters))]
        st = [min(q[s] for q in prof) for s in range(4)]
        ab = p.info["alg_bytes"]
        print(json.dumps({"config": cfg.name, "method": args.method, "m": args.m, "opts": opts,
                          "stage_ms": [round(v, 4) for v in st],
                          "hbm_frac": [round(ab[s] / (st[s] * 1e-3) / 6534.5e9, 3) if st[s] > 0 else None
                                       for s in range(4)]}))


if __name__ == "__main__":
    main()
