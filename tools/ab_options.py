#!/usr/bin/env python
"""Whole-layer time of plan-option variants (conv_plan_options), L2 flushed before every
step, per-step CUDA events, median and min of 20 steps (not the bench contract line).

    OPT_CASES="k5:regular_fft:14:,k5:regular_fft:14:complex_mode=0;single_cta_mma=1" \
        python tools/ab_options.py

Each case is config:method:m:options, options "name=value" joined by ';' (empty: defaults).
AB_LIB=expt/lib_x.so times an experiment build instead of the product library.
"""
from __future__ import annotations

import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if os.environ.get("AB_LIB"):  # an experiment build (tools/ab_stages.py) instead of the product library
    from paper_1809_07851_b200 import _build
    _build.LIB = os.path.abspath(os.environ["AB_LIB"])

import torch  # noqa: E402

import synth  # noqa: E402
import paper_1809_07851_b200 as fc  # noqa: E402


def main() -> None:
    cases = [c.split(":") for c in os.environ["OPT_CASES"].split(",") if c]
    flushbuf = torch.empty(2 * 126 * 2**20 // 4, device="cuda")
    for name, method, m, optstr in cases:
        cfg = synth.CONFIGS[name]
        I, W = synth.make_inputs(cfg)
        x, w = I.cuda(), W.cuda()
        opts = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in optstr.split(";") if kv}
        p = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, int(m), "auto", **opts)
        ws = p.alloc_workspace()
        out = torch.empty(p.out_shape, device="cuda")
        for _ in range(3):
            p.forward(x, w, out, ws)
        ts = []
        for _ in range(20):
            flushbuf.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            p.forward(x, w, out, ws)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        print(json.dumps({"lib": os.path.basename(os.environ.get("AB_LIB", "product")),
                          "case": "%s/%s/%s" % (name, method, m), "opts": opts,
                          "ms_median": round(statistics.median(ts), 4), "ms_min": round(min(ts), 4)}), flush=True)
        del p, ws, out, x, w
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
