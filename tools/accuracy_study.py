#!/usr/bin/env python
"""Accuracy of every method and tile size against the fp64 oracle (the paper's
accuracy discussion; SURVEY 8(f) row 4 for 8x8 Winograd
tiles).  Reduced BASELINE configs (1-2 images, full channels and image size),
max-abs error / max|O| (the north_star metric) and relative L2 error (SPEC's).
Writes profiles/<tag>_accuracy.json.  Test-infrastructure use of oracle/."""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_1809_07851_b200 as fc  # noqa: E402

RUNS = {"winograd": (2, 3, 4, 5, 6), "regular_fft": (2, 4, 6, 8, 14, 22, 30), "gauss_fft": (6, 14, 30),
        "direct": (0,)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--gemm", default="auto", choices=["auto", "f16x3", "tcgen05", "ffma"])
    ap.add_argument("--out", default=None, help="also copy the JSON here (e.g. gpurun_out/)")
    args = ap.parse_args()
    fc.load()
    out = {}
    for name, nb in (("tiny", 1), ("vgg3_2", 2), ("k5", 2), ("deep", 2)):
        cfg = synth.CONFIGS[name]
        I, W = synth.make_inputs(cfg)
        I = I[:nb].contiguous()
        O = oracle.conv_fp64(I, W)
        x, w = I.cuda(), W.cuda()
        res = {}
        for method, ms in RUNS.items():
            for m in ms:
                t = m + cfg.r - 1
                if method == "winograd" and (t > 8 or m < 2):
                    continue
                if method != "direct" and (t > 64 or m > cfg.Ho):
                    continue
                p = fc.Plan(nb, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m,
                            args.gemm if method != "direct" else "auto")
                y = p.forward(x, w).double().cpu().numpy()
                res["%s/m=%d" % (method, m)] = {
                    "t": t, "max_rel": float(np.abs(y - O).max() / np.abs(O).max()),
                    "l2_rel": float(np.linalg.norm(y - O) / np.linalg.norm(O))}
        out[name] = res
        print(name, {k: "%.2e" % v["max_rel"] for k, v in res.items()}, flush=True)
    out["_gemm"] = args.gemm
    path = os.path.join(ROOT, "profiles", "%s_accuracy_%s.json" % (args.tag, args.gemm))
    json.dump(out, open(path, "w"), indent=1)
    if args.out:
        json.dump(out, open(os.path.join(args.out, os.path.basename(path)), "w"), indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
