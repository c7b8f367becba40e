#!/usr/bin/env python
"""A/B per-stage timing of experiment builds of the library (not the bench contract line;
bench.py is).  The round-2 transform experiments in DESIGN.md §11 were measured with it.

Build a variant with compile-time switches into expt/ (git-ignored, travels with gpurun):

    python -c "from paper_1809_07851_b200 import _build; _build.build(extra_flags=['-DX=1'], out='expt/lib_x.so')"

then time the product library against every expt/*.so on (config, method, m) cases:

    AB_CASES=vgg1_2:regular_fft:25,k5:regular_fft:14 python tools/ab_stages.py [lib]

Per case and library: per-stage ms (min of 8 conv_forward_profiled runs, NK1 not
overlapped with NK2 so each stage is timed alone), the fraction of the measured HBM copy
peak, and max|out - ref| / max|ref| on up to 4 images against an fp64 torch conv2d on the
host (a smoke check of the variant; the parity tests are tests/test_gpu_*.py).  With a
library argument only that library runs (one process per library: ctypes cannot unload).
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CASES = [c.split(":") for c in os.environ.get("AB_CASES", "").split(",") if c]
HBM_GBS = 6534.5  # measured copy peak (MEASURED_PEAKS.json on the pool's B200s)


def child(lib: str) -> None:
    from paper_1809_07851_b200 import _build
    if lib != "product":
        _build.LIB = os.path.abspath(lib)
    import torch
    import synth
    import paper_1809_07851_b200 as fc
    for name, method, m in CASES:
        cfg = synth.CONFIGS[name]
        I, W = synth.make_inputs(cfg)
        x, w = I.cuda(), W.cuda()
        p = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, int(m), "auto",
                    overlap_kernel_transform=0)
        ws = p.alloc_workspace()
        out = torch.empty(p.out_shape, device="cuda")
        for _ in range(3):
            p.forward(x, w, out, ws)
        torch.cuda.synchronize()
        idx = torch.tensor(sorted({0, 1 % cfg.B, max(cfg.B - 2, 0), cfg.B - 1}), device="cuda")
        ref = torch.nn.functional.conv2d(x[idx].double().cpu(), w.double().cpu()).cuda()
        err = ((out[idx].double() - ref).abs().max() / ref.abs().max()).item()
        del ref
        prof = [p.forward_profiled(x, w, out, ws) for _ in range(8)]
        st = [min(q[s] for q in prof) for s in range(4)]
        ab = p.info["alg_bytes"]
        print(json.dumps({"lib": os.path.basename(lib), "case": "%s/%s/%s" % (name, method, m),
                          "ms": [round(v * 1000, 1) for v in st], "err4": float("%.3g" % err),
                          "frac": [round(ab[s] / (st[s] * 1e-3) / (HBM_GBS * 1e9), 3) if st[s] > 0 else None
                                   for s in range(4)]}), flush=True)
        del p, ws, out, x, w
        torch.cuda.empty_cache()


if __name__ == "__main__":
    if len(sys.argv) > 1:
        child(sys.argv[1])
    else:
        d = os.path.join(ROOT, "expt")
        libs = sorted(os.path.join(d, f) for f in os.listdir(d) if f.endswith(".so")) if os.path.isdir(d) else []
        for lib in ["product"] + libs:
            subprocess.run([sys.executable, __file__, lib])
