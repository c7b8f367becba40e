"""Out-of-bounds guards (compute-sanitizer is unavailable on the GPU pool): every buffer the
library touches sits inside a larger allocation whose margins hold sentinels.

* output and workspace margins must come back bit-identical (no stray writes);
* input and weight margins hold NaN, so a read past either tensor that reaches the result
  turns the output non-finite; the output must also match the oracle.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

fc = None
G = 4096  # guard floats on each side (16 KB: keeps every view 16-byte aligned)
SENT = -12345.678


def setup_module(module):
    global fc
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1809_07851_b200 as _fc
    _fc.load()
    fc = _fc


def _guarded(n, fill, dtype=torch.float32):
    buf = torch.full((n + 2 * G,), fill, dtype=dtype, device="cuda")
    return buf, buf[G:G + n]


CASES = [
    # (B, C, C', H, W, r): ragged tiles, odd sizes, C' % 32 == 0 (Gauss combine), M > 128 with
    # few tiles (128-column contraction tiles), single-CTA tiles
    (2, 5, 7, 19, 23, 3),
    (3, 16, 160, 18, 17, 3),
    (1, 24, 64, 21, 21, 5),
    (2, 8, 300, 10, 11, 3),
]
RUNS = [("winograd", 2), ("winograd", 4), ("winograd", 6), ("regular_fft", 6), ("regular_fft", 9),
        ("gauss_fft", 6), ("gauss_fft", 14), ("direct", 0)]


VARIANTS = [("auto", None), ("tcgen05", None), ("ffma", None), ("auto", "generic_transforms"),
            ("auto", "chunk_images"), ("auto", "single_cta_mma")]


@pytest.mark.parametrize("gemm,opt", VARIANTS)
@pytest.mark.parametrize("shape", CASES)
def test_no_out_of_bounds_access(shape, gemm, opt):
    opts = {opt: 1} if opt else {}  # runtime-t transforms / one-image chunks / single-CTA MMA tiles
    cfg = synth.custom(*shape, seed=97, dist="normal")
    I, W = synth.make_inputs(cfg)
    O = oracle.conv_fp64(I, W)
    for method, m in RUNS:
        if method == "winograd" and m + cfg.r - 1 > 8:
            continue
        if method == "direct" and gemm != "auto":
            continue
        p = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m, gemm if method != "direct" else "auto",
                    **opts)
        xb, x = _guarded(I.numel(), float("nan"))
        wb, w = _guarded(W.numel(), float("nan"))
        x.copy_(I.reshape(-1))
        w.copy_(W.reshape(-1))
        ob, o = _guarded(int(np.prod(p.out_shape)), SENT)
        nws = max(p.workspace_bytes, 16)
        wsb = torch.full((nws + 8 * G,), 0x5A, dtype=torch.uint8, device="cuda")
        ws = wsb[4 * G:4 * G + nws]
        y = p.forward(x.view(p.in_shape), w.view(p.w_shape), o.view(p.out_shape), ws)
        torch.cuda.synchronize()
        assert torch.all(ob[:G] == SENT) and torch.all(ob[G + o.numel():] == SENT), (method, m, "output margin")
        assert torch.all(wsb[:4 * G] == 0x5A) and torch.all(wsb[4 * G + nws:] == 0x5A), (method, m, "workspace margin")
        assert torch.isfinite(y).all(), (method, m, "read past an input")
        yn = y.double().cpu().numpy()
        err = np.abs(yn - O).max() / np.abs(O).max()
        bar = 1e-5 if method.endswith("fft") or method == "direct" else (5e-4 if m + cfg.r - 1 >= 8 else 1e-4)
        assert err <= bar, (method, m, gemm, err)
