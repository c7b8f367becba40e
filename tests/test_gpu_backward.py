"""Backward passes (conv_plan_backward) on the CUDA path against the
fp64 gradient oracles (oracle.conv_bwd_data_fp64 / conv_bwd_filter_fp64, pinned by the exact
adjoint identities and torch's fp64 autograd routines in tests/test_oracle.py).  The gradients
run through the forward pipeline on re-laid-out operands, so the forward bars apply, relative
to the gradient's max|.|: FFT 1e-5, Winograd 1e-4 (5e-4 at t = 8), direct 1e-5."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

fc = None


def setup_module(module):
    global fc
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1809_07851_b200 as _fc
    _fc.load()
    fc = _fc


def _rel(y, ref):
    return float(np.abs(y - ref).max() / np.abs(ref).max())


SHAPES = [(3, 16, 24, 20, 18, 3), (2, 8, 12, 17, 23, 5), (2, 32, 64, 30, 30, 3)]


@pytest.mark.parametrize("gemm", ["auto", "tcgen05", "ffma"])
@pytest.mark.parametrize("shape", SHAPES)
def test_backward_data(shape, gemm):
    B, C, Co, H, W, r = shape
    I, Wt = synth.make_inputs(synth.custom(*shape, seed=141, dist="normal"))
    dY = torch.randn(B, Co, H - r + 1, W - r + 1, generator=torch.Generator().manual_seed(142))
    ref = oracle.conv_bwd_data_fp64(dY, Wt, H, W)
    for method, m, bar in (("winograd", 2, 1e-4), ("winograd", 4 if r == 3 else 2, 1e-4), ("regular_fft", 8, 1e-5),
                           ("gauss_fft", 6, 1e-5), ("direct", 0, 1e-5)):
        if method == "direct" and gemm != "auto":
            continue
        p = fc.BackwardPlan("data", B, C, Co, H, W, r, method, m, gemm if method != "direct" else "auto")
        dx = p.data(dY.cuda(), Wt.cuda())
        torch.cuda.synchronize()
        err = _rel(dx.cpu().double().numpy(), ref)
        assert err <= bar, (method, m, err)


@pytest.mark.parametrize("gemm", ["auto", "tcgen05", "ffma"])
@pytest.mark.parametrize("shape", SHAPES)
def test_backward_filter(shape, gemm):
    B, C, Co, H, W, r = shape
    I, Wt = synth.make_inputs(synth.custom(*shape, seed=143, dist="normal"))
    dY = torch.randn(B, Co, H - r + 1, W - r + 1, generator=torch.Generator().manual_seed(144))
    ref = oracle.conv_bwd_filter_fp64(I, dY, r)
    for method in ("regular_fft", "gauss_fft", "direct"):
        if method == "direct" and gemm != "auto":
            continue
        p = fc.BackwardPlan("filter", B, C, Co, H, W, r, method, 0, gemm if method != "direct" else "auto")
        dw = p.filter(I.cuda(), dY.cuda())
        torch.cuda.synchronize()
        err = _rel(dw.cpu().double().numpy(), ref)
        assert err <= 1e-5, (method, err)


def test_backward_plans_reject_misuse():
    p = fc.BackwardPlan("data", 1, 4, 4, 10, 10, 3, "winograd", 2)
    x = torch.zeros(1, 4, 10, 10, device="cuda")
    with pytest.raises(fc.ConvError):
        fc.load()  # keep the library loaded
        import ctypes
        ws = p.alloc_workspace()
        st = fc.load().conv_forward(p._h, x.data_ptr(), x.data_ptr(), x.data_ptr(), ws.data_ptr(), ws.numel(),
                                    None)
        fc._check(st)
    with pytest.raises(fc.ConvError):
        fc.BackwardPlan("filter", 1, 4, 4, 10, 10, 3, "winograd", 2)
