"""Dynamic-range behaviour of the tensor-core contractions (readings R11, R16).

F16X3 scales V per output channel (s_v[c'] from max|W[c']|) and U per image
(s_u[b] from max|U_b|) by exact powers of two before the fp16 hi/lo split; 3xTF32
splits in the fp32 exponent range.  Both are therefore exactly equivariant under
power-of-two rescaling of the inputs, and F16X3 keeps every output channel
accurate relative to its own magnitude however different the channels' scales are.
"""
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


RUNS = [("winograd", 2), ("winograd", 4), ("winograd", 6), ("regular_fft", 6), ("gauss_fft", 8)]


def _bar(method, m, r):
    if method == "winograd":
        return 5e-4 if m + r - 1 >= 8 else 1e-4
    return 1e-5


def _run(I, W, method, m, gemm):
    p = fc.Plan(I.shape[0], I.shape[1], W.shape[0], I.shape[2], I.shape[3], W.shape[2], method, m, gemm)
    y = p.forward(I.cuda(), W.cuda())
    torch.cuda.synchronize()
    return y.cpu()


@pytest.mark.parametrize("gemm", ["f16x3", "tcgen05"])
@pytest.mark.parametrize("method,m", RUNS)
@pytest.mark.parametrize("ki,kw", [(60, -40), (-50, 30), (90, -60), (-30, -30)])
def test_power_of_two_equivariance_is_exact(method, m, gemm, ki, kw):
    """conv(2^a I, 2^b W) == 2^(a+b) conv(I, W) bit for bit: every scale the contraction
    chooses moves with the data, and no fp32 / fp16 intermediate leaves its normal range."""
    cfg = synth.custom(2, 24, 40, 20, 19, 3, seed=91, dist="normal")
    I, W = synth.make_inputs(cfg)
    y0 = _run(I, W, method, m, gemm)
    y1 = _run(I * 2.0 ** ki, W * 2.0 ** kw, method, m, gemm)
    assert torch.equal(y1, y0 * 2.0 ** (ki + kw)), (method, m, gemm, ki, kw)


@pytest.mark.parametrize("method,m", RUNS)
def test_output_channels_of_wildly_different_scale(method, m):
    """Rows of W scaled by 2^-60 .. 2^60 (and one all-zero row): with per-c' scales each
    output channel meets the bar relative to its own maximum."""
    cfg = synth.custom(2, 16, 12, 18, 18, 3, seed=92, dist="normal")
    I, W = synth.make_inputs(cfg)
    f = torch.tensor([2.0 ** k for k in (-60, -30, -12, 0, 7, 20, 40, 60, -1, 3, 1, 0)], dtype=torch.float32)
    f[-1] = 0.0  # a zero output channel
    Ws = (W * f[:, None, None, None]).contiguous()
    O = oracle.conv_fp64(I, Ws)
    y = _run(I, Ws, method, m, "f16x3").double().numpy()
    assert np.all(y[:, -1] == 0.0)
    for co in range(cfg.Cout - 1):
        ref = O[:, co]
        err = np.abs(y[:, co] - ref).max() / np.abs(ref).max()
        assert err <= _bar(method, m, cfg.r), (method, m, co, err)


@pytest.mark.parametrize("method,m", RUNS)
def test_input_channels_of_different_scale(method, m):
    """Half the input channels 2^-20 smaller: one per-forward s_u serves them all; the error
    stays within the bar relative to max|O| (small channels lose only absolute precision
    below 2^-25 of the scaled range, R16)."""
    cfg = synth.custom(2, 16, 8, 20, 20, 3, seed=93, dist="normal")
    I, W = synth.make_inputs(cfg)
    I[:, ::2] *= 2.0 ** -20
    O = oracle.conv_fp64(I, W)
    y = _run(I, W, method, m, "f16x3").double().numpy()
    err = np.abs(y - O).max() / np.abs(O).max()
    assert err <= _bar(method, m, cfg.r), (method, m, err)


def test_f16x3_not_less_accurate_than_3xtf32():
    """On the VGG-3.2 shape (2 images) F16X3's error is at most 3xTF32's, per method."""
    cfg = synth.CONFIGS["vgg3_2"]
    I, W = synth.make_inputs(cfg)
    I = I[:2].contiguous()
    O = oracle.conv_fp64(I, W)
    for method, m in (("winograd", 4), ("regular_fft", 14), ("gauss_fft", 14)):
        e = {}
        for gemm in ("f16x3", "tcgen05"):
            y = _run(I, W, method, m, gemm).double().numpy()
            e[gemm] = np.abs(y - O).max() / np.abs(O).max()
        print(method, m, e)
        assert e["f16x3"] <= 1.25 * e["tcgen05"], (method, m, e)


@pytest.mark.parametrize("shape", [(2, 24, 64, 20, 19, 3), (3, 16, 160, 18, 18, 3), (2, 32, 96, 17, 23, 5),
                                   (1, 8, 32, 12, 12, 3)])
@pytest.mark.parametrize("m", [2, 6, 9])
def test_gauss_epilogue_combine_equals_three_planes(shape, m):
    """with C' % 32 == 0 the F16X3 contraction stores Re = T1 - T3 and
    Im = T1 + T2 instead of T1, T2, T3.  Scaling by 1/(s_u s_v) is a power of
    two, so combining before or after it rounds identically: the output equals the
    three-plane path (gauss_combine = 0) bit for bit, and meets the oracle bar."""
    cfg = synth.custom(*shape, seed=94, dist="normal")
    I, W = synth.make_inputs(cfg)
    p = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, "gauss_fft", m, "f16x3", gauss_combine=1)
    assert p.info["x_planes"] == 2
    y = p.forward(I.cuda(), W.cuda()).cpu()
    p3 = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, "gauss_fft", m, "f16x3", gauss_combine=0)
    assert p3.info["x_planes"] == 3 and p3.info["bytes_X"] * 2 == p.info["bytes_X"] * 3
    y3 = p3.forward(I.cuda(), W.cuda()).cpu()
    torch.cuda.synchronize()
    assert torch.equal(y, y3)
    O = oracle.conv_fp64(I, W)
    err = np.abs(y.double().numpy() - O).max() / np.abs(O).max()
    assert err <= 1e-5, err


@pytest.mark.parametrize("gemm", ["f16x3", "tcgen05", "ffma"])
@pytest.mark.parametrize("method,m", [("winograd", 4), ("winograd", 6), ("regular_fft", 6), ("regular_fft", 14),
                                      ("gauss_fft", 8)])
def test_per_image_precision_and_batch_independence(method, m, gemm):
    """The F16X3 U scale is per image (NK2 reduces max|U_b| per image b): images 2^-20 and
    2^-30 below their batch-mates each meet the bar against their OWN max|O_b|, and every
    image's output is bit-identical to the image convolved alone (batch of one) -- so
    batch sharding and chunking change no arithmetic.  Images span several
    128-tile blocks and share blocks with their neighbours (N = 100 tiles at m = 2)."""
    cfg = synth.custom(4, 32, 64, 22, 22, 3, seed=95, dist="normal")
    I, W = synth.make_inputs(cfg)
    I[1] *= 2.0 ** -20
    I[2] *= 2.0 ** -30
    I[3] *= 2.0 ** 12
    y = _run(I, W, method, m, gemm)
    O = oracle.conv_fp64(I, W)
    bar = _bar(method, m, cfg.r)
    for b in range(cfg.B):
        e = np.abs(y[b].double().numpy() - O[b]).max() / np.abs(O[b]).max()
        assert e <= bar, (b, e)
        yb = _run(I[b:b + 1].contiguous(), W, method, m, gemm)
        assert torch.equal(yb[0], y[b]), b
