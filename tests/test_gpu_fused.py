"""Fused NK2-NK4 Winograd F(2,3) kernel (conv_plan_options.fused) against
the fp64 oracle, every output, through the C-ABI.

The fused kernel computes the same F(2x2, 3x3) algorithm as the staged path (U = B^T d B,
3xTF32 products, Y = A^T M A) with U and X kept on chip, so the Winograd bar applies:
err = max|y - O| / max|O| <= 1e-4 (reading R10).  Shapes cover every tile-block
width the launcher picks (8, 16, 32 tiles), ragged tile blocks and ragged 2 x 2 tiles (odd
Ho / Wo), C not a multiple of the 8-channel K step, C' not a multiple of the 32-channel
block, odd W (4-byte input copies) and more tasks than SMs (the persistent loop).
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


CASES = [  # (B, C, C', H, W)
    (1, 8, 32, 18, 34),      # one tile block of 8 x 16 tiles, one K step, one channel block
    (2, 13, 40, 21, 37),     # ragged everything, odd W (4-byte copies), C' = 32 + 8
    (2, 64, 64, 30, 30),     # 14 x 14 tiles -> 16-wide blocks, several K steps
    (1, 24, 96, 58, 58),     # VGG-3.2-like 28 x 28 tiles -> 4 x 32 blocks
    (3, 16, 16, 66, 12),     # tall narrow image -> 16 x 8 blocks, C' < 32
    (1, 3, 5, 3, 3),         # single output pixel
    (4, 32, 64, 114, 114),   # 56 x 56 tiles: more tasks than SMs (persistent loop)
]


@pytest.mark.parametrize("case", CASES)
def test_fused_parity(case):
    B, C, Co, H, W = case
    cfg = synth.custom(B, C, Co, H, W, 3, seed=700 + H + W, dist="normal")
    I, Wt = synth.make_inputs(cfg)
    O = oracle.conv_fp64(I, Wt)
    p = fc.Plan(B, C, Co, H, W, 3, "winograd", 2, "auto", fused=1)
    info = p.info
    assert info["fused"] == 1 and info["gemm"] == fc.GEMMS["tcgen05"]
    assert info["bytes_U"] == 0 and info["bytes_X"] == 0
    y = p.forward(I.cuda(), Wt.cuda())
    torch.cuda.synchronize()
    err = float(np.abs(y.cpu().double().numpy() - O).max() / np.abs(O).max())
    print("FUSED %s err=%.3e" % (case, err))
    assert err <= 1e-4, err


def test_fused_paths_and_guards():
    """Cached weights and the pipelined host path give the same bits as conv_forward; NaN-filled
    outputs are fully overwritten; ineligible layers are refused with CONV_ERR_UNSUPPORTED."""
    B, C, Co, H, W = 3, 20, 48, 40, 44
    cfg = synth.custom(B, C, Co, H, W, 3, seed=777, dist="normal")
    I, Wt = synth.make_inputs(cfg)
    x, w = I.cuda(), Wt.cuda()
    p = fc.Plan(B, C, Co, H, W, 3, "winograd", 2, "tcgen05", fused=1)
    out = torch.full(p.out_shape, float("nan"), device="cuda")
    ws = p.alloc_workspace()
    p.forward(x, w, out, ws)
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()
    ref = out.clone()
    p.transform_weights(w, ws)
    assert torch.equal(p.forward_cached(x, ws), ref)
    hi, hw = I.pin_memory(), Wt.pin_memory()
    ho = torch.empty(p.out_shape).pin_memory()
    di, dw, do = torch.empty_like(x), torch.empty_like(w), torch.empty(p.out_shape, device="cuda")
    p.forward_host(hi, hw, ho, di, dw, do, ws)
    torch.cuda.synchronize()
    assert torch.equal(ho, ref.cpu())
    # each image's output is independent of its batch-mates (per-image arithmetic)
    p1 = fc.Plan(1, C, Co, H, W, 3, "winograd", 2, "auto", fused=1)
    assert torch.equal(p1.forward(x[1:2].contiguous(), w), ref[1:2])
    for bad in (dict(method="winograd", m=4, gemm="auto"), dict(method="regular_fft", m=6, gemm="auto"),
                dict(method="winograd", m=2, gemm="f16x3")):
        with pytest.raises(fc.ConvError):
            fc.Plan(B, C, Co, H, W, 3, bad["method"], bad["m"], bad["gemm"], fused=1)
    with pytest.raises(fc.ConvError):
        fc.Plan(B, C, Co, H, W, 5, "winograd", 2, "auto", fused=1)
