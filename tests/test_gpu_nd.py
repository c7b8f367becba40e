"""N-dimensional and non-isotropic layers on the CUDA path (conv_plan_nd; PAPER.md P:926-929:
"an arbitrary number of dimensions, as well as non-isotropic kernels") against the N-D fp64
oracle (oracle.conv_nd_fp64), every method x contraction mode, with ragged tiles on every
axis.  Bars as for 2-D: FFT 1e-5, Winograd 1e-4 (5e-4 when any axis has t = 8); relative to
max|O|."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

fc = None


def setup_module(module):
    global fc
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1809_07851_b200 as _fc
    _fc.load()
    fc = _fc


def _inputs(ishape, wshape, seed):
    g = torch.Generator().manual_seed(seed)
    I = torch.randn(ishape, generator=g)
    W = torch.randn(wshape, generator=g) * (2.0 / (wshape[1] * np.prod(wshape[2:]))) ** 0.5
    return I.contiguous(), W.contiguous()


def _bar(method, ts):
    if method == "winograd":
        return 5e-4 if max(ts) >= 8 else 1e-4
    return 1e-5


CASES = [  # (input shape, kernel shape, {method: tiles})
    ((3, 8, 37), (12, 8, 3), {"winograd": (4,), "regular_fft": (14,), "gauss_fft": (9,), "direct": None}),
    ((2, 6, 29), (5, 6, 5), {"winograd": (2,), "regular_fft": (12,), "gauss_fft": (28,), "direct": None}),
    ((2, 8, 11, 19), (16, 8, 1, 3), {"winograd": (3, 4), "regular_fft": (5, 8), "gauss_fft": (4, 6),
                                     "direct": None}),
    ((2, 4, 14, 17), (8, 4, 5, 3), {"winograd": (2, 4), "regular_fft": (6, 10), "gauss_fft": (8, 7),
                                    "direct": None}),
    ((2, 8, 10, 12, 13), (16, 8, 3, 3, 3), {"winograd": (2, 4, 4), "regular_fft": (6, 6, 6),
                                            "gauss_fft": (4, 5, 6), "direct": None}),
    ((1, 5, 9, 7, 11), (6, 5, 2, 3, 4), {"winograd": (3, 2, 4), "regular_fft": (4, 5, 8), "gauss_fft": (8, 3, 5),
                                         "direct": None}),
]


@pytest.mark.parametrize("gemm", ["auto", "tcgen05", "ffma"])
@pytest.mark.parametrize("ci", range(len(CASES)))
def test_nd_parity(ci, gemm):
    ishape, wshape, runs = CASES[ci]
    I, W = _inputs(ishape, wshape, 200 + ci)
    O = oracle.conv_nd_fp64(I, W)
    x, w = I.cuda(), W.cuda()
    B, C = ishape[:2]
    for method, m in runs.items():
        if method == "direct" and gemm != "auto":
            continue
        p = fc.Plan.nd(B, C, wshape[0], ishape[2:], wshape[2:], method, m, gemm if method != "direct" else "auto")
        assert p.out_shape == O.shape
        y = p.forward(x, w)
        torch.cuda.synchronize()
        err = float(np.abs(y.cpu().double().numpy() - O).max() / np.abs(O).max())
        ts = p.info["t_shape"]
        print("ND %s %s m=%s %s err=%.2e" % (ishape, method, m, gemm, err))
        assert err <= (1e-5 if method == "direct" else _bar(method, ts)), (method, m, err)


def test_nd_paths_and_info():
    """The N-D plans run through the same entry points: cached weight transforms (bit-identical),
    batch chunks (bit-identical: per-image arithmetic), the pipelined host path, and the
    per-image F16X3 scale (an image 2^-24 below its batch-mate keeps its own accuracy)."""
    ishape, wshape = (4, 8, 10, 12, 13), (16, 8, 3, 3, 3)
    I, W = _inputs(ishape, wshape, 301)
    I[1] *= 2.0 ** -24
    O = oracle.conv_nd_fp64(I, W)
    x, w = I.cuda(), W.cuda()
    for method, m in (("winograd", (2, 4, 4)), ("regular_fft", (6, 6, 6)), ("gauss_fft", (4, 5, 6))):
        p = fc.Plan.nd(4, 8, 16, ishape[2:], wshape[2:], method, m)
        assert p.info["nd"] == 3
        ref = p.forward(x, w)
        ws = p.alloc_workspace()
        p.transform_weights(w, ws)
        assert torch.equal(p.forward_cached(x, ws), ref)
        pc = fc.Plan.nd(4, 8, 16, ishape[2:], wshape[2:], method, m, chunk_images=3)
        assert torch.equal(pc.forward(x, w), ref)
        hi, hw = I.pin_memory(), W.pin_memory()
        ho = torch.empty(p.out_shape).pin_memory()
        di, dw, do = torch.empty_like(x), torch.empty_like(w), torch.empty(p.out_shape, device="cuda")
        p.forward_host(hi, hw, ho, di, dw, do, ws)
        torch.cuda.synchronize()
        assert torch.equal(ho, ref.cpu())
        y = ref.cpu().double().numpy()
        for b in range(4):
            e = np.abs(y[b] - O[b]).max() / np.abs(O[b]).max()
            assert e <= _bar(method, p.info["t_shape"]), (method, b, e)
