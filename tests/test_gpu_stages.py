"""Stage-level checks of NK1 / NK2 / NK3 / NK4 on the GPU against fp64 NumPy
stage models (test aids built from library routines: numpy.fft.rfft2 per tile,
the plan's exact Winograd matrices, numpy matmul).  They localise a failing
stage; the end-to-end oracle parity lives in test_gpu_parity.py."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1809_07851_b200 as m
    m.load()
    return m


def _tiles(I, m, r, n_h, n_w):
    """[B][C][N][t][t] zero-padded overlapping tiles."""
    B, C, H, W = I.shape
    t = m + r - 1
    P = np.zeros((B, C, n_h * m + r - 1, n_w * m + r - 1))
    P[:, :, :H, :W] = I
    T = np.empty((B, C, n_h * n_w, t, t))
    for i in range(n_h):
        for j in range(n_w):
            T[:, :, i * n_w + j] = P[:, :, i * m:i * m + t, j * m:j * m + t]
    return T


def _ws_view(ws, off, count):
    return ws[off:off + 4 * count].view(torch.float32)


@pytest.mark.parametrize("shape", [(2, 4, 3, 16, 14, 3), (3, 72, 160, 21, 19, 3)])
@pytest.mark.parametrize("gemm", ["ffma", "tcgen05", "f16x3"])
@pytest.mark.parametrize("method,m", [("winograd", 2), ("winograd", 4), ("regular_fft", 6), ("gauss_fft", 6),
                                      ("regular_fft", 5)])
def test_stages(fc, method, m, gemm, shape):
    cfg = synth.custom(*shape, seed=41)
    I, W = synth.make_inputs(cfg)
    p = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m, gemm)
    info = p.info
    t, h, E, N, BN, BNp = info["t"], info["h"], info["E"], info["N"], info["BN"], info["BN_pad"]
    Z, M, K = info["gemm_Z"], info["gemm_M"], info["gemm_K"]
    Kp = (K + 7) // 8 * 8 if gemm == "f16x3" else (K + 3) // 4 * 4
    x, w = I.cuda(), W.cuda()
    ws = p.alloc_workspace()
    out = torch.empty(p.out_shape, device="cuda")
    p.run_stage(0, w=w, workspace=ws)
    p.run_stage(1, x=x, workspace=ws)
    torch.cuda.synchronize()
    if gemm == "f16x3":  # scaled fp16 pair: V = (V'_hi + V'_lo) / s_v[c'], s_v a power of two
        hv = lambda off: ws[off:off + 2 * Z * M * Kp].view(torch.float16).reshape(Z, M, Kp)[:, :, :K]
        Vh, Vl = hv(p.layout["V"]), hv(p.layout["Vlo"])
        vs = ws[p.layout["vscale"]:p.layout["vscale"] + 8 * cfg.Cout].view(torch.float32).cpu()
        sv, inv = vs[:cfg.Cout].double().numpy(), vs[cfg.Cout:].double().numpy()
        assert np.all(sv * inv == 1.0) and np.all(np.log2(sv) == np.round(np.log2(sv)))
        assert torch.isfinite(Vh).all() and Vh.abs().max().item() <= 2.0 ** 14
        rows = np.arange(M) % cfg.Cout
        V = (Vh.double().cpu().numpy() + Vl.double().cpu().numpy()) * inv[rows][None, :, None]
    else:
        V = _ws_view(ws, p.layout["V"], Z * M * Kp).reshape(Z, M, Kp)[:, :, :K].double().cpu().numpy()
    if gemm == "tcgen05":  # NK1 stores the 3xTF32 split: V = V_hi + V_lo, V_hi exactly TF32
        Vhi = _ws_view(ws, p.layout["V"], Z * M * Kp).reshape(Z, M, Kp)[:, :, :K].cpu()
        assert torch.all((Vhi.view(torch.int32) & 0x1FFF) == 0)
        V = V + _ws_view(ws, p.layout["Vlo"], Z * M * Kp).reshape(Z, M, Kp)[:, :, :K].double().cpu().numpy()
    # U is blocked by 128 tiles: [BN_pad / 128][Z][K][128] (fc_u_off) -> [Z][K][BN]
    U = (_ws_view(ws, p.layout["U"], Z * K * BNp).reshape(BNp // 128, Z, K, 128).permute(1, 2, 0, 3)
         .reshape(Z, K, BNp)[:, :, :BN].double().cpu().numpy())
    if gemm == "f16x3":  # NK2's per-image reduction: exactly max|U_b| (Winograd), a bound |re|+|im| (FFT)
        umax = ws[p.layout["umax"]:p.layout["umax"] + 4 * cfg.B].view(torch.float32).double().cpu().numpy()
        for b in range(cfg.B):
            ub = np.abs(U[:, :, b * N:(b + 1) * N]).max()
            if method == "winograd":
                assert umax[b] == ub, b
            else:
                assert ub <= umax[b] <= 2.0 * ub, b
    In = I.double().numpy()
    Wn = W.double().numpy()
    tiles = _tiles(In, m, cfg.r, info["n_h"], info["n_w"])  # [B][C][N][t][t]
    C, Co = cfg.C, cfg.Cout
    if method == "winograd":
        AT, BT, G = p.winograd_matrices()
        AT = np.array(AT).reshape(m, t)
        BT = np.array(BT).reshape(t, t)
        G = np.array(G).reshape(t, cfg.r)
        Uref = np.einsum("ka,xcnay,ly->klcxn", BT, tiles, BT).reshape(E, C, BN)
        Vref = np.einsum("kp,ocpq,lq->kloc", G, Wn, G).reshape(E, Co, C)
        np.testing.assert_allclose(U, Uref, atol=2e-5 * np.abs(Uref).max())
        np.testing.assert_allclose(V, Vref, atol=2e-6 * np.abs(Vref).max())
    else:
        F = np.fft.rfft2(tiles)  # [B][C][N][t][h]
        Fu = F.reshape(cfg.B, C, N, E).transpose(3, 1, 0, 2).reshape(E, C, cfg.B * N)  # [E][C][BN]
        Wpad = np.zeros((Co, C, t, t))
        Wpad[:, :, :cfg.r, :cfg.r] = Wn
        Vc = np.conj(np.fft.rfft2(Wpad)) / (t * t)  # [Co][C][t][h]
        Vc = np.moveaxis(Vc.reshape(Co, C, E), 2, 0)  # [E][Co][C]
        sc = np.abs(Fu).max()
        sv = np.abs(Vc).max()
        if method == "regular_fft":
            np.testing.assert_allclose(U[:, :C], Fu.real, atol=1e-5 * sc)
            np.testing.assert_allclose(U[:, C:], Fu.imag, atol=1e-5 * sc)
            np.testing.assert_allclose(V[:, :Co, :C], Vc.real, atol=1e-6 * sv)
            np.testing.assert_allclose(V[:, :Co, C:], -Vc.imag, atol=1e-6 * sv)
            np.testing.assert_allclose(V[:, Co:, :C], Vc.imag, atol=1e-6 * sv)
            np.testing.assert_allclose(V[:, Co:, C:], Vc.real, atol=1e-6 * sv)
        else:
            np.testing.assert_allclose(U[:E], Fu.real + Fu.imag, atol=1e-5 * sc)
            np.testing.assert_allclose(U[E:2 * E], Fu.real, atol=1e-5 * sc)
            np.testing.assert_allclose(U[2 * E:], Fu.imag, atol=1e-5 * sc)
            np.testing.assert_allclose(V[:E], Vc.real, atol=1e-6 * sv)
            np.testing.assert_allclose(V[E:2 * E], Vc.imag - Vc.real, atol=1e-6 * sv)
            np.testing.assert_allclose(V[2 * E:], Vc.real + Vc.imag, atol=1e-6 * sv)
    # NK3: X_z = V_z U_z (fp64 matmul of the same operands)
    p.run_stage(2, workspace=ws)
    torch.cuda.synchronize()
    Xref = np.matmul(V, U)
    if info["x_planes"] == 2 and method == "gauss_fft":
        # Gauss combined in NK3's epilogue: X [E][2C'][BN_pad] holds
        # Re = T1 - T3 in rows [0, C') and Im = T1 + T2 in rows [C', 2C')
        assert gemm == "f16x3" and Co % 32 == 0 and info["bytes_X"] == E * 2 * Co * BNp * 4
        Xref = np.concatenate([Xref[:E] - Xref[2 * E:], Xref[:E] + Xref[E:2 * E]], axis=1)
    X = _ws_view(ws, p.layout["X"], Xref.size // BN * BNp).reshape(Xref.shape[0], Xref.shape[1], BNp)
    X = X[:, :, :BN].double().cpu().numpy()
    np.testing.assert_allclose(X, Xref, atol=1e-5 * np.abs(Xref).max())
    # NK4 against the oracle-free direct reference through torch fp64 conv2d
    p.run_stage(3, out=out, workspace=ws)
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(I.double(), W.double()).numpy()
    np.testing.assert_allclose(out.cpu().double().numpy(), ref, atol=1e-4 * np.abs(ref).max())
