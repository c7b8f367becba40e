"""CPU-only checks of the product's host side: the C-ABI library loads and exports
every function include/fastconv.h declares; argument validation; plan geometry
(PAPER.md P:956-965); algorithmic byte/FLOP counts (Table
layer-stuff); the exact Winograd matrices (Eq. 1)."""
import ctypes
from fractions import Fraction

import numpy as np
import pytest

import paper_1809_07851_b200 as fc


@pytest.fixture(scope="module")
def lib():
    from paper_1809_07851_b200 import _build
    _build.build()
    return fc.load()


def test_exports_every_header_symbol(lib):
    names = fc.header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    # the binding wires exactly these names
    for n in ("conv_plan", "conv_forward", "conv_destroy", "conv_plan_query", "conv_workspace_bytes"):
        assert n in names


def test_status_strings(lib):
    for k, v in fc.STATUS.items():
        assert lib.conv_status_string(k).decode() == v
    assert lib.conv_status_string(99).decode() == "CONV_ERR_UNKNOWN"
    lib.conv_destroy(None)  # NULL-safe


@pytest.mark.parametrize("args,status", [
    ((0, 4, 4, 16, 16, 3, "winograd", 2), 1),
    ((1, 4, 4, 2, 16, 3, "winograd", 2), 1),      # H < r
    ((1, 4, 4, 16, 16, 3, "regular_fft", -1), 1),  # m < 0 (m = 0: the planner picks)
    ((1, 4, 4, 16, 16, 3, "winograd", 7), 2),     # t = 9 > 8
    ((1, 4, 4, 16, 16, 1, "winograd", 4), 2),     # r < 2
    ((1, 4, 4, 99, 99, 3, "regular_fft", 63), 2),  # t = 65 > 64
])
def test_plan_query_rejects(lib, args, status):
    with pytest.raises(fc.ConvError) as ei:
        fc.plan_query(*args)
    assert ei.value.status == status


def test_direct_ignores_m(lib):
    info = fc.plan_query(2, 3, 4, 10, 10, 3, "direct", -5)
    assert info["Ho"] == 8 and info["workspace_bytes"] == 0


@pytest.mark.parametrize("x,r,m,t,N", [(58, 3, 4, 6, 196), (6, 3, 4, 6, 1), (7, 3, 4, 6, 4),
                                       (58, 3, 14, 16, 16), (31, 5, 27, 31, 1), (16, 3, 7, 9, 4),
                                       (226, 3, 25, 27, 81)])
def test_geometry(lib, x, r, m, t, N):
    # N = ceil((x-r+1)/m)^2; SPEC S:46-48 worked examples for the first three
    for method in ("winograd", "regular_fft", "gauss_fft"):
        if method == "winograd" and t > 8:
            continue
        info = fc.plan_query(2, 3, 5, x, x, r, method, m)
        assert info["t"] == t and info["N"] == N
        assert info["n_h"] * info["n_w"] == N
        if method == "winograd":
            assert info["E"] == t * t and info["planes"] == 1
        else:
            assert info["h"] == (t + 1 + 1) // 2 and info["E"] == t * ((t + 2) // 2)  # t*ceil((t+1)/2)
            assert info["planes"] == (2 if method == "regular_fft" else 3)
        assert info["BN"] == 2 * N and info["BN_pad"] % 128 == 0 and info["BN_pad"] >= info["BN"]


def test_half_spectrum_size_t3(lib):
    # P:1065 / SPEC S:363: t = 3 -> t * ceil((t+1)/2) = 6 stored complex numbers
    info = fc.plan_query(1, 1, 1, 5, 5, 2, "regular_fft", 2)
    assert info["t"] == 3 and info["E"] == 6


def test_rectangular_geometry(lib):
    info = fc.plan_query(1, 1, 1, 20, 33, 3, "winograd", 4)
    assert (info["n_h"], info["n_w"]) == (5, 8)


def test_algorithmic_costs_vgg32(lib):
    B, C, Co, x, r = 64, 256, 256, 58, 3
    w4 = fc.plan_query(B, C, Co, x, x, r, "winograd", 4)
    t, N = 6, 196
    assert w4["alg_bytes"][1] == pytest.approx(4 * B * C * x * x + 4 * B * C * N * t * t)
    assert w4["alg_bytes"][0] == pytest.approx(4 * C * Co * (r * r + t * t))
    assert w4["alg_bytes"][3] == pytest.approx(4 * B * Co * N * (t * t + 16))
    assert w4["alg_flops"][2] == pytest.approx(2 * t * t * B * N * C * Co)
    assert w4["direct_flops"] == pytest.approx(2 * B * C * Co * 56 * 56 * 9)
    f14 = fc.plan_query(B, C, Co, x, x, r, "regular_fft", 14)
    g14 = fc.plan_query(B, C, Co, x, x, r, "gauss_fft", 14)
    th = 16 * 9
    assert f14["alg_flops"][2] == pytest.approx(8 * th * B * 16 * C * Co)
    assert g14["alg_flops"][2] == pytest.approx(6 * th * B * 16 * C * Co)
    assert g14["alg_bytes"][1] - 4 * B * C * x * x == pytest.approx(1.5 * (f14["alg_bytes"][1] - 4 * B * C * x * x))
    # X planes: on VGG-3.2 the stage-sum model keeps Gauss's three planes (T1, T2, T3): the
    # combine's 128-column contraction tiles would cost more than the X plane saves
    assert (w4["x_planes"], f14["x_planes"], g14["x_planes"]) == (1, 2, 3)
    assert g14["alg_bytes"][2] == pytest.approx(4 * 3 * th * (B * 16 * C + C * Co + B * 16 * Co))


def test_gauss_epilogue_combine_choice(lib):
    """where the plan combines Gauss in the contraction's epilogue (X at w = 2)
    NK4 moves what Regular-FFT's does and NK3 writes 2/3 of the three-plane X."""
    B, C, Co, x, r, th = 64, 64, 64, 226, 3, 16 * 9  # VGG-1.2, m = 14: HBM-bound, combined
    g = fc.plan_query(B, C, Co, x, x, r, "gauss_fft", 14)
    f = fc.plan_query(B, C, Co, x, x, r, "regular_fft", 14)
    BN = B * 16 * 16
    assert g["x_planes"] == 2 and g["bytes_X"] == 2 * th * Co * g["BN_pad"] * 4
    assert g["alg_bytes"][3] == pytest.approx(f["alg_bytes"][3])
    assert g["alg_bytes"][2] == pytest.approx(4 * 3 * th * (BN * C + C * Co) + 4 * 2 * th * BN * Co)
    g3 = fc.plan_query(B, C, Co, x, x, r, "gauss_fft", 14, gauss_combine=0)
    assert g3["x_planes"] == 3 and g3["bytes_X"] == 3 * th * Co * g3["BN_pad"] * 4
    assert fc.plan_query(64, 256, 256, 58, 58, 3, "gauss_fft", 14, gauss_combine=1)["x_planes"] == 2
    # the combine needs the F16X3 contraction: 3xTF32 / FFMA plans keep three planes
    assert fc.plan_query(B, C, Co, x, x, r, "gauss_fft", 14, gemm="tcgen05")["x_planes"] == 3
    assert fc.plan_query(B, C, Co, x, x, r, "gauss_fft", 14, gemm="ffma", gauss_combine=1)["x_planes"] == 3
    # C' % 32 != 0: never combined
    g_odd = fc.plan_query(2, 8, 40, 20, 20, 3, "gauss_fft", 6)
    assert g_odd["x_planes"] == 3 and g_odd["bytes_X"] == 3 * g_odd["E"] * 40 * g_odd["BN_pad"] * 4


def _frac(v):
    return Fraction(v).limit_denominator(1 << 16)


@pytest.mark.parametrize("m,r", [(2, 3), (4, 3), (6, 3), (2, 5), (3, 2), (2, 2), (4, 5), (3, 4)])
def test_winograd_exact_identity(lib, m, r):
    """A^T [(G g) . (B^T d)] equals the valid correlation exactly in rationals (Eq. 1),
    and the 2-D nesting A^T[(G g G^T) . (B^T d B)]A (Eq. 4) likewise."""
    AT, BT, G = fc.winograd_matrices(m, r)
    t = m + r - 1
    AT = [[_frac(v) for v in row] for row in AT]
    BT = [[_frac(v) for v in row] for row in BT]
    G = [[_frac(v) for v in row] for row in G]
    rng = np.random.default_rng(m * 10 + r)
    for _ in range(5):
        d = [Fraction(int(v)) for v in rng.integers(-9, 10, t)]
        g = [Fraction(int(v)) for v in rng.integers(-9, 10, r)]
        Gg = [sum(G[i][j] * g[j] for j in range(r)) for i in range(t)]
        Bd = [sum(BT[i][j] * d[j] for j in range(t)) for i in range(t)]
        y = [sum(AT[i][k] * Gg[k] * Bd[k] for k in range(t)) for i in range(m)]
        assert y == [sum(g[p] * d[i + p] for p in range(r)) for i in range(m)]
    D = [[Fraction(int(v)) for v in row] for row in rng.integers(-5, 6, (t, t))]
    K = [[Fraction(int(v)) for v in row] for row in rng.integers(-5, 6, (r, r))]
    mm = lambda A, Bm: [[sum(A[i][k] * Bm[k][j] for k in range(len(Bm))) for j in range(len(Bm[0]))]
                        for i in range(len(A))]
    tr = lambda A: [list(c) for c in zip(*A)]
    GK = mm(mm(G, K), tr(G))
    BD = mm(mm(BT, D), tr(BT))
    Y = mm(mm(AT, [[GK[i][j] * BD[i][j] for j in range(t)] for i in range(t)]), tr(AT))
    ref = [[sum(K[p][q] * D[i + p][j + q] for p in range(r) for q in range(r)) for j in range(m)]
           for i in range(m)]
    assert Y == ref


def test_winograd_f23_matches_lavin_form(lib):
    # SPEC S:288 F(2,3) (Lavin form) -- equal up to the sign of the infinity row/column
    AT, BT, G = fc.winograd_matrices(2, 3)
    assert np.allclose(np.abs(BT), np.abs([[1, 0, -1, 0], [0, 1, 1, 0], [0, -1, 1, 0], [0, 1, 0, -1]]))
    assert np.allclose(G, [[1, 0, 0], [.5, .5, .5], [.5, -.5, .5], [0, 0, 1]])
    assert np.allclose(np.abs(AT), np.abs([[1, 1, 1, 0], [0, 1, -1, -1]]))


def test_winograd_matrices_reject(lib):
    with pytest.raises(fc.ConvError):
        fc.winograd_matrices(7, 3)


def test_plan_without_gpu_fails_cleanly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    st = lib.conv_plan_ex(ctypes.byref(h), 1, 4, 4, 16, 16, 3, 1, 2, 0)
    assert st == 4 and not h.value  # CONV_ERR_CUDA, no plan returned


def test_library_reads_no_environment():
    """Every plan choice comes from the arguments and conv_plan_options (no getenv in csrc/)."""
    import glob
    import os
    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1809_07851_b200", "csrc")
    for f in glob.glob(os.path.join(root, "*")):
        assert "getenv" not in open(f).read(), f


def test_plan_options_validation(lib):
    o = fc.options()
    assert (o.gemm, o.gauss_combine, o.complex_mode, o.chunk_images, o.generic_transforms, o.single_cta_mma,
            o.e2e_chunks, o.overlap_kernel_transform) == (0, -1, -1, 0, 0, 0, 0, -1)
    info = fc.PlanInfo()
    bad = fc.options(gauss_combine=2)
    assert lib.conv_plan_query_opts(1, 4, 4, 16, 16, 3, 1, 4, ctypes.byref(bad), ctypes.byref(info)) == 1
    bad = fc.options()
    bad.struct_size = 4
    assert lib.conv_plan_query_opts(1, 4, 4, 16, 16, 3, 1, 4, ctypes.byref(bad), ctypes.byref(info)) == 1
    # NULL options = defaults
    assert lib.conv_plan_query_opts(1, 4, 4, 16, 16, 3, 1, 4, None, ctypes.byref(info)) == 0
    # complex mode off: the Regular-FFT V holds the real embedding (4x the (V_r, V_i) planes' entries)
    on = fc.plan_query(64, 256, 256, 58, 58, 3, "regular_fft", 14)
    off = fc.plan_query(64, 256, 256, 58, 58, 3, "regular_fft", 14, complex_mode=0)
    assert off["bytes_V"] > on["bytes_V"]
    # batch chunks
    ch = fc.plan_query(64, 256, 256, 58, 58, 3, "winograd", 4, chunk_images=8)
    assert (ch["chunk"], ch["nchunks"]) == (8, 8)


def test_best_m_model(lib):
    """conv_plan_best_m: the paper's stage-sum model over every compiled tile,
    the argmin returned; m = 0 in conv_plan_query resolves to it."""
    for method in ("winograd", "regular_fft", "gauss_fft"):
        m, ms, cand = fc.best_m(64, 256, 256, 58, 58, 3, method)
        assert m in cand and ms == pytest.approx(min(cand.values()))
        assert all(cand[k] > ms or k >= m for k in cand)  # ties keep the smaller m
        assert fc.plan_query(64, 256, 256, 58, 58, 3, method, 0)["m"] == m
    # Winograd candidates: the compiled (t, m) pairs with t <= 8 for r = 3
    _, _, cw = fc.best_m(64, 256, 256, 58, 58, 3, "winograd")
    assert sorted(cw) == [2, 3, 4, 6]
    # FFT candidates: every codelet t <= 32
    _, _, cf = fc.best_m(64, 64, 64, 226, 226, 3, "regular_fft")
    assert sorted(k + 2 for k in cf) == [4, 5, 6, 7, 8, 9, 10, 12, 13, 14, 15, 16, 18, 20, 21, 24, 25, 27, 28, 30,
                                         31, 32]
    with pytest.raises(fc.ConvError):
        fc.best_m(1, 4, 4, 16, 16, 3, "direct")
    with pytest.raises(fc.ConvError):
        fc.plan_query(1, 4, 4, 16, 16, 3, "winograd", -1)


def test_plan_query_nd_geometry(lib):
    """conv_plan_query_nd: per-axis tiles t_d = m_d + r_d - 1, tiles per axis
    ceil((n_d - r_d + 1) / m_d), E = prod t_d (Winograd) or prod_{d<nd-1} t_d (t_last/2 + 1)
    (FFT half spectrum on the last axis), and the Table layer-stuff costs with volumes."""
    B, C, Co = 2, 8, 16
    q = fc.plan_query_nd(B, C, Co, (10, 12, 14), (3, 3, 3), "winograd", (2, 2, 4))
    assert q["nd"] == 3 and list(q["t_shape"]) == [4, 4, 6] and list(q["tiles"]) == [4, 5, 3]
    assert q["E"] == 4 * 4 * 6 and q["N"] == 60 and q["BN"] == B * 60
    assert list(q["out_shape"]) == [8, 10, 12]
    assert q["direct_flops"] == 2.0 * B * C * Co * 8 * 10 * 12 * 27
    assert q["alg_bytes"][1] == pytest.approx(4 * B * C * 10 * 12 * 14 + 4 * q["E"] * B * C * 60)
    f = fc.plan_query_nd(B, C, Co, (10, 12, 14), (3, 3, 3), "regular_fft", (6, 6, 6))
    assert f["E"] == 8 * 8 * 5 and f["planes"] == 2
    one = fc.plan_query_nd(B, C, Co, (30,), (5,), "gauss_fft", (10,))
    assert one["nd"] == 1 and one["E"] == 14 // 2 + 1 and one["N"] == 3
    # non-isotropic 2-D kernel (1 x 3): the r = 1 axis is an identity Winograd axis, t = m
    ni = fc.plan_query_nd(B, C, Co, (9, 12), (1, 3), "winograd", (3, 4))
    assert list(ni["t_shape"])[1:] == [3, 6] and ni["E"] == 18
    # nd = 2, square kernel, equal tiles: the 2-D plan itself
    assert fc.plan_query_nd(B, C, Co, (20, 20), (3, 3), "winograd", (4, 4))["E"] == \
        fc.plan_query(B, C, Co, 20, 20, 3, "winograd", 4)["E"]
    with pytest.raises(fc.ConvError):
        fc.plan_query_nd(B, C, Co, (10, 12, 14), (3, 3, 3), "winograd", (2, 2, 7))  # t = 9 > 8
    with pytest.raises(fc.ConvError):
        fc.plan_query_nd(B, C, Co, (2, 12, 14), (3, 3, 3), "regular_fft", (2, 2, 2))  # input < kernel


def test_best_method(lib):
    """conv_plan_best_method: the fastest method at its best m on the calibrated model -- the
    measured-best family on B200 for the BASELINE layers (profiles/r02j_flushed_configs.json)."""
    assert fc.best_method(64, 256, 256, 58, 58, 3)[:2] == ("winograd", 4)      # VGG-3.2
    assert fc.best_method(64, 64, 64, 226, 226, 3)[:2] == ("regular_fft", 14)  # VGG-1.2
    assert fc.best_method(128, 96, 256, 31, 31, 5)[0].endswith("fft")         # 5x5
    assert fc.best_method(64, 512, 512, 16, 16, 3)[:2] == ("winograd", 4)      # deep


def test_fused_option_query():
    """conv_plan_options.fused: eligible only for 2-D Winograd F(2,3) with the
    3xTF32 contraction; the plan then has no U / X in its workspace and one fused stage carrying
    input + V + output bytes (the transforms' element-wise FLOPs are unchanged)."""
    B, C, Co, x = 4, 64, 64, 58
    staged = fc.plan_query(B, C, Co, x, x, 3, "winograd", 2, "tcgen05")
    fused = fc.plan_query(B, C, Co, x, x, 3, "winograd", 2, "auto", fused=1)
    assert staged["fused"] == 0 and fused["fused"] == 1
    assert fused["gemm"] == fc.GEMMS["tcgen05"]  # AUTO resolves to 3xTF32 for fused plans
    assert fused["bytes_U"] == 0 and fused["bytes_X"] == 0 and fused["x_planes"] == 0
    assert fused["workspace_bytes"] < staged["workspace_bytes"]
    assert fused["alg_bytes"][1] == 0 and fused["alg_bytes"][3] == 0
    Ho = x - 2
    assert fused["alg_bytes"][2] == 4.0 * (B * C * x * x + 16 * C * Co + B * Co * Ho * Ho)
    assert fused["alg_flops"][2] == staged["alg_flops"][2]
    for bad in (dict(method="winograd", m=4), dict(method="regular_fft", m=6), dict(method="gauss_fft", m=6)):
        with pytest.raises(fc.ConvError):
            fc.plan_query(B, C, Co, x, x, 3, bad["method"], bad["m"], "auto", fused=1)
    with pytest.raises(fc.ConvError):  # F16X3 / FFMA contractions, chunking, other kernel sizes
        fc.plan_query(B, C, Co, x, x, 3, "winograd", 2, "f16x3", fused=1)
    with pytest.raises(fc.ConvError):
        fc.plan_query(B, C, Co, x, x, 3, "winograd", 2, "ffma", fused=1)
    with pytest.raises(fc.ConvError):
        fc.plan_query(B, C, Co, x, x, 3, "winograd", 2, "auto", fused=1, chunk_images=2)
    with pytest.raises(fc.ConvError):
        fc.plan_query(B, C, Co, x, x, 5, "winograd", 2, "auto", fused=1)
    with pytest.raises(fc.ConvError):  # out of range
        fc.plan_query(B, C, Co, x, x, 3, "winograd", 2, "auto", fused=2)


def test_peer_exchange_arg_checks(lib):
    """conv_eshard_forward_*_peer and conv_ipc_*: argument errors come back as statuses before any
    device work (no GPU needed)."""
    import ctypes
    vp = ctypes.c_void_p
    arr = (vp * 2)(None, None)
    assert lib.conv_eshard_forward_a_peer(None, None, None, None, None, None, 0, None) == 1
    assert lib.conv_eshard_forward_a_peer(None, None, None, arr, None, None, 0, None) == 1  # NULL plan
    assert lib.conv_eshard_forward_b_peer(None, None, None, None, None, 0, None) == 1
    p = vp()
    h = (ctypes.c_char * 64)()
    assert lib.conv_ipc_alloc(0, ctypes.byref(p), h) == 1
    assert lib.conv_ipc_alloc(16, None, h) == 1
    assert lib.conv_ipc_open(None, ctypes.byref(p)) == 1
    assert lib.conv_ipc_free(None) == 0 and lib.conv_ipc_close(None) == 0  # NULL-safe
