"""Parity of the CUDA path (through the C-ABI) against the fp64 oracle.

Error metric (BASELINE.json north_star; reading R10):
    err = max |y_gpu - O| / max |O|     over the compared outputs.
Bars: Regular/Gauss-FFT <= 1e-5; Winograd t <= 6 (F(2,3), F(4,3), F(2,5)) <= 1e-4;
Winograd F(6,3) (t = 8, "6x6 output tiles", reading R9) <= 5e-4; direct <= 1e-5.

* reduced configs (full oracle, every output): each BASELINE config with its
  batch cut to 1-2 images (channels, image size, kernel and tiles kept, so the
  contraction spans several K-steps and tiles, and partial tiles are ragged);
* full BASELINE sizes, in the launch configuration bench.py times: every output
  against the full oracle tensor (cached on disk by (config, seed));
* edge cases: single output, C = 1, rectangular images, ragged tails, m > Ho,
  zero weights.
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


def tol(method, m, r):
    if method == "winograd":
        return 5e-4 if m + r - 1 >= 8 else 1e-4
    return 1e-5


GEMMS = ["ffma", "tcgen05", "f16x3"]


def _gemm_ok(gemm):
    if gemm in ("tcgen05", "f16x3"):
        try:
            fc.Plan(1, 4, 4, 8, 8, 3, "winograd", 2, gemm)
        except fc.ConvError as e:
            pytest.skip("tcgen05 path unavailable: %s" % e)


def run_gpu(I, W, method, m, gemm="auto"):
    x, w = I.cuda(), W.cuda()
    B, C, H, Wd = x.shape
    p = fc.Plan(B, C, W.shape[0], H, Wd, W.shape[2], method, m, gemm)
    y = p.forward(x, w)
    torch.cuda.synchronize()
    return y.cpu().numpy().astype(np.float64)


def rel_err(y, O):
    return float(np.abs(y - O).max() / max(np.abs(O).max(), 1e-30))


# ---------------------------------------------------------------- reduced ---
REDUCED_B = {"tiny": 1, "vgg3_2": 2, "vgg1_2": 1, "k5": 2, "deep": 2}


def _reduced_cases():
    for name, cfg in synth.CONFIGS.items():
        for (method, m) in cfg.runs + (("direct", 0),):
            yield name, method, m


_oracle_cache = {}


def _reduced(name):
    if name not in _oracle_cache:
        cfg = synth.CONFIGS[name]
        I, W = synth.make_inputs(cfg)
        I = I[:REDUCED_B[name]].contiguous()
        _oracle_cache[name] = (I, W, oracle.conv_fp64(I, W))
    return _oracle_cache[name]


@pytest.mark.parametrize("gemm", GEMMS)
@pytest.mark.parametrize("name,method,m", list(_reduced_cases()))
def test_reduced_full_oracle(name, method, m, gemm):
    if method == "direct" and gemm != "ffma":
        pytest.skip("direct path has no contraction variant")
    _gemm_ok(gemm)
    I, W, O = _reduced(name)
    y = run_gpu(I, W, method, m, gemm)
    err = rel_err(y, O)
    bar = tol(method, m, W.shape[2])
    print("%s %s m=%d %s err=%.3e (bar %.0e)" % (name, method, m, gemm, err, bar))
    assert err <= bar


# ------------------------------------------------------------- full size ---
# Every output of the four large BASELINE configs against the full oracle tensor (cached on
# disk by (config, seed), tests/oracle_cache.py), in the launch configuration bench.py times.
_full_cache = {}


def _full(name):
    if name not in _full_cache:
        _full_cache.clear()
        torch.cuda.empty_cache()
        import oracle_cache
        cfg = synth.CONFIGS[name]
        I, W, O = oracle_cache.full_output(cfg)
        Od = torch.from_numpy(np.ascontiguousarray(O)).cuda()
        _full_cache[name] = (cfg, I, W, Od, float(Od.abs().max()))
    return _full_cache[name]


def _full_cases():
    for name in ("vgg3_2", "vgg1_2", "k5", "deep"):
        cfg = synth.CONFIGS[name]
        for (method, m) in cfg.runs:
            for gemm in ("auto", "tcgen05"):
                yield name, method, m, gemm
        if cfg.r == 3:  # the fused NK2-NK4 F(2,3) kernel (conv_plan_options.fused) at full size
            yield name, "winograd", 2, "fused"


@pytest.mark.parametrize("name,method,m,gemm", list(_full_cases()))
def test_full_size_full_tensor(name, method, m, gemm):
    cfg, I, W, Od, omax = _full(name)
    if gemm == "fused":
        p = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m, "auto", fused=1)
    else:
        p = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m, gemm)  # bench.py's launch config
    y = p.forward(I.cuda(), W.cuda())
    torch.cuda.synchronize()
    assert torch.isfinite(y).all()
    err = float((y.double() - Od).abs().max()) / omax
    bar = tol(method, m, cfg.r)
    print("FULL %s %s m=%d %s err=%.3e bar=%.0e margin=%.2f" % (name, method, m, gemm, err, bar, err / bar))
    assert err <= bar
    del y


# ----------------------------------------------------------------- edges ---
EDGE = [
    ("single_output", synth.custom(1, 3, 2, 3, 3, 3, seed=21)),
    ("c1", synth.custom(2, 1, 3, 11, 9, 3, seed=22)),
    ("rect_ragged", synth.custom(3, 6, 5, 19, 33, 3, seed=23)),
    ("r5_ragged", synth.custom(2, 7, 9, 23, 17, 5, seed=24)),
    ("r2", synth.custom(2, 5, 6, 12, 12, 2, seed=25)),
    ("odd_channels", synth.custom(3, 13, 11, 20, 20, 3, seed=26)),
    ("many_cout", synth.custom(1, 8, 300, 10, 10, 3, seed=27)),
]
EDGE_RUNS = [("winograd", 2), ("winograd", 4), ("winograd", 6), ("regular_fft", 2), ("regular_fft", 5),
             ("regular_fft", 13), ("gauss_fft", 3), ("gauss_fft", 8), ("regular_fft", 40),
             ("direct", 0)]


@pytest.mark.parametrize("gemm", GEMMS)
@pytest.mark.parametrize("ename,cfg", EDGE)
def test_edge_cases(ename, cfg, gemm):
    _gemm_ok(gemm)
    I, W = synth.make_inputs(cfg)
    O = oracle.conv_fp64(I, W)
    for method, m in EDGE_RUNS:
        if method == "winograd" and (m + cfg.r - 1 > 8 or cfg.r < 2):
            continue
        if method != "winograd" and m + cfg.r - 1 > 64:
            continue
        y = run_gpu(I, W, method, m, gemm)
        err = rel_err(y, O)
        assert err <= tol(method, m, cfg.r), (ename, method, m, err)


@pytest.mark.parametrize("method,m", [("winograd", 4), ("regular_fft", 6), ("gauss_fft", 6), ("direct", 0)])
def test_zero_weights_give_zero(method, m):
    cfg = synth.CONFIGS["tiny"]
    I, W = synth.make_inputs(cfg)
    y = run_gpu(I, torch.zeros_like(W), method, m)
    assert np.all(y == 0.0)


def test_regular_vs_gauss_agree():
    cfg = synth.custom(2, 32, 16, 30, 30, 3, seed=31, dist="normal")
    I, W = synth.make_inputs(cfg)
    for m in (6, 14):
        a = run_gpu(I, W, "regular_fft", m)
        b = run_gpu(I, W, "gauss_fft", m)
        assert rel_err(a, b) <= 2e-6


def test_linearity_gpu():
    cfg = synth.custom(2, 16, 8, 20, 20, 3, seed=32, dist="normal")
    I1, W = synth.make_inputs(cfg)
    I2, _ = synth.make_inputs(cfg, seed=33)
    for method, m in (("winograd", 4), ("regular_fft", 8), ("gauss_fft", 8)):
        y = run_gpu(I1 + I2, W, method, m)
        y12 = run_gpu(I1, W, method, m) + run_gpu(I2, W, method, m)
        assert rel_err(y, y12) <= 2e-5


def test_abi_errors_on_gpu():
    cfg = synth.CONFIGS["tiny"]
    I, W = synth.make_inputs(cfg)
    x, w = I.cuda(), W.cuda()
    p = fc.Plan(1, 4, 4, 16, 16, 3, "winograd", 2)
    ws = p.alloc_workspace()
    out = torch.empty(p.out_shape, device="cuda")
    lib = fc.load()
    s = torch.cuda.current_stream().cuda_stream
    # misaligned input pointer
    st = lib.conv_forward(p._h, x.data_ptr() + 4, w.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(), s)
    assert st == 1
    # host pointer
    st = lib.conv_forward(p._h, I.data_ptr(), w.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(), s)
    assert st == 1
    # short workspace
    st = lib.conv_forward(p._h, x.data_ptr(), w.data_ptr(), out.data_ptr(), ws.data_ptr(), 16, s)
    assert st == 1
    # NULL output
    st = lib.conv_forward(p._h, x.data_ptr(), w.data_ptr(), None, ws.data_ptr(), ws.numel(), s)
    assert st == 1
    with pytest.raises(ValueError):
        p.forward(x[:, :2].contiguous(), w)
    assert p.launches == 4
    assert fc.Plan(1, 4, 4, 16, 16, 3, "winograd", 2, "tcgen05").launches == 4
    assert fc.Plan(1, 4, 4, 16, 16, 3, "winograd", 2, "ffma").launches == 4


def test_forward_host_and_profiled():
    cfg = synth.CONFIGS["tiny"]
    I, W = synth.make_inputs(cfg)
    O = oracle.conv_fp64(I, W)
    p = fc.Plan(1, 4, 4, 16, 16, 3, "gauss_fft", 6)
    hi, hw = I.pin_memory(), W.pin_memory()
    ho = torch.empty(p.out_shape).pin_memory()
    di, dw = torch.empty_like(I, device="cuda"), torch.empty_like(W, device="cuda")
    do = torch.empty(p.out_shape, device="cuda")
    ws = p.alloc_workspace()
    p.forward_host(hi, hw, ho, di, dw, do, ws)
    torch.cuda.synchronize()
    assert rel_err(ho.numpy().astype(np.float64), O) <= 1e-5
    ms = p.forward_profiled(di, dw, do, ws)
    assert len(ms) == 4 and all(v >= 0 for v in ms)


@pytest.mark.parametrize("chunk", [1, 3, 0])
@pytest.mark.parametrize("method,m", [("winograd", 4), ("winograd", 6), ("regular_fft", 8), ("gauss_fft", 5)])
def test_l2_chunking(method, m, chunk):
    """conv_forward processes the batch in chunks of images (ragged last chunk); the per-image
    arithmetic (per-image F16X3 scales) makes the result bit-identical to the unchunked one."""
    cfg = synth.custom(7, 24, 40, 22, 19, 3, seed=51, dist="normal")
    I, W = synth.make_inputs(cfg)
    O = oracle.conv_fp64(I, W)
    p = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m, chunk_images=chunk)
    assert p.info["chunk"] == (chunk if chunk else cfg.B)
    assert p.launches == (1 if method == "winograd" else 2) + 3 * p.info["nchunks"]  # F16X3 FFT: scale prologue
    y = p.forward(I.cuda(), W.cuda())
    ref = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m).forward(I.cuda(), W.cuda())
    torch.cuda.synchronize()
    assert torch.equal(y, ref)
    assert rel_err(y.cpu().double().numpy(), O) <= tol(method, m, cfg.r)


@pytest.mark.parametrize("method,m", [("winograd", 4), ("regular_fft", 6), ("gauss_fft", 8)])
def test_cached_weight_transform(method, m):
    """conv_transform_weights + conv_forward_cached (inference with V computed once)
    equals conv_forward bit for bit, for several inputs against one V."""
    cfg = synth.custom(3, 16, 24, 20, 20, 3, seed=61, dist="normal")
    I, W = synth.make_inputs(cfg)
    I2, _ = synth.make_inputs(cfg, seed=62)
    p = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m)
    x, x2, w = I.cuda(), I2.cuda(), W.cuda()
    ref, ref2 = p.forward(x, w), p.forward(x2, w)
    ws = p.alloc_workspace()
    p.transform_weights(w, ws)
    y = p.forward_cached(x, ws)
    y2 = p.forward_cached(x2, ws)
    torch.cuda.synchronize()
    assert torch.equal(y, ref) and torch.equal(y2, ref2)
    assert rel_err(y.cpu().double().numpy(), oracle.conv_fp64(I, W)) <= tol(method, m, cfg.r)


@pytest.mark.parametrize("gemm", ["tcgen05", "f16x3"])
def test_regular_complex_mode_matches_embedding(gemm):
    """Regular-FFT complex mode ((V_r, V_i) planes, A-negate for -V_i) gives exactly the
    real-embedding result ([[V_r, -V_i], [V_i, V_r]] stored), and both match the oracle."""
    cfg = synth.custom(2, 64, 256, 18, 18, 3, seed=71, dist="normal")
    I, W = synth.make_inputs(cfg)
    O = oracle.conv_fp64(I, W)
    x, w = I.cuda(), W.cuda()
    p = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, "regular_fft", 6, gemm)
    y = p.forward(x, w)
    pe = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, "regular_fft", 6, gemm, complex_mode=0)
    ye = pe.forward(x, w)
    torch.cuda.synchronize()
    assert p.info["bytes_V"] < pe.info["bytes_V"]  # half the V bytes
    assert torch.equal(y, ye)
    assert rel_err(y.cpu().double().numpy(), O) <= 1e-5


def test_accuracy_orderings():
    """The paper's accuracy claims as orderings:
    Winograd error grows with the tile t, the FFT error is flat in t and below Winograd's."""
    I, W, O = _reduced("vgg3_2")
    ew = {m: rel_err(run_gpu(I, W, "winograd", m), O) for m in (2, 4, 6)}
    ef = {m: rel_err(run_gpu(I, W, "regular_fft", m), O) for m in (8, 14, 22, 30)}
    assert ew[2] < ew[4] < ew[6]
    assert max(ef.values()) <= 10 * min(ef.values())
    assert ef[14] <= ew[6]


@pytest.mark.parametrize("method,m", [("winograd", 4), ("gauss_fft", 6), ("direct", 0)])
def test_forward_host_pipelined(method, m):
    """conv_forward_host pipelines H2D / kernels / D2H over image chunks on plan-owned
    copy streams; the host result equals the device-resident forward bit for bit."""
    cfg = synth.custom(7, 12, 20, 21, 17, 3, seed=81, dist="normal")
    I, W = synth.make_inputs(cfg)
    p = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m)
    ref = p.forward(I.cuda(), W.cuda())
    hi, hw = I.pin_memory(), W.pin_memory()
    ho = torch.full(p.out_shape, float("nan")).pin_memory()
    di, dw = torch.empty_like(I, device="cuda"), torch.empty_like(W, device="cuda")
    do = torch.empty(p.out_shape, device="cuda")
    ws = p.alloc_workspace()
    for _ in range(2):
        p.forward_host(hi, hw, ho, di, dw, do, ws)
    torch.cuda.current_stream().synchronize()
    assert torch.equal(ho, ref.cpu())


@pytest.mark.parametrize("name", ["tiny", "vgg3_2", "k5", "deep"])
def test_generic_transforms_option(name):
    """conv_plan_options.generic_transforms = 1 (runtime-t transform kernels) meets the same
    bars as the compile-time-t codelets it stands beside."""
    I, W, O = _reduced(name)
    cfg = synth.CONFIGS[name]
    for method, m in cfg.runs[:4]:
        x, w = I.cuda(), W.cuda()
        p = fc.Plan(I.shape[0], cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m, generic_transforms=1)
        y = p.forward(x, w).cpu().double().numpy()
        assert rel_err(y, O) <= tol(method, m, cfg.r), (name, method, m)


@pytest.mark.parametrize("name", ["vgg3_2", "k5", "deep"])
def test_planner_m0(name):
    """m = 0: the plan takes conv_plan_best_m's tile and meets that tile's bar."""
    I, W, O = _reduced(name)
    cfg = synth.CONFIGS[name]
    for method in ("winograd", "regular_fft", "gauss_fft"):
        if method == "winograd" and cfg.r > 3:
            continue
        m_best, _, _ = fc.best_m(I.shape[0], cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method)
        p = fc.Plan(I.shape[0], cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, 0)
        assert p.info["m"] == m_best
        y = p.forward(I.cuda(), W.cuda()).cpu().double().numpy()
        assert rel_err(y, O) <= tol(method, m_best, cfg.r)


@pytest.mark.parametrize("method,m", [("winograd", 4), ("regular_fft", 6), ("gauss_fft", 8), ("direct", 0)])
def test_cuda_graph_forward(method, m):
    """conv_graph_create / conv_graph_launch: a captured forward (1 and 3 steps per graph)
    equals the eager conv_forward bit for bit, and a replay picks up new input contents."""
    cfg = synth.custom(3, 16, 24, 20, 20, 3, seed=101, dist="normal")
    I, W = synth.make_inputs(cfg)
    I2, _ = synth.make_inputs(cfg, seed=102)
    p = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m)
    x, w = I.cuda(), W.cuda()
    ref = p.forward(x, w).clone()
    ref2 = p.forward(I2.cuda(), w).clone()
    ws = p.alloc_workspace()
    out = torch.full(p.out_shape, float("nan"), device="cuda")
    for steps in (1, 3):
        g = p.capture(x, w, out, ws, steps=steps)
        g.launch()
        torch.cuda.synchronize()
        assert torch.equal(out, ref)
        x.copy_(I2)
        g.launch()
        torch.cuda.synchronize()
        assert torch.equal(out, ref2)
        x.copy_(I)
    if method != "direct":  # cached-weights graph
        wsc = p.alloc_workspace()
        p.transform_weights(w, wsc)
        g = p.capture(x, None, out, wsc, cached=True)
        out.fill_(float("nan"))
        g.launch()
        torch.cuda.synchronize()
        assert torch.equal(out, ref)


def test_cuda_graph_errors():
    p = fc.Plan(1, 4, 4, 16, 16, 3, "winograd", 2)
    lib = fc.load()
    import ctypes
    h = ctypes.c_void_p()
    assert lib.conv_graph_create(p._h, None, None, None, None, 0, 1, 0, ctypes.byref(h)) == 1
    assert lib.conv_graph_launch(None, None) == 1
    lib.conv_graph_destroy(None)


@pytest.mark.parametrize("method", ["regular_fft", "gauss_fft"])
@pytest.mark.parametrize("shape", [(3, 16, 64, 37, 33, 3), (2, 12, 32, 35, 29, 5)])
def test_every_fft_codelet(method, shape):
    """Every compiled FFT tile edge t <= 32 (the three codelet translation units, the tiles the
    planner's sweep and conv_plan_best_m choose from) meets the oracle bar, Regular and Gauss
    (three planes and combined in the contraction's epilogue)."""
    cfg = synth.custom(*shape, seed=121, dist="normal")
    I, W = synth.make_inputs(cfg)
    O = oracle.conv_fp64(I, W)
    x, w = I.cuda(), W.cuda()
    for t in [4, 5, 6, 7, 8, 9, 10, 12, 13, 14, 15, 16, 18, 20, 21, 24, 25, 27, 28, 30, 31, 32]:
        m = t - cfg.r + 1
        if m < 1:
            continue
        for gcomb in ((-1,) if method == "regular_fft" else (0, 1)):
            kw = {} if gcomb < 0 else {"gauss_combine": gcomb}
            p = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m, **kw)
            y = p.forward(x, w)
            torch.cuda.synchronize()
            assert rel_err(y.cpu().double().numpy(), O) <= 1e-5, (t, gcomb)
