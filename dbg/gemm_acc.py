import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_1809_07851_b200 as fc, synth
cfg = synth.custom(4, 256, 256, 58, 58, 3, seed=2, dist="normal")
I, W = synth.make_inputs(cfg)
x, w = I.cuda(), W.cuda()
for method, m in (("winograd", 2), ("winograd", 4), ("regular_fft", 14), ("gauss_fft", 14)):
    res = {}
    for gemm in ("tcgen05", "ffma"):
        os.environ["FASTCONV_NO_CPLX"] = "1"
        p = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m, gemm)
        info = p.info; Z, M, K, BNp, BN = info["gemm_Z"], info["gemm_M"], info["gemm_K"], info["BN_pad"], info["BN"]
        Kp = (K + 3) // 4 * 4
        ws = p.alloc_workspace(); ws.zero_()
        p.run_stage(0, w=w, workspace=ws); p.run_stage(1, x=x, workspace=ws); p.run_stage(2, workspace=ws)
        torch.cuda.synchronize()
        V = ws[p.layout["V"]:p.layout["V"] + 4 * Z * M * Kp].view(torch.float32).reshape(Z, M, Kp)[:, :, :K].double()
        if gemm == "tcgen05":
            V = V + ws[p.layout["Vlo"]:p.layout["Vlo"] + 4 * Z * M * Kp].view(torch.float32).reshape(Z, M, Kp)[:, :, :K].double()
        U = ws[p.layout["U"]:p.layout["U"] + 4 * Z * K * BNp].view(torch.float32).reshape(Z, K, BNp)[:, :, :BN].double()
        X = ws[p.layout["X"]:p.layout["X"] + 4 * Z * M * BNp].view(torch.float32).reshape(Z, M, BNp)[:, :, :BN].double()
        ref = torch.matmul(V, U)
        err = ((X - ref).abs().max() / ref.abs().max()).item()
        # error relative to the sum of |terms| (conditioning-free)
        scale = torch.matmul(V.abs(), U.abs())
        err2 = ((X - ref).abs() / scale.clamp_min(1e-30)).max().item()
        res[gemm] = (err, err2)
    print(method, m, "K=%d" % K, {k: ("%.2e" % v[0], "%.2e" % v[1]) for k, v in res.items()})
