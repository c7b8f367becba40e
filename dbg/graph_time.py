"""Eager conv_forward vs CUDA-graph replay (1 and 10 steps per graph), ms per step."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_1809_07851_b200 as fc
fc.load()
for name, method, m in (("tiny", "winograd", 2), ("deep", "winograd", 4), ("vgg3_2", "winograd", 4),
                        ("k5", "regular_fft", 14)):
    cfg = synth.CONFIGS[name]
    I, W = synth.make_inputs(cfg)
    x, w = I.cuda(), W.cuda()
    p = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m)
    ws = p.alloc_workspace()
    out = torch.empty(p.out_shape, device="cuda")
    def timeit(fn, n):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        b.record(); b.synchronize()
        return a.elapsed_time(b) / n
    n = 200
    e = timeit(lambda: p.forward(x, w, out, ws), n)
    g1 = p.capture(x, w, out, ws, steps=1)
    t1 = timeit(g1.launch, n)
    g10 = p.capture(x, w, out, ws, steps=10)
    t10 = timeit(g10.launch, n // 10) / 10
    print("%-7s %-12s m=%d  eager %.4f ms  graph(1) %.4f ms  graph(10) %.4f ms" % (name, method, m, e, t1, t10))
