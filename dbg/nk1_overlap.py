"""Does running NK1 (kernel transform) concurrently with NK2 (input transform) on a second
stream shorten the layer?  Sequential conv_forward vs stage calls with NK1 on a side stream."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_1809_07851_b200 as fc
fc.load()
for name, method, m in (("vgg3_2", "winograd", 4), ("vgg3_2", "regular_fft", 14), ("deep", "winograd", 4)):
    cfg = synth.CONFIGS[name]
    I, W = synth.make_inputs(cfg)
    x, w = I.cuda(), W.cuda()
    p = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m)
    ws = p.alloc_workspace()
    out = torch.empty(p.out_shape, device="cuda")
    main = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    def seq():
        p.forward(x, w, out, ws)
    def conc():
        ev0 = torch.cuda.Event()
        ev0.record(main)
        side.wait_event(ev0)
        p.run_stage(0, w=w, workspace=ws, stream=side)
        ev1 = torch.cuda.Event()
        ev1.record(side)
        p.run_stage(1, x=x, workspace=ws, stream=main)
        main.wait_event(ev1)
        p.run_stage(2, workspace=ws, stream=main)
        p.run_stage(3, out=out, workspace=ws, stream=main)
    def t(fn, n=200):
        for _ in range(5): fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main)
        for _ in range(n): fn()
        b.record(main); b.synchronize()
        return a.elapsed_time(b) / n
    ref = out.clone(); seq(); torch.cuda.synchronize(); r1 = out.clone(); conc(); torch.cuda.synchronize()
    print(name, method, m, "seq %.4f ms  conc %.4f ms  same=%s" % (t(seq), t(conc), torch.equal(r1, out)))
