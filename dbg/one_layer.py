"""Run a few forwards of one config (for ncu captures): python dbg/one_layer.py vgg3_2 winograd 4 [iters]"""
import sys
import torch
sys.path.insert(0, ".")
import synth
import paper_1809_07851_b200 as fc

name, method, m = sys.argv[1], sys.argv[2], int(sys.argv[3])
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 3
cfg = synth.CONFIGS[name]
I, W = synth.make_inputs(cfg)
x, w = I.cuda(), W.cuda()
p = fc.Plan(cfg.B, cfg.C, cfg.Cout, cfg.H, cfg.W, cfg.r, method, m)
ws = p.alloc_workspace()
out = torch.empty(p.out_shape, device="cuda")
for _ in range(iters):
    p.forward(x, w, out, ws)
torch.cuda.synchronize()
print("ok", out.abs().max().item())
