import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_1809_07851_b200 as fc
p = fc.Plan(1, 4, 3, 16, 14, 3, "winograd", 2, "tcgen05")
info = p.info
print({k: info[k] for k in ("gemm_Z","gemm_M","gemm_K","BN","BN_pad")}, p.layout)
ws = p.alloc_workspace(); ws.zero_()
x = torch.randn(1,4,16,14,device="cuda"); w = torch.randn(3,4,3,3,device="cuda")
p.run_stage(0, w=w, workspace=ws); p.run_stage(1, x=x, workspace=ws); torch.cuda.synchronize()
p.run_stage(2, workspace=ws); torch.cuda.synchronize()
Z,M,K,NP = info["gemm_Z"],info["gemm_M"],info["gemm_K"],info["BN_pad"]
X = ws[p.layout["X"]:p.layout["X"]+4*Z*M*NP].view(torch.float32).reshape(Z,M,NP)
print("X[0,:,:4]", X[0,:,:4])
