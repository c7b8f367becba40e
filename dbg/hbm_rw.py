"""HBM bandwidth by access mix on this box: write-only (fill), read-only (sum), copy."""
import torch
n = 1 << 28  # 1 GiB of fp32
x = torch.empty(n, device="cuda")
y = torch.empty(n, device="cuda")
x.fill_(1.0)
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        a.record(); fn(); b.record(); b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best
ms = t(lambda: x.fill_(2.0)); print("write-only %.0f GB/s" % (n * 4 / ms / 1e6))
ms = t(lambda: x.sum()); print("read-only  %.0f GB/s" % (n * 4 / ms / 1e6))
ms = t(lambda: y.copy_(x)); print("copy       %.0f GB/s (r+w)" % (2 * n * 4 / ms / 1e6))
z = torch.empty(n // 2, device="cuda")
ms = t(lambda: torch.add(x[: n // 2], x[n // 2:], out=z)); print("2r:1w      %.0f GB/s" % (1.5 * n * 4 / ms / 1e6))
