"""Pinned host <-> device copy bandwidth on this box (H2D alone, D2H alone, both at once)."""
import torch
n = 223 * 1000 * 1000 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
h2 = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
d2 = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); b.record(); b.synchronize()
    return a.elapsed_time(b) / reps
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
ms = t(lambda: d.copy_(h, non_blocking=True)); print("H2D %.1f GB/s (%.2f ms)" % (n * 4 / ms / 1e6, ms))
ms = t(lambda: h2.copy_(d2, non_blocking=True)); print("D2H %.1f GB/s (%.2f ms)" % (n * 4 / ms / 1e6, ms))
ms = t(both); print("both %.2f ms -> %.1f GB/s each" % (ms, n * 4 / ms / 1e6))
