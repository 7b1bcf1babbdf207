"""How long does torch's caching host allocator take to hand out page-locked
output buffers of the sizes fused_sweep returns (ping-pong: the previous
result is still alive while the next is allocated)?"""
import time
import torch
torch.cuda.init()
for mb in (2, 6, 19, 38):
    n = mb * (1 << 20) // 8
    prev = None
    ts = []
    for it in range(6):
        t0 = time.perf_counter()
        a = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
        ts.append((time.perf_counter() - t0) * 1e3)
        prev = a
    print(mb, "MB:", " ".join(f"{t:.2f}" for t in ts), "ms")
