"""H2D/D2H bandwidth of pinned host memory on this box (context for the e2e number)."""
import torch

dev = torch.device("cuda", 0)
for mb in (1, 10, 100):
    n = mb * 2**20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        d.copy_(h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10
    print(f"H2D {mb:4d} MB: {t * 1e3:8.1f} us  {n / t / 1e6:6.1f} GB/s")
