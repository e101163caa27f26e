"""Host->device bandwidth of the e2e trace upload (pinned, 5.9 GB) on this box."""
import time
import torch
n = 5_900_000_000 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
for _ in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"H2D {n * 8 / dt / 1e9:.1f} GB/s ({dt * 1e3:.0f} ms for 5.9 GB)")
