"""Dev probe (GPU): pinned H2D / D2H bandwidth and latency at e2e sizes."""
import time, torch
for nb in (400_000, 800_000, 8_000_000, 64_000_000):
    h = torch.empty(nb, dtype=torch.uint8).pin_memory(); d = torch.empty(nb, dtype=torch.uint8, device="cuda")
    for direction in ("h2d", "d2h"):
        for _ in range(5):
            (d.copy_(h) if direction == "h2d" else h.copy_(d)); torch.cuda.synchronize()
        n = 50; t = time.perf_counter()
        for _ in range(n):
            (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True)); torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / n
        print(f"{direction} {nb/1e6:.1f} MB sync each: {dt*1e6:.1f} us  {nb/dt/1e9:.1f} GB/s")
