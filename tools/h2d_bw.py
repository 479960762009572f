"""Pinned host -> device copy bandwidth for the C2 batch size (diagnostics for the e2e number)."""
import time, torch
n = 1 << 22  # 16.8 MB of float32
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
for chunks in (1, 4):
    t = time.perf_counter()
    for _ in range(50):
        for c in range(chunks):
            sl = slice(c * n // chunks, (c + 1) * n // chunks)
            d[sl].copy_(h[sl], non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 50
    print(f"H2D {n * 4 / 1e6:.1f} MB in {chunks} chunk(s): {dt * 1e3:.3f} ms -> {n * 4 / dt / 1e9:.1f} GB/s")
