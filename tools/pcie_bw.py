"""Raw pinned-host <-> HBM copy bandwidth: H2D alone, D2H alone, both at once."""
import time

import torch

n = 256 << 20
h_in = torch.empty(n // 4, dtype=torch.float32).pin_memory()
h_out = torch.empty(n // 4, dtype=torch.float32).pin_memory()
d_a = torch.empty(n // 4, dtype=torch.float32, device="cuda")
d_b = torch.empty(n // 4, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d_a.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_out.copy_(d_b, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    return reps * n * (h2d + d2h) / dt / 1e9


run(1, 1, 2)
print(f"H2D {run(1, 0):.1f} GB/s  D2H {run(0, 1):.1f} GB/s  both {run(1, 1):.1f} GB/s total")
