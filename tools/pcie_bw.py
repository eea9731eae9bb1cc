"""Raw pinned-host <-> HBM copy bandwidth: H2D alone, D2H alone, both at once,
with one frame-sized copy per direction split over 1, 2 or 4 streams (copy
engines) and into chunks. usage: python tools/pcie_bw.py"""
import time

import torch

n = 256 << 20  # bytes per direction per repetition (one 8192^2 fp32 frame)
h_in = torch.empty(n // 4, dtype=torch.float32).pin_memory()
h_out = torch.empty(n // 4, dtype=torch.float32).pin_memory()
d_a = torch.empty(n // 4, dtype=torch.float32, device="cuda")
d_b = torch.empty(n // 4, dtype=torch.float32, device="cuda")
up = [torch.cuda.Stream() for _ in range(4)]
dn = [torch.cuda.Stream() for _ in range(4)]


def run(h2d, d2h, nstreams=1, chunks=1, reps=10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m = n // 4 // chunks
    for _ in range(reps):
        for c in range(chunks):
            sl = slice(c * m, (c + 1) * m)
            if h2d:
                with torch.cuda.stream(up[c % nstreams]):
                    d_a[sl].copy_(h_in[sl], non_blocking=True)
            if d2h:
                with torch.cuda.stream(dn[c % nstreams]):
                    h_out[sl].copy_(d_b[sl], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    return reps * n * (h2d + d2h) / dt / 1e9


run(1, 1, 2)
for ns, ch in ((1, 1), (1, 4), (2, 2), (2, 8), (4, 4), (4, 16)):
    print(f"streams {ns} chunks {ch:2d}: H2D {run(1, 0, ns, ch):.1f} GB/s  D2H {run(0, 1, ns, ch):.1f} GB/s  "
          f"both {run(1, 1, ns, ch):.1f} GB/s total", flush=True)
