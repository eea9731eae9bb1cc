"""Timing of the drop-in call gpf_filter_gpf on one frame (host fp64 in/out):
call time vs device filter time vs a pinned 2-way copy of the same bytes."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1505_00077_b200 import _lib, gpf, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
cfg = synth.scaled(synth.CONFIGS[3], n, n)
img = gpf.Image.from_array(synth.make(cfg).astype(np.float64))
L = _lib.lib()
for ss in (2.0, 5.0):
    sp, rp = gpf.spatial_params(ss), gpf.range_params(30.0, 20)
    for rep in range(4):
        out = C.c_void_p()
        fb = C.c_longlong()
        t0 = time.perf_counter()
        assert L.gpf_filter_gpf(img.h, C.byref(sp), C.byref(rp), 1, 1, C.byref(fb), C.byref(out)) == 0
        t1 = time.perf_counter()
        L.gpf_image_destroy(out)
        print(f"sigma_s {ss} call {rep}: {1e3 * (t1 - t0):.2f} ms, device {gpf.last_device_ms():.2f} ms, "
              f"{gpf.last_precision()}")
h = torch.empty((n, n), dtype=torch.float64).pin_memory()
d = torch.empty((n, n), dtype=torch.float64, device="cuda")
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"pinned H2D {h.numel() * 8 / (t1 - t0) / 1e9:.1f} GB/s, D2H {h.numel() * 8 / (t2 - t1) / 1e9:.1f} GB/s")
