"""Concurrent gpf_filter_gpf callers (dropin.cpp call slots): frames per second
with 1..T host threads on C3 frames, per-call latency, and the pinned PCIe
copy rates one way and both ways at once for the same bytes.
usage: GPF_B200_DROPIN_SLOTS=k python tools/dropin_concurrency.py [n] [threads]"""
import ctypes as C
import os
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1505_00077_b200 import _lib, gpf, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
T = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = synth.scaled(synth.CONFIGS[3], n, n)
frames = [synth.make(cfg, frame=k) for k in range(T)]
imgs = [gpf.Image.from_array(np.asarray(f, dtype=np.float64)) for f in frames]
L = _lib.lib()
sigmas = [2.0, 5.0, 10.0, 20.0, 50.0]
rp = gpf.range_params(30.0, 20)
lat = []


def call(i):
    sp = gpf.spatial_params(sigmas[i % len(sigmas)])
    out = C.c_void_p()
    fb = C.c_longlong()
    t0 = time.perf_counter()
    assert L.gpf_filter_gpf(imgs[i].h, C.byref(sp), C.byref(rp), 1, 1, C.byref(fb), C.byref(out)) == 0
    lat.append(time.perf_counter() - t0)
    L.gpf_image_destroy(out)


def run(threads, reps):
    def w(i):
        for _ in range(reps):
            call(i)
    ths = [threading.Thread(target=w, args=(i,)) for i in range(threads)]
    t0 = time.perf_counter()
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    return time.perf_counter() - t0


run(T, 1)
for threads in sorted({1, 2, 3, T}):
    lat.clear()
    sec = run(threads, 4)
    print(f"slots {os.environ.get('GPF_B200_DROPIN_SLOTS', 'default')} threads {threads}: "
          f"{threads * 4 * n * n / sec / 1e6:.0f} Mpix/s, {1e3 * sec / (threads * 4):.1f} ms/frame, "
          f"call latency median {1e3 * sorted(lat)[len(lat) // 2]:.1f} ms", flush=True)
h1 = torch.empty((n, n), dtype=torch.float64).pin_memory()
h2 = torch.empty((n, n), dtype=torch.float64).pin_memory()
d1 = torch.empty((n, n), dtype=torch.float64, device="cuda")
d2 = torch.empty((n, n), dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    b = n * n * 8
    print(f"pinned H2D alone {b / (t1 - t0) / 1e9:.1f} GB/s; H2D + D2H at once {2 * b / (t2 - t1) / 1e9:.1f} GB/s total")
