"""Device time of the direct (windowed) backend on one frame, beside the
recursive backend's (not the hot path; recorded for DESIGN.md 7).
usage: python tools/direct_time.py [size] [sigma_s]"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1505_00077_b200 as g  # noqa: E402
from paper_1505_00077_b200 import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
ss = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0
img = synth.rects_image(n, n, max(n // 8, 1), 10.0, 1).astype(np.float64)
res = {"frame": f"{n}x{n}", "sigma_s": ss, "sigma_r": 30.0, "degree": 20}
for name, backend in (("direct", 0), ("recursive_fp64", 1)):
    if backend == 1:
        g.set_precision("fp64")
    for _ in range(2):
        t0 = time.perf_counter()
        out, fb = g.gpf_filter_gpf(img, g.spatial_params(ss), g.range_params(30.0, 20), backend=backend)
        wall = time.perf_counter() - t0
    res[name] = {"device_ms": round(g.last_device_ms(), 3), "wall_ms": round(wall * 1e3, 2),
                 "Mpix_s_device": round(n * n / g.last_device_ms() / 1e3, 1), "fallbacks": fb}
g.set_precision("auto")
t0 = time.perf_counter()
g.gpf_gaussian_direct(img, g.spatial_params(ss))
res["gaussian_direct_wall_ms"] = round((time.perf_counter() - t0) * 1e3, 2)
print(json.dumps(res))
