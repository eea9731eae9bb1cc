"""One gpf_filter_gpf call in the reference-exact fp64 mode on a BASELINE frame
(for ncu launch lists of the fp64 kernels). Usage: python tools/fp64_one.py [cid] [reps]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1505_00077_b200 as g  # noqa: E402
from paper_1505_00077_b200 import synth  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = synth.CONFIGS[cid]
img = synth.make(cfg).astype(np.float64)
g.set_precision("fp64")
for _ in range(reps):
    out, fb = g.gpf_filter_gpf(img, g.spatial_params(cfg.sigma_s[0]), g.range_params(cfg.sigma_r, cfg.degree))
    print(f"C{cid} fp64: device {g.last_device_ms():.3f} ms, fallbacks {fb}, out[0,0] {out[0, 0]:.6f}")
