"""Probe of non-finite fp32 outputs (forced fp32 through gpf_filter_gpf) on the
calibration frames: per case, the count of non-finite outputs and the H range of
those pixels. usage: GPF_B200_LIB=... python tools/gs_probe.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1505_00077_b200 as g  # noqa: E402
from paper_1505_00077_b200 import synth  # noqa: E402

n = 768
base = synth.rects_image(n, n, 64, 10.0, 7).astype(np.float64)
cases = [("rects_dark", np.floor(base * 0.4), 8.0), ("rects", base, 18.0), ("rects", base, 10.0)]
g.set_precision("fp32")
for name, img, sr in cases:
    for ss in (2.0, 30.0):
        out, fb = g.gpf_filter_gpf(img, g.spatial_params(ss), g.range_params(sr, 20))
        tc = img.mean()
        H = (img - tc) / sr
        bad = ~np.isfinite(out)
        print(name, sr, ss, "hmax", round(float(np.abs(H).max()), 3), "nonfinite", int(bad.sum()),
              "H of those", (round(float(H[bad].min()), 3), round(float(H[bad].max()), 3)) if bad.any() else None,
              "max|out|", float(np.nanmax(np.abs(np.where(bad, 0, out)))), flush=True)
