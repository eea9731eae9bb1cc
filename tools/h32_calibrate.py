"""Calibration of the fp32 envelope (kH32Limit, dropin.cpp).

Runs the fp32 plane kernels (gpf_filter_gpf forced to FP32) and the unmodified
reference (oracle/_ref) on generator frames over a grid of sigma_r / sigma_s /
intensity layouts, and prints, per case, max|H| = max(f_max - t_c, t_c - f_min)
/ sigma_r against max |gpu - reference| over all pixels and over pixels whose
reference output stays in the input range. Usage (GPU box):
  python tools/h32_calibrate.py [size] > gpurun_out/h32.jsonl
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference  # noqa: E402
import paper_1505_00077_b200 as g  # noqa: E402
from paper_1505_00077_b200 import synth  # noqa: E402


def images(n):
    base = synth.rects_image(n, n, 64, 10.0, 7).astype(np.float64)
    yield "rects", base
    yield "rects_dark", np.floor(base * 0.4)
    yield "rects_inv", 255.0 - base
    yield "checker", synth.checker_image(n, n, 5.0, 3).astype(np.float64)
    lo = synth.checker_image(n, n, 5.0, 4).astype(np.float64)
    yield "checker_30_200", 30.0 + lo * (170.0 / 255.0)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 768
    ref = Reference()
    ref.set_num_threads(os.cpu_count() or 1)
    g.set_precision("fp32")
    for name, img in images(n):
        for sr in (6.0, 8.0, 10.0, 12.0, 15.0, 18.0, 20.0, 25.0, 30.0, 40.0):
            for ss in (2.0, 8.0, 30.0):
                st, r, rfb = ref.gpf(img, ss, sr, 20)
                out, fb = g.gpf_filter_gpf(img, g.spatial_params(ss), g.range_params(sr, 20))
                tc = img.mean()
                hmax = max(img.max() - tc, tc - img.min()) / sr
                d = np.abs(out - r)
                inr = (r >= img.min()) & (r <= img.max())
                print(json.dumps({"img": name, "sr": sr, "ss": ss, "hmax": round(hmax, 3),
                                  "max": float(d.max()),
                                  "max_in": float(d[inr].max()) if inr.any() else 0.0,
                                  "outside": int((~inr).sum()), "fb": [fb, rfb]}), flush=True)


if __name__ == "__main__":
    main()
