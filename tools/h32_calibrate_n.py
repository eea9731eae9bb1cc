"""fp32 envelope per degree N: like tools/h32_calibrate.py, over
degrees 0-48, on 256x256 frames of the calibration layouts (and a single-row
strip), sigma_r swept so max|H| covers 0.5-12; the fp32 kernels are forced and
compared with the unmodified reference. One JSON line per case.
Usage (GPU box): python tools/h32_calibrate_n.py > gpurun_out/h32n.jsonl"""
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
    base = synth.rects_image(n, n, 16, 10.0, 7).astype(np.float64)
    yield "rects", base
    yield "rects_inv", 255.0 - base
    yield "checker", synth.checker_image(n, n, 5.0, 3).astype(np.float64)
    lo = synth.checker_image(n, n, 5.0, 4).astype(np.float64)
    yield "checker_30_200", 30.0 + lo * (170.0 / 255.0)
    yield "checker_row", synth.checker_image(4 * n, 1, 5.0, 5).astype(np.float64)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    ref = Reference()
    ref.set_num_threads(os.cpu_count() or 1)
    g.set_precision("fp32")
    for name, img in images(n):
        tc = img.mean()
        span = max(img.max() - tc, tc - img.min())
        for deg in (0, 1, 2, 3, 5, 8, 10, 12, 15, 20, 25, 30, 40, 48):
            for hm in (0.5, 1.0, 1.5, 2.0, 2.5, 3.0, 3.5, 4.0, 5.0, 6.0, 7.0, 8.0, 10.0, 12.0):
                sr = span / hm
                for ss in (2.0, 8.0):
                    st, r, rfb = ref.gpf(img, ss, sr, deg)
                    out, fb = g.gpf_filter_gpf(img, g.spatial_params(ss), g.range_params(sr, deg))
                    d = np.abs(out - r)
                    inr = (r >= img.min()) & (r <= img.max())
                    print(json.dumps({"img": name, "deg": deg, "sr": round(sr, 4), "ss": ss, "hmax": hm,
                                      "max": float(np.nan_to_num(d, nan=1e30).max()),
                                      "max_in": float(d[inr].max()) if inr.any() else 0.0,
                                      "outside": int((~inr).sum()), "fb": [fb, rfb]}), flush=True)


if __name__ == "__main__":
    main()
