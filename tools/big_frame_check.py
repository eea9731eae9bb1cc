"""Maximum-size check: fp32 plan path and the drop-in call on frames larger than the BASELINE
ones (V above 2^31 floats, 512 strips / 1024 bands), every pixel against the unmodified
reference on the host cores. Usage (GPU box): python tools/big_frame_check.py [W H sigma_s]...
Default: 16384x8192 at sigma_s 5 and 8192x16384 at sigma_s 20. Prints one JSON line per frame."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import Reference  # noqa: E402
import paper_1505_00077_b200 as g  # noqa: E402
from paper_1505_00077_b200 import synth  # noqa: E402


def main():
    a = sys.argv[1:]
    cases = [(int(a[i]), int(a[i + 1]), float(a[i + 2])) for i in range(0, len(a) - 2, 3)] or \
        [(16384, 8192, 5.0), (8192, 16384, 20.0)]
    ref = Reference()
    ref.set_num_threads(os.cpu_count() or 1)
    for w, h, ss in cases:
        img32 = synth.rects_image(w, h, 2048, 10.0, 9000 + w // 1024)
        img = img32.astype(np.float64)
        t0 = time.time()
        st, r, rfb = ref.gpf(img, ss, 30.0, 20)
        t_ref = time.time() - t0
        assert st == 0
        plan = g.Plan(w, h, ss, 30.0, 20)
        o32, fbs = plan.filter_host(img32)
        ws = plan.workspace_bytes
        plan.close()
        out, fb = g.gpf_filter_gpf(img, g.spatial_params(ss), g.range_params(30.0, 20))
        print(json.dumps({"shape": [h, w], "sigma_s": ss, "ref_seconds": round(t_ref, 1),
                          "host_threads": os.cpu_count(), "plan_workspace_GiB": round(ws / 2**30, 2),
                          "fp32_plan_max_abs": float(np.abs(o32 - r).max()), "fp32_plan_fallbacks": fbs[0],
                          "dropin_precision": g.last_precision(), "dropin_max_abs": float(np.abs(out - r).max()),
                          "dropin_fallbacks": fb, "ref_fallbacks": rfb,
                          "ref_range": [float(r.min()), float(r.max())]}), flush=True)
        del r, out, o32, img, img32
        g.dropin_release()


if __name__ == "__main__":
    main()
