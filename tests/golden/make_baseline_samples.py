"""Generates tests/golden/baseline_samples.npz: the UNMODIFIED reference's
output (oracle/_ref/libgpfilter_ref.so, built from /root/reference/proj by
oracle/Makefile) on the full-size BASELINE frames, sampled on a regular grid.

The GPU box has no /root/reference, and the reference needs about a minute of
CPU per 8192^2 frame, so bench.py checks its own full-size outputs against
these samples (max |gpu - reference| over the grid, outside the timed region),
while tests/test_gpu_fullsize.py compares every pixel against the reference
run on the box. Stored per (config, sigma_s): the grid stride, the sampled
reference output, the reference's fallback count and t_c-independent stats of
the whole reference frame (min, max, pixels outside the input range).

Run here:  python tests/golden/make_baseline_samples.py   (about 10 min on 8 cores)
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference  # noqa: E402
from paper_1505_00077_b200 import synth  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "baseline_samples.npz")
STRIDE = {1: 8, 2: 16, 3: 64, 4: 32, 5: 32}


def frames(cid):
    cfg = synth.CONFIGS[cid]
    if cid == 4:
        return [(f"c4_f{f}_ch{c}", synth.make(cfg, f, c), cfg.sigma_s[0]) for f, c in ((0, 0), (31, 1), (63, 2))]
    if cid == 3:  # bench.py filters frame k of the C3 batch at sigma_s[k]
        return [(f"c3_f{k}_ss{int(ss)}", synth.make(cfg, k), ss) for k, ss in enumerate(cfg.sigma_s)]
    return [(f"c{cid}_ss{int(ss)}", synth.make(cfg), ss) for ss in cfg.sigma_s]


def main() -> None:
    ref = Reference()
    ref.set_num_threads(os.cpu_count() or 1)
    data = {}
    names = []
    for cid in (1, 2, 5, 4, 3):
        cfg = synth.CONFIGS[cid]
        for name, img32, ss in frames(cid):
            t0 = time.time()
            img = img32.astype(np.float64)
            st, out, fb = ref.gpf(img, ss, cfg.sigma_r, cfg.degree)
            assert st == 0, (name, st)
            s = STRIDE[cid]
            lo, hi = float(img.min()), float(img.max())
            outside = (out < lo) | (out > hi)
            data[f"{name}/samples"] = out[::s, ::s].copy()
            data[f"{name}/meta"] = np.array([s, fb, out.min(), out.max(), outside.sum(), ss, cfg.sigma_r,
                                             cfg.degree, cid])
            names.append(name)
            print(f"{name}: {time.time() - t0:.1f} s, fb {fb}, out [{out.min():.4g}, {out.max():.4g}], "
                  f"outside input range {int(outside.sum())}", flush=True)
    data["__names__"] = np.array(names)
    np.savez_compressed(OUT, **data)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
