"""Seeded random sweep of the drop-in entry (gpf_filter_gpf, AUTO precision)
against the oracle (pinned to the reference, tests/test_oracle.py): frame
shapes from 1x1 to a few hundred pixels (partial chunks and strips on both
axes), sigma_s 0.5-60, sigma_r 8-80, degrees 0-22 and the large-N kernels,
both centering modes and non-unit kernel_scale, on the three image families
of the BASELINE generator. Bar: max |d| <= 1e-3 and equal fallback counts.
(GPF_FUZZ_N sets the number of cases; 40 by default.)"""
import os

import numpy as np
import pytest

from paper_1505_00077_b200 import synth

pytestmark = pytest.mark.gpu

TOL = 1e-3


def _cases(n=int(os.environ.get("GPF_FUZZ_N", "40")), seed=20261021):
    rng = np.random.default_rng(seed)
    for i in range(n):
        w = int(rng.choice([1, 2, 7, 31, 32, 33, 63, 64, 65, 97, 130, 257]))
        h = int(rng.choice([1, 3, 16, 17, 31, 32, 33, 48, 95, 129, 200]))
        ss = float(np.round(np.exp(rng.uniform(np.log(0.5), np.log(60.0))), 3))
        sr = float(np.round(rng.uniform(8.0, 80.0), 2))
        deg = int(rng.choice([0, 1, 2, 5, 10, 19, 20, 21, 22, 30, 48]))
        cen = int(rng.choice([0, 1]))
        ks = float(rng.choice([1.0, 0.5, 3.0]))
        kind = ("rects", "checker", "noise")[i % 3]
        yield pytest.param(i, w, h, ss, sr, deg, cen, ks, kind,
                           id=f"{i}-{kind}-{w}x{h}-ss{ss:g}-sr{sr:g}-n{deg}-c{cen}-k{ks:g}")


def _image(kind, w, h, seed):
    if kind == "rects":
        return synth.rects_image(w, h, max(1, w * h // 4096), 10.0, seed).astype(np.float64)
    if kind == "checker":
        return synth.checker_image(w, h, 5.0, seed).astype(np.float64)
    rng = np.random.default_rng(seed)
    return np.clip(rng.normal(128.0, 40.0, (h, w)), 0.0, 255.0)


@pytest.mark.parametrize("i,w,h,ss,sr,deg,cen,ks,kind", list(_cases()))
def test_fuzz_dropin_vs_oracle(gpu, oracle, i, w, h, ss, sr, deg, cen, ks, kind):
    img = _image(kind, w, h, 7000 + i)
    ref, rfb, _ = oracle.gpf(img, ss, sr, deg, centering=cen, kernel_scale=ks)
    out, fb = gpu.gpf_filter_gpf(img, gpu.spatial_params(ss, kernel_scale=ks), gpu.range_params(sr, deg),
                                 centering=cen)
    d = float(np.abs(out - ref).max())
    assert fb == rfb and d <= TOL, (d, fb, rfb, gpu.last_precision())
