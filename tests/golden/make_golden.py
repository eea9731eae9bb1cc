"""Generates tests/golden/gpf_golden.npz by running the UNMODIFIED reference
library (oracle/_ref/libgpfilter_ref.so, compiled from /root/reference/proj by
oracle/Makefile) through its own C ABI.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The GPU box never reads /root/reference; it reads the committed .npz.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference  # noqa: E402
from paper_1505_00077_b200 import synth  # noqa: E402


def mt_uniform_image(seed: int, w: int, h: int, hi: float) -> np.ndarray:
    """uniform_noise_image of proj/tests/noise.hpp:46-56 (mt19937, (x+0.5)/2^32)."""
    # numpy's legacy RandomState is MT19937 seeded like std::mt19937 for a
    # 32-bit seed; its raw 32-bit outputs are the standard stream.
    rs = np.random.RandomState(seed)
    raw = rs.randint(0, 2**32, size=w * h, dtype=np.uint32).astype(np.float64)
    u = (raw + 0.5) / 4294967296.0 * hi
    return (np.floor(u) if hi > 1.0 else u).reshape(h, w)


def cases():
    two_level = np.zeros((8, 8))
    two_level[:, 4:] = 255.0
    yield "fallback_sr1_n5", two_level, dict(sigma_s=2.0, sigma_r=1.0, degree=5)
    yield "two_level_sr30", two_level, dict(sigma_s=2.0, sigma_r=30.0, degree=20)
    yield "constant_42", np.full((16, 16), 42.0), dict(sigma_s=2.0, sigma_r=30.0, degree=20)
    yield "constant_frac", np.full((32, 32), 187.34719982), dict(sigma_s=5.0, sigma_r=10.0, degree=20)
    yield "px_1x1", np.array([[77.0]]), dict(sigma_s=2.0, sigma_r=30.0, degree=20)
    yield "row_1x7", np.arange(7, dtype=np.float64)[None, :] * 30.0, dict(sigma_s=2.0, sigma_r=30.0, degree=20)
    yield "col_5x1", np.arange(5, dtype=np.float64)[:, None] * 50.0, dict(sigma_s=2.0, sigma_r=30.0, degree=20)
    u = mt_uniform_image(61, 48, 32, 256.0)
    yield "uniform_48x32_n10", u, dict(sigma_s=2.0, sigma_r=30.0, degree=10)
    c1 = synth.rects_image(96, 80, 4, 10.0, 1001)
    for ss in (0.5, 2.0, 3.0, 10.0, 50.0):
        yield f"rects_96x80_ss{ss:g}", c1, dict(sigma_s=ss, sigma_r=30.0, degree=20)
    for n in (0, 1, 5, 30):
        yield f"rects_96x80_deg{n}", c1, dict(sigma_s=3.0, sigma_r=30.0, degree=n)
    yield "rects_96x80_nocenter", c1, dict(sigma_s=3.0, sigma_r=30.0, degree=20, centering=0)
    yield "rects_96x80_kscale", c1, dict(sigma_s=3.0, sigma_r=30.0, degree=20, kernel_scale=5.25)
    yield "rects_128x128_ss8_sr25", synth.rects_image(128, 128, 8, 8.0, 4001), dict(sigma_s=8.0, sigma_r=25.0, degree=20)
    yield "checker_128_ss6_sr10", synth.checker_image(128, 128, 5.0, 5500), dict(sigma_s=6.0, sigma_r=10.0, degree=20)
    yield "rects_160x96_ss5_sr20", synth.rects_image(160, 96, 4, 15.0, 2001), dict(sigma_s=5.0, sigma_r=20.0, degree=20)


def main() -> None:
    ref = Reference()
    ref.set_num_threads(1)
    out = {}
    names = []
    for name, img, kw in cases():
        st, res, fb = ref.gpf(img, kw["sigma_s"], kw["sigma_r"], kw.get("degree", 20),
                              kw.get("centering", 1), kw.get("kernel_scale", 1.0))
        assert st == 0, (name, st, ref.last_error())
        out[f"{name}/in"] = np.asarray(img, np.float64)
        out[f"{name}/out"] = res
        out[f"{name}/fb"] = np.array(fb)
        out[f"{name}/params"] = np.array([kw["sigma_s"], kw["sigma_r"], kw.get("degree", 20),
                                          kw.get("centering", 1), kw.get("kernel_scale", 1.0)])
        names.append(name)
    # gpf_gaussian_recursive single-plane outputs
    lib = ref.lib
    import ctypes as C
    for name, img, sigma, scale in [("gauss_64x48_s2", mt_uniform_image(55, 64, 48, 255.0), 2.0, 1.0),
                                    ("gauss_32x32_s3", np.full((32, 32), 7.0), 3.0, 1.0),
                                    ("gauss_81_impulse_s3", np.pad(np.ones((1, 1)), 40), 3.0, 1.0),
                                    ("gauss_24x24_s2_k025", mt_uniform_image(41, 24, 24, 255.0), 2.0, 0.25),
                                    ("gauss_40x30_s0.5", mt_uniform_image(7, 40, 30, 255.0), 0.5, 1.0),
                                    ("gauss_40x30_s50", mt_uniform_image(8, 40, 30, 255.0), 50.0, 1.0)]:
        src = ref._img(img)
        o = C.c_void_p()
        assert lib.gpf_gaussian_recursive(src, sigma, scale, C.byref(o)) == 0
        lib.gpf_image_destroy(src)
        out[f"{name}/in"] = img
        out[f"{name}/out"] = ref._take(o, img.shape)
        out[f"{name}/params"] = np.array([sigma, scale])
    out["__names__"] = np.array(names)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "gpf_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(names)} gpf cases, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
