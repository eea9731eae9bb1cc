"""The reference unit suite's pins on the GPF path, restated for the GPU library
(proj/tests/test_bilateral.cpp:141-289, proj/tests/test_spatial.cpp:206-306).
The reference's own fixtures are absent (doctest is not vendored), so inputs
come from `_mt_uniform` -- the reference's uniform noise generator restated
(mt19937, (x + 0.5) / 2^32, proj/tests/noise.hpp:46-56) -- and the expected
numbers from the reference library itself (oracle/_ref) where the pin is a
value rather than a property.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _mt_uniform(seed, w, h, hi):
    raw = np.random.RandomState(seed).randint(0, 2**32, size=w * h, dtype=np.uint32).astype(np.float64)
    u = (raw + 0.5) / 4294967296.0 * hi
    return (np.floor(u) if hi > 1.0 else u).reshape(h, w)


def _run(gpu, img, ss, sr, deg=20, cen=1, ks=1.0, mode="auto"):
    gpu.set_precision(mode)
    try:
        return gpu.gpf_filter_gpf(img, gpu.spatial_params(ss, kernel_scale=ks), gpu.range_params(sr, deg),
                                  centering=cen)
    finally:
        gpu.set_precision("auto")


def test_gpf_error_vs_exact_is_the_references(gpu, reference):
    """test_bilateral.cpp:203-216 and 218-232 on the recursive backend: the
    GPU's dB error against the exact filter equals the reference's (σr 80 and
    the degree sweep 5/10/20/30 at σr 30), and is non-increasing in N."""
    img = _mt_uniform(2, 32, 32, 256.0)
    ex = gpu.gpf_filter_exact(img, gpu.spatial_params(2.0), gpu.range_params(80.0))
    out, fb = _run(gpu, img, 2.0, 80.0)
    st, ref, rfb = reference.gpf(img, 2.0, 80.0, 20)
    assert st == 0 and fb == rfb == 0
    db, rdb = gpu.gpf_compare(ex, out)["mse_db"], gpu.gpf_compare(ex, ref)["mse_db"]
    assert abs(db - rdb) <= 0.01, (db, rdb)
    img = _mt_uniform(5, 32, 32, 256.0)
    ex = gpu.gpf_filter_exact(img, gpu.spatial_params(2.0), gpu.range_params(30.0))
    prev = 1e300
    for deg in (5, 10, 20, 30):
        out, _ = _run(gpu, img, 2.0, 30.0, deg)
        _, ref, _ = reference.gpf(img, 2.0, 30.0, deg)
        db, rdb = gpu.gpf_compare(ex, out)["mse_db"], gpu.gpf_compare(ex, ref)["mse_db"]
        assert abs(db - rdb) <= 0.01, (deg, db, rdb)
        assert db <= prev + 0.1
        prev = db


@pytest.mark.parametrize("mode,tol", [("fp64", 0.0), ("fp32", 1e-4)])
def test_centering_consistency(gpu, oracle, mode, tol):
    """test_bilateral.cpp:234-258: centred filtering equals filtering the image
    shifted by t_c with centering off, plus t_c -- bitwise in the fp64 mode
    (the reference's arithmetic), within fp32 rounding on the fp32 kernels."""
    img = _mt_uniform(13, 16, 16, 256.0)
    t_c = oracle.mean(img)
    centred, fb0 = _run(gpu, img, 2.0, 30.0, mode=mode)
    raw, fb1 = _run(gpu, img - t_c, 2.0, 30.0, cen=0, mode=mode)
    assert fb0 == fb1 == 0
    d = np.abs(centred - (raw + t_c)).max()
    assert d <= tol, d


@pytest.mark.parametrize("mode,tol", [("fp64", 1e-10), ("fp32", 0.0)])
def test_kernel_scale_invariance(gpu, mode, tol):
    """test_bilateral.cpp:272-289: kernel_scale cancels in P/Q (<= 1e-10)."""
    img = _mt_uniform(43, 16, 16, 256.0)
    base, _ = _run(gpu, img, 2.0, 30.0, mode=mode)
    scaled, _ = _run(gpu, img, 2.0, 30.0, ks=5.25, mode=mode)
    assert np.abs(base - scaled).max() <= tol


def test_recursive_gaussian_properties(gpu, oracle):
    """test_spatial.cpp:206-306 on gpf_gaussian_recursive: DC gain equals
    mass(sigma, ceil(3 sigma))^2 within 1e-6, linearity, kernel_scale,
    sigma 0.5 accepted."""
    for sigma in (0.5, 1.5, 4.0):
        m = oracle.kernel_mass_1d(sigma, int(np.ceil(3 * sigma)))
        ones = gpu.gpf_gaussian_recursive(np.ones((24, 20)), sigma)
        assert np.abs(ones - m * m).max() <= 1e-6 * m * m
    a, b = _mt_uniform(3, 20, 16, 255.0), _mt_uniform(4, 20, 16, 255.0)
    fa, fb = gpu.gpf_gaussian_recursive(a, 2.0), gpu.gpf_gaussian_recursive(b, 2.0)
    fab = gpu.gpf_gaussian_recursive(2.0 * a - 0.5 * b, 2.0)
    assert np.abs(fab - (2.0 * fa - 0.5 * fb)).max() <= 1e-9 * np.abs(fab).max()
    f3 = gpu.gpf_gaussian_recursive(a, 2.0, 3.0)
    assert np.abs(f3 - 3.0 * fa).max() <= 1e-12 * np.abs(f3).max()
