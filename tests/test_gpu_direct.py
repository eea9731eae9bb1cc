"""The direct (windowed) spatial backend on the GPU (csrc/direct.cu) against the
unmodified reference library: gpf_gaussian_direct is bitwise the reference's
direct_gaussian (proj/src/core/spatial.cpp:112-129) for every boundary mode,
window radius and ragged size; gpf_filter_gpf(..., GPF_BACKEND_DIRECT) follows
the reference's direct-backend GPF (apply_spatial, bilateral.cpp:58-62) to the
one ulp of exp() the fp64 mode allows. Property pins restated from
proj/tests/test_spatial.cpp:128-204 and proj/tests/test_capi.cpp:164-182."""
import math

import numpy as np
import pytest

from paper_1505_00077_b200 import synth

pytestmark = pytest.mark.gpu


def _noise(w, h, seed):
    return np.random.RandomState(seed).uniform(0.0, 255.0, size=(h, w))


@pytest.mark.parametrize("boundary", [0, 1, 2])
@pytest.mark.parametrize("w,h,ss,radius,ks", [
    (1, 1, 2.0, 0, 1.0), (1, 17, 2.0, 0, 1.0), (19, 1, 1.5, 3, 1.0), (37, 29, 2.0, 0, 1.0),
    (257, 33, 0.3, 1, 1.0), (300, 70, 5.0, 0, 0.5), (23, 31, 4.0, 40, 2.0),   # window wider than the image
    (64, 48, 50.0, 0, 1.0), (40, 24, 100.0, 600, 1.0),                         # apron too wide for shared memory
    (33, 20, 300.0, 2100, 1.0),                                                # taps read from global memory
])
def test_gaussian_direct_bitwise_vs_reference(gpu, reference, boundary, w, h, ss, radius, ks):
    img = _noise(w, h, 7 * w + h + boundary)
    st, ref = reference.gaussian_direct(img, ss, radius, boundary, ks)
    assert st == 0
    out = gpu.gpf_gaussian_direct(img, gpu.spatial_params(ss, radius, boundary, ks))
    np.testing.assert_array_equal(out, ref)


def test_gaussian_direct_full_hd_bitwise(gpu, reference):
    img = synth.rects_image(1920, 1080, 64, 10.0, 3).astype(np.float64)
    st, ref = reference.gaussian_direct(img, 3.0, 0, 0, 1.0)
    out = gpu.gpf_gaussian_direct(img, gpu.spatial_params(3.0))
    assert st == 0
    np.testing.assert_array_equal(out, ref)


def test_gaussian_direct_pins(gpu):
    # test_capi.cpp:164-182 / test_spatial.cpp:128-137: constants map to mass^2 (replicate)
    out = gpu.gpf_gaussian_direct(np.full((10, 12), 5.0))
    mass = sum(math.exp(-k * k / 8.0) for k in range(-6, 7))
    assert out.shape == (10, 12)
    assert np.allclose(out, 5.0 * mass * mass, rtol=1e-12, atol=0)
    # test_spatial.cpp:139-153: the impulse response is the kernel (zero boundary, centre of a 15x15)
    imp = np.zeros((15, 15))
    imp[7, 7] = 1.0
    out = gpu.gpf_gaussian_direct(imp, gpu.spatial_params(1.5, 4, 2))
    for dy in range(-4, 5):
        for dx in range(-4, 5):
            assert out[7 + dy, 7 + dx] == pytest.approx(math.exp(-(dx * dx + dy * dy) / 4.5), rel=1e-14)
    assert out[7, 7 + 5] == 0.0 and out[7 - 5, 7] == 0.0
    # 169-181: kernel_scale multiplies the output; 183-204: linearity
    a, b = _noise(21, 17, 1), _noise(21, 17, 2)
    sp = gpu.spatial_params(2.0, 5, 1)
    fa, fb = gpu.gpf_gaussian_direct(a, sp), gpu.gpf_gaussian_direct(b, sp)
    assert np.allclose(gpu.gpf_gaussian_direct(a, gpu.spatial_params(2.0, 5, 1, 3.0)), 3.0 * fa, rtol=1e-14)
    assert np.allclose(gpu.gpf_gaussian_direct(2.0 * a - 0.5 * b, sp), 2.0 * fa - 0.5 * fb, rtol=0, atol=1e-10)


@pytest.mark.parametrize("ss,sr,deg,radius,boundary,cen,ks", [
    (2.0, 30.0, 20, 0, 0, 1, 1.0), (0.4, 40.0, 10, 2, 1, 1, 1.0), (3.0, 30.0, 20, 7, 2, 0, 1.0),
    (1.0, 60.0, 5, 0, 0, 1, 0.5), (4.0, 20.0, 30, 0, 1, 1, 1.0),
])
def test_gpf_direct_backend_vs_reference(gpu, reference, ss, sr, deg, radius, boundary, cen, ks):
    img = synth.rects_image(96, 71, 8, 10.0, 21 + deg).astype(np.float64)
    st, ref, rfb = reference.gpf(img, ss, sr, deg, centering=cen, kernel_scale=ks, backend=0,
                                 window_radius=radius, boundary=boundary)
    assert st == 0
    out, fb = gpu.gpf_filter_gpf(img, gpu.spatial_params(ss, radius, boundary, ks), gpu.range_params(sr, deg),
                                 backend=0, centering=cen)
    assert gpu.last_precision() == "fp64"
    assert fb == rfb
    scale = max(1.0, float(np.abs(ref).max()))
    assert float(np.abs(out - ref).max()) <= 1e-9 * scale


def test_gpf_direct_backend_fallback_pixels(gpu, reference):
    """sigma_r 2 on a 0/255 edge: every Q underflows -> all pixels fall back, like the reference."""
    two = np.zeros((16, 16))
    two[:, 8:] = 255.0
    st, ref, rfb = reference.gpf(two, 2.0, 2.0, 20, backend=0)
    out, fb = gpu.gpf_filter_gpf(two, gpu.spatial_params(2.0), gpu.range_params(2.0, 20), backend=0)
    assert st == 0 and fb == rfb
    fell = out == two
    assert fell.sum() >= rfb
    np.testing.assert_allclose(out, ref, rtol=1e-9, atol=1e-9)


def test_gpf_direct_backend_needs_fp64_mode(gpu):
    gpu.set_precision("fp32")
    try:
        with pytest.raises(gpu.GpfError, match="fp64"):
            gpu.gpf_filter_gpf(np.zeros((8, 8)), backend=0)
    finally:
        gpu.set_precision("auto")
    out, fb = gpu.gpf_filter_gpf(np.full((8, 8), 9.0), backend=0)
    assert fb == 0 and np.allclose(out, 9.0, atol=1e-12)


def test_recursive_tracks_wide_direct_window(gpu):
    """test_spatial.cpp:234-261: the recursive Gaussian agrees with a wide direct
    window (W = 5 sigma) to the Deriche fit's accuracy, both on the GPU."""
    img = _noise(80, 60, 11)
    ss = 3.0
    wide = gpu.gpf_gaussian_direct(img, gpu.spatial_params(ss, 15))
    mass15 = sum(math.exp(-k * k / (2 * ss * ss)) for k in range(-15, 16))
    mass9 = sum(math.exp(-k * k / (2 * ss * ss)) for k in range(-9, 10))
    rec = gpu.gpf_gaussian_recursive(img, ss)
    rel = np.abs(rec / mass9 ** 2 - wide / mass15 ** 2).max() / 255.0
    assert rel <= 5e-3, rel


# --- the reference unit suite's direct-backend pins (proj/tests/test_bilateral.cpp), restated.
# Inputs: the reference's own generators restated (proj/tests/noise.hpp): the pins on noise
# images hold for those images, not for any image (the degree sweep below fails in the
# reference itself on a numpy-normal image of the same moments).

def _mt_uniform(seed, w, h, hi):
    # proj/tests/noise.hpp:46-56 restated: mt19937, (x + 0.5) / 2^32 * hi, floored for hi > 1
    raw = np.random.RandomState(seed).randint(0, 2**32, size=w * h, dtype=np.uint32).astype(np.float64)
    u = (raw + 0.5) / 4294967296.0 * hi
    return (np.floor(u) if hi > 1.0 else u).reshape(h, w)


def _gauss_noise(seed, w, h, mean=128.0, sigma=40.0):
    # proj/tests/noise.hpp:22-44 restated: Box-Muller pairs from the mt19937 stream,
    # clamp(round(mean + sigma z)) to [0, 255]
    n = w * h
    m = n + (n & 1)
    raw = np.random.RandomState(seed).randint(0, 2**32, size=m, dtype=np.uint32).astype(np.float64)
    u = (raw + 0.5) / 4294967296.0
    r = np.sqrt(-2.0 * np.log(u[0::2]))
    z = np.empty(m)
    z[0::2] = r * np.cos(6.283185307179586 * u[1::2])
    z[1::2] = r * np.sin(6.283185307179586 * u[1::2])
    return np.clip(np.floor(mean + sigma * z + 0.5), 0.0, 255.0)[:n].reshape(h, w)


def _gpf_direct(gpu, img, ss=2.0, sr=30.0, deg=20, cen=1, ks=1.0, radius=0):
    return gpu.gpf_filter_gpf(img, gpu.spatial_params(ss, radius, 0, ks), gpu.range_params(sr, deg),
                              backend=0, centering=cen)


def test_pin_constants_preserved_exactly(gpu):
    """test_bilateral.cpp:141-152."""
    out, fb = _gpf_direct(gpu, np.full((32, 32), 137.0))
    assert fb == 0 and (out == 137.0).all()


def test_pin_approaches_exact_for_large_sigma_r(gpu):
    """test_bilateral.cpp:203-216: matched direct windows, sigma_r 80 -> <= -20 dB."""
    img = _mt_uniform(2, 32, 32, 256.0)
    ex = gpu.gpf_filter_exact(img, gpu.spatial_params(2.0), gpu.range_params(80.0))
    out, fb = _gpf_direct(gpu, img, sr=80.0)
    assert fb == 0 and gpu.gpf_compare(ex, out)["mse_db"] <= -20.0


def test_pin_error_non_increasing_in_degree(gpu):
    """test_bilateral.cpp:218-232."""
    img = _gauss_noise(2, 32, 32)
    ex = gpu.gpf_filter_exact(img, gpu.spatial_params(2.0), gpu.range_params(30.0))
    prev = 1e300
    for deg in (5, 10, 20, 30):
        db = gpu.gpf_compare(ex, _gpf_direct(gpu, img, deg=deg)[0])["mse_db"]
        assert db <= prev + 0.1
        prev = db


def test_pin_centering_consistency_bitwise(gpu, oracle):
    """test_bilateral.cpp:234-258: centred == shift by t_c, centering off, add t_c back (bitwise)."""
    img = _mt_uniform(13, 16, 16, 256.0)
    out, fb = _gpf_direct(gpu, img)
    t_c = oracle.mean(img)
    raw, rfb = _gpf_direct(gpu, img - t_c, cen=0)
    assert fb == rfb == 0
    np.testing.assert_array_equal(out, raw + t_c)


def test_pin_kernel_scale_invariance(gpu):
    """test_bilateral.cpp:272-289: kernel_scale cancels in P/Q to 1e-10."""
    img = _mt_uniform(43, 16, 16, 256.0)
    base, _ = _gpf_direct(gpu, img)
    scaled, _ = _gpf_direct(gpu, img, ks=5.25)
    assert np.abs(base - scaled).max() <= 1e-10


def test_pin_backends_agree_away_from_border(gpu):
    """test_bilateral.cpp:291-315: direct (W = 4 sigma) vs recursive within 0.5 inside the 3 sigma band."""
    img = _gauss_noise(9, 64, 64)
    for sigma in (2.0, 5.0):
        d, _ = _gpf_direct(gpu, img, ss=sigma, radius=int(math.ceil(4.0 * sigma)))
        r, _ = gpu.gpf_filter_gpf(img, gpu.spatial_params(sigma), gpu.range_params(30.0, 20))
        b = int(math.ceil(3.0 * sigma))
        assert np.abs(d[b:64 - b, b:64 - b] - r[b:64 - b, b:64 - b]).max() <= 0.5


def test_pin_fallback_count_and_values(gpu):
    """test_bilateral.cpp:317-333: sigma_r 1, degree 5 on a two-level image: all 64 pixels fall back."""
    img = np.zeros((8, 8))
    img[:, 4:] = 255.0
    out, fb = _gpf_direct(gpu, img, sr=1.0, deg=5)
    assert fb == 64
    np.testing.assert_array_equal(out, img)


def test_pin_taylor_direct(gpu):
    """test_bilateral.cpp:335-356 (constants), 358-374 (K = 0 is num / den of direct_gaussian,
    bitwise), 376-391 (worse than gpf on noise), 393-409 (falls back on the two-level image)."""
    sp = gpu.spatial_params(2.0)
    one, fb = gpu.gpf_filter_taylor(np.full((8, 8), 1.0), sp, gpu.range_params(30.0, 20), backend=0)
    assert fb == 0 and np.abs(one - 1.0).max() <= 1e-12
    mid, fb = gpu.gpf_filter_taylor(np.full((8, 8), 100.0), sp, gpu.range_params(30.0, 20), backend=0)
    assert fb == 0 and np.abs(mid - 100.0).max() <= 1e-6
    img = _mt_uniform(47, 16, 16, 256.0)
    num = gpu.gpf_gaussian_direct(img, sp)
    den = gpu.gpf_gaussian_direct(np.ones((16, 16)), sp)
    for deg in (0, 1):
        out, fb = gpu.gpf_filter_taylor(img, sp, gpu.range_params(30.0, deg), backend=0)
        assert fb == 0
        np.testing.assert_array_equal(out, num / den)
    noisy = _gauss_noise(2, 32, 32)
    ex = gpu.gpf_filter_exact(noisy, sp, gpu.range_params(30.0))
    gp, _ = _gpf_direct(gpu, noisy)
    ty, _ = gpu.gpf_filter_taylor(noisy, sp, gpu.range_params(30.0, 20), backend=0)
    assert np.isfinite(ty).all()
    assert gpu.gpf_compare(ex, ty)["mse_db"] > gpu.gpf_compare(ex, gp)["mse_db"]
    two = np.zeros((8, 8))
    two[:, 4:] = 255.0
    out, fb = gpu.gpf_filter_taylor(two, sp, gpu.range_params(1.0, 2), backend=0)
    assert fb > 0 and np.isfinite(out).all()


def test_tiled_and_simple_kernels_agree_bitwise(gpu, reference, monkeypatch):
    """W <= 512 runs the register-tiled passes (R outputs per thread); GPF_B200_DIRECT_SIMPLE=1
    forces the one-output-per-thread kernels. Both are the reference's bits."""
    img = _noise(1100, 37, 5)
    for ss, radius, boundary in [(2.0, 0, 0), (2.0, 0, 2), (4.0, 12, 1), (4.5, 13, 2), (30.0, 90, 1), (170.0, 512, 0)]:
        st, ref = reference.gaussian_direct(img, ss, radius, boundary, 1.0)
        assert st == 0
        monkeypatch.delenv("GPF_B200_DIRECT_SIMPLE", raising=False)
        tiled = gpu.gpf_gaussian_direct(img, gpu.spatial_params(ss, radius, boundary))
        monkeypatch.setenv("GPF_B200_DIRECT_SIMPLE", "1")
        simple = gpu.gpf_gaussian_direct(img, gpu.spatial_params(ss, radius, boundary))
        monkeypatch.delenv("GPF_B200_DIRECT_SIMPLE")
        np.testing.assert_array_equal(tiled, ref)
        np.testing.assert_array_equal(simple, ref)
    tall = _noise(37, 1100, 6)
    st, ref = reference.gaussian_direct(tall, 6.0, 0, 1, 1.0)
    np.testing.assert_array_equal(gpu.gpf_gaussian_direct(tall, gpu.spatial_params(6.0, 0, 1)), ref)
