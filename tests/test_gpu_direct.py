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
