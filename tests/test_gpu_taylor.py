"""Taylor-polynomial baseline on the GPU (gpf_filter_taylor) against the
unmodified reference library: bitwise equal outputs and equal fallback counts
(the fp64 path replicates taylor_bilateral, bilateral.cpp:160-220, in the
reference's operation order with explicitly rounded operations)."""
import numpy as np
import pytest

from paper_1505_00077_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("degree,ss,sr", [(0, 2.0, 30.0), (4, 2.0, 30.0), (10, 3.0, 50.0),
                                          (20, 2.5, 30.0), (21, 1.5, 80.0)])
def test_taylor_bitwise_vs_reference(gpu, reference, degree, ss, sr):
    img = synth.rects_image(48, 37, 6, 10.0, 11 + degree).astype(np.float64)
    st, ref, rfb = reference.taylor(img, ss, sr, degree)
    assert st == 0
    out, fb = gpu.gpf_filter_taylor(img, gpu.spatial_params(ss), gpu.range_params(sr, degree))
    assert fb == rfb
    np.testing.assert_array_equal(out, ref)


def test_taylor_fallbacks_and_constant(gpu, reference):
    two = np.zeros((8, 8))
    two[:, 4:] = 255.0
    st, ref, rfb = reference.taylor(two, 2.0, 10.0, 20)
    out, fb = gpu.gpf_filter_taylor(two, gpu.spatial_params(2.0), gpu.range_params(10.0, 20))
    assert st == 0 and fb == rfb
    np.testing.assert_array_equal(out, ref)
    c = np.full((9, 11), 40.0)
    st, ref, rfb = reference.taylor(c, 2.0, 30.0, 6)
    out, fb = gpu.gpf_filter_taylor(c, gpu.spatial_params(2.0), gpu.range_params(30.0, 6))
    np.testing.assert_array_equal(out, ref)
    assert fb == rfb


@pytest.mark.parametrize("degree,ss,radius,boundary", [(4, 2.0, 0, 0), (10, 0.4, 2, 1), (20, 3.0, 5, 2)])
def test_taylor_direct_backend_bitwise_vs_reference(gpu, reference, degree, ss, radius, boundary):
    """filt = direct_gaussian (bilateral.cpp:168-172)."""
    img = synth.rects_image(41, 30, 5, 10.0, 3 + degree).astype(np.float64)
    sp = reference.SpatialParams(ss, radius, boundary, 1.0)
    rp = reference.RangeParams(30.0, degree)
    import ctypes as C
    src, outp, rfb = reference._img(img), C.c_void_p(), C.c_longlong(-1)
    reference.lib.gpf_filter_taylor.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                                C.POINTER(C.c_longlong), C.POINTER(C.c_void_p)]
    assert reference.lib.gpf_filter_taylor(src, C.byref(sp), C.byref(rp), 0, C.byref(rfb), C.byref(outp)) == 0
    reference.lib.gpf_image_destroy(src)
    ref = reference._take(outp, img.shape)
    out, fb = gpu.gpf_filter_taylor(img, gpu.spatial_params(ss, radius, boundary), gpu.range_params(30.0, degree),
                                    backend=0)
    assert fb == rfb.value
    np.testing.assert_array_equal(out, ref)
