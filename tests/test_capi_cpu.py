"""CPU: the C-ABI library loads, exports every declared symbol, and validates
arguments exactly like the reference C ABI (no device needed: validation runs
before any device work). Mirrors proj/tests/test_capi.cpp for the GPF path.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_1505_00077_b200 import _lib, gpf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for hdr in ("gpfilter.h", "gpfilter_b200.h"):
        text = open(os.path.join(ROOT, "include", "gpfilter", hdr)).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names |= set(re.findall(r"\b(gpf_\w+)\s*\(", text))
    return names


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    decl = declared_functions()
    assert decl == set(_lib.EXPORTED)
    for name in decl:
        assert hasattr(L, name), name


REFERENCE_ABI = [  # every function of proj/include/gpfilter/gpfilter.h (28)
    "gpf_compare", "gpf_decode_pgm", "gpf_encode_pgm", "gpf_filter_exact", "gpf_filter_gpf",
    "gpf_filter_taylor", "gpf_free_bytes", "gpf_gaussian_direct", "gpf_gaussian_recursive",
    "gpf_get_num_threads", "gpf_image_cdata", "gpf_image_create", "gpf_image_data",
    "gpf_image_destroy", "gpf_image_height", "gpf_image_width", "gpf_kernel_gauss",
    "gpf_kernel_gauss_poly", "gpf_kernel_sup_error", "gpf_kernel_taylor", "gpf_last_error",
    "gpf_range_params_init", "gpf_read_pgm", "gpf_set_num_threads", "gpf_spatial_params_init",
    "gpf_status_name", "gpf_version", "gpf_write_pgm",
]


def test_library_exports_the_whole_reference_abi():
    """Link-level drop-in: every function the reference header declares is exported
    (and, when the reference tree is present, the list above is the header's)."""
    L = _lib.lib()
    assert len(REFERENCE_ABI) == 28
    for name in REFERENCE_ABI:
        assert hasattr(L, name), name
    hdr = "/root/reference/proj/include/gpfilter/gpfilter.h"
    if os.path.exists(hdr):
        text = re.sub(r"/\*.*?\*/", "", open(hdr).read(), flags=re.S)
        assert sorted(set(re.findall(r"\b(gpf_\w+)\s*\(", text))) == REFERENCE_ABI


def test_version_and_status_names():
    L = _lib.lib()
    assert L.gpf_version().decode().startswith("1.0.0")
    assert L.gpf_status_name(0) == b"GPF_OK"
    assert L.gpf_status_name(3) == b"GPF_ERR_SIGMA_TOO_SMALL"
    assert L.gpf_status_name(9) == b"GPF_ERR_UNKNOWN"


def test_parameter_defaults():
    sp, rp = _lib.SpatialParams(), _lib.RangeParams()
    _lib.lib().gpf_spatial_params_init(C.byref(sp))
    _lib.lib().gpf_range_params_init(C.byref(rp))
    assert (sp.sigma_s, sp.window_radius, sp.boundary, sp.kernel_scale) == (2.0, 0, 0, 1.0)
    assert (rp.sigma_r, rp.degree) == (30.0, 20)
    _lib.lib().gpf_spatial_params_init(None)  # NULL is a no-op
    _lib.lib().gpf_range_params_init(None)


def test_image_lifecycle_and_null_safety():
    L = _lib.lib()
    h = C.c_void_p(1)
    assert L.gpf_image_create(0, 5, C.byref(h)) == _lib.GPF_ERR_INVALID_ARGUMENT
    assert h.value is None
    assert len(L.gpf_last_error()) > 0
    assert L.gpf_image_create(4, 4, None) == _lib.GPF_ERR_INVALID_ARGUMENT
    assert L.gpf_image_create(3, 2, C.byref(h)) == 0
    assert (L.gpf_image_width(h), L.gpf_image_height(h)) == (3, 2)
    data = np.ctypeslib.as_array(L.gpf_image_data(h), shape=(6,))
    assert (data == 0).all()
    L.gpf_image_destroy(h)
    L.gpf_image_destroy(None)
    assert L.gpf_image_width(None) == 0 and L.gpf_image_height(None) == 0
    assert not L.gpf_image_data(None) and not L.gpf_image_cdata(None)


def _call(img, sp, rp, backend=1, centering=1, out_ptr=True):
    L = _lib.lib()
    src = gpf.Image.from_array(img)
    out = C.c_void_p(1)
    fb = C.c_longlong(-7)
    st = L.gpf_filter_gpf(src.h, C.byref(sp) if sp is not None else None,
                          C.byref(rp) if rp is not None else None, backend, centering,
                          C.byref(fb), C.byref(out) if out_ptr else None)
    return st, out, fb, L.gpf_last_error().decode()


@pytest.mark.parametrize("case,status,needle", [
    (dict(sigma_s=-1.0), 1, "sigma_s"),
    (dict(sigma_s=0.0), 1, "sigma_s"),
    (dict(kernel_scale=0.0), 1, "kernel_scale"),
    (dict(sigma_r=0.0), 1, "sigma_r"),
    (dict(degree=-1), 1, "degree"),
    (dict(degree=63), 1, "degree"),
    (dict(boundary=9), 1, "boundary"),
    (dict(backend=7), 1, "backend"),
    (dict(backend=0, sigma_s=0.0), 1, "sigma_s"),
    (dict(backend=0, degree=-1), 1, "degree"),
    (dict(sigma_s=0.49), 3, "direct"),
    (dict(sigma_s=0.3), 3, "direct"),
])
def test_validation_statuses(case, status, needle):
    sp = gpf.spatial_params(case.get("sigma_s", 2.0), boundary=case.get("boundary", 0),
                            kernel_scale=case.get("kernel_scale", 1.0))
    rp = gpf.range_params(case.get("sigma_r", 30.0), case.get("degree", 20))
    st, out, fb, msg = _call(np.zeros((8, 8)), sp, rp, backend=case.get("backend", 1))
    assert st == status
    assert needle in msg
    assert out.value is None          # *out set to NULL before work
    assert fb.value == -7             # fallback_count untouched on error


def test_direct_backend_passes_validation():
    """GPF_BACKEND_DIRECT is provided (fp64 mode on the GPU) and takes any
    sigma_s > 0: validation passes, so the only failure left is a missing
    device (no CPU path: GPF_ERR_UNKNOWN, never INVALID_ARGUMENT / SIGMA_TOO_SMALL)."""
    sp, rp = gpf.spatial_params(0.3), gpf.range_params(30.0, 4)
    st, out, fb, msg = _call(np.zeros((8, 8)), sp, rp, backend=0)
    assert st in (0, 9), (st, msg)
    if st != 0:
        assert "CUDA" in msg and out.value is None


def test_gaussian_direct_and_kernel_null_and_validation():
    L = _lib.lib()
    src = gpf.Image.from_array(np.ones((8, 8)))
    out = C.c_void_p(1)
    sp = gpf.spatial_params(2.0)
    assert L.gpf_gaussian_direct(None, C.byref(sp), C.byref(out)) == 1
    assert L.gpf_gaussian_direct(src.h, None, C.byref(out)) == 1
    assert L.gpf_gaussian_direct(src.h, C.byref(sp), None) == 1
    for bad, needle in [(gpf.spatial_params(0.0), "sigma_s"), (gpf.spatial_params(2.0, kernel_scale=-1.0), "kernel_scale"),
                        (gpf.spatial_params(2.0, boundary=5), "boundary")]:
        out = C.c_void_p(1)
        assert L.gpf_gaussian_direct(src.h, C.byref(bad), C.byref(out)) == 1
        assert needle in L.gpf_last_error().decode() and out.value is None


def test_null_arguments():
    sp, rp = gpf.spatial_params(), gpf.range_params()
    for args in [(sp, None), (None, rp)]:
        st, _, _, msg = _call(np.zeros((4, 4)), *args)
        assert st == 1 and msg == "null argument"
    st, _, _, _ = _call(np.zeros((4, 4)), sp, rp, out_ptr=False)
    assert st == 1
    L = _lib.lib()
    out = C.c_void_p()
    assert L.gpf_filter_gpf(None, C.byref(sp), C.byref(rp), 1, 1, None, C.byref(out)) == 1


def test_gaussian_recursive_validation():
    L = _lib.lib()
    src = gpf.Image.from_array(np.ones((8, 8)))
    out = C.c_void_p()
    assert L.gpf_gaussian_recursive(src.h, 0.3, 1.0, C.byref(out)) == 3
    assert "direct" in L.gpf_last_error().decode()
    assert L.gpf_gaussian_recursive(src.h, -1.0, 1.0, C.byref(out)) == 1
    assert L.gpf_gaussian_recursive(None, 2.0, 1.0, C.byref(out)) == 1


def test_thread_count_plumbing():
    L = _lib.lib()
    assert L.gpf_get_num_threads() == 1
    assert L.gpf_set_num_threads(0) == 1
    assert L.gpf_get_num_threads() == 1
    assert L.gpf_set_num_threads(4) == 0
    assert L.gpf_get_num_threads() == 4
    assert L.gpf_set_num_threads(1) == 0


def test_plan_validation():
    with pytest.raises(gpf.GpfError) as e:
        gpf.Plan(64, 64, 0.4, 30.0)
    assert e.value.status == 3
    with pytest.raises(gpf.GpfError) as e:
        gpf.Plan(0, 64, 2.0, 30.0)
    assert e.value.status == 1


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(gpf.GpfError) as e:
        gpf.gpf_filter_gpf(np.full((8, 8), 3.0))
    assert e.value.status == 9 and "no CUDA device" in e.value.detail


def test_exact_and_compare_validation_before_device():
    """gpf_filter_exact / gpf_compare reject bad arguments with the reference's
    statuses and messages before touching the device."""
    import ctypes as C

    from paper_1505_00077_b200 import _lib, gpf
    L = _lib.lib()
    img = gpf.Image.from_array(np.zeros((4, 5)))
    out = C.c_void_p()
    sp, rp = gpf.spatial_params(), gpf.range_params()
    assert L.gpf_filter_exact(None, C.byref(sp), C.byref(rp), C.byref(out)) == _lib.GPF_ERR_INVALID_ARGUMENT
    sp.sigma_s = 0.0
    assert L.gpf_filter_exact(img.h, C.byref(sp), C.byref(rp), C.byref(out)) == _lib.GPF_ERR_INVALID_ARGUMENT
    assert b"sigma_s must be > 0" in L.gpf_last_error()
    sp = gpf.spatial_params()
    rp.sigma_r = -1.0
    assert L.gpf_filter_exact(img.h, C.byref(sp), C.byref(rp), C.byref(out)) == _lib.GPF_ERR_INVALID_ARGUMENT
    assert b"sigma_r must be > 0" in L.gpf_last_error()
    rep = _lib.ErrorReport()
    other = gpf.Image.from_array(np.zeros((4, 6)))
    assert L.gpf_compare(img.h, other.h, 0, C.byref(rep)) == _lib.GPF_ERR_INVALID_ARGUMENT
    assert b"differ in size" in L.gpf_last_error()
    assert L.gpf_compare(img.h, img.h, -1, C.byref(rep)) == _lib.GPF_ERR_INVALID_ARGUMENT
    assert L.gpf_compare(img.h, img.h, 2, C.byref(rep)) == _lib.GPF_ERR_INVALID_ARGUMENT
    assert b"no interior" in L.gpf_last_error()


def test_fp32_envelope_per_degree():
    """The AUTO precision envelope (dropin.cpp fp32_h_limit, calibrated by
    tools/h32_calibrate_n.py): 7.0 at the default degree, smaller at low and odd
    degrees where the reference's truncated series cancels sooner, the smaller
    neighbour for unsampled degrees, 0 where the fp32 kernels do not run."""
    import paper_1505_00077_b200 as g
    assert g.fp32_h_limit() == 7.0 == g.fp32_h_limit(20)
    sampled = {0: 3.5, 1: 1.5, 2: 4.0, 3: 2.5, 5: 3.5, 8: 6.0, 10: 7.0, 12: 7.0, 15: 5.0,
               25: 6.0, 30: 8.0, 40: 8.0, 48: 10.0}
    for n, lim in sampled.items():
        assert g.fp32_h_limit(n) == lim, n
    assert g.fp32_h_limit(4) == 2.5 and g.fp32_h_limit(19) == 5.0 and g.fp32_h_limit(21) == 6.0
    assert g.fp32_h_limit(-1) == 0.0 and g.fp32_h_limit(49) == 0.0
