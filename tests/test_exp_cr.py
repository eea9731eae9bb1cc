"""csrc/exp_cr.h -- the exp() of the reference-exact fp64 mode (F_0 of GpfState::init).
CPU: its host instantiation (tests/cxx/libexp_cr_host.so, -ffp-contract=off) against the
host libm the reference calls (math.exp) and, where mpmath is importable, against the
correctly rounded value. GPU: the device instantiation returns the same bits as the host one."""
import ctypes as C
import math
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HOST = os.path.join(ROOT, "tests", "cxx", "libexp_cr_host.so")


def _inputs(n=200000, seed=5):
    r = np.random.RandomState(seed)
    edge = np.array([0.0, -0.0, 1.0, -1.0, -745.0, -744.5, -708.4, -709.0, -720.3, -746.0, -1e-300, -5e-324,
                     709.7, 710.0, -0.34657359027997264, 0.34657359027997264, float("nan")])
    return np.concatenate([-r.uniform(0, 100, n // 2), -r.uniform(0, 745, n // 4), -r.uniform(0, 1, n // 8) ** 4,
                           r.uniform(0, 700, n // 8), edge])


def _host(x):
    if not os.path.exists(HOST):
        pytest.skip("tests/cxx/libexp_cr_host.so not built")
    lib = C.CDLL(HOST)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    lib.exp_cr_host(x.ctypes.data_as(C.c_void_p), y.ctypes.data_as(C.c_void_p), C.c_longlong(x.size))
    return y


def test_host_instantiation_vs_libm_and_correct_rounding():
    x = _inputs()
    y = _host(x)
    g = np.array([math.exp(v) if v < 709.78 else float("inf") for v in x[:-1]] + [float("nan")])
    same = (y == g) | (np.isnan(y) & np.isnan(g))
    rate = 1.0 - same.mean()
    assert rate <= 3e-3, rate                      # glibc misrounds ~1 argument in 1,000
    assert np.all(np.abs(y[~same] - g[~same]) <= np.spacing(np.abs(g[~same])))   # one ulp apart there
    e = y[-17:]   # the edge arguments
    assert e[0] == 1.0 and e[1] == 1.0 and e[9] == 0.0 and e[13] == float("inf") and e[11] == 1.0
    try:
        import mpmath as mp
    except ImportError:
        return
    mp.mp.prec = 200
    r = np.random.RandomState(7)
    idx = list(np.nonzero(~same)[0][:150]) + list(r.choice(x.size - 1, 1500, replace=False))
    for i in idx:
        assert float(mp.exp(mp.mpf(float(x[i])))) == y[i], (x[i], y[i].hex())   # correctly rounded


@pytest.mark.gpu
def test_device_instantiation_equals_host(gpu):
    from paper_1505_00077_b200 import _lib
    x = np.ascontiguousarray(_inputs(400000, 9))
    y = np.empty_like(x)
    assert _lib.lib().gpf_b200_exp_cr(x.ctypes.data_as(C.c_void_p), y.ctypes.data_as(C.c_void_p), x.size) == 0
    h = _host(x)
    assert np.array_equal(y[:-1], h[:-1]) and np.isnan(y[-1])


@pytest.mark.gpu
def test_gpf_state_f0_is_the_correctly_rounded_exp(gpu, reference):
    """The fp64 drop-in output against the reference with the correctly rounded F_0."""
    from paper_1505_00077_b200 import synth
    img = synth.checker_image(256, 192, 5.0, 7).astype(np.float64)
    gpu.set_precision("fp64")
    try:
        out, fb = gpu.gpf_filter_gpf(img, gpu.spatial_params(6.0), gpu.range_params(10.0, 20))
    finally:
        gpu.set_precision("auto")
    st, ref, rfb = reference.gpf(img, 6.0, 10.0, 20)
    assert st == 0 and fb == rfb
    scale = max(1.0, float(np.abs(ref).max()))
    # ~0.1 % of the F_0 values differ by an ulp and the IIR spreads each over its row and column,
    # so the outputs agree to rounding level rather than bitwise
    assert float(np.abs(out - ref).max()) <= 1e-11 * scale
