"""Scalar range-kernel evaluators of the C ABI (gpf_kernel_gauss / _gauss_poly /
_taylor / _sup_error; host fp64, csrc/range_kernel.cpp) against the unmodified
reference library (proj/src/capi.cpp:230-286): bitwise equal values and equal
statuses, over the cases of proj/tests/test_capi.cpp:184-209 and
proj/tests/test_range_kernel.cpp:27-232 (validation, tau = 0 collapse, symmetry,
degree 0, endpoints of the sup grid, monotone convergence in the degree)."""
import itertools
import math

import pytest

from paper_1505_00077_b200 import gpf


def test_values_bitwise_vs_reference(reference):
    ts = [-40.0, 0.0, 1.0, 37.5, 100.0, 255.0]
    for t, tau, sr in itertools.product(ts, [0.0, 40.0, -100.0, 127.5], [5.0, 30.0, 80.0]):
        assert gpf.kernel_gauss(t, tau, sr) == reference.kernel("gauss", t, tau, sr)[1]
        for deg in (0, 1, 5, 12, 20, 41):
            assert gpf.kernel_gauss_poly(t, tau, sr, deg) == reference.kernel("gauss_poly", t, tau, sr, deg)[1]
            assert gpf.kernel_taylor(t, tau, sr, deg) == reference.kernel("taylor", t, tau, sr, deg)[1]


@pytest.mark.parametrize("which", [0, 1])
def test_sup_error_bitwise_vs_reference(reference, which):
    for sr, deg, tau, lo, hi, step in [(30.0, 12, 40.0, 0.0, 255.0, 1.0), (30.0, 20, 0.0, -127.5, 127.5, 0.5),
                                       (10.0, 20, 127.5, 0.0, 255.0, 0.7), (50.0, 4, -60.0, 0.0, 1.0, 0.3),
                                       (30.0, 0, 10.0, 0.0, 10.0, 20.0)]:
        st, ref = reference.kernel("sup_error", sr, deg, tau, lo, hi, step, which)
        assert st == 0
        assert gpf.kernel_sup_error(sr, deg, tau, lo, hi, step, which) == ref


def test_properties():
    # test_range_kernel.cpp:34-46, 48-59, 61-74, 85-89
    assert gpf.kernel_gauss(5.0, 5.0, 3.0) == 1.0
    assert gpf.kernel_gauss(30.0, 0.0, 30.0) == pytest.approx(math.exp(-0.5), rel=1e-15)
    for t in (-50.0, 0.0, 80.0):
        assert gpf.kernel_gauss_poly(t, 0.0, 30.0, 7) == gpf.kernel_gauss(t, 0.0, 30.0)
    assert gpf.kernel_gauss_poly(60.0, 25.0, 30.0, 9) == gpf.kernel_gauss_poly(25.0, 60.0, 30.0, 9)
    assert gpf.kernel_gauss_poly(60.0, 25.0, 30.0, 0) == pytest.approx(
        gpf.kernel_gauss(60.0, 0.0, 30.0) * gpf.kernel_gauss(25.0, 0.0, 30.0), rel=1e-15)
    assert gpf.kernel_gauss_poly(100.0, -100.0, 30.0, 3) < 0.0          # 91-100: odd truncation dips negative
    assert gpf.kernel_taylor(10.0, 10.0, 30.0, 8) == 1.0
    assert abs(gpf.kernel_taylor(255.0, 0.0, 30.0, 20)) > 1e3           # 119-127: diverges far from tau
    # 129-135: exact at tau = 0; 169-184: monotone in the degree; 198-220: centering pays off
    assert gpf.kernel_sup_error(30.0, 10, 0.0, 0.0, 255.0, 1.0) == 0.0
    errs = [gpf.kernel_sup_error(40.0, n, 60.0, 0.0, 127.0, 1.0) for n in (2, 6, 10, 20, 30)]
    assert all(a >= b for a, b in zip(errs, errs[1:])) and errs[-1] < 1e-9
    assert gpf.kernel_sup_error(30.0, 20, 127.5, -127.5, 127.5, 1.0) < gpf.kernel_sup_error(30.0, 20, 255.0, 0.0, 255.0, 1.0)


def test_validation_matches_reference(reference):
    cases = [("gauss", (1.0, 2.0, 0.0)), ("gauss", (1.0, 2.0, -3.0)), ("gauss_poly", (1.0, 2.0, 30.0, -1)),
             ("taylor", (1.0, 2.0, 0.0, 4)), ("sup_error", (30.0, 12, 40.0, 255.0, 0.0, 1.0, 1)),
             ("sup_error", (30.0, 12, 40.0, 0.0, 255.0, 0.0, 0)), ("sup_error", (30.0, 12, 40.0, 0.0, 255.0, 1.0, 7)),
             ("sup_error", (0.0, 12, 40.0, 0.0, 255.0, 1.0, 0)), ("sup_error", (30.0, -2, 40.0, 0.0, 255.0, 1.0, 0))]
    for name, args in cases:
        st, _ = reference.kernel(name, *args)
        rmsg = reference.last_error()
        with pytest.raises(gpf.GpfError) as e:
            getattr(gpf, "kernel_" + name)(*args)
        assert e.value.status == st == 1
        assert rmsg in str(e.value)


def test_null_out():
    from paper_1505_00077_b200 import _lib
    L = _lib.lib()
    assert L.gpf_kernel_gauss(1.0, 2.0, 3.0, None) == 1
    assert L.gpf_last_error().decode() == "out is null"
    assert L.gpf_kernel_sup_error(30.0, 12, 40.0, 0.0, 255.0, 1.0, 0, None) == 1
