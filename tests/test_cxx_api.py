"""The C++ entry point gpfilter::gpf (include/gpfilter/gpfilter.hpp) against the
reference's own C++ core (proj/src/core/bilateral.hpp:73-75, built unmodified
into oracle/_ref by oracle/Makefile): tests/cxx/gpf_cxx_driver.cpp is compiled
against each, and both binaries get the same arguments and input.

CPU: the exceptions (type and message) of the validation path, which runs
before any device work. GPU: the filtered images, including the midpoint
centering mode that only the C++ API reaches (ref bilateral.hpp:15-21).
"""
import os
import subprocess
import tempfile

import numpy as np
import pytest

from paper_1505_00077_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OURS = os.path.join(ROOT, "tests", "cxx", "gpf_cxx_driver_b200")
REF = os.path.join(ROOT, "oracle", "_ref", "gpf_cxx_driver_ref")


def drive(binary, img, ss=3.0, sr=30.0, deg=20, cen=1, mode="mean", low=0.0, high=255.0,
          backend="recursive", ks=1.0, radius=9, state=None, fn=None):
    if not os.path.exists(binary):
        pytest.skip(f"{binary} not built")
    with tempfile.TemporaryDirectory() as d:
        src, dst = os.path.join(d, "in.raw"), os.path.join(d, "out.raw")
        h, w = img.shape if img is not None else (0, 0)
        if img is not None:
            np.ascontiguousarray(img, dtype="<f8").tofile(src)
        out = subprocess.run([binary, src, str(w), str(h), dst, repr(ss), repr(sr), str(deg), str(cen),
                              mode, repr(low), repr(high), backend, repr(ks), str(radius)]
                             + ([f"state:{state}"] if state is not None else [])
                             + ([f"fn:{fn}"] if fn is not None else []),
                             capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr
        line = out.stdout.strip()
        if line.startswith("ok") and state is not None:
            raw = np.fromfile(dst, dtype="<f8")
            names = ["G", "F", "Fbar", "P", "Q", "H", "out"]
            res = {"t_c": raw[0], "c": raw[1], "n": int(raw[2])}
            res.update({k: raw[3 + i * h * w: 3 + (i + 1) * h * w].reshape(h, w) for i, k in enumerate(names)})
            return int(line.split()[1]), res
        if line.startswith("ok") and fn == "misc":
            return int(line.split()[1]), np.fromfile(dst, dtype="<f8")
        if line.startswith("ok"):
            return int(line.split()[1]), np.fromfile(dst, dtype="<f8").reshape(h, w)
        _, kind, msg = line.split(" ", 2)
        return kind, msg


ERROR_CASES = [
    dict(ss=0.4),                    # SigmaTooSmallError, "direct" in the message
    dict(ss=0.0),                    # SpatialParams: sigma_s must be > 0
    dict(radius=0),                  # SpatialParams: window_radius must be >= 1
    dict(ks=0.0),                    # SpatialParams: kernel_scale must be > 0
    dict(sr=0.0),                    # RangeParams: sigma_r must be > 0
    dict(deg=-1),                    # RangeParams: degree must be >= 0
    dict(low=200.0, high=100.0),     # GpfOptions: range.low must be < range.high
    dict(low=5.0, high=5.0, cen=0),  # checked even with centering off
]


@pytest.mark.parametrize("case", ERROR_CASES, ids=[str(c) for c in ERROR_CASES])
def test_exceptions_match_reference(case):
    img = synth.rects_image(16, 12, 2, 10.0, 1).astype(np.float64)
    ref = drive(REF, img, **case)
    ours = drive(OURS, img, **case)
    assert isinstance(ref[0], str) and ref == ours, (ref, ours)


def test_empty_image_rejected_like_reference():
    ref = drive(REF, None)
    ours = drive(OURS, None)
    assert ref == ours == ("invalid_argument", "Image dimensions must be >= 1")


def test_direct_backend_validates_like_reference():
    """SpatialBackend::direct: same parameter exceptions as the reference, and
    no SigmaTooSmallError below 0.5 (only the recursive backend has that limit)."""
    img = synth.rects_image(16, 12, 2, 10.0, 1).astype(np.float64)
    for case in [dict(ss=0.0), dict(radius=0), dict(ks=0.0), dict(deg=-1)]:
        ref = drive(REF, img, backend="direct", **case)
        ours = drive(OURS, img, backend="direct", **case)
        assert isinstance(ref[0], str) and ref == ours, (ref, ours)
    ours = drive(OURS, img, backend="direct", ss=0.4)
    assert ours[0] not in ("SigmaTooSmallError", "invalid_argument"), ours


@pytest.mark.gpu
@pytest.mark.parametrize("case", [dict(ss=2.0, radius=6), dict(ss=0.4, radius=2),
                                  dict(ss=3.0, radius=9, mode="midpoint", ks=0.5)])
def test_direct_backend_matches_reference_core(case):
    """gpfilter::gpf(..., SpatialBackend::direct) against the reference's C++ core."""
    img = synth.rects_image(40, 28, 3, 10.0, 5).astype(np.float64)
    rfb, ref = drive(REF, img, backend="direct", **case)
    fb, out = drive(OURS, img, backend="direct", **case)
    assert fb == rfb
    assert np.abs(out - ref).max() <= 1e-9


@pytest.mark.gpu
@pytest.mark.parametrize("opts", [
    dict(),                                        # mean centering (gpf_filter_gpf's default)
    dict(mode="midpoint"),                         # t_c = 127.5
    dict(mode="midpoint", low=20.0, high=120.0),   # t_c = 70
    dict(cen=0),                                   # no centering (t_c = 0)
    dict(ks=2.5, ss=5.0, sr=25.0),                 # kernel_scale cancels, fallback threshold moves
    dict(sr=10.0, ss=6.0),                         # outside the fp32 envelope: fp64 mode
    dict(deg=8, sr=40.0),
])
def test_gpf_matches_reference_cxx(gpu, opts):
    img = synth.rects_image(320, 240, 12, 10.0, 11).astype(np.float64)
    rfb, ref = drive(REF, img, **opts)
    fb, out = drive(OURS, img, **opts)
    assert fb == rfb
    assert np.abs(out - ref).max() <= 1e-3, opts


def test_gpf_state_validates_like_reference():
    """GpfState::init (bilateral.cpp:64-72): the same exceptions as the reference."""
    img = synth.rects_image(16, 12, 2, 10.0, 1).astype(np.float64)
    for case in [dict(ss=0.4), dict(ss=0.0), dict(radius=0), dict(sr=0.0), dict(deg=-1),
                 dict(low=200.0, high=100.0)]:
        ref = drive(REF, img, state=2, **case)
        ours = drive(OURS, img, state=2, **case)
        assert isinstance(ref[0], str) and ref == ours, (ref, ours)


@pytest.mark.gpu
@pytest.mark.parametrize("backend,steps,opts", [
    ("direct", 0, dict()), ("direct", 6, dict()), ("recursive", 3, dict()),
    ("recursive", 21, dict()), ("direct", 21, dict(mode="midpoint")), ("recursive", 11, dict(cen=0, deg=10)),
])
def test_gpf_state_stepping_matches_reference_core(backend, steps, opts):
    """GpfState (ref bilateral.hpp:38-68; test_bilateral.cpp:154-201): every state image after
    K steps against the reference's own GpfState -- t_c, c and n equal, G and H bitwise (pure
    fp64 products of the input), F / Fbar / P / Q to the ulp of exp() -- and finalize()."""
    img = synth.rects_image(40, 28, 3, 10.0, 5).astype(np.float64)
    rfb, ref = drive(REF, img, backend=backend, state=steps, radius=9, **opts)
    fb, out = drive(OURS, img, backend=backend, state=steps, radius=9, **opts)
    assert fb == rfb
    assert out["n"] == ref["n"] == steps and out["c"] == ref["c"] and out["t_c"] == ref["t_c"]
    np.testing.assert_array_equal(out["H"], ref["H"])
    np.testing.assert_array_equal(out["G"], ref["G"])
    for k in ("F", "Fbar", "P", "Q"):
        scale = max(float(np.abs(ref[k]).max()), 1e-300)
        assert float(np.abs(out[k] - ref[k]).max()) <= 1e-13 * scale, k
    assert float(np.abs(out["out"] - ref["out"]).max()) <= 1e-9


@pytest.mark.gpu
def test_gpf_state_full_run_equals_gpf():
    """init + (degree + 1) steps + finalize is gpf() (bilateral.cpp:150-158): against the
    reference's gpf on the reference side, and ours within 1e-9 of it."""
    img = synth.rects_image(40, 28, 3, 10.0, 7).astype(np.float64)
    rfb, ref = drive(REF, img, deg=12)
    fb, st = drive(OURS, img, deg=12, state=13)
    assert fb == rfb and float(np.abs(st["out"] - ref).max()) <= 1e-9


def test_core_functions_validate_like_reference():
    """exact_bilateral / taylor_bilateral / direct_gaussian / recursive_gaussian: the reference
    core's exceptions (type and message) for bad parameters, before any device work."""
    img = synth.rects_image(16, 12, 2, 10.0, 1).astype(np.float64)
    for fn, case in [("exact", dict(ss=0.0)), ("exact", dict(sr=0.0)), ("exact", dict(radius=0)),
                     ("taylor", dict(deg=-1)), ("taylor", dict(ss=0.3)), ("direct", dict(ks=0.0)),
                     ("recursive", dict(ss=0.4)), ("recursive", dict(ss=-1.0))]:
        ref = drive(REF, img, fn=fn, **case)
        ours = drive(OURS, img, fn=fn, **case)
        assert isinstance(ref[0], str) and ref == ours, (fn, case, ref, ours)


@pytest.mark.gpu
@pytest.mark.parametrize("fn,case,tol", [
    ("exact", dict(ss=2.0, radius=6), 1e-10), ("taylor", dict(ss=2.5, deg=10), 0.0),
    ("taylor", dict(ss=2.0, deg=8, backend="direct", radius=5), 0.0),
    ("direct", dict(ss=3.0, radius=7, ks=0.5), 0.0), ("recursive", dict(ss=4.0, ks=2.0), 0.0),
])
def test_core_functions_match_reference_core(fn, case, tol):
    """The other C++ entry points against the reference's C++ core: the Gaussians and the Taylor
    baseline bitwise (fallback counts equal), the exact filter to 1e-10."""
    img = synth.rects_image(40, 28, 3, 10.0, 5).astype(np.float64)
    rfb, ref = drive(REF, img, fn=fn, **case)
    fb, out = drive(OURS, img, fn=fn, **case)
    assert fb == rfb
    if tol == 0.0:
        np.testing.assert_array_equal(out, ref)
    else:
        assert float(np.abs(out - ref).max()) <= tol


@pytest.mark.gpu
def test_core_scalars_and_metrics_match_reference_core():
    """mean_intensity, kernel_mass_1d, compare, max_abs_diff, the range-kernel evaluators."""
    img = synth.rects_image(40, 28, 3, 10.0, 5).astype(np.float64)
    _, ref = drive(REF, img, fn="misc", deg=12)
    _, out = drive(OURS, img, fn="misc", deg=12)
    names = ["mean", "mass", "mse", "mse_db", "max_abs", "pixels", "max_abs_diff", "gauss", "gauss_poly",
             "taylor", "sup_gp", "sup_taylor"]
    for k, a, b in zip(names, out, ref):
        if k in ("mse", "mse_db"):
            assert a == pytest.approx(b, rel=1e-12), k
        else:
            assert a == b, (k, a, b)
