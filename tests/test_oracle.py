"""CPU: pin the oracle (plain-C fp64 restatement) against the reference.

The golden fixtures in tests/golden/gpf_golden.npz were produced by the
unmodified reference library (tests/golden/make_golden.py); the restatement
must reproduce them bitwise. Where oracle/_ref is present (it is built here from
/root/reference), the two are also compared live on fresh inputs.
"""
import numpy as np
import pytest

from paper_1505_00077_b200 import synth


def _gpf_cases(golden):
    return [str(n) for n in golden["__names__"]]


def test_oracle_matches_golden_bitwise(golden, oracle):
    for name in _gpf_cases(golden):
        img = golden[f"{name}/in"]
        ss, sr, deg, cen, ks = golden[f"{name}/params"]
        out, fb, _ = oracle.gpf(img, ss, sr, int(deg), int(cen), ks)
        assert fb == int(golden[f"{name}/fb"]), name
        np.testing.assert_array_equal(out, golden[f"{name}/out"], err_msg=name)


def test_oracle_gaussian_matches_golden_bitwise(golden, oracle):
    names = sorted({k.split("/")[0] for k in golden.files if k.startswith("gauss_")})
    assert len(names) == 6
    for name in names:
        sigma, scale = golden[f"{name}/params"]
        out = oracle.recursive_gaussian(golden[f"{name}/in"], sigma, scale)
        np.testing.assert_array_equal(out, golden[f"{name}/out"], err_msg=name)


def test_survey_pins(golden, oracle):
    # proj/tests/test_bilateral.cpp:317-333 on the recursive backend: 64/64
    # fallbacks, output == input bitwise.
    img = golden["fallback_sr1_n5/in"]
    out, fb, _ = oracle.gpf(img, 2.0, 1.0, 5)
    assert fb == 64
    np.testing.assert_array_equal(out, img)
    # same image, sigma_r 30, N 20 (SURVEY 8(c) probe values)
    out, fb, _ = oracle.gpf(img, 2.0, 30.0, 20)
    assert fb == 0
    assert abs(out.ravel()[0] - 0.527253) < 1e-6
    assert abs(out.ravel()[63] - 254.472747) < 1e-6


def test_mean_examples(oracle):
    # SPEC.md mean_intensity examples
    assert oracle.mean(np.zeros((2, 2))) == 0.0
    assert oracle.mean(np.array([[0.0, 100.0], [100.0, 200.0]])) == 100.0


def test_kernel_mass_and_radius(oracle):
    for s in (0.5, 2.0, 3.0, 50.0):
        r = int(np.ceil(3 * s))
        ks = np.arange(-r, r + 1)
        assert abs(oracle.kernel_mass_1d(s, r) - np.exp(-ks * ks / (2 * s * s)).sum()) < 1e-12


def test_oracle_equals_reference_live(reference, oracle):
    rng = np.random.default_rng(3)
    for (w, h, ss, sr, deg, cen, ks) in [(64, 48, 2.0, 30.0, 20, 1, 1.0), (37, 53, 7.5, 12.0, 12, 1, 1.0),
                                         (50, 50, 0.5, 45.0, 3, 0, 2.0), (16, 200, 25.0, 30.0, 20, 1, 1.0)]:
        img = np.floor(rng.uniform(0, 256, size=(h, w)))
        st, ref_out, ref_fb = reference.gpf(img, ss, sr, deg, cen, ks)
        assert st == 0
        out, fb, _ = oracle.gpf(img, ss, sr, deg, cen, ks)
        assert fb == ref_fb
        np.testing.assert_array_equal(out, ref_out)


def test_oracle_thread_count_bitwise(oracle):
    img = synth.rects_image(64, 40, 4, 10.0, 7)
    a, fa, _ = oracle.gpf(img, 3.0, 30.0, 20, threads=1)
    b, fb, _ = oracle.gpf(img, 3.0, 30.0, 20, threads=4)
    assert fa == fb
    np.testing.assert_array_equal(a, b)


def test_reference_error_strings(reference):
    img = np.zeros((8, 8))
    st, _, _ = reference.gpf(img, 0.49, 30.0, 20)
    assert st == 3 and "direct" in reference.last_error()
    st, _, _ = reference.gpf(img, 2.0, 30.0, -1)
    assert st == 1 and "degree" in reference.last_error()
    st, _, _ = reference.gpf(img, 2.0, 30.0, 20, kernel_scale=0.0)
    assert st == 1 and "kernel_scale" in reference.last_error()


def test_synth_is_deterministic():
    a = synth.make(synth.scaled(synth.CONFIGS[1], 64, 64))
    b = synth.make(synth.scaled(synth.CONFIGS[1], 64, 64))
    assert a.dtype == np.float32 and a.min() >= 0 and a.max() <= 255
    np.testing.assert_array_equal(a, b)
    c = synth.make(synth.scaled(synth.CONFIGS[5], 128, 128))
    assert set(np.unique(np.round(c[c > 200] / 255.0))) <= {1.0}


@pytest.mark.parametrize("cid", [1, 2, 5])
def test_synth_shapes(cid):
    cfg = synth.CONFIGS[cid]
    small = synth.scaled(cfg, 96, 64)
    img = synth.make(small)
    assert img.shape == (64, 96)
