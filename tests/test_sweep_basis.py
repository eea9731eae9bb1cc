"""CPU: the sweep realisation the kernels use, emulated in
fp64 numpy, against the reference's direct-form Deriche filter (the oracle's
restatement of spatial.cpp:186-251, pinned bitwise to the reference).

Each conjugate pole pair p_k of the reference's 4th-order recurrences is one
complex first-order section per direction, with residues A_k (causal) and B_k
(anticausal) from the partial-fraction expansion of nc / na over d. The kernels
keep each section in the output-aligned basis u1 = Re w - tau Im w,
u2 = Im w / Im p (tau = Im R / Re R, clamped to |tau Im p| <= 1), advance it as
u2' = m22 u2 + u1, u1' = m11 u1 + m12 u2 + x and emit Re R u1 (+ a u2 term only
where tau was clamped), with every emit weight divided by S = Re A_0 and the
input scaled by S. Same transfer function, so the emulation must reproduce the
oracle's row filter to fp64 rounding, across the clamp window near
sigma_s = 1.07 and out to wide kernels.
"""
import cmath
import math

import numpy as np
import pytest

L = (1.7830, 1.7230)  # pole decay constants (spatial.cpp:141-142)
W = (0.6318, 1.9970)  # pole frequencies


def sections(nc, na, d, sigma):
    p = [cmath.rect(math.exp(-L[k] / sigma), W[k] / sigma) for k in range(2)]
    p4 = p + [c.conjugate() for c in p]
    out = []
    for k in range(2):
        q = 1.0 / p[k]
        den = 1.0
        for j in range(4):
            if j != k:
                den *= 1.0 - p4[j] * q
        poly = lambda c: c[0] + q * (c[1] + q * (c[2] + q * c[3]))  # noqa: E731
        out.append((p[k], 2.0 * poly(nc) / den, 2.0 * poly(na) / den))
    return out


def basis(p, R):
    a, b = p.real, p.imag
    tau = R.imag / R.real
    if abs(tau * b) > 1.0:
        tau = math.copysign(1.0 / b, tau)
    m11, m22, m12 = a - tau * b, a + tau * b, -b * b * (1.0 + tau * tau)
    v = b * (R.real * tau - R.imag)  # u2 emit weight (0 unless clamped)
    return tau, m11, m12, m22, R.real, v


def sweep_line(x, secs):
    """Causal + anticausal outputs of one line, replicate warm starts."""
    n = len(x)
    S = secs[0][1].real  # emit normalisation
    xs = x * S
    y = np.zeros(n)
    for p, A, B in secs:
        g = 1.0 / (1.0 - p)
        for R, causal in ((A, True), (B, False)):
            tau, m11, m12, m22, er, v = basis(p, R)
            er, v = er / S, v / S
            w0 = (xs[0] if causal else xs[-1]) * g
            u1, u2 = w0.real - tau * w0.imag, w0.imag / p.imag
            order = range(n) if causal else range(n - 1, -1, -1)
            for i in order:
                if not causal:  # anticausal: emit, then take x[i]
                    y[i] += er * u1 + v * u2
                u1, u2 = m11 * u1 + m12 * u2 + xs[i], u1 + m22 * u2
                if causal:
                    y[i] += er * u1 + v * u2
    return y


@pytest.mark.parametrize("sigma", [0.5, 0.8, 0.96, 1.0, 1.07, 1.12, 1.17, 1.5, 2.0, 5.0, 20.0, 50.0])
def test_output_aligned_sections_match_direct_form(oracle, sigma):
    rng = np.random.default_rng(int(sigma * 1000))
    n = 160
    x = rng.uniform(0.0, 255.0, n)
    nc, na, d = oracle.deriche_coeffs(sigma)
    y = sweep_line(x, sections(nc, na, d, sigma))
    # oracle: the 2-D recursive Gaussian of a 1 x n image = row filter x mass^2
    ref = oracle.recursive_gaussian(x[None, :], sigma)[0]
    mass = oracle.kernel_mass_1d(sigma, math.ceil(3.0 * sigma))
    err = np.abs(y * mass * mass - ref).max() / np.abs(ref).max()
    assert err < 1e-9, err


def test_clamp_window_is_where_expected(oracle):
    """Only B_1's basis is clamped, and only for sigma_s in about [0.96, 1.17]."""
    clamped = []
    for sigma in np.arange(0.5, 5.0, 0.01):
        nc, na, d = oracle.deriche_coeffs(sigma)
        for k, (p, A, B) in enumerate(sections(nc, na, d, sigma)):
            for name, R in (("A", A), ("B", B)):
                if abs(R.imag / R.real * p.imag) > 1.0:
                    clamped.append((name, k, round(float(sigma), 2)))
    assert {(n, k) for n, k, _ in clamped} == {("B", 1)}
    s = [c[2] for c in clamped]
    assert 0.95 <= min(s) and max(s) <= 1.18
