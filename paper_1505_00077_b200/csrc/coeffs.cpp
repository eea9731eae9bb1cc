// Host-side filter constants (fp64), see gpf_internal.h.
#include <algorithm>
#include <cmath>
#include <complex>
#include <string>

#include "gpf_internal.h"

namespace gpfb {

using cd = std::complex<double>;

// proj/src/core/spatial.cpp:14-16
int default_window_radius(double sigma_s) { return static_cast<int>(std::ceil(3.0 * sigma_s)); }

// proj/src/core/spatial.cpp:43-50 (same summation order)
double kernel_mass_1d(double sigma_s, int radius) {
  double mass = 0.0;
  for (int k = -radius; k <= radius; ++k)
    mass += std::exp(-(static_cast<double>(k) * k) / (2.0 * sigma_s * sigma_s));
  return mass;
}

namespace {

struct Deriche {
  double nc[4], na[4], d[4];
};

// The reference's 4th-order Deriche fit, proj/src/core/spatial.cpp:140-181:
// causal numerator nc, anticausal numerator na, shared denominator d, both
// numerators normalised to exact unit DC gain.
Deriche deriche(double s) {
  const double a1 = 1.6800, c1 = 3.7350, l1 = 1.7830, w1 = 0.6318;
  const double a2 = -0.6803, c2 = -0.2598, l2 = 1.7230, w2 = 1.9970;
  const double e1 = std::exp(-l1 / s), e2 = std::exp(-l2 / s);
  const double cw1 = std::cos(w1 / s), sw1 = std::sin(w1 / s);
  const double cw2 = std::cos(w2 / s), sw2 = std::sin(w2 / s);
  Deriche k{};
  k.nc[0] = a1 + a2;
  k.nc[1] = e2 * (c2 * sw2 - (a2 + 2.0 * a1) * cw2) + e1 * (c1 * sw1 - (2.0 * a2 + a1) * cw1);
  k.nc[2] = 2.0 * e1 * e2 * ((a1 + a2) * cw2 * cw1 - c1 * cw2 * sw1 - c2 * cw1 * sw2) +
            a2 * e1 * e1 + a1 * e2 * e2;
  k.nc[3] = e2 * e1 * e1 * (c2 * sw2 - a2 * cw2) + e1 * e2 * e2 * (c1 * sw1 - a1 * cw1);
  k.d[0] = -2.0 * e2 * cw2 - 2.0 * e1 * cw1;
  k.d[1] = 4.0 * cw2 * cw1 * e1 * e2 + e1 * e1 + e2 * e2;
  k.d[2] = -2.0 * cw1 * e1 * e2 * e2 - 2.0 * cw2 * e2 * e1 * e1;
  k.d[3] = e1 * e1 * e2 * e2;
  for (int i = 0; i < 3; ++i) k.na[i] = k.nc[i + 1] - k.d[i] * k.nc[0];
  k.na[3] = -k.d[3] * k.nc[0];
  double num = 0.0, den = 1.0;
  for (int i = 0; i < 4; ++i) {
    num += k.nc[i] + k.na[i];
    den += k.d[i];
  }
  const double dc = num / den;
  for (int i = 0; i < 4; ++i) {
    k.nc[i] /= dc;
    k.na[i] /= dc;
  }
  return k;
}

cd poly3(const double c[4], cd q) { return c[0] + q * (c[1] + q * (c[2] + q * c[3])); }

float2 dup(double v) { return make_float2(static_cast<float>(v), static_cast<float>(v)); }

}  // namespace

void deriche_coeffs_f64(double sigma, double nc[4], double na[4], double d[4]) {
  const Deriche k = deriche(sigma);
  for (int i = 0; i < 4; ++i) {
    nc[i] = k.nc[i];
    na[i] = k.na[i];
    d[i] = k.d[i];
  }
}

FilterConsts make_filter_consts(double s) {
  const Deriche k = deriche(s);
  // Denominator 1 + d0 q + d1 q^2 + d2 q^3 + d3 q^4 = prod_j (1 - p_j q) with
  // p = e^{-l/s} e^{+-i w/s} (the damped cosines of spatial.cpp:186-216).
  const cd p[4] = {std::polar(std::exp(-1.7830 / s), 0.6318 / s),
                   std::polar(std::exp(-1.7230 / s), 1.9970 / s),
                   std::polar(std::exp(-1.7830 / s), -0.6318 / s),
                   std::polar(std::exp(-1.7230 / s), -1.9970 / s)};
  FilterConsts fc{};
  double are[2], bre[2], aev = 0.0;  // emit weights before normalisation
  for (int sec = 0; sec < 2; ++sec) {
    const cd pk = p[sec];
    const cd q = 1.0 / pk;
    cd den = 1.0;
    for (int j = 0; j < 4; ++j)
      if (j != sec) den *= (1.0 - p[j] * q);
    // causal: sum_m nc_m z^-m / D(z^-1); residue at z^-1 = q
    const cd A = 2.0 * poly3(k.nc, q) / den;
    // anticausal: z * sum_m na_m z^m / D(z), expanded as sum_k B_k z/(1 - p_k z)
    const cd B = 2.0 * poly3(k.na, q) / den;
    const cd g = 1.0 / (1.0 - pk);
    const double pr = pk.real(), si = pk.imag();
    fc.pr2[sec] = dup(pr);
    fc.gr2[sec] = dup(g.real());
    fc.gi2[sec] = dup(g.imag());
    fc.gs2[sec] = dup(g.imag() / si);
    fc.ips2[sec] = dup(1.0 / si);
    // sweep bases (see FilterConsts): tau = Im R / Re R, clamped to |tau Im p| <= 1
    auto basis = [&](const cd& R, float2* m11, float2* m12, float2* m22, double& tau) {
      tau = R.imag() / R.real();
      if (!(std::fabs(tau * si) <= 1.0)) tau = std::copysign(1.0 / si, tau);
      m11[sec] = dup(pr - tau * si);
      m22[sec] = dup(pr + tau * si);
      m12[sec] = dup(-si * si * (1.0 + tau * tau));
    };
    double tc = 0.0, ta = 0.0;
    basis(A, fc.cm11, fc.cm12, fc.cm22, tc);
    basis(B, fc.am11, fc.am12, fc.am22, ta);
    // Re(R w) = Re R u1 + Im p (Re R tau - Im R) u2
    are[sec] = A.real();
    bre[sec] = B.real();
    const double cv = si * (A.real() * tc - A.imag()), av = si * (B.real() * ta - B.imag());
    if (std::fabs(cv) > 1e-12 * std::abs(A) || (sec == 0 && std::fabs(av) > 1e-12 * std::abs(B)))
      throw Error{9, "sweep basis: unsupported residue (sigma_s " + std::to_string(s) + ")"};
    // exactly zero unless B_1's basis was clamped (rounding leaves ~1e-18 otherwise),
    // so the sweep kernels' no-u2-term instantiation is selected
    if (sec == 1) aev = std::fabs(av) > 1e-12 * std::abs(B) ? av : 0.0;
    fc.ntau_a[sec] = dup(-ta);
    fc.cgu1[sec] = dup(g.real() - tc * g.imag());
  }
  // emit normalisation (see FilterConsts): S = Re A_0 > 0 for every sigma_s
  const double S = are[0];
  for (int sec = 0; sec < 2; ++sec) {
    fc.ce[sec] = dup(are[sec] / S);
    fc.ae[sec] = dup(bre[sec] / S);
  }
  fc.aev = dup(aev / S);
  fc.seed_log2 = 2.0 * std::log2(S);
  return fc;
}

TileConsts make_tile_consts(double s, int width, int height) {
  const cd p[2] = {std::polar(std::exp(-1.7830 / s), 0.6318 / s),
                   std::polar(std::exp(-1.7230 / s), 1.9970 / s)};
  TileConsts tc{};
  const int last_y = height - (height - 1) / kTile * kTile;  // rows in the last row chunk
  const int last_x = width - (width - 1) / kTile * kTile;    // columns in the last strip
  for (int j = 0; j < kTile; ++j) {
    const cd w0 = std::pow(p[0], j), w1 = std::pow(p[1], j);
    tc.w4[j] = make_float4(static_cast<float>(w0.real()), static_cast<float>(w0.imag()),
                           static_cast<float>(w1.real()), static_cast<float>(w1.imag()));
  }
  for (int k = 0; k < 2; ++k) {
    const cd pt = std::pow(p[k], kTile), py = std::pow(p[k], last_y), px = std::pow(p[k], last_x);
    tc.pTr2[k] = dup(pt.real());
    tc.pTi2[k] = dup(pt.imag());
    tc.pYr2[k] = dup(py.real());
    tc.pYi2[k] = dup(py.imag());
    tc.pXr2[k] = dup(px.real());
    tc.pXi2[k] = dup(px.imag());
  }
  return tc;
}

RangeConsts make_range_consts(const Params& p) {
  RangeConsts rc{};
  rc.sigma_r = p.sigma_r;
  rc.inv_sr = 1.0 / p.sigma_r;
  rc.inv2s2 = 1.0 / (2.0 * p.sigma_r * p.sigma_r);
  rc.degree = p.degree;
  rc.planes = p.degree + 2;
  rc.pairs = (rc.planes + 1) / 2;
  rc.centering = p.centering;
  rc.tc_fixed = p.tc_fixed;
  // Plane scaling s_n = s0 - k n. |F_n| = |H^n exp(-H^2/2)| <= (n/e)^(n/2);
  // pick the smallest k that keeps the last (padded) plane at or below 2^s0.
  const int n_max = 2 * rc.pairs - 1;
  const double lb = n_max > 0 ? 0.5 * n_max * std::log2(n_max / std::exp(1.0)) : 0.0;
  int k = static_cast<int>(std::ceil(lb / std::max(1, n_max)));
  if (k < 1) k = 1;
  const int s0 = 100;
  rc.e_scale = std::ldexp(1.0, s0);
  rc.e_log2 = s0;
  rc.exp2_k = 1.4426950408889634 / (2.0 * p.sigma_r * p.sigma_r);
  rc.h_step = static_cast<float>(std::ldexp(1.0, -k));
  rc.c0 = static_cast<float>(std::ldexp(1.0, -s0));
  rc.p_scale = static_cast<float>(std::ldexp(1.0, k));
  for (int n = 0; n < kMaxPlanes; ++n)
    rc.w_step[n] = static_cast<float>(std::ldexp(1.0, k) / (n + 1));
  double kc = std::ldexp(1.0, -s0);  // c0
  for (int n = 0; n < kMaxPlanes; ++n) {
    rc.k_coef[n] = static_cast<float>(kc);
    kc *= std::ldexp(1.0, k) / (n + 1);
  }
  const double mass = kernel_mass_1d(p.sigma_s, default_window_radius(p.sigma_s));
  rc.q_thresh = static_cast<float>(1e-8 / (mass * mass * p.kernel_scale));
  finalize_range_consts(rc);
  return rc;
}

void fill_gscale_consts(TileConsts& tc, RangeConsts& rc) {
  // K_n = prod_{i<n} w_i = 2^{kn}/n! takes plane n from the seed chain
  // (es m^n = F_n 2^{s0-kn} S^2) to G units (F_n 2^{s0} S^2 / n!), times
  // 2^-kGsShift: G units are 2^{s0-64} = 2^36 times the true plane / n!, so
  // the contraction's Q and P (which reach ~1e8 in true units just past the
  // fp32 envelope, where the truncated series diverges) stay far from the fp32
  // maximum, while every significant plane value stays normal
  constexpr int kGsShift = 64;
  double K[34];
  K[0] = std::ldexp(1.0, -kGsShift);
  for (int n = 1; n < 34; ++n) K[n] = K[n - 1] * rc.w_step[n - 1];
  for (int g = 0; g < 16; ++g) {
    tc.gstep[g] = make_float2(static_cast<float>(static_cast<double>(rc.w_step[2 * g]) * rc.w_step[2 * g + 1]),
                              static_cast<float>(static_cast<double>(rc.w_step[2 * g + 1]) * rc.w_step[2 * g + 2]));
    tc.gpre[g] = static_cast<float>(K[2 * g]);
    tc.gw[g] = rc.w_step[2 * g];
    tc.gcar[g] = make_float2(static_cast<float>(K[2 * g]), static_cast<float>(K[2 * g + 1]));
  }
  rc.q_thresh_g = static_cast<float>(static_cast<double>(rc.q_thresh) * rc.e_scale * K[0]);
}

void finalize_range_consts(RangeConsts& rc) {
  const double ei = std::floor(rc.e_log2);
  rc.e_int = static_cast<int>(ei);
  const double ef = rc.e_log2 - ei;
  rc.e_frac_hi = static_cast<float>(ef);
  rc.e_frac_lo = static_cast<float>(ef - rc.e_frac_hi);
  rc.k_hi = static_cast<float>(rc.exp2_k);
  rc.k_lo = static_cast<float>(rc.exp2_k - rc.k_hi);
  rc.inv_sr_f = static_cast<float>(rc.inv_sr);
}

}  // namespace gpfb
