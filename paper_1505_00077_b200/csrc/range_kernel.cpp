// Scalar range-kernel evaluators of the reference C ABI (ref.h:123-143,
// proj/src/capi.cpp:230-286 -> proj/src/core/range_kernel.cpp:31-89): the exact
// Gaussian range kernel, its degree-N Gauss-polynomial and Taylor
// approximations, and the sup of their absolute error over an intensity grid.
//
// Host fp64 by nature (one number in, one number out: the analysis side of the
// paper's Fig. 1, nothing a GPU helps with); they are here so that the library
// exports every symbol of the reference header. The operation order of each
// expression is the reference's, so the values are bitwise the reference's on
// the same libm.
#include <cmath>
#include <string>

#include "gpf_internal.h"

namespace gpfb {

namespace {

void check_range_params(double sigma_r, int degree) {  // RangeParams::validate (range_kernel.cpp:22-29)
  if (!(sigma_r > 0.0)) throw Error{1, "RangeParams: sigma_r must be > 0"};
  if (degree < 0) throw Error{1, "RangeParams: degree must be >= 0"};
}

// exp(-x^2 / 2 sigma_r^2); one expression for every caller (range_kernel.cpp:16-18)
double half_gauss(double x, double sigma_r) { return std::exp(-(x * x) / (2.0 * sigma_r * sigma_r)); }

// sum_{n <= terms} prod_{i <= n} (step / i): the truncated exponential series
// both approximations share (range_kernel.cpp:39-44, 53-58)
double truncated_exp(double step, int terms) {
  double term = 1.0, sum = 1.0;
  for (int i = 1; i <= terms; ++i) {
    term *= step / i;
    sum += term;
  }
  return sum;
}

}  // namespace

double kernel_gauss(double t, double tau, double sigma_r) {
  check_range_params(sigma_r, 20);
  return half_gauss(t - tau, sigma_r);
}

// exp(-tau^2/2s^2) exp(-t^2/2s^2) sum_{n<=N} (t tau / s^2)^n / n!   (Eq. (4) of the paper)
double kernel_gauss_poly(double t, double tau, double sigma_r, int degree) {
  check_range_params(sigma_r, degree);
  const double z = (t / sigma_r) * (tau / sigma_r);
  const double series = truncated_exp(z, degree);
  return (half_gauss(tau, sigma_r) * half_gauss(t, sigma_r)) * series;
}

// sum_{k <= N/2} (-(t - tau)^2 / 2s^2)^k / k!
double kernel_taylor(double t, double tau, double sigma_r, int degree) {
  check_range_params(sigma_r, degree);
  const double d = t - tau;
  const double u = (d * d) / (2.0 * sigma_r * sigma_r);
  return truncated_exp(-u, degree / 2);
}

// range_kernel.cpp:61-89: grid low + k step, k = 0..floor(span/step + 1e-9),
// closed with `high` when the last grid point falls short of it
double kernel_sup_error(double sigma_r, int degree, double tau, double low, double high, double step,
                        int taylor) {
  check_range_params(sigma_r, degree);
  if (!(low < high)) throw Error{1, "sup_error: range.low must be < range.high"};
  if (!(step > 0.0)) throw Error{1, "sup_error: step must be > 0"};
  auto err_at = [&](double t) {
    const double a = taylor ? kernel_taylor(t, tau, sigma_r, degree) : kernel_gauss_poly(t, tau, sigma_r, degree);
    return std::abs(half_gauss(t - tau, sigma_r) - a);
  };
  const long long last_k = static_cast<long long>(std::floor((high - low) / step + 1e-9));
  double worst = 0.0, t = low;
  for (long long k = 0; k <= last_k; ++k) {
    t = low + static_cast<double>(k) * step;
    worst = std::fmax(worst, err_at(t));
  }
  if (t < high - 1e-9 * step) worst = std::fmax(worst, err_at(high));
  return worst;
}

}  // namespace gpfb
