// TEST INFRASTRUCTURE: the host instantiation of csrc/exp_cr.h behind a C entry,
// built with -ffp-contract=off (tests/test_exp_cr.py compares it with libm and
// mpmath here, and with the device instantiation on the GPU).
#include "../../paper_1505_00077_b200/csrc/exp_cr.h"

extern "C" void exp_cr_host(const double* x, double* y, long long n) {
  for (long long i = 0; i < n; ++i) y[i] = gpfb::exp_cr(x[i]);
}
