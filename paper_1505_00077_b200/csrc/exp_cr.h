// exp(x) for the reference-exact fp64 mode, evaluated in double-double and
// rounded once: the result is the correctly rounded exp(x) (up to ties closer
// than ~2^-96 relative, i.e. never in practice), so F_0 = exp(-h^2 / 2 sigma_r^2)
// (GpfState::init, bilateral.cpp:99-100) equals the reference's std::exp
// wherever the host libm is itself correctly rounded -- glibc's exp errs by at
// most ~0.51 ulp, so the two agree except on arguments whose exact result lies
// within ~0.01 ulp of a rounding boundary. CUDA's exp() is only within one ulp.
//
// Every operation is an explicitly rounded IEEE add / multiply / fma, so the
// host instantiation (tests/cxx/exp_cr_host.cpp, built with -ffp-contract=off)
// returns the same bits as the device one and can be checked against libm and
// mpmath without a GPU.
//   x = k ln2 + r, |r| <= ln2 / 2, ln2 = L1 + L2 + L3 (L1: 32 bits, k L1 exact)
//   exp(r) = exp(r / 256)^256: degree-9 Taylor (orders 0-4 in double-double, the
//   tail in double; truncation < 2^-117), then eight double-double squarings
//   result = round(E_hi + E_lo) 2^k, one rounding also when the result is subnormal
#ifndef GPFB_EXP_CR_H
#define GPFB_EXP_CR_H

#ifdef __CUDA_ARCH__
#define GPFB_XADD(a, b) __dadd_rn((a), (b))
#define GPFB_XMUL(a, b) __dmul_rn((a), (b))
#define GPFB_XFMA(a, b, c) __fma_rn((a), (b), (c))
#define GPFB_XRINT(a) rint(a)
#else
#include <cmath>
#define GPFB_XADD(a, b) ((a) + (b))
#define GPFB_XMUL(a, b) ((a) * (b))
#define GPFB_XFMA(a, b, c) std::fma((a), (b), (c))
#define GPFB_XRINT(a) std::nearbyint(a)
#endif

#ifdef __CUDACC__
#define GPFB_HD __host__ __device__ __forceinline__
#else
#define GPFB_HD inline
#endif

namespace gpfb {
namespace expcr {

struct DD {
  double hi, lo;
};

GPFB_HD DD fast_two_sum(double a, double b) {  // |a| >= |b|
  const double s = GPFB_XADD(a, b);
  return DD{s, GPFB_XADD(b, -GPFB_XADD(s, -a))};
}
GPFB_HD DD two_sum(double a, double b) {
  const double s = GPFB_XADD(a, b);
  const double bb = GPFB_XADD(s, -a);
  return DD{s, GPFB_XADD(GPFB_XADD(a, -GPFB_XADD(s, -bb)), GPFB_XADD(b, -bb))};
}
GPFB_HD DD dd_mul(DD a, DD b) {
  const double p = GPFB_XMUL(a.hi, b.hi);
  double e = GPFB_XFMA(a.hi, b.hi, -p);
  e = GPFB_XFMA(a.hi, b.lo, e);
  e = GPFB_XFMA(a.lo, b.hi, e);
  return fast_two_sum(p, e);
}
GPFB_HD DD dd_add(DD a, DD b) {
  DD s = two_sum(a.hi, b.hi);
  const DD t = two_sum(a.lo, b.lo);
  s = fast_two_sum(s.hi, GPFB_XADD(s.lo, t.hi));
  return fast_two_sum(s.hi, GPFB_XADD(s.lo, t.lo));
}

GPFB_HD double pow2(int k) {  // 2^k, -1022 <= k <= 1023
  union {
    unsigned long long u;
    double d;
  } v;
  v.u = static_cast<unsigned long long>(k + 1023) << 52;
  return v.d;
}

}  // namespace expcr

GPFB_HD double exp_cr(double x) {
  using namespace expcr;
  if (x != x) return x;
  if (x > 709.782712893384) return x * 8.98846567431158e307;  // overflow -> +inf
  if (x < -745.2) return 0.0;
  const double kd = GPFB_XRINT(GPFB_XMUL(x, 0x1.71547652b82fep+0));
  const int k = static_cast<int>(kd);
  // r = x - k ln2 as a double-double (the first product and difference are exact)
  const double t1 = GPFB_XFMA(-kd, 0x1.62e42fee00000p-1, x);
  const double ph = GPFB_XMUL(kd, 0x1.a39ef35793c76p-33);
  const double pl = GPFB_XFMA(kd, 0x1.a39ef35793c76p-33, -ph);
  DD r = two_sum(t1, -ph);
  r = fast_two_sum(r.hi, GPFB_XADD(GPFB_XADD(r.lo, -pl), -GPFB_XMUL(kd, 0x1.cc01f97b57a08p-87)));
  const DD s = DD{GPFB_XMUL(r.hi, 0.00390625), GPFB_XMUL(r.lo, 0.00390625)};  // r / 256, exact
  // exp(s) = 1 + s (1 + s (1/2 + s (1/3! + s (1/4! + s T)))), |s| <= 0.00136.
  // T = 1/5! + s/6! + ... + s^4/9! in plain double: its term enters the sum below 2^-54, so a
  // 2^-52 relative error in T is below 2^-106 of the result; truncation after s^9/9! < 2^-117
  const double sh = s.hi;
  double t = 0x1.71de3a556c734p-19;                              // 1/9!
  t = GPFB_XFMA(t, sh, 0x1.a01a01a01a01ap-16);                   // 1/8!
  t = GPFB_XFMA(t, sh, 0x1.a01a01a01a01ap-13);                   // 1/7!
  t = GPFB_XFMA(t, sh, 0x1.6c16c16c16c17p-10);                   // 1/6!
  t = GPFB_XFMA(t, sh, 0x1.1111111111111p-7);                    // 1/5!
  // the low orders in double-double: 1/4!, 1/3!, 1/2
  const DD c4{0x1.5555555555555p-5, 0x1.5555555555555p-59}, c3{0x1.5555555555555p-3, 0x1.5555555555555p-57};
  DD q = dd_add(dd_mul(DD{t, 0.0}, s), c4);
  q = dd_add(dd_mul(q, s), c3);
  q = dd_add(dd_mul(q, s), DD{0.5, 0.0});
  q = dd_add(dd_mul(q, s), DD{1.0, 0.0});
  DD e = dd_add(dd_mul(q, s), DD{1.0, 0.0});  // exp(r / 256)
  for (int i = 0; i < 8; ++i) e = dd_mul(e, e);
  if (k > 1000) return GPFB_XMUL(GPFB_XMUL(e.hi, pow2(k - 100)), pow2(100));  // k may be 1024
  if (k >= -1021) return GPFB_XMUL(e.hi, pow2(k));  // e.hi = round(e.hi + e.lo): the pair is normalised
  // subnormal result: scale the pair exactly into range, then one rounding
  const double a = GPFB_XMUL(e.hi, pow2(k + 1000)), b = GPFB_XMUL(e.lo, pow2(k + 1000));
  return GPFB_XFMA(a, pow2(-1000), GPFB_XMUL(b, pow2(-1000)));
}

}  // namespace gpfb

#endif  // GPFB_EXP_CR_H
