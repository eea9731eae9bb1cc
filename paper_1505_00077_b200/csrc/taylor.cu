// Taylor-polynomial bilateral baseline (reference taylor_bilateral,
// proj/src/core/bilateral.cpp:160-220; C ABI gpf_filter_taylor,
// proj/src/capi.cpp:194-207), on the GPU, bitwise equal to the reference.
//
// Moments M_m = f^m (m = 0 .. 2K+1, K = degree / 2, no centring or scaling:
// f^21 reaches 1e50, so this path is fp64 throughout) are each smoothed by
// the same recursive Gaussian as gpf_gaussian_recursive (run_gaussian_f64:
// the reference's deriche_line with explicitly rounded, never-contracted
// operations), then every pixel recombines them with the binomial expansion of
// exp(-(f(q) - f(p))^2 / 2 sigma_r^2) truncated at order K, in the reference's
// operation order. A pixel whose denominator is <= 1e-8 (or negative: the
// truncation broke down) keeps its input value and is counted.
#include <algorithm>
#include <cstdint>
#include <string>

#include <cuda_runtime.h>

#include "gpf_internal.h"

namespace gpfb {

namespace {

__device__ __forceinline__ double m_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double a_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double d_(double a, double b) { return __ddiv_rn(a, b); }

// moment m+1 = moment m * f (bilateral.cpp:181-183), one plane per launch
__global__ void k_moment_next(const double* __restrict__ f, const double* __restrict__ prev,
                              double* __restrict__ next, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    next[i] = m_(prev[i], f[i]);
}

__global__ void k_fill(double* __restrict__ p, double v, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}

// per-pixel recombination (bilateral.cpp:189-217); mbar = [2K+2][n]
__global__ void k_taylor_combine(const double* __restrict__ f, const double* __restrict__ mbar,
                                 double* __restrict__ out, long long n, int K, double sr2x2,
                                 unsigned long long* __restrict__ fallbacks) {
  unsigned my_fb = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    // Order-K Taylor weight of the range Gaussian, sum_k a_k (f(q) - t)^{2k},
    // expanded binomially over the smoothed moments f^m. Evaluated with the
    // reference's recurrences and operation order (bitwise parity): the
    // series coefficient a_k, the binomial C(2k, m) walked from m = 2k down,
    // and the power (-t)^(2k-m) walked up alongside.
    const double t = f[i];
    double num = 0.0, den = 0.0;
    double a = 1.0;
    for (int k = 0; k <= K; ++k) {
      double binom = 1.0;
      double pw = 1.0;
      for (int m = 2 * k; m >= 0; --m) {
        const double coef = m_(m_(a, binom), pw);
        den = a_(den, m_(coef, mbar[(size_t)m * n + i]));
        num = a_(num, m_(coef, mbar[(size_t)(m + 1) * n + i]));
        if (m > 0) {
          binom = d_(m_(binom, static_cast<double>(m)), static_cast<double>(2 * k - m + 1));
          pw = m_(pw, -t);
        }
      }
      a = m_(a, d_(-1.0, m_(sr2x2, static_cast<double>(k + 1))));
    }
    if (den <= 1e-8) {  // kQMin (bilateral.hpp:85): a vanishing or negative
      out[i] = t;       // denominator keeps the input sample
      ++my_fb;
    } else {
      out[i] = d_(num, den);
    }
  }
  for (int o = 16; o; o >>= 1) my_fb += __shfl_xor_sync(0xffffffffu, my_fb, o);
  if ((threadIdx.x & 31) == 0 && my_fb) atomicAdd(fallbacks, (unsigned long long)my_fb);
}

void check_(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();  // clear a non-sticky error (e.g. a failed allocation) for the caller
    throw Error{9, std::string(what) + ": " + cudaGetErrorString(e)};
  }
}

}  // namespace

// d_in (w x h fp64) -> d_out; d_fb (one counter, zeroed here); workspace
// allocated here: (2K+2) filtered moments + two moment/temp planes.
void run_taylor_f64(const double* d_in, double* d_out, const Params& p, unsigned long long* d_fb,
                    cudaStream_t st) {
  const int w = p.width, h = p.height, degree = p.degree;
  const double sigma_s = p.sigma_s, kernel_scale = p.kernel_scale, sigma_r = p.sigma_r;
  const long long n = (long long)w * h;
  const int K = degree / 2;
  const int planes = 2 * K + 2;
  double *mbar = nullptr, *mom = nullptr, *mom2 = nullptr, *tmp = nullptr;
  cudaError_t e = cudaMallocAsync(&mbar, sizeof(double) * n * planes, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&mom, sizeof(double) * n, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&mom2, sizeof(double) * n, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&tmp, sizeof(double) * n, st);
  if (e != cudaSuccess) {  // release what was allocated before the failure
    for (double* p : {mbar, mom, mom2, tmp})
      if (p) cudaFreeAsync(p, st);
    check_(e, "cudaMallocAsync (Taylor workspace)");
  }
  const double mass = kernel_mass_1d(sigma_s, default_window_radius(sigma_s));
  const double scale = mass * mass * kernel_scale;  // recursive_gaussian's output scale
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148 * 8);
  k_fill<<<blocks, 256, 0, st>>>(mom, 1.0, n);
  for (int m = 0; m < planes; ++m) {
    // filt (bilateral.cpp:168-172)
    if (p.backend == 0)
      run_direct_gaussian_f64(mom, mbar + (size_t)m * n, tmp, w, h, 1, sigma_s, kernel_scale,
                              p.window_radius, p.boundary, st);
    else
      run_gaussian_f64(mom, mbar + (size_t)m * n, tmp, w, h, sigma_s, scale, st);
    if (m + 1 < planes) {
      k_moment_next<<<blocks, 256, 0, st>>>(d_in, mom, mom2, n);
      std::swap(mom, mom2);
    }
  }
  check_(cudaMemsetAsync(d_fb, 0, sizeof(unsigned long long), st), "cudaMemsetAsync");
  const double sr2x2 = 2.0 * sigma_r * sigma_r;
  k_taylor_combine<<<blocks, 256, 0, st>>>(d_in, mbar, d_out, n, K, sr2x2, d_fb);
  check_(cudaGetLastError(), "kernel launch");
  cudaFreeAsync(mbar, st);
  cudaFreeAsync(mom, st);
  cudaFreeAsync(mom2, st);
  cudaFreeAsync(tmp, st);
}

}  // namespace gpfb
