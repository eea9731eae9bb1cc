// Direct O(sigma_s^2) bilateral filter (reference exact_bilateral,
// proj/src/core/bilateral.cpp:14-56) and the error metrics of
// metrics::compare (proj/src/core/metrics.cpp:20-56), on the GPU.
//
// The exact filter is the MSE yardstick of the GPF path (north_star: "MSE
// against a direct O(sigma_s^2) bilateral filter is reported alongside";
// SURVEY.md 8(f) row 1). Per output pixel (offset form, Eq. (1)):
//   out = f_c + sum w d / sum w,  d = f(q) - f_c,
//   w = exp(-(a^2 + b^2) / 2 sigma_s^2) exp(-d^2 / 2 sigma_r^2)
// over the (2W+1)^2 window with the reference's boundary_index mapping
// (replicate / reflect / zero: zero-padded taps contribute nothing). The
// kernel_scale factor of the spatial weight cancels in num/den and is not
// applied. A warp owns one output row segment of 32 pixels (lane = column);
// for every row offset a it stages the boundary-mapped input row segment
// (32 + 2W values) in its own smem slice, then sweeps b with one exp2 per tap
// (spatial and range exponents folded). Sums run in fp32 over one row of taps
// (<= 2W+1 terms) and in fp64 across rows.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>

#include <cuda_runtime.h>

#include "gpf_internal.h"

namespace gpfb {

namespace {

constexpr int kExactWarps = 8;  // output rows per CTA

__device__ __forceinline__ int bidx(int i, int n, int boundary) {  // spatial.cpp:52-70
  if (i >= 0 && i < n) return i;
  if (boundary == 0) return i < 0 ? 0 : n - 1;  // replicate
  if (boundary == 1) {                           // reflect (half-sample symmetric)
    const int period = 2 * n;
    int m = i % period;
    if (m < 0) m += period;
    return m < n ? m : period - 1 - m;
  }
  return -1;  // zero
}

template <typename T, bool ZERO>
__global__ void __launch_bounds__(32 * kExactWarps) k_exact(const T* __restrict__ in_all,
                                                            T* __restrict__ out_all, int w, int h,
                                                            int W, int boundary, float ks2,
                                                            float kr2) {
  extern __shared__ float seg_all[];  // [warps][32 + 2W]
  const int lane = threadIdx.x, warp = threadIdx.y, f = blockIdx.z;
  const int span = 32 + 2 * W;
  float* seg = seg_all + warp * span;
  const int x0 = blockIdx.x * 32, x = x0 + lane;
  const int r = blockIdx.y * kExactWarps + warp;
  if (r >= h) return;  // warp-uniform; no CTA barrier below
  const T* in = in_all + (size_t)f * w * h;
  T* out = out_all + (size_t)f * w * h;
  const float fc = static_cast<float>(in[(size_t)r * w + min(x, w - 1)]);
  // ks2 = log2(e) / (2 sigma_s^2), kr2 = log2(e) / (2 sigma_r^2):
  // w = 2^-(ks2 (a^2 + b^2) + kr2 d^2)
  double num = 0.0, den = 0.0;
  for (int a = -W; a <= W; ++a) {
    const int rr = bidx(r + a, h, boundary);
    if (rr < 0) continue;  // zero padding: the whole row of taps contributes nothing
    const T* src = in + (size_t)rr * w;
    __syncwarp();
    for (int j = lane; j < span; j += 32) {
      const int cc = bidx(x0 - W + j, w, boundary);
      seg[j] = cc >= 0 ? static_cast<float>(src[cc]) : __int_as_float(0x7fc00000);  // NaN: no tap
    }
    __syncwarp();
    const float sa = ks2 * static_cast<float>(a * a);
    float nr = 0.f, dr = 0.f;
#pragma unroll 4
    for (int b = -W; b <= W; ++b) {
      const float v = seg[lane + W + b];
      float d = v - fc;
      if (ZERO) d = (v == v) ? d : 0.f;  // zero-padded tap (NaN marker)
      const float e = fmaf(kr2 * d, d, fmaf(ks2, static_cast<float>(b * b), sa));
      float wt = exp2f(-e);
      if (ZERO) wt = (v == v) ? wt : 0.f;
      nr = fmaf(wt, d, nr);
      dr += wt;
    }
    num += nr;
    den += dr;
  }
  if (x < w) out[(size_t)r * w + x] = static_cast<T>(static_cast<double>(fc) + num / den);
}

// fp64 form for the reference-facing gpf_filter_exact: the reference's own
// operation sequence per pixel (bilateral.cpp:31-52) with explicitly rounded,
// never-contracted fp64 operations; the spatial weight table ws[a][b] =
// kernel_scale * spatial_weight(a, b, sigma_s) is the reference's own
// expression evaluated once on the host (spatial.cpp:37-41), so only the range
// factor's exp() is CUDA's instead of glibc's (<= 1 ulp). A warp owns 32
// output pixels of one row and stages each boundary-mapped input row segment
// in shared memory (coalesced loads); taps of zero padding are skipped.
__device__ __forceinline__ double dm_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da_(double a, double b) { return __dadd_rn(a, b); }

__global__ void __launch_bounds__(32 * kExactWarps) k_exact64(const double* __restrict__ in_all,
                                                              double* __restrict__ out_all, int w,
                                                              int h, int W, int boundary,
                                                              const double* __restrict__ ws,
                                                              double inv2s2) {
  extern __shared__ double seg64_all[];  // [warps][32 + 2W]
  const int lane = threadIdx.x, warp = threadIdx.y, f = blockIdx.z;
  const int span = 32 + 2 * W;
  double* seg = seg64_all + warp * span;
  int* ok = reinterpret_cast<int*>(seg64_all + kExactWarps * span) + warp * span;
  const int x0 = blockIdx.x * 32, x = x0 + lane;
  const int r = blockIdx.y * kExactWarps + warp;
  if (r >= h) return;  // warp-uniform; no CTA barrier below
  const double* in = in_all + (size_t)f * w * h;
  double* out = out_all + (size_t)f * w * h;
  const double fc = in[(size_t)r * w + min(x, w - 1)];
  const int n = 2 * W + 1;
  double num = 0.0, den = 0.0;
  for (int a = -W; a <= W; ++a) {
    const int rr = bidx(r + a, h, boundary);
    if (rr < 0) continue;  // zero padding contributes nothing (bilateral.cpp:39)
    const double* src = in + (size_t)rr * w;
    __syncwarp();
    for (int j = lane; j < span; j += 32) {
      const int cc = bidx(x0 - W + j, w, boundary);
      seg[j] = cc >= 0 ? src[cc] : 0.0;
      ok[j] = cc >= 0;
    }
    __syncwarp();
    const double* wrow = ws + (size_t)(a + W) * n;
    for (int b = -W; b <= W; ++b) {
      if (!ok[lane + W + b]) continue;  // bilateral.cpp:42
      const double d = __dsub_rn(seg[lane + W + b], fc);
      const double wgt = dm_(wrow[b + W], exp(dm_(-dm_(d, d), inv2s2)));
      num = da_(num, dm_(wgt, d));
      den = da_(den, wgt);
    }
  }
  if (x < w) out[(size_t)r * w + x] = da_(fc, __ddiv_rn(num, den));
}

// ---------------------------------------------------------------- metrics
// sum (ref - test)^2 and max |ref - test| over the interior, as exact
// double-double partial sums per CTA (order-independent up to the final tree,
// which is fixed), so the result is deterministic.
constexpr int kCmpThreads = 256;

__device__ __forceinline__ void two_sum_(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}

template <typename T>
__global__ void __launch_bounds__(kCmpThreads) k_cmp_partial(const T* __restrict__ ref,
                                                             const T* __restrict__ test, int w,
                                                             int h, int border,
                                                             double* __restrict__ partials) {
  __shared__ double shi[kCmpThreads], slo[kCmpThreads], smx[kCmpThreads];
  const int iw = w - 2 * border, ih = h - 2 * border;
  const long long n = (long long)iw * ih;
  double hi = 0.0, lo = 0.0, mx = 0.0;
  for (long long i = (long long)blockIdx.x * kCmpThreads + threadIdx.x; i < n;
       i += (long long)gridDim.x * kCmpThreads) {
    const int r = border + (int)(i / iw), c = border + (int)(i % iw);
    const double d = static_cast<double>(ref[(size_t)r * w + c]) - static_cast<double>(test[(size_t)r * w + c]);
    double s, e;
    const double sq = d * d;
    two_sum_(hi, sq, s, e);
    hi = s;
    lo += e + fma(d, d, -sq);  // the square's rounding error too
    mx = fmax(mx, fabs(d));
  }
  const int t = threadIdx.x;
  shi[t] = hi;
  slo[t] = lo;
  smx[t] = mx;
  __syncthreads();
  for (int off = kCmpThreads / 2; off > 0; off >>= 1) {
    if (t < off) {
      double s, e;
      two_sum_(shi[t], shi[t + off], s, e);
      shi[t] = s;
      slo[t] += slo[t + off] + e;
      smx[t] = fmax(smx[t], smx[t + off]);
    }
    __syncthreads();
  }
  if (t == 0) {
    partials[3 * blockIdx.x] = shi[0];
    partials[3 * blockIdx.x + 1] = slo[0];
    partials[3 * blockIdx.x + 2] = smx[0];
  }
}

void check_(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();  // clear a non-sticky error (e.g. a failed allocation) for the caller
    throw Error{9, std::string(what) + ": " + cudaGetErrorString(e)};
  }
}

template <typename T>
void run_exact(const T* d_in, T* d_out, int w, int h, int count, int W, int boundary, double sigma_s,
               double sigma_r, cudaStream_t st) {
  if (count <= 0) return;
  const double log2e = 1.4426950408889634;
  const float ks2 = static_cast<float>(log2e / (2.0 * sigma_s * sigma_s));
  const float kr2 = static_cast<float>(log2e / (2.0 * sigma_r * sigma_r));
  const size_t smem = sizeof(float) * kExactWarps * (32 + 2 * (size_t)W);
  if (smem > 227 * 1024) throw Error{1, "exact filter: window radius too large for the GPU kernel"};
  auto k = boundary == 2 ? k_exact<T, true> : k_exact<T, false>;
  check_(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
         "cudaFuncSetAttribute");
  const dim3 grid((w + 31) / 32, (h + kExactWarps - 1) / kExactWarps, count);
  k<<<grid, dim3(32, kExactWarps), smem, st>>>(d_in, d_out, w, h, W, boundary, ks2, kr2);
  check_(cudaGetLastError(), "kernel launch");
}

}  // namespace

void run_exact_f32(const float* d_in, float* d_out, int w, int h, int count, int W, int boundary,
                   double sigma_s, double sigma_r, cudaStream_t st) {
  run_exact<float>(d_in, d_out, w, h, count, W, boundary, sigma_s, sigma_r, st);
}

void run_exact_f64(const double* d_in, double* d_out, int w, int h, int count, int W, int boundary,
                   double sigma_s, double sigma_r, double kernel_scale, cudaStream_t st) {
  if (count <= 0) return;
  const int n = 2 * W + 1;
  // ws[a][b] = kernel_scale * spatial_weight(a, b, sigma_s) (bilateral.cpp:23-28, spatial.cpp:37-41)
  double* hws = nullptr;
  check_(cudaMallocHost(&hws, sizeof(double) * n * n), "cudaMallocHost");
  for (int a = -W; a <= W; ++a)
    for (int b = -W; b <= W; ++b) {
      const double r2 = static_cast<double>(a) * a + static_cast<double>(b) * b;
      hws[(a + W) * n + (b + W)] = kernel_scale * std::exp(-r2 / (2.0 * sigma_s * sigma_s));
    }
  double* dws = nullptr;
  cudaError_t e = cudaMallocAsync(&dws, sizeof(double) * n * n, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dws, hws, sizeof(double) * n * n, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) {
    cudaFreeHost(hws);
    check_(e, "exact filter weights");
  }
  const double inv2s2 = 1.0 / (2.0 * sigma_r * sigma_r);  // bilateral.cpp:29
  const size_t smem = (sizeof(double) + sizeof(int)) * kExactWarps * (32 + 2 * (size_t)W);
  if (smem > 227 * 1024) {
    cudaFreeAsync(dws, st);
    cudaStreamSynchronize(st);
    cudaFreeHost(hws);
    throw Error{1, "exact filter: window radius too large for the GPU kernel"};
  }
  check_(cudaFuncSetAttribute(k_exact64, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
         "cudaFuncSetAttribute");
  const dim3 grid((w + 31) / 32, (h + kExactWarps - 1) / kExactWarps, count);
  k_exact64<<<grid, dim3(32, kExactWarps), smem, st>>>(d_in, d_out, w, h, W, boundary, dws, inv2s2);
  e = cudaGetLastError();
  cudaFreeAsync(dws, st);
  const cudaError_t e2 = cudaStreamSynchronize(st);  // the pinned table may be released
  cudaFreeHost(hws);
  check_(e, "kernel launch");
  check_(e2, "exact filter");
}

// mse / max_abs / pixels of (ref, test) over the interior (metrics.cpp:20-56);
// synchronises `st`.
template <typename T>
static ErrorStats compare_dev(const T* d_ref, const T* d_test, int w, int h, int border,
                              cudaStream_t st) {
  const long long n = (long long)(w - 2 * border) * (h - 2 * border);
  const int blocks = (int)std::min<long long>((n + kCmpThreads - 1) / kCmpThreads, 148 * 4);
  double* d_part = nullptr;
  check_(cudaMallocAsync(&d_part, sizeof(double) * 3 * blocks, st), "cudaMallocAsync");
  k_cmp_partial<T><<<blocks, kCmpThreads, 0, st>>>(d_ref, d_test, w, h, border, d_part);
  check_(cudaGetLastError(), "kernel launch");
  std::string err;
  double* part = new double[3 * blocks];
  const cudaError_t e1 = cudaMemcpyAsync(part, d_part, sizeof(double) * 3 * blocks,
                                         cudaMemcpyDeviceToHost, st);
  const cudaError_t e2 = cudaStreamSynchronize(st);
  cudaFreeAsync(d_part, st);
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    delete[] part;
    check_(e1 != cudaSuccess ? e1 : e2, "compare");
  }
  // fixed-order combination of the CTA partials (double-double)
  double hi = 0.0, lo = 0.0, mx = 0.0;
  for (int b = 0; b < blocks; ++b) {
    double s, e;
    s = hi + part[3 * b];
    const double bb = s - hi;
    e = (hi - (s - bb)) + (part[3 * b] - bb);
    hi = s;
    lo += e + part[3 * b + 1];
    mx = std::max(mx, part[3 * b + 2]);
  }
  delete[] part;
  ErrorStats r;
  r.pixels = n;
  r.mse = (hi + lo) / static_cast<double>(n);
  r.max_abs = mx;
  return r;
}

ErrorStats compare_f32(const float* d_ref, const float* d_test, int w, int h, int border,
                       cudaStream_t st) {
  return compare_dev<float>(d_ref, d_test, w, h, border, st);
}

ErrorStats compare_f64(const double* d_ref, const double* d_test, int w, int h, int border,
                       cudaStream_t st) {
  return compare_dev<double>(d_ref, d_test, w, h, border, st);
}

}  // namespace gpfb
