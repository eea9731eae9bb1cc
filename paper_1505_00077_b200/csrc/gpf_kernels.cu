// sm_100a kernels of the Gauss-polynomial bilateral filter (GPF) hot path.
//
// Reference path (proj/src/core/bilateral.cpp:150-158, gpf()):
//   t_c = mean(f)                                   -> k_mean_*        (K0)
//   N+2 planes F_n = H^n exp(-h^2/2sr^2), each
//   filtered by the separable Deriche IIR           -> k_colpass       (K1, columns)
//                                                      k_rowpass       (K2, rows)
//   Q = sum c G Fbar_n, P = sum c G Fbar_{n+1},
//   out = sr P/Q + t_c, |Q| <= 1e-8 -> input        -> k_combine       (K3)
//
// Data layout in HBM: plane pair g (planes 2g, 2g+1) of the intermediate is a
// row-major float2 image [pairs][h][w]; one thread owns one (line, pair).
#include <cuda_runtime.h>

#include "gpf_internal.h"

namespace gpfb {

// ----------------------------------------------------------------------------
// K0: t_c = mean(f), deterministic double-double reduction. Replaces the
// Neumaier loop of mean_intensity (proj/src/core/image.cpp:20-37): the
// compensated (hi, lo) pair carries the exact rounding error of every add, so
// a constant image returns its value exactly for power-of-two pixel counts,
// as the reference's compensated sum does.
// ----------------------------------------------------------------------------
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}

__device__ __forceinline__ void dd_add(double& hi, double& lo, double bhi, double blo) {
  double s, e;
  two_sum(hi, bhi, s, e);
  e += lo + blo;
  hi = s + e;
  lo = e - (hi - s);
}

constexpr int kMeanThreads = 256;

__device__ void block_dd_reduce(double& hi, double& lo) {
  __shared__ double shi[kMeanThreads], slo[kMeanThreads];
  const int t = threadIdx.x;
  shi[t] = hi;
  slo[t] = lo;
  __syncthreads();
  for (int off = kMeanThreads / 2; off > 0; off >>= 1) {
    if (t < off) {
      double h = shi[t], l = slo[t];
      dd_add(h, l, shi[t + off], slo[t + off]);
      shi[t] = h;
      slo[t] = l;
    }
    __syncthreads();
  }
  hi = shi[0];
  lo = slo[0];
}

template <typename T>
__global__ void __launch_bounds__(kMeanThreads) k_mean_partial(const T* __restrict__ in,
                                                               long long n,
                                                               double* __restrict__ partials) {
  double hi = 0.0, lo = 0.0;
  const long long stride = (long long)gridDim.x * kMeanThreads;
  for (long long i = (long long)blockIdx.x * kMeanThreads + threadIdx.x; i < n; i += stride) {
    double s, e;
    two_sum(hi, static_cast<double>(in[i]), s, e);
    hi = s;
    lo += e;
  }
  block_dd_reduce(hi, lo);
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = hi;
    partials[2 * blockIdx.x + 1] = lo;
  }
}

__global__ void __launch_bounds__(kMeanThreads) k_mean_final(const double* __restrict__ partials,
                                                             int nblocks, long long n,
                                                             int centering,
                                                             double* __restrict__ scalars) {
  double hi = 0.0, lo = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += kMeanThreads)
    dd_add(hi, lo, partials[2 * b], partials[2 * b + 1]);
  block_dd_reduce(hi, lo);
  if (threadIdx.x == 0) scalars[0] = centering ? (hi + lo) / static_cast<double>(n) : 0.0;
}

// ----------------------------------------------------------------------------
// Plane generation (bilateral.cpp:92-101 and the F <- H F recursion of
// step(), bilateral.cpp:117-120): for pixel value f,
//   h = f - t_c, H = h / sr, E = exp(-h^2 / 2 sr^2)      (fp64, like the ref)
//   plane n (scaled) = E 2^s0 * (H 2^-k)^n              (fp32 chain)
// ----------------------------------------------------------------------------
struct PixelRange {
  float es;  // E * 2^s0
  float m;   // H * 2^-k
};

__device__ __forceinline__ PixelRange pixel_range(double f, double t_c, const RangeConsts& rc) {
  const double h = f - t_c;
  PixelRange r;
  r.es = static_cast<float>(exp(-(h * h) * rc.inv2s2) * rc.e_scale);
  r.m = static_cast<float>(h * rc.inv_sr) * rc.h_step;
  return r;
}

// planes (2g, 2g+1) of a pixel: es * m^(2g), es * m^(2g+1). g is warp-uniform.
__device__ __forceinline__ float2 pair_values(const PixelRange& r, int g) {
  float base = r.m * r.m, acc = r.es;
  for (int e = g; e; e >>= 1) {
    if (e & 1) acc *= base;
    base *= base;
  }
  return make_float2(acc, acc * r.m);
}

// ----------------------------------------------------------------------------
// One complex first-order section pair for two planes (see FilterConsts).
// ----------------------------------------------------------------------------
struct PairState {
  float wr[2][2], wi[2][2];  // [plane][section]
};

__device__ __forceinline__ void warm_start(PairState& s, float2 x, const FilterConsts& fc) {
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    s.wr[0][k] = x.x * fc.gr[k];
    s.wi[0][k] = x.x * fc.gi[k];
    s.wr[1][k] = x.y * fc.gr[k];
    s.wi[1][k] = x.y * fc.gi[k];
  }
}

// w <- p w + x
__device__ __forceinline__ void advance(PairState& s, float2 x, const FilterConsts& fc) {
#pragma unroll
  for (int k = 0; k < 2; ++k) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const float xv = q == 0 ? x.x : x.y;
      const float nr = fmaf(fc.pr[k], s.wr[q][k], fmaf(-fc.pi[k], s.wi[q][k], xv));
      const float ni = fmaf(fc.pr[k], s.wi[q][k], fc.pi[k] * s.wr[q][k]);
      s.wr[q][k] = nr;
      s.wi[q][k] = ni;
    }
  }
}

// sum_k Re(c_k w_k) with residues (cr, ci)
__device__ __forceinline__ float2 emit(const PairState& s, const float* cr, const float* ci) {
  float2 o;
  o.x = fmaf(cr[0], s.wr[0][0], fmaf(-ci[0], s.wi[0][0], fmaf(cr[1], s.wr[0][1], -ci[1] * s.wi[0][1])));
  o.y = fmaf(cr[0], s.wr[1][0], fmaf(-ci[0], s.wi[1][0], fmaf(cr[1], s.wr[1][1], -ci[1] * s.wi[1][1])));
  return o;
}

// ----------------------------------------------------------------------------
// K1: column pass (deriche_line over columns, spatial.cpp:240-243), fused with
// the plane generator. Thread = (column x, plane pair g); block = 32 columns x
// pairs. Causal sweep writes its output, anticausal sweep adds to it.
// ----------------------------------------------------------------------------
template <typename Tin>
__global__ void k_colpass(const Tin* __restrict__ in, float2* __restrict__ planes,
                          const double* __restrict__ scalars, int w, int h,
                          FilterConsts fc, RangeConsts rc) {
  const int x = blockIdx.x * 32 + threadIdx.x;
  const int g = threadIdx.y;
  if (x >= w) return;
  const double t_c = scalars[0];
  float2* out = planes + (size_t)g * h * w + x;

  PairState s;
  {
    const float2 x0 = pair_values(pixel_range(static_cast<double>(in[x]), t_c, rc), g);
    warm_start(s, x0, fc);
  }
  for (int y = 0; y < h; ++y) {
    const float2 xv = pair_values(pixel_range(static_cast<double>(in[(size_t)y * w + x]), t_c, rc), g);
    advance(s, xv, fc);
    out[(size_t)y * w] = emit(s, fc.ar, fc.ai);
  }
  {
    const float2 xl = pair_values(pixel_range(static_cast<double>(in[(size_t)(h - 1) * w + x]), t_c, rc), g);
    warm_start(s, xl, fc);
  }
  for (int y = h - 1; y >= 0; --y) {
    const float2 a = emit(s, fc.br, fc.bi);
    float2 o = out[(size_t)y * w];
    o.x += a.x;
    o.y += a.y;
    out[(size_t)y * w] = o;
    if (y > 0) {
      const float2 xv = pair_values(pixel_range(static_cast<double>(in[(size_t)y * w + x]), t_c, rc), g);
      advance(s, xv, fc);
    }
  }
}

// ----------------------------------------------------------------------------
// K2: row pass (deriche_line over rows, spatial.cpp:235-239) on the
// intermediate planes. Thread = (row y, pair g).
// ----------------------------------------------------------------------------
__global__ void k_rowpass(const float2* __restrict__ src, float2* __restrict__ dst, int w, int h,
                          FilterConsts fc) {
  const int y = blockIdx.x * 32 + threadIdx.x;
  const int g = threadIdx.y;
  if (y >= h) return;
  const float2* row = src + ((size_t)g * h + y) * w;
  float2* orow = dst + ((size_t)g * h + y) * w;
  PairState s;
  warm_start(s, row[0], fc);
  for (int x = 0; x < w; ++x) {
    advance(s, row[x], fc);
    orow[x] = emit(s, fc.ar, fc.ai);
  }
  warm_start(s, row[w - 1], fc);
  for (int x = w - 1; x >= 0; --x) {
    const float2 a = emit(s, fc.br, fc.bi);
    float2 o = orow[x];
    o.x += a.x;
    o.y += a.y;
    orow[x] = o;
    if (x > 0) advance(s, row[x], fc);
  }
}

// ----------------------------------------------------------------------------
// K3: P/Q recombination and normalisation (bilateral.cpp:117-126, 139-146):
//   Q = sum_{n<=N} c_n Fbar_n, P = sum_{n<=N} c_n Fbar_{n+1}, c_n = H^n/n!
// (scaled by 2^-s_n so c_n Fbar_n,scaled is in reference units / S), then
// out = sr P/Q + t_c, or the input where |Q| <= 1e-8/S.
// ----------------------------------------------------------------------------
template <typename Tin, typename Tout>
__global__ void k_combine(const Tin* __restrict__ in, const float2* __restrict__ planes,
                          Tout* __restrict__ out, const double* __restrict__ scalars,
                          unsigned long long* __restrict__ fb_count, int w, int h,
                          RangeConsts rc) {
  const long long npx = (long long)w * h;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  int fell = 0;
  if (i < npx) {
    const double t_c = scalars[0];
    const double f = static_cast<double>(in[i]);
    const float H = static_cast<float>((f - t_c) * rc.inv_sr);
    float c = rc.c0, P = 0.f, Q = 0.f;
    float2 cur = planes[i];
    for (int g = 0; g < rc.pairs; ++g) {
      const int n = 2 * g;
      const float2 nxt = (g + 1 < rc.pairs) ? planes[(size_t)(g + 1) * npx + i] : make_float2(0.f, 0.f);
      if (n <= rc.degree) {
        Q = fmaf(c, cur.x, Q);
        P = fmaf(c, cur.y, P);
        c = c * (H * rc.w_step[n]);
      }
      if (n + 1 <= rc.degree) {
        Q = fmaf(c, cur.y, Q);
        P = fmaf(c, nxt.x, P);
        c = c * (H * rc.w_step[n + 1]);
      }
      cur = nxt;
    }
    double o;
    if (!(fabsf(Q) > rc.q_thresh)) {
      o = f;
      fell = 1;
    } else {
      o = rc.sigma_r * ((static_cast<double>(P) * rc.p_scale) / static_cast<double>(Q)) + t_c;
    }
    out[i] = static_cast<Tout>(o);
  }
  const unsigned ballot = __ballot_sync(0xffffffffu, fell);
  if ((threadIdx.x & 31) == 0 && ballot) atomicAdd(fb_count, (unsigned long long)__popc(ballot));
}

// ----------------------------------------------------------------------------
// Host launchers
// ----------------------------------------------------------------------------
static void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error{9, std::string(what) + ": " + cudaGetErrorString(e)};
}

void plan_init(Plan& plan, const Params& p, int device) {
  plan.p = p;
  plan.device = device;
  plan.fc = make_filter_consts(p.sigma_s);
  plan.rc = make_range_consts(p);
  const size_t npx = (size_t)p.width * p.height;
  const size_t plane_bytes = (size_t)plan.rc.pairs * npx * sizeof(float2);
  plan.mean_blocks = (int)std::min<size_t>((npx + kMeanThreads - 1) / kMeanThreads, 148 * 8);
  if (plan.mean_blocks < 1) plan.mean_blocks = 1;
  check(cudaMalloc(&plan.planes_v, plane_bytes), "cudaMalloc(planes_v)");
  check(cudaMalloc(&plan.planes_b, plane_bytes), "cudaMalloc(planes_b)");
  check(cudaMalloc(&plan.d_scalars, 4 * sizeof(double)), "cudaMalloc(scalars)");
  check(cudaMalloc(&plan.d_partials, 2 * sizeof(double) * plan.mean_blocks), "cudaMalloc(partials)");
  plan.bytes = 2 * plane_bytes + 4 * sizeof(double) + 2 * sizeof(double) * plan.mean_blocks;
  plan.launches_per_frame = 5;
}

void plan_free(Plan& plan) {
  cudaFree(plan.planes_v);
  cudaFree(plan.planes_b);
  cudaFree(plan.d_scalars);
  cudaFree(plan.d_partials);
  plan.planes_v = plan.planes_b = nullptr;
  plan.d_scalars = plan.d_partials = nullptr;
}

template <typename Tin, typename Tout>
static void run_frame(Plan& plan, const Tin* d_in, Tout* d_out, unsigned long long* d_fb,
                      cudaStream_t st) {
  const int w = plan.p.width, h = plan.p.height;
  const long long npx = (long long)w * h;
  k_mean_partial<Tin><<<plan.mean_blocks, kMeanThreads, 0, st>>>(d_in, npx, plan.d_partials);
  k_mean_final<<<1, kMeanThreads, 0, st>>>(plan.d_partials, plan.mean_blocks, npx,
                                           plan.rc.centering, plan.d_scalars);
  const dim3 blk(32, plan.rc.pairs);
  float2* pv = reinterpret_cast<float2*>(plan.planes_v);
  float2* pb = reinterpret_cast<float2*>(plan.planes_b);
  k_colpass<Tin><<<(w + 31) / 32, blk, 0, st>>>(d_in, pv, plan.d_scalars, w, h, plan.fc, plan.rc);
  k_rowpass<<<(h + 31) / 32, blk, 0, st>>>(pv, pb, w, h, plan.fc);
  k_combine<Tin, Tout><<<(unsigned)((npx + 255) / 256), 256, 0, st>>>(
      d_in, pb, d_out, plan.d_scalars, d_fb, w, h, plan.rc);
  check(cudaGetLastError(), "kernel launch");
}


// ----------------------------------------------------------------------------
// gpf_gaussian_recursive (proj/src/capi.cpp:219-228 -> spatial.cpp:220-251):
// the reference's direct-form deriche_line in fp64 with explicitly rounded,
// never-contracted IEEE operations in the reference's evaluation order, so the
// single-plane exposure is bitwise equal to the x86-64 reference build.
// Not on the hot path (one plane, fp64); rows are one thread per row.
// ----------------------------------------------------------------------------
struct DericheD {
  double nc[4], na[4], d[4];
};

__device__ __forceinline__ double m_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double a_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double s_(double a, double b) { return __dsub_rn(a, b); }

__device__ void deriche_line_f64(const double* src, double* dst, int n, long long stride,
                                 const DericheD& k) {
  const double den_sum = a_(a_(a_(a_(1.0, k.d[0]), k.d[1]), k.d[2]), k.d[3]);
  const double x0 = src[0];
  double ss = __ddiv_rn(m_(x0, a_(a_(a_(k.nc[0], k.nc[1]), k.nc[2]), k.nc[3])), den_sum);
  double xm1 = x0, xm2 = x0, xm3 = x0, ym1 = ss, ym2 = ss, ym3 = ss, ym4 = ss;
  for (int i = 0; i < n; ++i) {
    const double xi = src[i * stride];
    double yi = m_(k.nc[0], xi);
    yi = a_(yi, m_(k.nc[1], xm1));
    yi = a_(yi, m_(k.nc[2], xm2));
    yi = a_(yi, m_(k.nc[3], xm3));
    yi = s_(yi, m_(k.d[0], ym1));
    yi = s_(yi, m_(k.d[1], ym2));
    yi = s_(yi, m_(k.d[2], ym3));
    yi = s_(yi, m_(k.d[3], ym4));
    dst[i * stride] = yi;
    xm3 = xm2; xm2 = xm1; xm1 = xi;
    ym4 = ym3; ym3 = ym2; ym2 = ym1; ym1 = yi;
  }
  const double xl = src[(long long)(n - 1) * stride];
  ss = __ddiv_rn(m_(xl, a_(a_(a_(k.na[0], k.na[1]), k.na[2]), k.na[3])), den_sum);
  double xp1 = xl, xp2 = xl, xp3 = xl, xp4 = xl, yp1 = ss, yp2 = ss, yp3 = ss, yp4 = ss;
  for (int i = n - 1; i >= 0; --i) {
    double yi = m_(k.na[0], xp1);
    yi = a_(yi, m_(k.na[1], xp2));
    yi = a_(yi, m_(k.na[2], xp3));
    yi = a_(yi, m_(k.na[3], xp4));
    yi = s_(yi, m_(k.d[0], yp1));
    yi = s_(yi, m_(k.d[1], yp2));
    yi = s_(yi, m_(k.d[2], yp3));
    yi = s_(yi, m_(k.d[3], yp4));
    dst[i * stride] = a_(dst[i * stride], yi);
    xp4 = xp3; xp3 = xp2; xp2 = xp1; xp1 = src[i * stride];
    yp4 = yp3; yp3 = yp2; yp2 = yp1; yp1 = yi;
  }
}

__global__ void k_gauss_rows(const double* __restrict__ in, double* __restrict__ tmp, int w, int h,
                             DericheD k) {
  const int y = blockIdx.x * blockDim.x + threadIdx.x;
  if (y < h) deriche_line_f64(in + (size_t)y * w, tmp + (size_t)y * w, w, 1, k);
}

__global__ void k_gauss_cols(const double* __restrict__ tmp, double* __restrict__ out, int w, int h,
                             DericheD k, double scale) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= w) return;
  deriche_line_f64(tmp + x, out + x, h, w, k);
  for (int y = 0; y < h; ++y) out[(size_t)y * w + x] = m_(out[(size_t)y * w + x], scale);
}

void run_gaussian_f64(const double* d_in, double* d_out, double* d_tmp, int w, int h,
                      double sigma_s, double scale, cudaStream_t st) {
  DericheD k;
  deriche_coeffs_f64(sigma_s, k.nc, k.na, k.d);
  cudaMemsetAsync(d_out, 0, sizeof(double) * (size_t)w * h, st);
  k_gauss_rows<<<(h + 127) / 128, 128, 0, st>>>(d_in, d_tmp, w, h, k);
  k_gauss_cols<<<(w + 127) / 128, 128, 0, st>>>(d_tmp, d_out, w, h, k, scale);
  check(cudaGetLastError(), "kernel launch");
}

void run_frame_f32(Plan& plan, const float* d_in, float* d_out, unsigned long long* d_fb,
                   cudaStream_t st) {
  run_frame<float, float>(plan, d_in, d_out, d_fb, st);
}

void run_frame_f64(Plan& plan, const double* d_in, double* d_out, unsigned long long* d_fb,
                   cudaStream_t st) {
  run_frame<double, double>(plan, d_in, d_out, d_fb, st);
}

}  // namespace gpfb
