// Reference-exact fp64 precision mode of the GPF path (gpf_filter_gpf's
// PRECISION_FP64).
//
// The fp32 plane pipeline (gpf_kernels.cu) meets the 1e-3 bar wherever the
// reference's degree-N series is well conditioned. Where it is not (small
// sigma_r with pixels far from t_c: BASELINE C2 and C5, whose reference
// outputs leave the input range and reach 1e5), no fp32 evaluation can follow
// the reference, so this mode replays the reference's own fp64 arithmetic on
// the GPU, operation for operation, with explicitly rounded, never-contracted
// IEEE operations:
//   GpfState::init  (proj/src/core/bilateral.cpp:64-106): H = (f - t_c)/sr,
//                   F_0 = exp(-(h h) inv2s2)                  -> k_f64_prologue
//   GpfState::step  (bilateral.cpp:108-129): F_{n+1} = H F_n, Fbar = filter(F)
//                   -> F_n regenerated per pixel by the same multiply chain
//                   recursive_gaussian (spatial.cpp:220-251), rows then columns,
//                   deriche_line (spatial.cpp:186-216)      -> k_f64_rows, k_f64_cols
//                   Q += (c G) Fbar_n, P += (c G) Fbar_{n+1}, G = H G, in step order
//   GpfState::finalize (bilateral.cpp:131-148)                -> k_f64_combine
// All N+2 planes are filtered concurrently (they are independent given H and
// F_0): one lane per (row, 2 planes) in the row pass, one thread per
// (column, plane) in the column pass. The only non-replayed operation is
// exp(): CUDA's exp (<= 1 ulp) instead of glibc's, so F_0 may differ from the
// reference by an ulp on some pixels; everything downstream is bitwise the
// reference's evaluation of those inputs. t_c comes from the deterministic
// double-double mean (K0), equal to the reference's Neumaier mean whenever the
// latter is correctly rounded (every BASELINE frame).
//
// HBM per frame (doubles): H, F_0 [w h]; R [planes][w h] row-pass output;
// C [planes][w h] column-pass output (the filtered planes Fbar_n).
#include <algorithm>
#include <string>

#include <cuda_runtime.h>

#include "gpf_internal.h"

namespace gpfb {

namespace {

__device__ __forceinline__ double m_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double a_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double s_(double a, double b) { return __dsub_rn(a, b); }

struct Deriche64 {
  double nc[4], na[4], d[4];
  double csum, asum, den;  // (nc0+nc1+nc2+nc3), (na0+...), 1+d0+d1+d2+d3 in the reference's order
};

constexpr int kGP = 2;  // planes per row-pass thread

// GpfState::init (bilateral.cpp:92-101)
__global__ void k_f64_prologue(const double* __restrict__ f, const double* __restrict__ scalars,
                               double* __restrict__ H, double* __restrict__ F0, long long n,
                               double sigma_r, double inv2s2) {
  const double t_c = scalars[0];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double hv = s_(f[i], t_c);
    H[i] = __ddiv_rn(hv, sigma_r);
    F0[i] = exp(m_(-m_(hv, hv), inv2s2));
  }
}

// Plane n0+k of a pixel: F_{n0+k} = H (H (... (H F_0))) as step() forms it.
template <int GP>
__device__ __forceinline__ void gen_planes(double hv, double v, int n0, double (&x)[GP]) {
  for (int j = 0; j < n0; ++j) v = m_(hv, v);
  x[0] = v;
#pragma unroll
  for (int k = 1; k < GP; ++k) x[k] = m_(hv, x[k - 1]);
}

// One deriche_line term sequence: nc0 x + nc1 xm1 + nc2 xm2 + nc3 xm3
// - d0 ym1 - d1 ym2 - d2 ym3 - d3 ym4, left to right (spatial.cpp:196-198).
__device__ __forceinline__ double deriche_step(const double (&c)[4], const double (&d)[4], double x0,
                                               double x1, double x2, double x3, double y1, double y2,
                                               double y3, double y4) {
  double y = m_(c[0], x0);
  y = a_(y, m_(c[1], x1));
  y = a_(y, m_(c[2], x2));
  y = a_(y, m_(c[3], x3));
  y = s_(y, m_(d[0], y1));
  y = s_(y, m_(d[1], y2));
  y = s_(y, m_(d[2], y3));
  y = s_(y, m_(d[3], y4));
  return y;
}

// Row pass of recursive_gaussian (spatial.cpp:235-239): CTA = one warp = 32
// rows x kGP planes, lane = row. The row is walked in chunks of 32 columns
// staged through shared memory, so every global access is a coalesced 256-B
// row segment: the (H, F_0) chunk is loaded row by row, each lane runs its
// row's recurrences out of the tile (planes regenerated from (H, F_0) by the
// reference's multiply chain), and the chunk of outputs leaves through a
// [plane][row][column] tile. The anticausal walk reloads the causal outputs
// the same way and adds its own (dst[i] += y-, spatial.cpp:211).
constexpr int kRowT = 32;  // rows per CTA == lanes
#ifndef GPF_F64_ROW_CHUNK
#define GPF_F64_ROW_CHUNK 32
#endif
// columns per staged chunk (32: 256-B row segments, 34 KB of tiles per one-warp
// CTA; 16 halves the tiles and doubles the CTAs per SM but measured slower:
// C5 8.15 vs 7.89 ms, C2 3.08 vs 2.73 ms)
constexpr int kRowC = GPF_F64_ROW_CHUNK;

__global__ void __launch_bounds__(32) k_f64_rows(const double* __restrict__ H,
                                                 const double* __restrict__ F0,
                                                 double* __restrict__ R, int w, int h, int planes,
                                                 Deriche64 k) {
  __shared__ double sH[kRowT][kRowC + 1], sF[kRowT][kRowC + 1];
  __shared__ double sR[kGP][kRowT][kRowC + 1];
  const int lane = threadIdx.x;
  const int y0 = blockIdx.x * kRowT, rows = min(kRowT, h - y0);
  const int n0 = blockIdx.y * kGP, np = min(kGP, planes - n0);
  const size_t ps = (size_t)w * h;
  const int nc = (w + kRowC - 1) / kRowC;
  // global -> shared copies as cp.async (LDGSTS): all of a chunk's row
  // segments in flight at once instead of one load latency per row
  auto cp8 = [](double* smem, const double* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
  };
  auto load_in = [&](int x0, int cols) {
    if (lane < cols)
      for (int r = 0; r < rows; ++r) {
        cp8(&sH[r][lane], H + (size_t)(y0 + r) * w + x0 + lane);
        cp8(&sF[r][lane], F0 + (size_t)(y0 + r) * w + x0 + lane);
      }
  };
  auto load_r = [&](int x0, int cols) {
    if (lane < cols)
      for (int p = 0; p < np; ++p)
        for (int r = 0; r < rows; ++r)
          cp8(&sR[p][r][lane], R + (size_t)(n0 + p) * ps + (size_t)(y0 + r) * w + x0 + lane);
  };
  auto wait_loads = [] {
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  };
  // base plane of this lane's row over the chunk: sF <- F_{n0} = H^{n0} F_0
  // (the reference's multiply chain), eight independent chains interleaved
  auto base_planes = [&](int cols) {
    if (n0 == 0 || !(lane < rows)) return;
    for (int j0 = 0; j0 < cols; j0 += 8) {
      double v[8], hv[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int j = min(j0 + q, cols - 1);
        v[q] = sF[lane][j];
        hv[q] = sH[lane][j];
      }
      for (int t = 0; t < n0; ++t) {
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = m_(hv[q], v[q]);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (j0 + q < cols) sF[lane][j0 + q] = v[q];
    }
  };
  auto store_r = [&](int x0, int cols) {
    if (lane < cols)
      for (int p = 0; p < np; ++p)
        for (int r = 0; r < rows; ++r)
          R[(size_t)(n0 + p) * ps + (size_t)(y0 + r) * w + x0 + lane] = sR[p][r][lane];
  };
  const bool live = lane < rows;
  double x[kGP], xm1[kGP], xm2[kGP], xm3[kGP], ym1[kGP], ym2[kGP], ym3[kGP], ym4[kGP];
  // causal (spatial.cpp:190-202): warm start from column 0
  for (int c = 0; c < nc; ++c) {
    const int x0 = c * kRowC, cols = min(kRowC, w - x0);
    load_in(x0, cols);
    wait_loads();
    __syncwarp();
    base_planes(cols);
    if (live) {
      if (c == 0) {
        gen_planes<kGP>(sH[lane][0], sF[lane][0], 0, x);
#pragma unroll
        for (int p = 0; p < kGP; ++p) {
          const double ss = __ddiv_rn(m_(x[p], k.csum), k.den);
          xm1[p] = xm2[p] = xm3[p] = x[p];
          ym1[p] = ym2[p] = ym3[p] = ym4[p] = ss;
        }
      }
      for (int j = 0; j < cols; ++j) {
        gen_planes<kGP>(sH[lane][j], sF[lane][j], 0, x);
#pragma unroll
        for (int p = 0; p < kGP; ++p) {
          const double yi = deriche_step(k.nc, k.d, x[p], xm1[p], xm2[p], xm3[p], ym1[p], ym2[p],
                                         ym3[p], ym4[p]);
          sR[p][lane][j] = yi;
          xm3[p] = xm2[p]; xm2[p] = xm1[p]; xm1[p] = x[p];
          ym4[p] = ym3[p]; ym3[p] = ym2[p]; ym2[p] = ym1[p]; ym1[p] = yi;
        }
      }
    }
    __syncwarp();
    store_r(x0, cols);
    __syncwarp();
  }
  // anticausal (spatial.cpp:204-215): xp = x[i+1..i+4], warm start from column w-1
  double xp4[kGP];
  for (int c = nc - 1; c >= 0; --c) {
    const int x0 = c * kRowC, cols = min(kRowC, w - x0);
    load_in(x0, cols);
    load_r(x0, cols);
    wait_loads();
    __syncwarp();
    base_planes(cols);
    if (live) {
      if (c == nc - 1) {
        gen_planes<kGP>(sH[lane][cols - 1], sF[lane][cols - 1], 0, x);
#pragma unroll
        for (int p = 0; p < kGP; ++p) {
          const double ss = __ddiv_rn(m_(x[p], k.asum), k.den);
          xm1[p] = xm2[p] = xm3[p] = xp4[p] = x[p];  // xp1..xp4
          ym1[p] = ym2[p] = ym3[p] = ym4[p] = ss;
        }
      }
      for (int j = cols - 1; j >= 0; --j) {
        gen_planes<kGP>(sH[lane][j], sF[lane][j], 0, x);
#pragma unroll
        for (int p = 0; p < kGP; ++p) {
          const double yi = deriche_step(k.na, k.d, xm1[p], xm2[p], xm3[p], xp4[p], ym1[p], ym2[p],
                                         ym3[p], ym4[p]);
          sR[p][lane][j] = a_(sR[p][lane][j], yi);
          xp4[p] = xm3[p]; xm3[p] = xm2[p]; xm2[p] = xm1[p]; xm1[p] = x[p];
          ym4[p] = ym3[p]; ym3[p] = ym2[p]; ym2[p] = ym1[p]; ym1[p] = yi;
        }
      }
    }
    __syncwarp();
    store_r(x0, cols);
    __syncwarp();
  }
}

// Column pass of recursive_gaussian (spatial.cpp:240-249), output scaled by
// mass^2 kernel_scale: thread = (column, plane), coalesced across columns.
__global__ void __launch_bounds__(128) k_f64_cols(const double* __restrict__ R, double* __restrict__ C,
                                                  int w, int h, Deriche64 k, double scale) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= w) return;
  const size_t ps = (size_t)w * h;
  const double* src = R + (size_t)blockIdx.y * ps + x;
  double* dst = C + (size_t)blockIdx.y * ps + x;
  const double x0 = src[0];
  double ss = __ddiv_rn(m_(x0, k.csum), k.den);
  double xm1 = x0, xm2 = x0, xm3 = x0, ym1 = ss, ym2 = ss, ym3 = ss, ym4 = ss;
  for (int i = 0; i < h; ++i) {
    const double xi = src[(size_t)i * w];
    const double yi = deriche_step(k.nc, k.d, xi, xm1, xm2, xm3, ym1, ym2, ym3, ym4);
    dst[(size_t)i * w] = yi;
    xm3 = xm2; xm2 = xm1; xm1 = xi;
    ym4 = ym3; ym3 = ym2; ym2 = ym1; ym1 = yi;
  }
  const double xl = src[(size_t)(h - 1) * w];
  ss = __ddiv_rn(m_(xl, k.asum), k.den);
  double xp1 = xl, xp2 = xl, xp3 = xl, xp4 = xl, yp1 = ss, yp2 = ss, yp3 = ss, yp4 = ss;
  for (int i = h - 1; i >= 0; --i) {
    const double xi = src[(size_t)i * w];
    const double yi = deriche_step(k.na, k.d, xp1, xp2, xp3, xp4, yp1, yp2, yp3, yp4);
    dst[(size_t)i * w] = m_(a_(dst[(size_t)i * w], yi), scale);
    xp4 = xp3; xp3 = xp2; xp2 = xp1; xp1 = xi;
    yp4 = yp3; yp3 = yp2; yp2 = yp1; yp1 = yi;
  }
}

// Accumulation in step order and finalize (bilateral.cpp:117-148).
struct Combine64 {
  double c[kMaxPlanes];  // c_n = c_{n-1} / n, as step() updates it
  double sigma_r;
  int degree;
};

__global__ void k_f64_combine(const double* __restrict__ f, const double* __restrict__ H,
                              const double* __restrict__ Cb, const double* __restrict__ scalars,
                              double* __restrict__ out, long long n, long long i0, long long i1,
                              Combine64 cb, unsigned long long* __restrict__ fallbacks) {
  const double t_c = scalars[0];
  unsigned my_fb = 0;
  for (long long i = i0 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < i1;
       i += (long long)gridDim.x * blockDim.x) {
    const double hv = H[i];
    double g = 1.0, q = 0.0, p = 0.0;
    double fb = Cb[i];
    for (int s = 0; s <= cb.degree; ++s) {
      const double cg = m_(cb.c[s], g);
      q = a_(q, m_(cg, fb));
      fb = Cb[(size_t)(s + 1) * n + i];
      p = a_(p, m_(cg, fb));
      g = m_(hv, g);
    }
    if (fabs(q) <= 1e-8) {  // kQMin (bilateral.hpp:85)
      out[i] = f[i];
      ++my_fb;
    } else {
      out[i] = a_(m_(cb.sigma_r, __ddiv_rn(p, q)), t_c);
    }
  }
  for (int o = 16; o; o >>= 1) my_fb += __shfl_xor_sync(0xffffffffu, my_fb, o);
  if ((threadIdx.x & 31) == 0 && my_fb) atomicAdd(fallbacks, (unsigned long long)my_fb);
}

void chk(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();  // clear a non-sticky error (e.g. a failed allocation) for the caller
    throw Error{9, std::string(what) + ": " + cudaGetErrorString(e)};
  }
}

}  // namespace

size_t f64_workspace_bytes(int w, int h, int degree) {
  const size_t n = (size_t)w * h;
  return sizeof(double) * (n * (2 + 2 * (size_t)(degree + 2)) + 2 + 4 * kF64MeanBlocks);
}

void F64Work::ensure(size_t bytes_needed) {
  if (bytes_needed <= cap) return;
  release();
  chk(cudaMalloc(&base, bytes_needed), "cudaMalloc(fp64 GPF workspace)");
  cap = bytes_needed;
}

void F64Work::release() {
  cudaFree(base);
  base = nullptr;
  cap = 0;
}

void run_gpf_f64_exact(const double* d_in, double* d_out, const Params& p, F64Work& ws,
                       unsigned long long* d_fb, cudaStream_t st, int ranges,
                       cudaEvent_t* range_done) {
  const int w = p.width, h = p.height, planes = p.degree + 2;
  if (planes > kMaxPlanes) throw Error{1, "RangeParams: degree must be <= 62 in the B200 library"};
  const long long n = (long long)w * h;
  ws.ensure(f64_workspace_bytes(w, h, p.degree));
  double* H = ws.base;
  double* F0 = H + n;
  double* R = F0 + n;
  double* Cb = R + (size_t)planes * n;
  double* scalars = Cb + (size_t)planes * n;
  double* partials = scalars + 2;
  launch_mean_f64(d_in, n, p.centering, p.tc_fixed, p.sigma_r, partials, kF64MeanBlocks, scalars, st);
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148 * 16);
  // GpfState::init: inv2s2 = 1.0 / (2.0 * sr * sr) (bilateral.cpp:92)
  const double inv2s2 = 1.0 / (2.0 * p.sigma_r * p.sigma_r);
  k_f64_prologue<<<blocks, 256, 0, st>>>(d_in, scalars, H, F0, n, p.sigma_r, inv2s2);
  Deriche64 k;
  deriche_coeffs_f64(p.sigma_s, k.nc, k.na, k.d);
  k.den = 1.0 + k.d[0] + k.d[1] + k.d[2] + k.d[3];
  k.csum = k.nc[0] + k.nc[1] + k.nc[2] + k.nc[3];
  k.asum = k.na[0] + k.na[1] + k.na[2] + k.na[3];
  k_f64_rows<<<dim3((h + kRowT - 1) / kRowT, (planes + kGP - 1) / kGP), kRowT, 0, st>>>(H, F0, R, w, h,
                                                                                        planes, k);
  const double mass = kernel_mass_1d(p.sigma_s, default_window_radius(p.sigma_s));
  const double scale = mass * mass * p.kernel_scale;
  k_f64_cols<<<dim3((w + 127) / 128, planes), 128, 0, st>>>(R, Cb, w, h, k, scale);
  Combine64 cb;
  cb.c[0] = 1.0;
  for (int s = 0; s + 1 < kMaxPlanes; ++s) cb.c[s + 1] = cb.c[s] / (s + 1);  // c = c / (n + 1)
  cb.sigma_r = p.sigma_r;
  cb.degree = p.degree;
  chk(cudaMemsetAsync(d_fb, 0, sizeof(unsigned long long), st), "cudaMemsetAsync");
  // pixel ranges (drop-in D2H overlap): event i once pixels [n i/R, n (i+1)/R) are final
  const int nr = (ranges > 1 && range_done) ? ranges : 1;
  for (int r = 0; r < nr; ++r) {
    const long long i0 = n * r / nr, i1 = n * (r + 1) / nr;
    const int rb = (int)std::min<long long>((i1 - i0 + 255) / 256, 148 * 16);
    k_f64_combine<<<std::max(rb, 1), 256, 0, st>>>(d_in, H, Cb, scalars, d_out, n, i0, i1, cb, d_fb);
    if (nr > 1) chk(cudaEventRecord(range_done[r], st), "cudaEventRecord");
  }
  chk(cudaGetLastError(), "kernel launch (fp64 GPF)");
}

}  // namespace gpfb
