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
// exp(): a correctly rounded double-double evaluation (exp_cr.h) instead of
// glibc's, which is itself correctly rounded on ~99.9 % of arguments -- F_0
// differs from the reference by one ulp on the rest (~1 pixel in 1,000);
// everything downstream is bitwise the reference's evaluation of those inputs. t_c comes from the deterministic
// double-double mean (K0), equal to the reference's Neumaier mean whenever the
// latter is correctly rounded (every BASELINE frame).
//
// HBM per frame (doubles): H, F_0 [w h]; R [planes][w h] row-pass output;
// C [planes][w h] column-pass output (the filtered planes Fbar_n).
#include <algorithm>
#include <cstdlib>
#include <string>

#include <cuda_runtime.h>

#include "exp_cr.h"
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
    F0[i] = exp_cr(m_(-m_(hv, hv), inv2s2));  // correctly rounded (exp_cr.h); CUDA's exp is within 1 ulp
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

// ----------------------------------------------------------------------------
// Chunked form of the same two passes (the default). The reference's line
// filter runs the causal recurrence over the whole line, then the anticausal
// one adding into it; replayed literally (k_f64_rows / k_f64_cols above) that
// is a read-modify-write of every plane per axis. Here a line is cut into
// chunks of kF64Chunk samples:
//   states kernel : the anticausal recurrence alone, walked from the far end
//                   of the line; its register state (x[i+1..i+4], y-[i+1..i+4])
//                   is recorded where it enters each chunk.
//   chunk kernel  : walks the chunks in causal order; per chunk the causal
//                   recurrence (state carried in registers), then the
//                   anticausal one restarted from the recorded state, summed
//                   and written once.
// Every output is produced by the same operations on the same operands in the
// same order as in the sequential form, so the two are bitwise equal
// (tests/test_gpu_dropin.py compares them); the planes cross HBM once per
// axis instead of being re-read and re-written.
// ----------------------------------------------------------------------------
constexpr int kF64Chunk = 32;  // samples per chunk of the column pass
#ifndef GPF_F64_RB
#define GPF_F64_RB 8
#endif
#ifndef GPF_F64_RCH
#define GPF_F64_RCH 32
#endif
constexpr int kRB2 = GPF_F64_RB;     // rows per CTA of the chunked row pass (4 or 8)
constexpr int kRowCh = GPF_F64_RCH;  // samples per chunk of the row pass (<= 32)
constexpr int kTP = kRowCh + 1;      // padded tile pitch (doubles)
// Y plane stride: a half-warp's 16 / kRB2 plane pairs land kRB2 doubles apart in the bank space
constexpr int kYP = kRB2 * kTP + ((kRB2 / 2 - (kRB2 * kTP) % 8 + 8) % 8);
static_assert(kRB2 == 4 || kRB2 == 8, "rows per CTA");
static_assert(kRowCh == 8 || kRowCh == 16 || kRowCh == 32, "row chunk");

__device__ __forceinline__ void cp8(double* smem, const double* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}

// Chunked row pass, shared by its two kernels. A CTA owns kRB2 rows and ALL
// planes: thread = (row, plane pair), so a chunk's (H, F_0) tile is loaded once
// for every plane and the even planes F_2g = H (H F_{2g-2}) are formed once per
// pixel by the reference's multiply chain (X2), the odd ones as H F_2g by their
// owner. Shared memory (doubles): sH, sF [kRB2][kTP]; X2 [pg][kRB2][kTP];
// Y [planes][kRB2][kTP] (chunk kernel only).
struct RowCtx {
  double *sH, *sF, *X2;
  int tid, nthr, row, pg, PG, rows, y0;
};

// Chunk pipeline: while a chunk's recurrences run, the next chunk's F_0 tile
// streams into sF by cp.async (sF is free once the even planes are formed) and
// its H values wait in registers (sH is still being read); rows_finish_load
// lands both. kHR H values per thread cover the tile for CTAs of >= 64 threads.
constexpr int kHR = 4;
struct RowPrefetch {
  double hreg[kHR];
};
__device__ __forceinline__ void rows_issue_load(const RowCtx& c, RowPrefetch& pf,
                                                const double* __restrict__ H,
                                                const double* __restrict__ F0, int w, int x0, int cols) {
#pragma unroll
  for (int q = 0; q < kHR; ++q) {
    const int e = c.tid + q * c.nthr;
    const int r = e / kRowCh, j = e % kRowCh;
    if (e < kRB2 * kRowCh && r < c.rows && j < cols) {
      const size_t g = (size_t)(c.y0 + r) * w + x0 + j;
      pf.hreg[q] = __ldg(H + g);
      cp8(&c.sF[r * kTP + j], F0 + g);
    }
  }
  asm volatile("cp.async.commit_group;\n" ::);
}
// lands the issued chunk in sH / sF and forms the even planes of its pixels
__device__ __forceinline__ void rows_finish_load(const RowCtx& c, const RowPrefetch& pf, int cols) {
#pragma unroll
  for (int q = 0; q < kHR; ++q) {
    const int e = c.tid + q * c.nthr;
    const int r = e / kRowCh, j = e % kRowCh;
    if (e < kRB2 * kRowCh && r < c.rows && j < cols) c.sH[r * kTP + j] = pf.hreg[q];
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  // even planes of every pixel of the chunk, four pixels' chains interleaved
  constexpr int kE = 4;
  for (int e0 = c.tid; e0 < kRB2 * kRowCh; e0 += c.nthr * kE) {
    double hv[kE], v[kE];
    int off[kE];
    bool ok[kE];
#pragma unroll
    for (int q = 0; q < kE; ++q) {
      const int e = e0 + q * c.nthr;
      const int r = e / kRowCh, j = e % kRowCh;
      ok[q] = e < kRB2 * kRowCh && r < c.rows && j < cols;
      off[q] = ok[q] ? r * kTP + j : 0;
      hv[q] = c.sH[off[q]];
      v[q] = c.sF[off[q]];
      if (ok[q]) c.X2[off[q]] = v[q];
    }
    for (int g = 1; g < c.PG; ++g) {
#pragma unroll
      for (int q = 0; q < kE; ++q) {
        v[q] = m_(hv[q], m_(hv[q], v[q]));
        if (ok[q]) c.X2[g * kRB2 * kTP + off[q]] = v[q];
      }
    }
  }
  __syncthreads();
}

// this thread's plane pair at column j of the chunk: (F_2pg, F_2pg+1); xe / hr
// are the thread's rows of X2 and sH (immediate offsets in the unrolled loops)
__device__ __forceinline__ void rows_x(const double* xe, const double* hr, int j, double (&x)[kGP]) {
  x[0] = xe[j];
  x[1] = m_(hr[j], x[0]);
}

struct Anti64 {  // anticausal register state of one line
  double xp1, xp2, xp3, xp4, yp1, yp2, yp3, yp4;
};
__device__ __forceinline__ void anti_warm(Anti64& a, double xl, const Deriche64& k) {
  const double ss = __ddiv_rn(m_(xl, k.asum), k.den);
  a.xp1 = a.xp2 = a.xp3 = a.xp4 = xl;
  a.yp1 = a.yp2 = a.yp3 = a.yp4 = ss;
}
__device__ __forceinline__ double anti_step(Anti64& a, double xi, const Deriche64& k) {
  const double yi = deriche_step(k.na, k.d, a.xp1, a.xp2, a.xp3, a.xp4, a.yp1, a.yp2, a.yp3, a.yp4);
  a.xp4 = a.xp3; a.xp3 = a.xp2; a.xp2 = a.xp1; a.xp1 = xi;
  a.yp4 = a.yp3; a.yp3 = a.yp2; a.yp2 = a.yp1; a.yp1 = yi;
  return yi;
}
struct Caus64 {
  double xm1, xm2, xm3, ym1, ym2, ym3, ym4;
};
__device__ __forceinline__ void caus_warm(Caus64& s, double x0, const Deriche64& k) {
  const double ss = __ddiv_rn(m_(x0, k.csum), k.den);
  s.xm1 = s.xm2 = s.xm3 = x0;
  s.ym1 = s.ym2 = s.ym3 = s.ym4 = ss;
}
__device__ __forceinline__ double caus_step(Caus64& s, double xi, const Deriche64& k) {
  const double yi = deriche_step(k.nc, k.d, xi, s.xm1, s.xm2, s.xm3, s.ym1, s.ym2, s.ym3, s.ym4);
  s.xm3 = s.xm2; s.xm2 = s.xm1; s.xm1 = xi;
  s.ym4 = s.ym3; s.ym3 = s.ym2; s.ym2 = s.ym1; s.ym1 = yi;
  return yi;
}
// recorded states: component k of line `line` at p[k * stride]
__device__ __forceinline__ void anti_store(const Anti64& a, double* p, size_t stride) {
  p[0] = a.xp1; p[stride] = a.xp2; p[2 * stride] = a.xp3; p[3 * stride] = a.xp4;
  p[4 * stride] = a.yp1; p[5 * stride] = a.yp2; p[6 * stride] = a.yp3; p[7 * stride] = a.yp4;
}
__device__ __forceinline__ void anti_load(Anti64& a, const double* p, size_t stride) {
  a.xp1 = p[0]; a.xp2 = p[stride]; a.xp3 = p[2 * stride]; a.xp4 = p[3 * stride];
  a.yp1 = p[4 * stride]; a.yp2 = p[5 * stride]; a.yp3 = p[6 * stride]; a.yp4 = p[7 * stride];
}

__device__ __forceinline__ RowCtx rows_ctx(double* smem, int h, int planes) {
  RowCtx c;
  c.sH = smem;
  c.sF = smem + kRB2 * kTP;
  c.X2 = smem + 2 * kRB2 * kTP;
  c.tid = threadIdx.x;
  c.nthr = blockDim.x;
  c.row = c.tid % kRB2;
  c.pg = c.tid / kRB2;
  c.PG = (planes + kGP - 1) / kGP;
  c.y0 = blockIdx.x * kRB2;
  c.rows = min(kRB2, h - c.y0);
  return c;
}

// S layout (row pass): [band][chunk][8 components][planes][kRB2 rows]
__global__ void k_f64_rows_states(const double* __restrict__ H, const double* __restrict__ F0,
                                  double* __restrict__ S, int w, int h, int planes, Deriche64 k) {
  extern __shared__ double smem_d[];
  const RowCtx c = rows_ctx(smem_d, h, planes);
  const int nc = (w + kRowCh - 1) / kRowCh;
  const bool live = c.pg < c.PG && c.row < c.rows;
  const size_t comp = (size_t)planes * kRB2;
  const double* xe = c.X2 + (c.pg < c.PG ? c.pg : 0) * kRB2 * kTP + c.row * kTP;
  const double* hr = c.sH + c.row * kTP;
  Anti64 a[kGP];
  double x[kGP];
  RowPrefetch pf;
  if (nc > 1) rows_issue_load(c, pf, H, F0, w, (nc - 1) * kRowCh, w - (nc - 1) * kRowCh);
  for (int ch = nc - 1; ch >= 1; --ch) {  // chunk 0's walk would record nothing
    const int x0 = ch * kRowCh, cols = min(kRowCh, w - x0);
    rows_finish_load(c, pf, cols);
    if (ch > 1) rows_issue_load(c, pf, H, F0, w, x0 - kRowCh, kRowCh);
    if (live) {
      if (ch == nc - 1) {
        rows_x(xe, hr, cols - 1, x);
#pragma unroll
        for (int p = 0; p < kGP; ++p) anti_warm(a[p], x[p], k);
      }
      if (cols == kRowCh) {  // full chunk: eight samples' inputs at a time, rotations rename registers
        for (int j0 = kRowCh - 8; j0 >= 0; j0 -= 8) {
          double xs[8], hs[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            xs[q] = xe[j0 + q];
            hs[q] = hr[j0 + q];
          }
#pragma unroll
          for (int q = 7; q >= 0; --q) {
            anti_step(a[0], xs[q], k);
            anti_step(a[1], m_(hs[q], xs[q]), k);
          }
        }
      } else {
        for (int j = cols - 1; j >= 0; --j) {
          rows_x(xe, hr, j, x);
#pragma unroll
          for (int p = 0; p < kGP; ++p) anti_step(a[p], x[p], k);
        }
      }
      double* dst = S + ((size_t)blockIdx.x * nc + (ch - 1)) * 8 * comp + c.row;
#pragma unroll
      for (int p = 0; p < kGP; ++p)
        if (c.pg * kGP + p < planes) anti_store(a[p], dst + (size_t)(c.pg * kGP + p) * kRB2, comp);
    }
    __syncthreads();  // sH and X2 are free again
  }
}

__global__ void k_f64_rows_chunked(const double* __restrict__ H, const double* __restrict__ F0,
                                   const double* __restrict__ S, double* __restrict__ R, int w, int h,
                                   int planes, Deriche64 k) {
  extern __shared__ double smem_d[];
  const RowCtx c = rows_ctx(smem_d, h, planes);
  double* Y = c.X2 + (size_t)c.PG * kRB2 * kTP;  // [planes][kRB2][kTP]
  const int nc = (w + kRowCh - 1) / kRowCh;
  const bool live = c.pg < c.PG && c.row < c.rows;
  const size_t comp = (size_t)planes * kRB2, ps = (size_t)w * h;
  const int lane = c.tid & 31, warp = c.tid >> 5;
  const double* xe = c.X2 + (c.pg < c.PG ? c.pg : 0) * kRB2 * kTP + c.row * kTP;
  const double* hr = c.sH + c.row * kTP;
  Caus64 cs[kGP];
  double x[kGP];
  RowPrefetch pf;
  rows_issue_load(c, pf, H, F0, w, 0, min(kRowCh, w));
  for (int ch = 0; ch < nc; ++ch) {
    const int x0 = ch * kRowCh, cols = min(kRowCh, w - x0);
    // the anticausal state entering this chunk, in flight under the even-plane chains
    Anti64 a[kGP], an[kGP];
    if (live && ch + 1 < nc) {
      const double* src = S + ((size_t)blockIdx.x * nc + ch) * 8 * comp + c.row;
#pragma unroll
      for (int p = 0; p < kGP; ++p)
        if (c.pg * kGP + p < planes) anti_load(an[p], src + (size_t)(c.pg * kGP + p) * kRB2, comp);
    }
    rows_finish_load(c, pf, cols);
    if (ch + 1 < nc) rows_issue_load(c, pf, H, F0, w, x0 + kRowCh, min(kRowCh, w - x0 - kRowCh));
    if (live) {
      double* yt = Y + (size_t)(c.pg * kGP) * kYP + c.row * kTP;
      const bool two = c.pg * kGP + 1 < planes;
      if (ch == 0) {
        rows_x(xe, hr, 0, x);
#pragma unroll
        for (int p = 0; p < kGP; ++p) caus_warm(cs[p], x[p], k);
      }
      if (ch + 1 == nc) {
        rows_x(xe, hr, cols - 1, x);
#pragma unroll
        for (int p = 0; p < kGP; ++p) anti_warm(a[p], x[p], k);
      } else {
#pragma unroll
        for (int p = 0; p < kGP; ++p) a[p] = an[p];
      }
      if (cols == kRowCh && two) {
        // full chunk, eight samples at a time: their inputs are read before the
        // outputs are stored (the tiles share one array, so the compiler keeps
        // loads behind earlier stores), and the state rotations rename registers
        for (int j0 = 0; j0 < kRowCh; j0 += 8) {
          double xs[8], hs[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            xs[q] = xe[j0 + q];
            hs[q] = hr[j0 + q];
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            yt[j0 + q] = caus_step(cs[0], xs[q], k);
            yt[kYP + j0 + q] = caus_step(cs[1], m_(hs[q], xs[q]), k);
          }
        }
        for (int j0 = kRowCh - 8; j0 >= 0; j0 -= 8) {
          double xs[8], hs[8], y0s[8], y1s[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            xs[q] = xe[j0 + q];
            hs[q] = hr[j0 + q];
            y0s[q] = yt[j0 + q];
            y1s[q] = yt[kYP + j0 + q];
          }
#pragma unroll
          for (int q = 7; q >= 0; --q) {
            yt[j0 + q] = a_(y0s[q], anti_step(a[0], xs[q], k));
            yt[kYP + j0 + q] = a_(y1s[q], anti_step(a[1], m_(hs[q], xs[q]), k));
          }
        }
      } else {
        for (int j = 0; j < cols; ++j) {
          rows_x(xe, hr, j, x);
          yt[j] = caus_step(cs[0], x[0], k);
          const double y1 = caus_step(cs[1], x[1], k);
          if (two) yt[kYP + j] = y1;
        }
        for (int j = cols - 1; j >= 0; --j) {
          rows_x(xe, hr, j, x);
          yt[j] = a_(yt[j], anti_step(a[0], x[0], k));
          const double y1 = anti_step(a[1], x[1], k);
          if (two) yt[kYP + j] = a_(yt[kYP + j], y1);
        }
      }
    }
    // The chunk leaves as coalesced row segments of kRowCh doubles. A warp owns whole
    // planes of Y (its plane pairs), so it stores them as soon as its own recurrences are
    // done; the CTA barrier below only guards the tiles the next chunk overwrites.
    __syncwarp();
    constexpr int kSW = 32 / kRowCh;       // row segments per warp and turn
    constexpr int kPW = kGP * 32 / kRB2;  // planes of one warp
    const int l = lane % kRowCh;
    const int n0w = warp * kPW, n1w = min(n0w + kPW, planes);
    for (int r = lane / kRowCh; r < c.rows; r += kSW) {
      const double* ys = Y + r * kTP + l;
      double* rd = R + (size_t)(c.y0 + r) * w + x0 + l;
      if (l < cols) {
#pragma unroll 4
        for (int n = n0w; n < n1w; ++n) rd[(size_t)n * ps] = ys[n * kYP];
      }
    }
    __syncthreads();
  }
}

size_t rows2_smem_bytes(int planes) {
  const int PG = (planes + kGP - 1) / kGP;
  return sizeof(double) * ((size_t)(2 + PG) * kRB2 * kTP + (size_t)planes * kYP);
}

// Chunked column pass: thread = (column, plane), coalesced across columns. A
// thread's chunk of inputs arrives in its own shared-memory column by
// cp.async, double-buffered: the next chunk's 32 loads are in flight while the
// current one is filtered, and no value waits in registers. No barriers: a
// thread only touches its own column of the tiles.
// S layout: [plane][chunk][8 components][w].
constexpr int kColT = 128;
struct ColTiles {
  double x[2][kF64Chunk][kColT];  // inputs, two chunks
  double y[kF64Chunk][kColT];     // causal outputs of the current chunk (chunk kernel)
};
__device__ __forceinline__ void cols_load_chunk(double (*sx)[kColT], const double* src, int w, int y0,
                                                int rows) {
#pragma unroll
  for (int j = 0; j < kF64Chunk; ++j)
    if (j < rows) cp8(&sx[j][threadIdx.x], src + (size_t)(y0 + j) * w);
  asm volatile("cp.async.commit_group;\n" ::);
}
__device__ __forceinline__ void cols_wait_chunk(bool newer_in_flight) {
  if (newer_in_flight) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
  else asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

__global__ void __launch_bounds__(kColT) k_f64_cols_states(const double* __restrict__ R,
                                                           double* __restrict__ S, int w, int h,
                                                           Deriche64 k) {
  extern __shared__ double smem_d[];
  double(*sx)[kF64Chunk][kColT] = reinterpret_cast<double(*)[kF64Chunk][kColT]>(smem_d);
  const int x = blockIdx.x * kColT + threadIdx.x;
  if (x >= w) return;
  const size_t ps = (size_t)w * h;
  const int ncy = (h + kF64Chunk - 1) / kF64Chunk;
  const double* src = R + (size_t)blockIdx.y * ps + x;
  Anti64 a;
  anti_warm(a, src[(size_t)(h - 1) * w], k);
  cols_load_chunk(sx[(ncy - 1) & 1], src, w, (ncy - 1) * kF64Chunk, h - (ncy - 1) * kF64Chunk);
  for (int cy = ncy - 1; cy >= 1; --cy) {  // chunk 0's walk would record nothing
    const int rows = min(kF64Chunk, h - cy * kF64Chunk);
    if (cy > 1) cols_load_chunk(sx[(cy - 1) & 1], src, w, (cy - 1) * kF64Chunk, kF64Chunk);
    cols_wait_chunk(cy > 1);
    const double* cx = &sx[cy & 1][0][threadIdx.x];
    if (rows == kF64Chunk) {
#pragma unroll 8
      for (int j = kF64Chunk - 1; j >= 0; --j) anti_step(a, cx[j * kColT], k);
    } else {
      for (int j = rows - 1; j >= 0; --j) anti_step(a, cx[j * kColT], k);
    }
    anti_store(a, S + ((size_t)blockIdx.y * ncy + (cy - 1)) * 8 * w + x, w);
  }
}

__global__ void __launch_bounds__(kColT) k_f64_cols_chunked(const double* __restrict__ R,
                                                            const double* __restrict__ S,
                                                            double* __restrict__ C, int w, int h,
                                                            Deriche64 k, double scale) {
  extern __shared__ double smem_d[];
  ColTiles& t = *reinterpret_cast<ColTiles*>(smem_d);
  const int x = blockIdx.x * kColT + threadIdx.x;
  if (x >= w) return;
  const size_t ps = (size_t)w * h;
  const int ncy = (h + kF64Chunk - 1) / kF64Chunk;
  const double* src = R + (size_t)blockIdx.y * ps + x;
  double* dst = C + (size_t)blockIdx.y * ps + x;
  Caus64 cs;
  cols_load_chunk(t.x[0], src, w, 0, min(kF64Chunk, h));
  for (int cy = 0; cy < ncy; ++cy) {
    const int y0 = cy * kF64Chunk, rows = min(kF64Chunk, h - y0);
    const bool more = cy + 1 < ncy;
    Anti64 a;
    if (more) {
      cols_load_chunk(t.x[(cy + 1) & 1], src, w, y0 + kF64Chunk, min(kF64Chunk, h - y0 - kF64Chunk));
      anti_load(a, S + ((size_t)blockIdx.y * ncy + cy) * 8 * w + x, w);
    }
    cols_wait_chunk(more);
    const double* cx = &t.x[cy & 1][0][threadIdx.x];
    double* cyo = &t.y[0][threadIdx.x];
    double* dd = dst + (size_t)y0 * w;
    if (cy == 0) caus_warm(cs, cx[0], k);
    if (!more) anti_warm(a, cx[(rows - 1) * kColT], k);
    if (rows == kF64Chunk) {  // eight samples' inputs read ahead of the outputs' stores
      for (int j0 = 0; j0 < kF64Chunk; j0 += 8) {
        double xs[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) xs[q] = cx[(j0 + q) * kColT];
#pragma unroll
        for (int q = 0; q < 8; ++q) cyo[(j0 + q) * kColT] = caus_step(cs, xs[q], k);
      }
      for (int j0 = kF64Chunk - 8; j0 >= 0; j0 -= 8) {
        double xs[8], ys[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          xs[q] = cx[(j0 + q) * kColT];
          ys[q] = cyo[(j0 + q) * kColT];
        }
#pragma unroll
        for (int q = 7; q >= 0; --q)
          dd[(size_t)(j0 + q) * w] = m_(a_(ys[q], anti_step(a, xs[q], k)), scale);
      }
    } else {
      for (int j = 0; j < rows; ++j) cyo[j * kColT] = caus_step(cs, cx[j * kColT], k);
      for (int j = rows - 1; j >= 0; --j) {
        const double yi = anti_step(a, cx[j * kColT], k);
        dd[(size_t)j * w] = m_(a_(cyo[j * kColT], yi), scale);
      }
    }
  }
}

size_t f64_state_doubles(int w, int h, int planes) {
  const size_t nc = (w + kRowCh - 1) / kRowCh, ncy = (h + kF64Chunk - 1) / kF64Chunk;
  const size_t bands = (h + kRB2 - 1) / kRB2;
  const size_t rows_s = bands * nc * 8 * planes * kRB2, cols_s = (size_t)planes * ncy * 8 * w;
  return std::max(rows_s, cols_s);
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
    // eight planes' loads in flight per pixel, then their steps in step order
    for (int s0 = 0; s0 <= cb.degree; s0 += 8) {
      double nx[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (s0 + k <= cb.degree) nx[k] = Cb[(size_t)(s0 + k + 1) * n + i];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (s0 + k <= cb.degree) {
          const double cg = m_(cb.c[s0 + k], g);
          q = a_(q, m_(cg, fb));
          fb = nx[k];
          p = a_(p, m_(cg, fb));
          g = m_(hv, g);
        }
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

// ---- GpfState stepping (cxxapi.cpp; bilateral.cpp:64-148), one call per phase
namespace {

__global__ void k_exp_cr(const double* __restrict__ x, double* __restrict__ y, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = exp_cr(x[i]);
}

// step(), first loop (bilateral.cpp:117-120): q += c g fbar; f = h f
__global__ void k_state_step_a(double* __restrict__ Q, double* __restrict__ F,
                               const double* __restrict__ G, const double* __restrict__ Fbar,
                               const double* __restrict__ H, double c, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    Q[i] = a_(Q[i], m_(m_(c, G[i]), Fbar[i]));
    F[i] = m_(H[i], F[i]);
  }
}

// step(), second loop (bilateral.cpp:123-126): p += c g fbar; g = h g
__global__ void k_state_step_b(double* __restrict__ P, double* __restrict__ G,
                               const double* __restrict__ Fbar, const double* __restrict__ H,
                               double c, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    P[i] = a_(P[i], m_(m_(c, G[i]), Fbar[i]));
    G[i] = m_(H[i], G[i]);
  }
}

// finalize() (bilateral.cpp:131-148)
__global__ void k_state_finalize(const double* __restrict__ in, const double* __restrict__ P,
                                 const double* __restrict__ Q, double* __restrict__ out, long long n,
                                 double sigma_r, double t_c, unsigned long long* __restrict__ fallbacks) {
  unsigned my_fb = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (fabs(Q[i]) <= 1e-8) {  // kQMin
      out[i] = in[i];
      ++my_fb;
    } else {
      out[i] = a_(m_(sigma_r, __ddiv_rn(P[i], Q[i])), t_c);
    }
  }
  for (int o = 16; o; o >>= 1) my_fb += __shfl_xor_sync(0xffffffffu, my_fb, o);
  if ((threadIdx.x & 31) == 0 && my_fb) atomicAdd(fallbacks, (unsigned long long)my_fb);
}

int state_blocks(long long n) { return (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, 148 * 16)); }

}  // namespace

// the device instantiation of exp_cr.h over n doubles (test hook: gpf_b200_exp_cr)
void run_exp_cr_f64(const double* d_x, double* d_y, long long n, cudaStream_t st) {
  k_exp_cr<<<state_blocks(n), 256, 0, st>>>(d_x, d_y, n);
  chk(cudaGetLastError(), "kernel launch (exp_cr)");
}

// t_c -> scalars[0] (scalars: 2 doubles; partials: 4 kF64MeanBlocks doubles), H, F_0
void state_init_f64(const double* d_in, double* H, double* F, double* scalars, double* partials,
                    const Params& p, cudaStream_t st) {
  const long long n = (long long)p.width * p.height;
  launch_mean_f64(d_in, n, p.centering, p.tc_fixed, p.sigma_r, partials, kF64MeanBlocks, scalars, st);
  const double inv2s2 = 1.0 / (2.0 * p.sigma_r * p.sigma_r);
  k_f64_prologue<<<state_blocks(n), 256, 0, st>>>(d_in, scalars, H, F, n, p.sigma_r, inv2s2);
  chk(cudaGetLastError(), "kernel launch (GpfState::init)");
}

// apply_spatial (bilateral.cpp:58-62): src -> dst through tmp
void state_spatial_f64(const double* src, double* dst, double* tmp, const Params& p, cudaStream_t st) {
  if (p.backend == 0) {
    run_direct_gaussian_f64(src, dst, tmp, p.width, p.height, 1, p.sigma_s, p.kernel_scale,
                            p.window_radius, p.boundary, st);
  } else {
    const double mass = kernel_mass_1d(p.sigma_s, default_window_radius(p.sigma_s));
    run_gaussian_f64(src, dst, tmp, p.width, p.height, p.sigma_s, mass * mass * p.kernel_scale, st);
  }
}

void state_step_a_f64(double* Q, double* F, const double* G, const double* Fbar, const double* H,
                      double c, long long n, cudaStream_t st) {
  k_state_step_a<<<state_blocks(n), 256, 0, st>>>(Q, F, G, Fbar, H, c, n);
  chk(cudaGetLastError(), "kernel launch (GpfState::step)");
}

void state_step_b_f64(double* P, double* G, const double* Fbar, const double* H, double c, long long n,
                      cudaStream_t st) {
  k_state_step_b<<<state_blocks(n), 256, 0, st>>>(P, G, Fbar, H, c, n);
  chk(cudaGetLastError(), "kernel launch (GpfState::step)");
}

void state_finalize_f64(const double* in, const double* P, const double* Q, double* out, long long n,
                        double sigma_r, double t_c, unsigned long long* d_fb, cudaStream_t st) {
  chk(cudaMemsetAsync(d_fb, 0, sizeof(unsigned long long), st), "cudaMemsetAsync");
  k_state_finalize<<<state_blocks(n), 256, 0, st>>>(in, P, Q, out, n, sigma_r, t_c, d_fb);
  chk(cudaGetLastError(), "kernel launch (GpfState::finalize)");
}

size_t f64_workspace_bytes(int w, int h, int degree) {
  const size_t n = (size_t)w * h;
  return sizeof(double) * (n * (2 + 2 * (size_t)(degree + 2)) + 2 + 4 * kF64MeanBlocks +
                           f64_state_doubles(w, h, degree + 2));
}

// GPF_B200_F64_SEQUENTIAL=1 runs the literal sequential replay instead of the
// chunked form (same bits; kept as the cross-check of tests/test_gpu_dropin.py)
static bool f64_sequential() {
  const char* e = std::getenv("GPF_B200_F64_SEQUENTIAL");
  return e != nullptr && e[0] != '\0' && e[0] != '0';
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
  if (p.backend == 0) {
    // SpatialBackend::direct: the planes are materialised (into C), filtered
    // rows-then-columns by the windowed passes (C -> R -> C)
    direct_gen_planes_f64(H, F0, Cb, n, planes, st);
    run_direct_gaussian_f64(Cb, Cb, R, w, h, planes, p.sigma_s, p.kernel_scale, p.window_radius,
                            p.boundary, st);
  }
  Deriche64 k = {};
  if (p.backend != 0) deriche_coeffs_f64(p.sigma_s, k.nc, k.na, k.d);
  k.den = 1.0 + k.d[0] + k.d[1] + k.d[2] + k.d[3];
  k.csum = k.nc[0] + k.nc[1] + k.nc[2] + k.nc[3];
  k.asum = k.na[0] + k.na[1] + k.na[2] + k.na[3];
  const double mass = kernel_mass_1d(p.sigma_s, default_window_radius(p.sigma_s));
  const double scale = mass * mass * p.kernel_scale;
  if (p.backend == 0) {
    // filtered above
  } else if (f64_sequential()) {
    k_f64_rows<<<dim3((h + kRowT - 1) / kRowT, (planes + kGP - 1) / kGP), kRowT, 0, st>>>(H, F0, R, w, h,
                                                                                          planes, k);
    k_f64_cols<<<dim3((w + 127) / 128, planes), 128, 0, st>>>(R, Cb, w, h, k, scale);
  } else {
    double* S = partials + 4 * kF64MeanBlocks;  // recorded anticausal states (rows, then columns)
    const size_t smA = rows2_smem_bytes(planes) - sizeof(double) * (size_t)planes * kYP;
    const size_t smB = rows2_smem_bytes(planes);
    chk(cudaFuncSetAttribute(k_f64_rows_states, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smA),
        "cudaFuncSetAttribute");
    chk(cudaFuncSetAttribute(k_f64_rows_chunked, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smB),
        "cudaFuncSetAttribute");
    const int PG = (planes + kGP - 1) / kGP;
    const int thr = std::max(64, ((PG * kRB2 + 31) / 32) * 32);  // >= 64: kHR loads per thread cover a tile
    const int bands = (h + kRB2 - 1) / kRB2;
    if (w > kRowCh) k_f64_rows_states<<<bands, thr, smA, st>>>(H, F0, S, w, h, planes, k);
    k_f64_rows_chunked<<<bands, thr, smB, st>>>(H, F0, S, R, w, h, planes, k);
    const dim3 cg((w + kColT - 1) / kColT, planes);
    const size_t smCA = sizeof(double) * 2 * kF64Chunk * kColT, smCB = sizeof(ColTiles);
    chk(cudaFuncSetAttribute(k_f64_cols_states, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smCA),
        "cudaFuncSetAttribute");
    chk(cudaFuncSetAttribute(k_f64_cols_chunked, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smCB),
        "cudaFuncSetAttribute");
    if (h > kF64Chunk) k_f64_cols_states<<<cg, kColT, smCA, st>>>(R, S, w, h, k);
    k_f64_cols_chunked<<<cg, kColT, smCB, st>>>(R, S, Cb, w, h, k, scale);
  }
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
