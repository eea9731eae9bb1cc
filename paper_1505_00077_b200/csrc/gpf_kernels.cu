// sm_100a kernels of the Gauss-polynomial bilateral filter (GPF) hot path.
//
// Reference path (proj/src/core/bilateral.cpp:150-158, gpf()):
//   t_c = mean(f)                                  -> k_mean_partial/final (K0)
//   N+2 planes F_n = H^n exp(-h^2/2sr^2), each filtered by the separable
//   4th-order Deriche IIR (spatial.cpp:220-251):
//     per-pixel plane seeds (E 2^s0, H 2^-k)       -> k_seed        (K1a)
//     column carries from the seeds                -> k_col_carry_tma (K1b; k_col_carry_reg /
//                                                     k_col_carry for larger N)
//     column pass (fused plane generator)          -> k_colpass_tma (K2; k_colpass for N > 30)
//     row carries (scan of K2's strip aggregates)  -> k_row_scan    (K3)
//     row pass + P/Q recombination + normalise     -> k_rowpass2    (K4; k_rowpass for N > 22)
//   Q = sum c G Fbar_n, P = sum c G Fbar_{n+1}, out = sr P/Q + t_c,
//   |Q| <= 1e-8 -> input (bilateral.cpp:117-148)
//
// Threads own (line, plane pair). Both passes sweep their lines in chunks of
// kTile samples, each complex section in its output-aligned basis
// (FilterConsts, device_common.cuh): the causal recurrence
// runs on across chunks; the anticausal one restarts every chunk from an exact
// carry (the anticausal state at the chunk's far end), so a chunk's two
// directions combine in registers and every intermediate plane crosses HBM
// exactly once (written by K2, read by K4).
//
// HBM layouts (per frame):
//   V  [pairs][h_pad/16][w][16]   column-pass output, BAND-MAJOR float2: the
//                                 16 rows of one column within a 16-row band
//                                 are 128 B, and a band's columns follow each
//                                 other, so a 32-column strip of a band is 4 KB
//                                 contiguous for both the writer (K2) and the
//                                 reader (K4)
//   CA [ny][pairs][w]   2xfloat4  column anticausal carries (from f, K1)
//   AH [nx][pairs][h]   2xfloat4  per-strip row aggregates sum_i p^i V (K2)
//   CH [nx][pairs][h]   2xfloat4  row anticausal carries (K3)
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "device_common.cuh"
#include "gpf_internal.h"
#include "sync.cuh"

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

__device__ void block_minmax_reduce(double& mn, double& mx) {
  for (int o = 16; o; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  __shared__ double smn[kMeanThreads / 32], smx[kMeanThreads / 32];
  if ((threadIdx.x & 31) == 0) {
    smn[threadIdx.x >> 5] = mn;
    smx[threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  mn = smn[0];
  mx = smx[0];
  for (int k = 1; k < kMeanThreads / 32; ++k) {
    mn = fmin(mn, smn[k]);
    mx = fmax(mx, smx[k]);
  }
}

// Per block: (hi, lo) of the double-double sum, and the min / max of f (for
// the conditioning measure max|H| of the frame).
template <typename T>
__global__ void __launch_bounds__(kMeanThreads) k_mean_partial(const T* __restrict__ in,
                                                               long long n,
                                                               double* __restrict__ partials) {
  in += (size_t)blockIdx.y * n;
  partials += (size_t)blockIdx.y * gridDim.x * 4;
  double hi = 0.0, lo = 0.0;
  float mn = INFINITY, mx = -INFINITY;
  double mnd = INFINITY, mxd = -INFINITY;
  const long long stride = (long long)gridDim.x * kMeanThreads;
  long long i0 = 0;
  if (sizeof(T) == 4 && (reinterpret_cast<uintptr_t>(in) & 15) == 0) {
    // four pixels per 16-B load; two_sum keeps every add's rounding error
    const float4* in4 = reinterpret_cast<const float4*>(in);
    const long long n4 = n / 4;
    for (long long i = (long long)blockIdx.x * kMeanThreads + threadIdx.x; i < n4; i += stride) {
      const float4 v = __ldg(in4 + i);
      const double e4[4] = {v.x, v.y, v.z, v.w};
      mn = fminf(fminf(mn, v.x), fminf(fminf(v.y, v.z), v.w));
      mx = fmaxf(fmaxf(mx, v.x), fmaxf(fmaxf(v.y, v.z), v.w));
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        double s, e;
        two_sum(hi, e4[k], s, e);
        hi = s;
        lo += e;
      }
    }
    i0 = n4 * 4;
  }
  for (long long i = i0 + (long long)blockIdx.x * kMeanThreads + threadIdx.x; i < n; i += stride) {
    const double v = static_cast<double>(in[i]);
    double s, e;
    two_sum(hi, v, s, e);
    hi = s;
    lo += e;
    mnd = fmin(mnd, v);
    mxd = fmax(mxd, v);
  }
  mnd = fmin(mnd, (double)mn);
  mxd = fmax(mxd, (double)mx);
  block_dd_reduce(hi, lo);
  block_minmax_reduce(mnd, mxd);
  if (threadIdx.x == 0) {
    partials[4 * blockIdx.x] = hi;
    partials[4 * blockIdx.x + 1] = lo;
    partials[4 * blockIdx.x + 2] = mnd;
    partials[4 * blockIdx.x + 3] = mxd;
  }
}

// scalars[2 f] = t_c, scalars[2 f + 1] = max|H| = max(f_max - t_c, t_c - f_min) / sigma_r;
// ill[f] (optional) = 1 when max|H| lies outside the fp32 envelope.
__global__ void __launch_bounds__(kMeanThreads) k_mean_final(const double* __restrict__ partials,
                                                             int nblocks, long long n,
                                                             int centering, double tc_fixed,
                                                             double inv_sr, double h_limit,
                                                             double* __restrict__ scalars,
                                                             int* __restrict__ ill) {
  partials += (size_t)blockIdx.x * nblocks * 4;
  double hi = 0.0, lo = 0.0, mn = INFINITY, mx = -INFINITY;
  for (int b = threadIdx.x; b < nblocks; b += kMeanThreads) {
    dd_add(hi, lo, partials[4 * b], partials[4 * b + 1]);
    mn = fmin(mn, partials[4 * b + 2]);
    mx = fmax(mx, partials[4 * b + 3]);
  }
  block_dd_reduce(hi, lo);
  block_minmax_reduce(mn, mx);
  if (threadIdx.x == 0) {
    // centering 1: mean; 2: a fixed t_c (CenteringMode::midpoint, bilateral.cpp:77-82); 0: none
    const double t_c =
        centering == 1 ? (hi + lo) / static_cast<double>(n) : (centering == 2 ? tc_fixed : 0.0);
    const double hmax = fmax(mx - t_c, t_c - mn) * inv_sr;
    scalars[2 * blockIdx.x] = t_c;
    scalars[2 * blockIdx.x + 1] = hmax;
    if (ill) ill[blockIdx.x] = !(hmax <= h_limit);
  }
}

// ----------------------------------------------------------------------------
// cp.async helpers (LDGSTS): global -> shared without staging in registers.
// ----------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
template <int BYTES>
__device__ __forceinline__ void cp_async_zfill(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(s), "l"(gmem), "n"(BYTES),
               "r"(valid ? BYTES : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

// f tile: the 32x32 image block at (x0, y0) into ftile[32 rows][33], zero
// outside the image. Issued by the whole CTA; caller commits/waits.
template <typename Tin>
__device__ __forceinline__ void issue_f_tile(Tin* ftile, const Tin* __restrict__ in, int w, int h,
                                             int x0, int y0) {
  const int nthr = blockDim.x * blockDim.y;
  const int tid = threadIdx.y * 32 + threadIdx.x;
  for (int p = tid; p < 1024; p += nthr) {
    const int r = p >> 5, c = p & 31;
    const bool ok = (y0 + r < h) && (x0 + c < w);
    const Tin* src = ok ? in + (size_t)(y0 + r) * w + x0 + c : in;
    cp_async_zfill<sizeof(Tin)>(ftile + r * 33 + c, src, ok);
  }
}

// Producer: all planes of a 32x32 pixel block into buf[pair][col][33 rows]
// (float2 = planes 2g, 2g+1), computed once per pixel from the smem f tile
// and shared by the `pairs` warps. Plane chain in fp32:
//   x_0 = E 2^s0,  x_{n+1} = x_n * (H 2^-k)      (bilateral.cpp:97-101, 117-120)
// A thread takes up to three pixels (1024 / (32 pairs) <= 3 for N <= 20) and
// runs their chains interleaved, so the dependent multiplies overlap.
template <typename Tin>
__device__ __forceinline__ void produce_planes(float2* buf, const Tin* ftile, double t_c,
                                               const RangeConsts& rc, float2* em = nullptr,
                                               int em_pitch = 0, int em_rows = 0, int em_cols = 0) {
  const int nthr = blockDim.x * blockDim.y, pairs = blockDim.y;
  const int tid = threadIdx.y * 32 + threadIdx.x;
  for (int p0 = tid; p0 < 1024; p0 += 3 * nthr) {
    float x[3], m[3];
    float2* dst[3];
    bool ok[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int pk = p0 + k * nthr;
      ok[k] = pk < 1024;
      const int pp = ok[k] ? pk : p0;
      const int j = pp >> 5, c = pp & 31;
      const float tc_hi = static_cast<float>(t_c), tc_lo = static_cast<float>(t_c - tc_hi);
      const float2 t = pixel_terms_t<Tin>(ftile[j * 33 + c], t_c, tc_hi, tc_lo, rc);
      x[k] = t.x;
      m[k] = t.y;
      dst[k] = buf + c * 33 + j;
      // K1 hands the per-pixel seeds to the column pass (coalesced: lanes = columns)
      if (em && ok[k] && j < em_rows && c < em_cols) em[(size_t)j * em_pitch + c] = t;
    }
#pragma unroll 2
    for (int gg = 0; gg < pairs; ++gg) {
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const float x1 = x[k] * m[k];
        if (ok[k]) dst[k][gg * 32 * 33] = make_float2(x[k], x1);
        x[k] = x1 * m[k];
      }
    }
  }
}

// ----------------------------------------------------------------------------
// K1: exact anticausal carries of the column pass, computed from f.
// Thread (column x, pair g) walks its column bottom-up over row chunks:
//   carry(last)   = x[h-1] / (1-p)                       (replicate, spatial.cpp:204-206)
//   carry(c - 1)  = sum_{j<L_c} p^j x[y0_c + j] + p^{L_c} carry(c)
// where carry(c) is the anticausal state at the last row of chunk c.
// ----------------------------------------------------------------------------
template <int MAXT, typename Tin>
__global__ void __launch_bounds__(MAXT, 2) k_col_carry(const Tin* __restrict__ in_all,
                                                       const double* __restrict__ scalars,
                                                       float4* __restrict__ CA_all,
                                                       float2* __restrict__ EM_all, int w, int h,
                                                       int w_pad, int ny, FilterConsts fc,
                                                       TileConsts tc, RangeConsts rc) {
  extern __shared__ float4 smem4[];
  float2* buf = reinterpret_cast<float2*>(smem4);                               // [pairs][32][33]
  Tin* ftiles = reinterpret_cast<Tin*>(buf + (size_t)blockDim.y * 32 * 33);  // [2][32*33]
  const int f = blockIdx.y, lane = threadIdx.x, g = threadIdx.y, pairs = blockDim.y;
  const int x0 = blockIdx.x * 32, x = x0 + lane;
  const Tin* in = in_all + (size_t)f * w * h;
  float4* CA = CA_all + (size_t)f * ny * pairs * w * 2;
  const double t_c = scalars[2 * f];
  const float2* mine = buf + ((size_t)g * 32 + lane) * 33;
  PairState C;
  ps_zero(C);
  issue_f_tile(ftiles + ((ny - 1) & 1) * 32 * 33, in, w, h, x0, (ny - 1) * kTile);
  cp_async_commit();
  for (int cy = ny - 1; cy >= 0; --cy) {
    const int y0 = cy * kTile, rows = min(kTile, h - y0);
    cp_async_wait_all();
    __syncthreads();
    if (cy > 0) {
      issue_f_tile(ftiles + ((cy - 1) & 1) * 32 * 33, in, w, h, x0, y0 - kTile);
      cp_async_commit();
    }
    produce_planes(buf, ftiles + (cy & 1) * 32 * 33, t_c, rc,
                   EM_all + ((size_t)f * h + y0) * w_pad + x0, w_pad, rows, min(32, w - x0));
    __syncthreads();
    if (x < w) {
      if (cy == ny - 1) ps_set_gain(C, mine[rows - 1], fc);
      ps_store(CA + ((size_t)cy * pairs + g) * w * 2 + (size_t)x * 2, C);
      if (cy > 0) {
        PairState agg;
        ps_zero(agg);
        if (rows == kTile) {
#pragma unroll
          for (int j = 0; j < kTile; ++j)
            ps_accum(agg, mine[j], tc.w4[j]);
        } else {
          for (int j = 0; j < rows; ++j)
            ps_accum(agg, mine[j], tc.w4[j]);
        }
        if (cy == ny - 1) ps_chain(C, agg, tc.pYr2, tc.pYi2);
        else ps_chain(C, agg, tc.pTr2, tc.pTi2);
      }
    }
  }
}

// ----------------------------------------------------------------------------
// K2: column pass (deriche_line over columns, spatial.cpp:240-243), fused with
// the plane generator.
//
// k_colpass_tma (N <= 24): per 32x32 chunk the producer writes every plane
// straight into a staging tile laid out exactly as one TMA box of V --
// [pair][16-row half][column][16 rows x float2], 128B-swizzled -- so that
// lanes = 32 columns touch 16-B chunks conflict-free when a thread moves two
// rows at once. Each thread lifts its column's 32 inputs into registers, runs
// the anticausal sweep from the K1 carry and then the causal sweep (state
// carried across chunks), both in place in the stage; one elected thread
// then writes the whole chunk with a single tensor store. Two stages
// alternate, so the store of chunk k drains while chunk k+1 is produced and
// swept. The chunk is finally reduced into the row-pass strip aggregates AH.
//
// k_colpass (larger N, where two stages do not fit): same sweeps on a padded
// [pair][column][33] tile, written to V by the warps.
// ----------------------------------------------------------------------------
constexpr int kStageAlign = 1024;  // SWIZZLE_128B atoms repeat every 1024 B

// float2 element (column of base_col, row j) of a stage tile; cm = column % 8
__device__ __forceinline__ float* stage_at(float* base_col, int j, int cm) {
  return base_col + (j >> 4) * 1024 + ((((j & 15) >> 1) ^ cm) << 2) + (j & 1) * 2;
}

constexpr int kColGroup = 4;  // pairs per column-pass CTA / carry warp

// m2^pair0 for pair0 in {0, 4, 8, 12} (kColGroup = 4, pairs <= 16): straight-line
// squarings and warp-uniform selects (shared by the producer and the carries)
__device__ __forceinline__ float pow_group(float m2, int pair0) {
  const float m4 = m2 * m2, m8 = m4 * m4;
  float r = (pair0 & 4) ? m8 : 1.f;
  if (pair0 & 8) r *= m8 * m8;
  return r;
}

// Producer into a stage tile for the pair group starting at plane n0 = 2*pair0,
// from the per-pixel seeds (es, m) K1 left in HBM (em tile [32 rows][32]):
// item = (column, row pair), four items (eight pixels) per thread in one
// straight-line pass, so eight independent multiply chains are in flight.
// x_{n0} = es m^{n0} by squarings, then the chain runs over the group's planes.
// 8-B shared store kept as issued (the compiler would fuse two adjacent ones
// into a 16-B store that needs an aligned register quad, i.e. register moves)
__device__ __forceinline__ void sts64(float2* p, float2 v) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};\n" ::"r"(smem_u32(p)), "f"(v.x), "f"(v.y) : "memory");
}

#ifndef GPF_GSCALE
#define GPF_GSCALE 1  // G-scaled planes + joint Horner contraction (TileConsts::gstep); 0: per-plane weights
#endif
#ifndef GPF_L2HINT
#define GPF_L2HINT 0  // evict-first L2 policies: 1 V stores, 2 V loads, 4 EM loads (column pass), 8 row-pass f/out
#endif
#ifndef GPF_COL_STS64
#define GPF_COL_STS64 1
#endif
#ifndef GPF_PROD_PAIRCHAIN
#define GPF_PROD_PAIRCHAIN 1
#endif
template <bool GS = false>
__device__ __forceinline__ void produce_group(float* stage, const float2* emt, int pair0,
                                              int npairs, const TileConsts* tcp = nullptr) {
  constexpr int kIt = 4;  // 512 items = 4 x 128 threads (4-warp CTAs)
  const int tid = threadIdx.y * 32 + threadIdx.x;
#if GPF_PROD_PAIRCHAIN
  // Pair chain: an item's two pixels (rows j, j+1) keep their current plane
  // pair (F_{2g}, F_{2g+1}) as float2 and step to the next pair with one
  // packed multiply by the broadcast m^2 (the carry walk forms its planes the
  // same way, carry_base). The pairs go to the stage as two 8-B stores, which
  // leaves the multiplies' register pairs in place (a 16-B store of the two
  // pixels needs an aligned quad and costs register moves).
  float2 a[kIt], b[kIt];
  float m2[2 * kIt];
  float2* dst[kIt];
#pragma unroll
  for (int k = 0; k < kIt; ++k) {
    const int it = tid + k * 128;
    const int c = it & 31, j = (it >> 5) * 2;  // rows j, j+1
    const float2 ta = emt[j * 32 + c], tb = emt[(j + 1) * 32 + c];
    m2[2 * k] = ta.y * ta.y;
    m2[2 * k + 1] = tb.y * tb.y;
    float xa = ta.x, xb = tb.x;
    if (pair0 > 0) {
      xa *= pow_group(m2[2 * k], pair0);
      xb *= pow_group(m2[2 * k + 1], pair0);
    }
    if constexpr (GS) {  // G units: plane n carries 1/n! (K_n = prod_{i<n} w_i)
      const float pre = tcp->gpre[pair0], w0 = tcp->gw[pair0];
      xa *= pre;
      xb *= pre;
      a[k] = make_float2(xa, xa * (ta.y * w0));
      b[k] = make_float2(xb, xb * (tb.y * w0));
    } else {
      a[k] = make_float2(xa, xa * ta.y);
      b[k] = make_float2(xb, xb * tb.y);
    }
    dst[k] = reinterpret_cast<float2*>(stage_at(stage + c * 32, j, c & 7));
  }
  // every pair slot of the stage is written (a group's missing pairs hold
  // finite values no warp sweeps, and the TMA store clips them), so the
  // chain is branch-free
  (void)npairs;
#pragma unroll
  for (int gg = 0; gg < kColGroup; ++gg) {
#pragma unroll
    for (int k = 0; k < kIt; ++k) {
      sts64(dst[k] + gg * 1024, a[k]);
      sts64(dst[k] + gg * 1024 + 1, b[k]);
      if (gg + 1 < kColGroup) {
        if constexpr (GS) {  // (G_{2g+2}, G_{2g+3}) = (G_2g, G_2g+1) * m^2 * gstep[g]
          const float2 st2 = tcp->gstep[pair0 + gg];
          a[k] = mul2(a[k], mul2(f2(m2[2 * k]), st2));
          b[k] = mul2(b[k], mul2(f2(m2[2 * k + 1]), st2));
        } else {
          a[k] = mul2(a[k], f2(m2[2 * k]));
          b[k] = mul2(b[k], f2(m2[2 * k + 1]));
        }
      }
    }
  }
#else
  float x[2 * kIt], m[2 * kIt];
  float4* dst[kIt];
#pragma unroll
  for (int k = 0; k < kIt; ++k) {
    const int it = tid + k * 128;
    const int c = it & 31, j = (it >> 5) * 2;  // rows j, j+1
    const float2 ta = emt[j * 32 + c], tb = emt[(j + 1) * 32 + c];
    x[2 * k] = ta.x;
    m[2 * k] = ta.y;
    x[2 * k + 1] = tb.x;
    m[2 * k + 1] = tb.y;
    dst[k] = reinterpret_cast<float4*>(stage_at(stage + c * 32, j, c & 7));
  }
  if (pair0 > 0) {
#pragma unroll
    for (int e = 0; e < 2 * kIt; ++e) x[e] *= pow_group(m[e] * m[e], pair0);
  }
#pragma unroll
  for (int gg = 0; gg < kColGroup; ++gg) {
    if (gg < npairs) {
#pragma unroll
      for (int k = 0; k < kIt; ++k) {
        const float a1 = x[2 * k] * m[2 * k], b1 = x[2 * k + 1] * m[2 * k + 1];
        dst[k][gg * 512] = make_float4(x[2 * k], a1, x[2 * k + 1], b1);
        x[2 * k] = a1 * m[2 * k];
        x[2 * k + 1] = b1 * m[2 * k + 1];
      }
    }
  }
#endif
}

// One CTA = 32 columns x kColGroup pairs (pair group blockIdx.z); several
// CTAs share an SM so one's producer / H-dot phases overlap another's sweeps.

#ifndef GPF_COL_STAGES
#define GPF_COL_STAGES 1
#endif
#ifndef GPF_COL_CTAS
#define GPF_COL_CTAS 4
#endif
#ifndef GPF_COL_XREG
#define GPF_COL_XREG 0
#endif
// GPF_COL_XREG: the full-chunk sweep keeps its inputs in registers for the
// second half (no re-reads from the stage; needs ~166 registers, 3 CTAs/SM)
constexpr bool kColXreg = GPF_COL_XREG != 0;
constexpr int kColStages = GPF_COL_STAGES;  // staging tiles per CTA (1: store drains under the H-dots)
#ifndef GPF_COL_EMBUFS
#define GPF_COL_EMBUFS 2
#endif
constexpr int kColEmBufs = GPF_COL_EMBUFS;  // EM seed tiles in flight (2: loaded two chunks ahead)

template <bool AEV, bool GS>
__global__ void __launch_bounds__(32 * kColGroup, GPF_COL_CTAS) k_colpass_tma(
    const float4* __restrict__ CA_all, float4* __restrict__ AH_all, int w, int h, int ny, int nx,
    int pairs, int groups, FilterConsts fc, TileConsts tc,
    const __grid_constant__ CUtensorMap emmap, const __grid_constant__ CUtensorMap vstore
#ifdef GPF_DIAG_EXTRA_VW
    , const __grid_constant__ CUtensorMap vstore_x
#endif
#ifdef GPF_DIAG_V_ONCE  // diagnostic: V stored on a plan's first call only (valid while it keeps its frame)
    , int vst
#endif
    ) {
  extern __shared__ float4 smem4[];
  __shared__ uint64_t em_full[kColEmBufs];
  const int f = blockIdx.y, lane = threadIdx.x, gl = threadIdx.y;
  const int tid = gl * 32 + lane;
  // pair group fastest in the grid: a strip's groups run together and share
  // its EM tiles in L2
  const int strip = blockIdx.x / groups, grp = blockIdx.x - strip * groups;
  const int pair0 = grp * kColGroup, npairs = min(kColGroup, pairs - pair0);
  const int g = pair0 + gl;           // this warp's pair
  const bool active = gl < npairs;
  // smem: [2 stages x kColGroup x 8 KB, 1024-aligned][EM tile 8 KB]. The
  // alignment is an offset from the smem base (not integer arithmetic on the
  // pointer) so the compiler keeps the accesses in the shared window.
  float* stages = reinterpret_cast<float*>(reinterpret_cast<char*>(smem4) +
                                           ((kStageAlign - smem_u32(smem4)) & (kStageAlign - 1)));
  constexpr int kStageFloats = kColGroup * 2048;
  float2* emts = reinterpret_cast<float2*>(stages + kColStages * kStageFloats);  // [kColEmBufs][32][32]
  const int x0 = strip * 32, x = x0 + lane;
  const int cols = min(32, w - x0);
  // EM tile of the chunk starting at row y into buffer b (TMA, completion on em_full[b])
  auto load_em = [&](int b, int y) {
    mbar_arrive_expect_tx(&em_full[b], 32 * 32 * sizeof(float2));
#ifdef GPF_DIAG_EM_L2  // diagnostic: EM tiles from a 256x256-pixel (L2-resident) region
    tma_load_3d(emts + b * 1024, &emmap, 2 * (x0 & 255), y & 255, f, &em_full[b]);
#else
    tma_load_3d(emts + b * 1024, &emmap, 2 * x0, y, f, &em_full[b]);
#endif
  };
  const float4* CA = CA_all + (size_t)f * ny * pairs * w * 2;
  float4* AH = AH_all + (size_t)f * nx * pairs * h * 2;
  const int cm = lane & 7;
  const int col_off = (gl * 64 + lane) * 32;  // this thread's column, half 0
  // H-dots: thread (pair, row lane) reads column c at hd_off + c*32 + ((hq ^ (c%8)) << 2)
  const int hq = (lane & 15) >> 1;
  const int hd_off = (gl * 64 + (lane >> 4) * 32) * 32 + (lane & 1) * 2;
  if (tid == 0) {
    for (int b = 0; b < kColEmBufs; ++b) mbar_init(&em_full[b], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0) {  // the first kColEmBufs chunks' seeds
    for (int b = 0; b < kColEmBufs && b < ny; ++b) load_em(b, b * kTile);
  }
  PairState cs;  // causal state, carried across chunks
  ps_zero(cs);
  // anticausal carries, prefetched one chunk ahead
  const float4* ca_ptr = CA + (size_t)min(g, pairs - 1) * w * 2 + (size_t)min(x, w - 1) * 2;
  const size_t ca_stride = (size_t)pairs * w * 2;
  float4 ca0 = __ldg(ca_ptr), ca1 = __ldg(ca_ptr + 1);
#ifdef GPF_DIAG_CLOCKS
  long long tph[6] = {0, 0, 0, 0, 0, 0};  // barA, waitEM, produce, barB, sweep, barC+store+hdot
  long long tq = clock64();
#define GPF_TICK(i) { const long long tn = clock64(); tph[i] += tn - tq; tq = tn; }
#else
#define GPF_TICK(i)
#endif
  for (int cy = 0; cy < ny; ++cy) {
    const int y0 = cy * kTile, rows = min(kTile, h - y0);
    float* stage = stages + (kColStages == 2 ? (cy & 1) : 0) * kStageFloats;
    if (tid == 0 && cy >= kColStages) {  // the store of chunk cy-kColStages (same stage) has read it
      if constexpr (kColStages == 2) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
      else asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    }
    __syncthreads();
    GPF_TICK(0);
    const int eb = cy % kColEmBufs;
    mbar_wait(&em_full[eb], (cy / kColEmBufs) & 1);  // this chunk's seeds have landed
    GPF_TICK(1);
#ifndef GPF_DIAG_NO_PROD
    produce_group<GS>(stage, emts + eb * 1024, pair0, npairs, &tc);
#endif
    GPF_TICK(2);
    PairState as;
    if constexpr (GS) {  // the carry walk's states are in seed-chain units: scale to G units
      const float2 kc = tc.gcar[min(g, 15)];
      ps_from_carry(as, make_float4(ca0.x * kc.x, ca0.y * kc.y, ca0.z * kc.x, ca0.w * kc.y),
                    make_float4(ca1.x * kc.x, ca1.y * kc.y, ca1.z * kc.x, ca1.w * kc.y), fc);
    } else {
      ps_from_carry(as, ca0, ca1, fc);
    }
    if (cy + 1 < ny) {
      ca0 = __ldg(ca_ptr + (size_t)(cy + 1) * ca_stride);
      ca1 = __ldg(ca_ptr + (size_t)(cy + 1) * ca_stride + 1);
    }
    __syncthreads();
    GPF_TICK(3);
    if (tid == 0 && cy + kColEmBufs < ny)  // EM buffer eb is free again: fetch chunk cy + kColEmBufs
      load_em(eb, y0 + kColEmBufs * kTile);
    float* mcol = stage + col_off;
    if (active && x < w && rows == kTile) {
      // full chunk: both directions in one branch-free loop (two independent
      // recurrences per step), two rows per smem access. Step t runs the
      // anticausal sections at rows 31-t, 30-t and the causal ones at rows
      // t, t+1. First-half outputs park in registers (pa: anticausal rows
      // 16..31, pc: causal rows 0..15) and the inputs stay in the stage, so
      // the second half re-reads its inputs there and writes each final
      // output once, in place.
      if (cy == 0) {
        const float4 v0 = *reinterpret_cast<const float4*>(stage_at(mcol, 0, cm));
        ps_set_gain_sweep(cs, make_float2(v0.x, v0.y), fc);
      }
      float2 pa[kTile / 2], pc[kTile / 2];
      [[maybe_unused]] float4 xa[kColXreg ? kTile / 4 : 1], xc[kColXreg ? kTile / 4 : 1];  // inputs kept for the second half
#pragma unroll
      for (int t = 0; t < kTile / 2; t += 2) {
        const float4 va = *reinterpret_cast<const float4*>(stage_at(mcol, 30 - t, cm));
        const float4 vc = *reinterpret_cast<const float4*>(stage_at(mcol, t, cm));
        if constexpr (kColXreg) {
          xa[t / 2] = va;  // rows 30-t, 31-t
          xc[t / 2] = vc;  // rows t, t+1
        }
        pa[15 - t] = ps_emit_a<AEV>(as, fc);  // row 31-t
        ps_advance_a(as, make_float2(va.z, va.w), fc);
        ps_advance_c(cs, make_float2(vc.x, vc.y), fc);
        pc[t] = ps_emit_c(cs, fc);  // row t
        pa[14 - t] = ps_emit_a<AEV>(as, fc);  // row 30-t
        ps_advance_a(as, make_float2(va.x, va.y), fc);
        ps_advance_c(cs, make_float2(vc.z, vc.w), fc);
        pc[t + 1] = ps_emit_c(cs, fc);  // row t+1
      }
      // second half: anticausal rows 15-u, 14-u; causal rows 16+u, 17+u; the
      // next step's inputs are read before this step's outputs are stored
      float4 va, vc;
      if constexpr (kColXreg) {
        va = xc[7];
        vc = xa[7];
      } else {
        va = *reinterpret_cast<const float4*>(stage_at(mcol, 14, cm));
        vc = *reinterpret_cast<const float4*>(stage_at(mcol, 16, cm));
      }
#pragma unroll
      for (int u = 0; u < kTile / 2; u += 2) {
        float4 na = va, nc = vc;
        if (u + 2 < kTile / 2) {
          if constexpr (kColXreg) {
            na = xc[(12 - u) / 2];  // rows 12-u, 13-u
            nc = xa[(12 - u) / 2];  // rows 18+u, 19+u
          } else {
            na = *reinterpret_cast<const float4*>(stage_at(mcol, 12 - u, cm));
            nc = *reinterpret_cast<const float4*>(stage_at(mcol, 18 + u, cm));
          }
        }
        const float2 yb = ps_emit_a_acc<AEV>(as, fc, pc[15 - u]);
        ps_advance_a(as, make_float2(va.z, va.w), fc);
        ps_advance_c(cs, make_float2(vc.x, vc.y), fc);
        const float2 yc0 = ps_emit_c_acc(cs, fc, pa[u]);
        const float2 ya = ps_emit_a_acc<AEV>(as, fc, pc[14 - u]);
        ps_advance_a(as, make_float2(va.x, va.y), fc);
        ps_advance_c(cs, make_float2(vc.z, vc.w), fc);
        const float2 yc1 = ps_emit_c_acc(cs, fc, pa[u + 1]);
#if GPF_COL_STS64
        {  // 8-B stores (fused back into 16-B ones by ptxas, without register moves)
          float2* pa2 = reinterpret_cast<float2*>(stage_at(mcol, 14 - u, cm));
          float2* pc2 = reinterpret_cast<float2*>(stage_at(mcol, 16 + u, cm));
          sts64(pa2, ya);
          sts64(pa2 + 1, yb);
          sts64(pc2, yc0);
          sts64(pc2 + 1, yc1);
        }
#else
        *reinterpret_cast<float4*>(stage_at(mcol, 14 - u, cm)) = make_float4(ya.x, ya.y, yb.x, yb.y);
        *reinterpret_cast<float4*>(stage_at(mcol, 16 + u, cm)) = make_float4(yc0.x, yc0.y, yc1.x, yc1.y);
#endif
        va = na;
        vc = nc;
      }
    } else if (active && x < w) {
      float2 xr[kTile];
#pragma unroll
      for (int j = 0; j < kTile; j += 2) {
        const float4 v = *reinterpret_cast<const float4*>(stage_at(mcol, j, cm));
        xr[j] = make_float2(v.x, v.y);
        xr[j + 1] = make_float2(v.z, v.w);
      }
      if (cy == 0) ps_set_gain_sweep(cs, xr[0], fc);
      {
#pragma unroll
        for (int j = kTile - 1; j >= 0; --j) {
          if (j < rows) {
            *reinterpret_cast<float2*>(stage_at(mcol, j, cm)) = ps_emit_a<AEV>(as, fc);
            ps_advance_a(as, xr[j], fc);
          }
        }
#pragma unroll
        for (int j = 0; j < kTile; ++j) {
          if (j < rows) {
            float2* p = reinterpret_cast<float2*>(stage_at(mcol, j, cm));
            ps_advance_c(cs, xr[j], fc);
            *p = add2(ps_emit_c(cs, fc), *p);
          }
        }
      }
    }
    GPF_TICK(4);
    fence_proxy_async();  // stage writes -> visible to the TMA store
    __syncthreads();
#ifndef GPF_DIAG_NO_STORE
#ifdef GPF_DIAG_V_ONCE
    if (tid == 0 && vst) {
#else
    if (tid == 0) {
#endif
      // pairs past the last one fall outside the tensor and are clipped
      if constexpr (GPF_L2HINT & 1) tma_store_5d_hint(&vstore, 0, x0, y0 >> 4, pair0, f, stage, l2_evict_first());
      else tma_store_5d(&vstore, 0, x0, y0 >> 4, pair0, f, stage);
#ifdef GPF_DIAG_EXTRA_VW  // diagnostic: the chunk is stored a second time, to a scratch copy of V
      tma_store_5d(&vstore_x, 0, x0, y0 >> 4, pair0, f, stage);
#endif
      bulk_commit();
    }
#endif
    // strip aggregates for the row pass: thread (pair, row lane)
#ifdef GPF_DIAG_NO_HDOT
    if (lane < 0) {
#else
    if (active && lane < rows) {
#endif
      PairState agg;
      ps_zero(agg);
      const float* sb = stage + hd_off;
      if (cols == 32) {
#pragma unroll
        for (int c = 0; c < 32; ++c)
          ps_accum(agg, *reinterpret_cast<const float2*>(sb + c * 32 + ((hq ^ (c & 7)) << 2)), tc.w4[c]);
      } else {
        for (int c = 0; c < cols; ++c)
          ps_accum(agg, *reinterpret_cast<const float2*>(sb + c * 32 + ((hq ^ (c & 7)) << 2)), tc.w4[c]);
      }
      ps_store(AH + ((size_t)strip * pairs + g) * h * 2 + (size_t)(y0 + lane) * 2, agg);
    }
    GPF_TICK(5);
  }
#ifdef GPF_DIAG_CLOCKS
  if ((blockIdx.x == 300 || blockIdx.x == 301) && (tid == 0 || tid == 96))
    printf("colpass cta %d tid %d: barA %lld waitEM %lld produce %lld barB %lld sweep %lld rest %lld (per chunk)\n",
           blockIdx.x, tid, tph[0] / ny, tph[1] / ny, tph[2] / ny, tph[3] / ny, tph[4] / ny, tph[5] / ny);
#endif
#undef GPF_TICK
  if (tid == 0) bulk_wait_all();  // V complete before the CTA retires
}

// ----------------------------------------------------------------------------
// K1a: per-pixel plane seeds EM = (E 2^s0, H 2^-k) (pixel_terms), written once
// per frame and read by the grouped carry and column passes via TMA.
// ----------------------------------------------------------------------------
template <typename Tin>
__global__ void __launch_bounds__(256) k_seed(const Tin* __restrict__ in_all,
                                              const double* __restrict__ scalars,
                                              float2* __restrict__ EM_all, int w, int h, int w_pad,
                                              RangeConsts rc) {
  // four pixels per thread: one 16-B load of f (fp32, w % 4 == 0), two 16-B stores
  const int f = blockIdx.z, x = (blockIdx.x * 256 + threadIdx.x) * 4;
  if (x >= w) return;
  const Tin* in = in_all + (size_t)f * w * h;
  float2* EM = EM_all + (size_t)f * h * w_pad;
  const double t_c = scalars[2 * f];
  const float tc_hi = static_cast<float>(t_c), tc_lo = static_cast<float>(t_c - tc_hi);
  // 16-B loads need a 16-B aligned frame base (a torch view may start at any float)
  const bool vec = sizeof(Tin) == 4 && (w & 3) == 0 && x + 4 <= w &&
                   (reinterpret_cast<uintptr_t>(in_all) & 15) == 0;
  for (int y = blockIdx.y; y < h; y += gridDim.y) {
    const Tin* src = in + (size_t)y * w + x;
    float2* dst = EM + (size_t)y * w_pad + x;
    if (vec) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(src));
#if defined(GPF_DIAG_SEED_COPY)  // diagnostic: the seed traffic without its arithmetic (wrong output)
      const float2 a = make_float2(v.x, v.x), b = make_float2(v.y, v.y);
      const float2 c = make_float2(v.z, v.z), d = make_float2(v.w, v.w);
#else
      const float2 a = pixel_terms_t<float>(v.x, t_c, tc_hi, tc_lo, rc);
      const float2 b = pixel_terms_t<float>(v.y, t_c, tc_hi, tc_lo, rc);
      const float2 c = pixel_terms_t<float>(v.z, t_c, tc_hi, tc_lo, rc);
      const float2 d = pixel_terms_t<float>(v.w, t_c, tc_hi, tc_lo, rc);
#endif
#if defined(GPF_DIAG_SEED_NOSTORE)  // diagnostic: the arithmetic without the EM stores (stale seeds)
      if (a.x == -1.f && b.x == -1.f && c.x == -1.f && d.x == -1.f)
#endif
      {
#ifdef GPF_SEED_STCS  // streaming stores (evict-first)
        __stcs(reinterpret_cast<float4*>(dst), make_float4(a.x, a.y, b.x, b.y));
        __stcs(reinterpret_cast<float4*>(dst) + 1, make_float4(c.x, c.y, d.x, d.y));
#else
        reinterpret_cast<float4*>(dst)[0] = make_float4(a.x, a.y, b.x, b.y);
        reinterpret_cast<float4*>(dst)[1] = make_float4(c.x, c.y, d.x, d.y);
#endif
      }
    } else {
      for (int k = 0; k < 4 && x + k < w; ++k) dst[k] = pixel_terms_t<Tin>(src[k], t_c, tc_hi, tc_lo, rc);
    }
  }
}

// ----------------------------------------------------------------------------
// K1b (registers only): chunk carries of the anticausal column recurrences.
// One warp = 16 columns x one group of kColGroup pairs (blockIdx.x = strip16 *
// groups + group); half-warp h owns pairs 2h, 2h + 1 of the group, so the row
// weights stay warp-uniform and no lane exchange is needed. Each lane walks its column
// bottom-up: it forms its group's planes from the per-pixel seeds (E 2^s0,
// H 2^-k) -- plane 2 pair0 by squarings, then packed multiplies -- and folds
// the chunk into the four-state dot products of every pair. No shared memory
// and no barriers; the seeds of the next chunk are in flight while the
// current one is folded. (Measured against the shared-memory tile kernel it
// replaces: 0.56 vs 0.62 ms per 8192^2 frame; thinner lanes -- one pair per
// lane, 8 columns per warp -- or 4-/8-way row splits with shuffle reductions
// are slower.)
// ----------------------------------------------------------------------------

__global__ void __launch_bounds__(32) k_col_carry_reg(const float2* __restrict__ EM_all,
                                                      float4* __restrict__ CA_all, int w, int h,
                                                      int w_pad, int ny, int pairs, int groups,
                                                      FilterConsts fc, TileConsts tc) {
  constexpr int kLanePairs = kColGroup / 2;  // pairs per lane
  const int lane = threadIdx.x, f = blockIdx.y;
  const int half = lane >> 4;  // pairs [pair0 + 2 half, pair0 + 2 half + 2)
  const int strip = blockIdx.x / groups, grp = blockIdx.x - strip * groups;
  const int pair0 = grp * kColGroup + half * kLanePairs;
  const int npairs = min(kLanePairs, pairs - pair0);
  const int x = strip * 16 + (lane & 15), xc = min(x, w - 1);
  const float2* src = EM_all + (size_t)f * h * w_pad + xc;
  float4* CA = CA_all + (size_t)f * ny * pairs * w * 2 + (size_t)x * 2;
  const size_t pair_stride = (size_t)w * 2, chunk_stride = (size_t)pairs * w * 2;
  static_assert(kColGroup == 4, "k_col_carry_reg: two pairs per lane, two lane halves");
  // plane pair (2 pair0, 2 pair0 + 1) of a seed: E m^{2 pair0} (m^2 squarings,
  // the half's extra m^4 by a select)
  auto base = [&](float2 s, float& m2) {
    m2 = s.y * s.y;
    const float m4 = m2 * m2;
    const float xb = s.x * pow_group(m2, grp * kColGroup) * (half ? m4 : 1.f);
    return make_float2(xb, xb * s.y);
  };
  PairState C[kLanePairs];
  {  // replicate boundary: steady state of the bottom row
    float m2;
    const float2 p0 = base(__ldg(src + (size_t)(h - 1) * w_pad), m2);
    ps_set_gain(C[0], p0, fc);
    ps_set_gain(C[1], mul2(p0, f2(m2)), fc);
  }
  float2 sd[kTile];
  {
    const int y0 = (ny - 1) * kTile, rows = h - y0;
#pragma unroll
    for (int j = 0; j < kTile; ++j)
      sd[j] = j < rows ? __ldg(src + (size_t)(y0 + j) * w_pad) : make_float2(0.f, 0.f);
  }
  for (int cy = ny - 1; cy >= 0; --cy) {
    if (x < w) {
#pragma unroll
      for (int gg = 0; gg < kLanePairs; ++gg)
        if (gg < npairs) ps_store(CA + cy * chunk_stride + (pair0 + gg) * pair_stride, C[gg]);
    }
    if (cy == 0) break;
    PairState agg[kLanePairs];
#pragma unroll
    for (int gg = 0; gg < kLanePairs; ++gg) ps_zero(agg[gg]);
    const float2* nxt = src + (size_t)(cy - 1) * kTile * w_pad;  // chunk cy-1 (full)
    // rows past the image (first, partial chunk) hold zero seeds: all their
    // planes vanish, so the loop is branch-free and rows interleave; pairs past
    // the last one are folded too but never stored
#pragma unroll
    for (int j = 0; j < kTile; ++j) {
      const float2 s = sd[j];
      sd[j] = __ldg(nxt + (size_t)j * w_pad);
      float m2;
      const float2 p0 = base(s, m2);
      ps_accum(agg[0], p0, tc.w4[j]);
      ps_accum(agg[1], mul2(p0, f2(m2)), tc.w4[j]);
    }
    const bool last = cy == ny - 1;
#pragma unroll
    for (int gg = 0; gg < kLanePairs; ++gg)
      ps_chain(C[gg], agg[gg], last ? tc.pYr2 : tc.pTr2, last ? tc.pYi2 : tc.pTi2);
  }
}

// K1b (TMA ring): the same carries, with each 32-row seed tile of a 64-column
// strip brought into shared memory by TMA, kCarrySlots chunks ahead, instead
// of a register prefetch of one chunk. CTA = 4 warps; warp wi takes columns
// 16 wi .. 16 wi + 15 of the strip with the lane mapping of k_col_carry_reg
// (half-warp = two pairs of the pair group). No register-resident seeds, so
// four CTAs fit an SM, and HBM latency is covered by the ring depth.
#ifndef GPF_CARRY_SLOTS
#define GPF_CARRY_SLOTS 2
#endif
constexpr int kCarrySlots = GPF_CARRY_SLOTS;
#ifndef GPF_CARRY_COLS
#define GPF_CARRY_COLS 64
#endif
#ifndef GPF_CARRY_LP
#define GPF_CARRY_LP 2
#endif
constexpr int kCarryLP = GPF_CARRY_LP;       // pairs per lane (2 or 4)
constexpr int kCarryCols = GPF_CARRY_COLS;  // columns per CTA
constexpr int kCarryWarps = kCarryCols / (8 * kCarryLP);

template <int GRP>
__device__ __forceinline__ float2 carry_base(float2 s, int half, float& m2) {
  // planes (2 pair0, 2 pair0 + 1) of a seed, pair0 = 4 GRP + 2 half:
  // E m^{8 GRP + 4 half} by squarings (GRP warp-uniform, half per lane)
  m2 = s.y * s.y;
  const float m4 = m2 * m2;
  float xb = s.x;
  if constexpr (GRP >= 1) {
    const float m8 = m4 * m4;
    xb *= (GRP == 2 ? m8 * m8 : m8);
  }
  xb *= half ? m4 : 1.f;
  return make_float2(xb, xb * s.y);
}

#ifndef GPF_CARRY_RS
#define GPF_CARRY_RS 0
#endif
// Row-split lanes (GPF_CARRY_RS, kCarryLP == 2 geometry: 16 columns per warp):
// lane = (column lane & 15, row half lane >> 4), every lane folds all four
// pairs of the group over its 16 rows of the chunk -- one power chain per
// seed and group instead of one per seed and half-warp -- and the two halves'
// partial dot products are summed with one shuffle per state word (the
// weights p^j already carry each row's absolute position in the chunk).
template <int GRP>
__device__ __forceinline__ void carry_walk_rs(float2* tiles, uint64_t* full, float4* CA,
                                              const CUtensorMap* emcmap, int w, int h, int ny,
                                              int pairs, int x0, int f, const FilterConsts& fc,
                                              const TileConsts& tc) {
  constexpr int kLanePairs = kColGroup;
  const int lane = threadIdx.x, wi = threadIdx.y, tid = wi * 32 + lane;
  const int rh = lane >> 4;
  const int col = wi * 16 + (lane & 15), x = x0 + col;
  const int pair0 = GRP * kColGroup;
  const int npairs = min(kLanePairs, pairs - pair0);
  const size_t pair_stride = (size_t)w * 2, chunk_stride = (size_t)pairs * w * 2;
  float4* ca = CA + (size_t)x * 2;
  PairState C[kLanePairs];
  for (int k = 0; k < ny; ++k) {
    const int cy = ny - 1 - k, s = k % kCarrySlots;
    const float2* tile = tiles + (size_t)s * 32 * kCarryCols + col;  // [32 rows][kCarryCols columns]
    mbar_wait(&full[s], (k / kCarrySlots) & 1);
    if (k == 0) {  // replicate boundary: steady state of the bottom row
      float m2;
      float2 pl = carry_base<GRP>(tile[(h - 1 - cy * kTile) * kCarryCols], 0, m2);
#pragma unroll
      for (int gg = 0; gg < kLanePairs; ++gg) {
        ps_set_gain(C[gg], pl, fc);
        pl = mul2(pl, f2(m2));
      }
    }
    if (x < w) {  // half 0 stores pairs 0, 1 and half 1 pairs 2, 3 (both hold every C)
#pragma unroll
      for (int gg = 0; gg < kLanePairs; ++gg)
        if ((gg >> 1) == rh && gg < npairs) ps_store(ca + cy * chunk_stride + (pair0 + gg) * pair_stride, C[gg]);
    }
    if (cy == 0) break;
    PairState agg[kLanePairs];
#pragma unroll
    for (int gg = 0; gg < kLanePairs; ++gg) ps_zero(agg[gg]);
    // rows past the image (last, partial chunk) read as zero seeds (TMA fill)
#pragma unroll
    for (int jj = 0; jj < kTile / 2; ++jj) {
      const int j = rh * (kTile / 2) + jj;
      float m2;
      float2 pl = carry_base<GRP>(tile[j * kCarryCols], 0, m2);
      const float4 wj = tc.w4[j];
#pragma unroll
      for (int gg = 0; gg < kLanePairs; ++gg) {
        ps_accum(agg[gg], pl, wj);
        if (gg + 1 < kLanePairs) pl = mul2(pl, f2(m2));
      }
    }
#pragma unroll
    for (int gg = 0; gg < kLanePairs; ++gg) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        agg[gg].wr[q].x += __shfl_xor_sync(0xffffffffu, agg[gg].wr[q].x, 16);
        agg[gg].wr[q].y += __shfl_xor_sync(0xffffffffu, agg[gg].wr[q].y, 16);
        agg[gg].wi[q].x += __shfl_xor_sync(0xffffffffu, agg[gg].wi[q].x, 16);
        agg[gg].wi[q].y += __shfl_xor_sync(0xffffffffu, agg[gg].wi[q].y, 16);
      }
    }
    const bool last = k == 0;
#pragma unroll
    for (int gg = 0; gg < kLanePairs; ++gg)
      ps_chain(C[gg], agg[gg], last ? tc.pYr2 : tc.pTr2, last ? tc.pYi2 : tc.pTi2);
    __syncthreads();  // every warp is done with slot s
    if (tid == 0 && k + kCarrySlots < ny) {
      mbar_arrive_expect_tx(&full[s], 32 * kCarryCols * sizeof(float2));
#ifdef GPF_DIAG_EMC_L2
      tma_load_3d(tiles + (size_t)s * 32 * kCarryCols, emcmap, 2 * (x0 & 255), ((cy - kCarrySlots) * kTile) & 255, f,
#else
      tma_load_3d(tiles + (size_t)s * 32 * kCarryCols, emcmap, 2 * x0, (cy - kCarrySlots) * kTile, f,
#endif
                  &full[s]);
    }
  }
}

template <int GRP>
__device__ __forceinline__ void carry_walk(float2* tiles, uint64_t* full,
                                           float4* CA, const CUtensorMap* emcmap, int w, int h,
                                           int ny, int pairs, int x0, int f, const FilterConsts& fc,
                                           const TileConsts& tc) {
  if constexpr (GPF_CARRY_RS && kCarryLP == 2) {
    carry_walk_rs<GRP>(tiles, full, CA, emcmap, w, h, ny, pairs, x0, f, fc, tc);
    return;
  }
  // kCarryLP pairs per lane: 2 (half-warp per two pairs, 16 columns per warp)
  // or 4 (the whole group, 32 columns per warp: one power chain per seed)
  constexpr int kLanePairs = kCarryLP;
  constexpr int kWarpCols = 8 * kCarryLP;  // 16 or 32
  const int lane = threadIdx.x, wi = threadIdx.y, tid = wi * 32 + lane;
  const int half = kCarryLP == 2 ? lane >> 4 : 0;
  const int col = wi * kWarpCols + (lane & (kWarpCols - 1)), x = x0 + col;
  const int pair0 = GRP * kColGroup + half * kLanePairs;
  const int npairs = min(kLanePairs, pairs - pair0);
  const size_t pair_stride = (size_t)w * 2, chunk_stride = (size_t)pairs * w * 2;
  float4* ca = CA + (size_t)x * 2;
  PairState C[kLanePairs];
  for (int k = 0; k < ny; ++k) {
    const int cy = ny - 1 - k, s = k % kCarrySlots;
    const float2* tile = tiles + (size_t)s * 32 * kCarryCols + col;  // [32 rows][kCarryCols columns]
    mbar_wait(&full[s], (k / kCarrySlots) & 1);
    if (k == 0) {  // replicate boundary: steady state of the bottom row
      float m2;
      float2 pl = carry_base<GRP>(tile[(h - 1 - cy * kTile) * kCarryCols], half, m2);
#pragma unroll
      for (int gg = 0; gg < kLanePairs; ++gg) {
        ps_set_gain(C[gg], pl, fc);
        pl = mul2(pl, f2(m2));
      }
    }
    if (x < w) {
#pragma unroll
      for (int gg = 0; gg < kLanePairs; ++gg)
        if (gg < npairs) ps_store(ca + cy * chunk_stride + (pair0 + gg) * pair_stride, C[gg]);
    }
    if (cy == 0) break;
    PairState agg[kLanePairs];
#pragma unroll
    for (int gg = 0; gg < kLanePairs; ++gg) ps_zero(agg[gg]);
    // rows past the image (last, partial chunk) read as zero seeds (TMA fill):
    // their planes vanish, so the loop is branch-free
#pragma unroll
    for (int j = 0; j < kTile; ++j) {
      float m2;
      float2 pl = carry_base<GRP>(tile[j * kCarryCols], half, m2);
#pragma unroll
      for (int gg = 0; gg < kLanePairs; ++gg) {
        ps_accum(agg[gg], pl, tc.w4[j]);
        if (gg + 1 < kLanePairs) pl = mul2(pl, f2(m2));
      }
    }
    const bool last = k == 0;
#pragma unroll
    for (int gg = 0; gg < kLanePairs; ++gg)
      ps_chain(C[gg], agg[gg], last ? tc.pYr2 : tc.pTr2, last ? tc.pYi2 : tc.pTi2);
    __syncthreads();  // every warp is done with slot s
    if (tid == 0 && k + kCarrySlots < ny) {
      mbar_arrive_expect_tx(&full[s], 32 * kCarryCols * sizeof(float2));
#ifdef GPF_DIAG_EMC_L2
      tma_load_3d(tiles + (size_t)s * 32 * kCarryCols, emcmap, 2 * (x0 & 255), ((cy - kCarrySlots) * kTile) & 255, f,
#else
      tma_load_3d(tiles + (size_t)s * 32 * kCarryCols, emcmap, 2 * x0, (cy - kCarrySlots) * kTile, f,
#endif
                  &full[s]);
    }
  }
}

__global__ void __launch_bounds__(32 * kCarryWarps, (GPF_CARRY_SLOTS == 2 ? (GPF_CARRY_RS ? 5 : 6) : 4) * (4 / kCarryWarps)) k_col_carry_tma(float4* __restrict__ CA_all, int w, int h,
                                                          int ny, int pairs, int groups,
                                                          FilterConsts fc, TileConsts tc,
                                                          const __grid_constant__ CUtensorMap emcmap) {
  extern __shared__ float4 smem4[];
  __shared__ uint64_t full[kCarrySlots];
  // [kCarrySlots][32][64] float2, 128-B aligned for TMA (offset from the smem base)
  float2* tiles = reinterpret_cast<float2*>(reinterpret_cast<char*>(smem4) +
                                            ((128u - smem_u32(smem4)) & 127u));
  const int f = blockIdx.y, tid = threadIdx.y * 32 + threadIdx.x;
  const int strip = blockIdx.x / groups, grp = blockIdx.x - strip * groups;
  const int x0 = strip * kCarryCols;
  if (tid == 0) {
    for (int s = 0; s < kCarrySlots; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (tid == 0) {
    for (int k = 0; k < kCarrySlots && k < ny; ++k) {
      mbar_arrive_expect_tx(&full[k], 32 * kCarryCols * sizeof(float2));
      tma_load_3d(tiles + (size_t)k * 32 * kCarryCols, &emcmap, 2 * x0, (ny - 1 - k) * kTile, f, &full[k]);
    }
  }
  float4* CA = CA_all + (size_t)f * ny * pairs * w * 2;
  if (grp == 0) carry_walk<0>(tiles, full, CA, &emcmap, w, h, ny, pairs, x0, f, fc, tc);
  else if (grp == 1) carry_walk<1>(tiles, full, CA, &emcmap, w, h, ny, pairs, x0, f, fc, tc);
  else carry_walk<2>(tiles, full, CA, &emcmap, w, h, ny, pairs, x0, f, fc, tc);
}

template <int MAXT, typename Tin>
__global__ void __launch_bounds__(MAXT, 1) k_colpass(const Tin* __restrict__ in_all,
                                                     const double* __restrict__ scalars,
                                                     const float4* __restrict__ CA_all,
                                                     float2* __restrict__ V_all,
                                                     float4* __restrict__ AH_all, int w, int h,
                                                     int h_pad, int ny, int nx, FilterConsts fc,
                                                     TileConsts tc, RangeConsts rc) {
  extern __shared__ float4 smem4[];
  float2* buf = reinterpret_cast<float2*>(smem4);                               // [pairs][32][33]
  Tin* ftiles = reinterpret_cast<Tin*>(buf + (size_t)blockDim.y * 32 * 33);  // [2][32*33]
  const int f = blockIdx.y, lane = threadIdx.x, g = threadIdx.y, pairs = blockDim.y;
  const int strip = blockIdx.x, x0 = strip * 32, x = x0 + lane;
  const int cols = min(32, w - x0);
  const Tin* in = in_all + (size_t)f * w * h;
  const float4* CA = CA_all + (size_t)f * ny * pairs * w * 2;
  float2* V = V_all + (size_t)f * pairs * w * h_pad;
  float4* AH = AH_all + (size_t)f * nx * pairs * h * 2;
  const double t_c = scalars[2 * f];
  float2* mine = buf + ((size_t)g * 32 + lane) * 33;
  PairState cs;  // causal state, carried across chunks
  ps_zero(cs);
  issue_f_tile(ftiles, in, w, h, x0, 0);
  cp_async_commit();
  const float4* ca_ptr = CA + (size_t)g * w * 2 + (size_t)min(x, w - 1) * 2;
  const size_t ca_stride = (size_t)pairs * w * 2;
  float4 ca0 = __ldg(ca_ptr), ca1 = __ldg(ca_ptr + 1);
  for (int cy = 0; cy < ny; ++cy) {
    const int y0 = cy * kTile, rows = min(kTile, h - y0);
    cp_async_wait_all();
    __syncthreads();
    if (cy + 1 < ny) {
      issue_f_tile(ftiles + ((cy + 1) & 1) * 32 * 33, in, w, h, x0, y0 + kTile);
      cp_async_commit();
    }
    produce_planes(buf, ftiles + (cy & 1) * 32 * 33, t_c, rc);
    PairState as;
    ps_from_carry(as, ca0, ca1, fc);
    if (cy + 1 < ny) {
      ca0 = __ldg(ca_ptr + (size_t)(cy + 1) * ca_stride);
      ca1 = __ldg(ca_ptr + (size_t)(cy + 1) * ca_stride + 1);
    }
    __syncthreads();
    if (x < w) {
      float2 xr[kTile];
#pragma unroll
      for (int j = 0; j < kTile; ++j) xr[j] = mine[j];
      if (cy == 0) ps_set_gain_sweep(cs, xr[0], fc);
#pragma unroll
      for (int j = kTile - 1; j >= 0; --j) {
        if (j < rows) {
          mine[j] = ps_emit_a(as, fc);
          ps_advance_a(as, xr[j], fc);
        }
      }
#pragma unroll
      for (int j = 0; j < kTile; ++j) {
        if (j < rows) {
          ps_advance_c(cs, xr[j], fc);
          mine[j] = add2(ps_emit_c(cs, fc), mine[j]);
        }
      }
    }
    __syncthreads();
    // write-out: warp g writes its pair's 32 columns; lanes = rows
    if (lane < rows) {
      // band-major: element (g, row y, column x) at ((g*nb + y/16)*w + x)*16 + y%16
      const int y = y0 + lane;
      float2* vdst = V + (((size_t)g * (h_pad >> 4) + (y >> 4)) * w + x0) * 16 + (y & 15);
      const float2* src = buf + (size_t)g * 32 * 33 + lane;
#pragma unroll 8
      for (int c = 0; c < cols; ++c, vdst += 16) *vdst = src[c * 33];
    }
    // strip aggregates for the row pass: thread (pair g, row lane)
    if (lane < rows) {
      PairState agg;
      ps_zero(agg);
      const float2* sg = buf + (size_t)g * 32 * 33 + lane;
      for (int c = 0; c < cols; ++c)
        ps_accum(agg, sg[c * 33], tc.w4[c]);
      ps_store(AH + ((size_t)strip * pairs + g) * h * 2 + (size_t)(y0 + lane) * 2, agg);
    }
  }
}

// ----------------------------------------------------------------------------
// K3: row anticausal carries: suffix scan of the strip aggregates.
//   carry(last strip) = V[w-1] / (1-p)
//   carry(b - 1)      = AH[b] + p^{L_b} carry(b)
// ----------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_row_scan(const float2* __restrict__ V_all,
                                                   const float4* __restrict__ AH_all,
                                                   float4* __restrict__ CH_all, int w, int h,
                                                   int h_pad, int nx, FilterConsts fc,
                                                   TileConsts tc) {
  const int f = blockIdx.y, g = threadIdx.y, pairs = blockDim.y;
  const int y = blockIdx.x * 32 + threadIdx.x;
  if (y >= h) return;
  const float2* V = V_all + (size_t)f * pairs * w * h_pad;
  const float4* AH = AH_all + (size_t)f * nx * pairs * h * 2;
  float4* CH = CH_all + (size_t)f * nx * pairs * h * 2;
  PairState C;
  ps_set_gain(C, V[(((size_t)g * (h_pad >> 4) + (y >> 4)) * w + (w - 1)) * 16 + (y & 15)], fc);
  const size_t sstride = (size_t)pairs * h * 2;
  const size_t off = (size_t)g * h * 2 + (size_t)y * 2;
  ps_store(CH + (size_t)(nx - 1) * sstride + off, C);
  for (int b = nx - 1; b >= 1; --b) {
    PairState agg;
    ps_load(agg, AH + (size_t)b * sstride + off);
    if (b == nx - 1) ps_chain(C, agg, tc.pXr2, tc.pXi2);
    else ps_chain(C, agg, tc.pTr2, tc.pTi2);
    ps_store(CH + (size_t)(b - 1) * sstride + off, C);
  }
}

}  // namespace gpfb

#include "rowpass.cuh"

namespace gpfb {

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

// ----------------------------------------------------------------------------
// Host side
// ----------------------------------------------------------------------------
static void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();  // clear a non-sticky error (e.g. a failed allocation) for the caller
    throw Error{9, std::string(what) + ": " + cudaGetErrorString(e)};
  }
}

template <typename Tin>
static size_t colpass_smem(int pairs) {  // k_colpass and k_col_carry
  return sizeof(float2) * (size_t)pairs * 32 * 33 + sizeof(Tin) * 2 * 32 * 33;
}
#ifndef GPF_COL_SMEM_KB
#define GPF_COL_SMEM_KB 0  // > 0: pad the column pass's shared memory (fewer CTAs per SM, room for others)
#endif
static size_t colpass_tma_smem() {  // stages of a pair group + EM tile + alignment slack
  const size_t need = kStageAlign + sizeof(float) * kColStages * kColGroup * 2048 + sizeof(float2) * 32 * 32 * kColEmBufs;
  return std::max<size_t>(need, (size_t)GPF_COL_SMEM_KB * 1024);
}
template <typename Tin, typename Tout>
static int rowpass_nbuf(int pairs) {  // deepest V ring that fits in 227 KB (0: none)
  for (int nb = kRowBufsMax; nb >= 2; --nb)
    if (rowpass_smem_bytes<Tin, Tout>(pairs, nb) <= 227 * 1024) return nb;
  return 0;
}

void run_gaussian_f64(const double* d_in, double* d_out, double* d_tmp, int w, int h,
                      double sigma_s, double scale, cudaStream_t st) {
  DericheD k;
  deriche_coeffs_f64(sigma_s, k.nc, k.na, k.d);
  check(cudaMemsetAsync(d_out, 0, sizeof(double) * (size_t)w * h, st), "cudaMemsetAsync");
  k_gauss_rows<<<(h + 127) / 128, 128, 0, st>>>(d_in, d_tmp, w, h, k);
  k_gauss_cols<<<(w + 127) / 128, 128, 0, st>>>(d_tmp, d_out, w, h, k, scale);
  check(cudaGetLastError(), "kernel launch");
}

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    check(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode),
                                  cudaEnableDefault, &q),
          "cudaGetDriverEntryPoint(cuTensorMapEncodeTiled)");
    if (q != cudaDriverEntryPointSuccess || !encode)
      throw Error{9, "cuTensorMapEncodeTiled unavailable"};
  }
  return encode;
}

// fp32 frames {w, h, count}, box {32 columns, 16 rows, 1}, 128B-swizzled: the
// row pass's output tile and f tile; requires w % 4 == 0 and a 16-B aligned base.
static void encode_out_map(CUtensorMap* m, void* d_out, int w, int h, int count, int band_rows) {
  const cuuint64_t dims[3] = {(cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)count};
  const cuuint64_t strides[2] = {(cuuint64_t)4 * w, (cuuint64_t)4 * w * h};
  const cuuint32_t box[3] = {32, (cuuint32_t)band_rows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = tensor_map_encoder()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d_out, dims, strides,
                                          box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw Error{9, "cuTensorMapEncodeTiled (output) failed (" + std::to_string((int)r) + ")"};
}

void plan_init(Plan& plan, const Params& p, int device, int batch) {
  plan.p = p;
  plan.device = device;
  plan.batch = std::max(1, batch);
  plan.fc = make_filter_consts(p.sigma_s);
  plan.tc = make_tile_consts(p.sigma_s, p.width, p.height);
  plan.rc = make_range_consts(p);
  plan.rc.e_log2 += plan.fc.seed_log2;  // column-pass input carries S^2 (emit normalisation)
  finalize_range_consts(plan.rc);
  fill_gscale_consts(plan.tc, plan.rc);
  const int pairs = plan.rc.pairs;
  if (rowpass_nbuf<double, double>(pairs) == 0 || colpass_smem<double>(pairs) > 227 * 1024)
    throw Error{1, "RangeParams: degree must be <= 48 in the B200 library"};
  const int w = p.width, h = p.height, B = plan.batch;
  plan.ny = (h + kTile - 1) / kTile;
  plan.nx = (w + kTile - 1) / kTile;
  const int h_pad = plan.ny * kTile;
  const size_t npx = (size_t)w * h;
  plan.mean_blocks = (int)std::min<size_t>((npx + kMeanThreads - 1) / kMeanThreads, 148 * 4);
  if (plan.mean_blocks < 1) plan.mean_blocks = 1;
  const size_t vb = sizeof(float2) * B * (size_t)pairs * w * h_pad;
  const size_t cab = sizeof(float4) * 2 * B * (size_t)plan.ny * pairs * w;
  const size_t ahb = sizeof(float4) * 2 * B * (size_t)plan.nx * pairs * h;
  plan.w_pad = (w + 1) & ~1;
  const size_t emb = sizeof(float2) * B * (size_t)h * plan.w_pad;
  plan.V = nullptr;
  plan.CA = plan.AH = plan.CH = nullptr;
  plan.EM = nullptr;
  plan.scalars = plan.partials = nullptr;
  try {
    check(cudaMalloc(&plan.EM, emb), "cudaMalloc(EM)");
    check(cudaMalloc(&plan.V, vb), "cudaMalloc(V)");
    check(cudaMalloc(&plan.CA, cab), "cudaMalloc(CA)");
    check(cudaMalloc(&plan.AH, ahb), "cudaMalloc(AH)");
    check(cudaMalloc(&plan.CH, ahb), "cudaMalloc(CH)");
    check(cudaMalloc(&plan.scalars, sizeof(double) * 2 * B), "cudaMalloc(scalars)");
    check(cudaMalloc(&plan.partials, sizeof(double) * 4 * B * plan.mean_blocks), "cudaMalloc(partials)");
  } catch (...) {
    plan_free(plan);
    throw;
  }
  plan.bytes = vb + cab + 2 * ahb + emb + sizeof(double) * 2 * B * (1 + 2 * plan.mean_blocks);
  // mean (2), [seed,] carries, column pass, row scan, row pass
  plan.launches_per_frame = 32 * pairs <= 512 ? 7 : 6;
  // TMA tensor maps of the band-major V: fp32 dims (inner first)
  // {32 = 16 rows x 2 planes, w, h_pad/16 bands, pairs, batch}.
  const auto encode = tensor_map_encoder();
  const cuuint64_t nb = (cuuint64_t)h_pad / 16;
  const cuuint64_t dims[5] = {32, (cuuint64_t)w, nb, (cuuint64_t)pairs, (cuuint64_t)B};
  const cuuint64_t strides[4] = {128, (cuuint64_t)128 * w, (cuuint64_t)128 * w * nb,
                                 (cuuint64_t)128 * w * nb * pairs};
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  // row pass: box {32, 32 columns, 1 band, pairs, 1} -> smem [pair][column][16 rows]
  const cuuint32_t box[5] = {32, 32, 1, (cuuint32_t)pairs, 1};
  const CUresult r = encode(&plan.vmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, plan.V, dims, strides, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    plan_free(plan);
    throw Error{9, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")"};
  }
  // 8-row-band row pass: box {16 (= 8 rows x 2 planes), 33 columns, 1 band, pairs, 1}
  const cuuint32_t box8[5] = {16, 33, 1, (cuuint32_t)pairs, 1};
  const CUresult r8 = encode(&plan.vmap8, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, plan.V, dims, strides, box8,
                             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r8 != CUDA_SUCCESS) {
    plan_free(plan);
    throw Error{9, "cuTensorMapEncodeTiled (8-row V) failed (" + std::to_string((int)r8) + ")"};
  }
  // column-pass chunk store: box {32, 32 columns, 2 bands, kColGroup pairs, 1}
  // = one 32x32 chunk of a pair group; smem [pair][band][column][128 B],
  // 128B-swizzled.
  const cuuint32_t sbox[5] = {32, 32, 2, (cuuint32_t)kColGroup, 1};
  const CUresult r2 = encode(&plan.vstore, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, plan.V, dims, strides,
                             sbox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
#ifdef GPF_DIAG_EXTRA_VW
  {
    float2* vx = nullptr;
    check(cudaMalloc(&vx, vb), "cudaMalloc(Vx)");  // diagnostic only: never freed
    encode(&plan.vmap8, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, vx, dims, strides, sbox, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
#endif
  if (r2 != CUDA_SUCCESS) {
    plan_free(plan);
    throw Error{9, "cuTensorMapEncodeTiled (store) failed (" + std::to_string((int)r2) + ")"};
  }
  // EM seeds for the column pass: fp32 {2*w_pad, h, batch}, box {64 (= 32
  // pixels), 32 rows, 1}; out-of-image pixels read as zero.
  const cuuint64_t edims[3] = {(cuuint64_t)2 * w, (cuuint64_t)h, (cuuint64_t)B};
  const cuuint64_t estrides[2] = {(cuuint64_t)8 * plan.w_pad, (cuuint64_t)8 * plan.w_pad * h};
  const cuuint32_t ebox[3] = {64, 32, 1};
  const cuuint32_t eestr[3] = {1, 1, 1};
  const CUresult r3 = encode(&plan.emmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, plan.EM, edims, estrides,
                             ebox, eestr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  // EM seeds for the carry walk: box {128 (= 64 pixels), 32 rows, 1}
  const cuuint32_t cbox[3] = {2 * kCarryCols, 32, 1};
  const CUresult r4 = encode(&plan.emcmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, plan.EM, edims, estrides,
                             cbox, eestr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r4 != CUDA_SUCCESS) {
    plan_free(plan);
    throw Error{9, "cuTensorMapEncodeTiled (EM carries) failed (" + std::to_string((int)r4) + ")"};
  }
  if (r3 != CUDA_SUCCESS) {
    plan_free(plan);
    throw Error{9, "cuTensorMapEncodeTiled (EM) failed (" + std::to_string((int)r3) + ")"};
  }
}

void plan_free(Plan& plan) {
  cudaFree(plan.V);
  cudaFree(plan.CA);
  cudaFree(plan.AH);
  cudaFree(plan.CH);
  cudaFree(plan.EM);
  cudaFree(plan.scalars);
  cudaFree(plan.partials);
  plan.V = nullptr;
  plan.CA = plan.AH = plan.CH = nullptr;
  plan.EM = nullptr;
  plan.scalars = plan.partials = nullptr;
}

// MAXT = the CTA size bound the kernels are compiled for (32 x pairs threads):
// 384 -> up to 168 registers/thread (N <= 22), 512 -> 128 (N <= 30), 1024 -> 64.
#ifndef GPF_ROW_BAND
#define GPF_ROW_BAND 16
#endif
#ifndef GPF_CARRY_TMA
#define GPF_CARRY_TMA 1
#endif

// G-scaled planes on the TMA column pass + k_rowpass2 path
#ifdef GPF_DIAG_V_ONCE
static int vonce_first(const void* v) {  // 1 on the first call of a plan (its V buffer)
  static std::vector<const void*> seen;
  if (std::find(seen.begin(), seen.end(), v) != seen.end()) return 0;
  seen.push_back(v);
  return 1;
}
#endif
static bool plan_gscale(const Plan& plan) { return GPF_GSCALE && plan.rc.pairs <= kGsPairs; }

template <int MAXT, typename Tin, typename Tout>
static void launch_passes(Plan& plan, const Tin* d_in, Tout* d_out, int count,
                          unsigned long long* d_fb, cudaStream_t st) {
  const int w = plan.p.width, h = plan.p.height, pairs = plan.rc.pairs;
  const int h_pad = plan.ny * kTile;
  const int csm = (int)colpass_smem<Tin>(pairs);
  // TMA-store column pass in pair groups (the large-N builds keep the padded one)
  constexpr bool kCanStage = MAXT <= 512;
  const bool staged = kCanStage;
  const int psm = (int)(staged ? colpass_tma_smem() : colpass_smem<Tin>(pairs));
  const int nbuf = rowpass_nbuf<Tin, Tout>(pairs);
  const int rsm = (int)rowpass_smem_bytes<Tin, Tout>(pairs, nbuf);
  check(cudaFuncSetAttribute(k_col_carry<MAXT, Tin>, cudaFuncAttributeMaxDynamicSharedMemorySize, csm),
        "cudaFuncSetAttribute");
  // row-pass CTA: (pairs+1)/2 sweep warps + kAux aux warps
  constexpr int RMAXT = MAXT <= 384 ? 384 : 640;
  check(cudaFuncSetAttribute(k_rowpass<RMAXT, Tin, Tout>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             rsm),
        "cudaFuncSetAttribute");
  const dim3 blk(32, pairs);
  const int groups = (pairs + kColGroup - 1) / kColGroup;
  stage_mark(plan, kStageColCarry, st);
  if constexpr (kCanStage) {
    // seeds once per pixel, then the carries in pair groups
#ifndef GPF_DIAG_NO_SEED  // diagnostic: reuse the previous call's seeds (bench-mix cost of K1a)
#ifndef GPF_SEED_ROWS
#define GPF_SEED_ROWS 1024
#endif
#ifdef GPF_DIAG_SEED_DUMMY  // diagnostic: the seed stores go to a scratch buffer (consumers read stale EM)
    static float2* dummy = nullptr;
    if (!dummy) check(cudaMalloc(&dummy, sizeof(float2) * (size_t)h * plan.w_pad * count), "cudaMalloc");
    k_seed<Tin><<<dim3((w + 1023) / 1024, std::min(h, GPF_SEED_ROWS), count), 256, 0, st>>>(
        d_in, plan.scalars, dummy, w, h, plan.w_pad, plan.rc);
#else
#ifdef GPF_DIAG_SEED_ONCE  // diagnostic: seeds only on a plan's first call (valid while it keeps its frame)
    static std::vector<const void*> seeded;
    const bool once = std::find(seeded.begin(), seeded.end(), (const void*)plan.EM) != seeded.end();
    if (!once) seeded.push_back(plan.EM);
    if (!once)
#endif
#ifdef GPF_DIAG_SEED_EXTRA  // diagnostic: a second seed pass into a scratch buffer (real data kept)
    static float2* dummy = nullptr;
    if (!dummy) check(cudaMalloc(&dummy, sizeof(float2) * (size_t)h * plan.w_pad * count), "cudaMalloc");
    k_seed<Tin><<<dim3((w + 1023) / 1024, std::min(h, GPF_SEED_ROWS), count), 256, 0, st>>>(
        d_in, plan.scalars, dummy, w, h, plan.w_pad, plan.rc);
#endif
    k_seed<Tin><<<dim3((w + 1023) / 1024, std::min(h, GPF_SEED_ROWS), count), 256, 0, st>>>(
        d_in, plan.scalars, plan.EM, w, h, plan.w_pad, plan.rc);
#endif
#endif
#ifndef GPF_DIAG_NO_CARRY  // diagnostic: skip the carries (wrong output; bench-mix cost)
#if GPF_CARRY_TMA
    if (groups <= 3) {
      const int csm2 = (int)(sizeof(float2) * kCarrySlots * 32 * kCarryCols + 128);
      check(cudaFuncSetAttribute(k_col_carry_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, csm2),
            "cudaFuncSetAttribute");
      k_col_carry_tma<<<dim3((w + kCarryCols - 1) / kCarryCols * groups, count), dim3(32, kCarryWarps), csm2, st>>>(
          plan.CA, w, h, plan.ny, pairs, groups, plan.fc, plan.tc, plan.emcmap);
    } else
#endif
    k_col_carry_reg<<<dim3((w + 15) / 16 * groups, count), 32, 0, st>>>(
        plan.EM, plan.CA, w, h, plan.w_pad, plan.ny, pairs, groups, plan.fc, plan.tc);
#endif
  } else {
    k_col_carry<MAXT, Tin><<<dim3(plan.nx, count), blk, csm, st>>>(
        d_in, plan.scalars, plan.CA, plan.EM, w, h, plan.w_pad, plan.ny, plan.fc, plan.tc, plan.rc);
  }
  stage_mark(plan, kStageColPass, st);
  if constexpr (kCanStage) {
    const bool gs = plan_gscale(plan);
    auto kc = plan.fc.aev.x != 0.f ? (gs ? k_colpass_tma<true, true> : k_colpass_tma<true, false>)
                                   : (gs ? k_colpass_tma<false, true> : k_colpass_tma<false, false>);
    check(cudaFuncSetAttribute(kc, cudaFuncAttributeMaxDynamicSharedMemorySize, psm),
          "cudaFuncSetAttribute");
    kc<<<dim3(plan.nx * groups, count), dim3(32, kColGroup), psm, st>>>(
        plan.CA, plan.AH, w, h, plan.ny, plan.nx, pairs, groups, plan.fc, plan.tc, plan.emmap,
        plan.vstore
#ifdef GPF_DIAG_EXTRA_VW
        , plan.vmap8
#endif
#ifdef GPF_DIAG_V_ONCE
        , vonce_first(plan.V)
#endif
        );
  }
  if (!staged) {
    check(cudaFuncSetAttribute(k_colpass<MAXT, Tin>, cudaFuncAttributeMaxDynamicSharedMemorySize, psm),
          "cudaFuncSetAttribute");
    k_colpass<MAXT, Tin><<<dim3(plan.nx, count), blk, psm, st>>>(d_in, plan.scalars, plan.CA, plan.V,
                                                                 plan.AH, w, h, h_pad, plan.ny, plan.nx,
                                                                 plan.fc, plan.tc, plan.rc);
  }
  if (plan.front_done) check(cudaEventRecord(plan.front_done, st), "cudaEventRecord");
  stage_mark(plan, kStageRowScan, st);
#ifndef GPF_DIAG_NO_ROWSCAN  // diagnostic: skip the row scan (wrong output; bench-mix cost)
  k_row_scan<<<dim3(plan.ny, count), blk, 0, st>>>(plan.V, plan.AH, plan.CH, w, h, h_pad, plan.nx,
                                                   plan.fc, plan.tc);
#endif
  stage_mark(plan, kStageRowPass, st);
  if (pairs <= 12) {
    constexpr int RB = GPF_ROW_BAND;  // rows per row-pass CTA (16 or 8)
    const int r2sm = (int)rowpass2_smem_bytes<Tin, Tout, RB>(pairs);
    // fp32 output with 16-B rows: TMA output store (tensor map of this call's d_out)
    const bool otma = sizeof(Tout) == 4 && sizeof(Tin) == 4 && (w % 4) == 0 &&
                      (reinterpret_cast<uintptr_t>(d_out) % 16) == 0 &&
                      (reinterpret_cast<uintptr_t>(d_in) % 16) == 0;
    alignas(64) CUtensorMap omap, imap;
    std::memset(&omap, 0, sizeof(omap));
    std::memset(&imap, 0, sizeof(imap));
    if (otma) {
      encode_out_map(&omap, d_out, w, h, count, RB);
      encode_out_map(&imap, const_cast<Tin*>(d_in), w, h, count, RB);  // same box shape for the f tiles
    }
    // the default degree (N = 20, reference RangeParams) has a fully static build
    const bool n20 = plan.rc.degree == 20;
    // the clamped-basis u2 emit term only for sigma_s in [0.96, 1.17]
    const bool aev = plan.fc.aev.x != 0.f;
    auto k = n20 ? (aev ? k_rowpass2<Tin, Tout, 20, false, RB, true> : k_rowpass2<Tin, Tout, 20, false, RB, false>)
                 : k_rowpass2<Tin, Tout, 0, false, RB, true>;
    if constexpr (sizeof(Tout) == 4) {
      if (otma)
        k = n20 ? (aev ? k_rowpass2<Tin, Tout, 20, true, RB, true> : k_rowpass2<Tin, Tout, 20, true, RB, false>)
                : k_rowpass2<Tin, Tout, 0, true, RB, true>;
    }
    check(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, r2sm),
          "cudaFuncSetAttribute");
    // Row ranges (single-frame host entries): the bands go out in plan.row_ranges
    // launches, each followed by plan.range_done[i], so the caller's D2H of
    // the finished rows overlaps the rest of the row pass.
    const int nbands = (h + RB - 1) / RB;
    const int nr = (count == 1 && plan.row_ranges > 1) ? std::min(plan.row_ranges, nbands) : 1;
    for (int i = 0; i < nr; ++i) {
      const int b0 = (int)((long long)nbands * i / nr), b1 = (int)((long long)nbands * (i + 1) / nr);
      k<<<dim3(b1 - b0, count), dim3(32, (pairs * RB + 31) / 32), r2sm, st>>>(
          d_in, plan.scalars, plan.CH, d_out, d_fb, w, h, plan.nx, pairs, plan.fc, plan.rc,
          RB == 8 ? plan.vmap8 : plan.vmap, omap, imap, b0);
      if (nr > 1) check(cudaEventRecord(plan.range_done[i], st), "cudaEventRecord");
    }
    plan.range_rows = RB;
    plan.ranges_launched = nr;
  } else {
    k_rowpass<RMAXT, Tin, Tout><<<dim3((h + kRowBand - 1) / kRowBand, count),
                                  dim3(32, (pairs + 1) / 2 + kAux), rsm, st>>>(
        d_in, plan.scalars, plan.CH, d_out, d_fb, w, h, plan.nx, pairs, nbuf, plan.fc, plan.rc,
        plan.vmap);
    plan.ranges_launched = 1;
  }
  stage_end(plan, st);
}

template <typename Tin, typename Tout>
static void run_frames(Plan& plan, const Tin* d_in, Tout* d_out, int count,
                       unsigned long long* d_fb, cudaStream_t st) {
  if (count <= 0) return;
  if (count > plan.batch) throw Error{1, "batch larger than the plan's workspace"};
  const long long npx = (long long)plan.p.width * plan.p.height;
  stage_mark(plan, kStageMean, st);
  k_mean_partial<Tin><<<dim3(plan.mean_blocks, count), kMeanThreads, 0, st>>>(d_in, npx, plan.partials);
  k_mean_final<<<count, kMeanThreads, 0, st>>>(plan.partials, plan.mean_blocks, npx,
                                               plan.rc.centering, plan.rc.tc_fixed, plan.rc.inv_sr,
                                               fp32_h_limit(plan.rc.degree), plan.scalars, plan.ill_out);
  const int nthr = 32 * plan.rc.pairs;
  if (nthr <= 352) launch_passes<352>(plan, d_in, d_out, count, d_fb, st);  // N <= 20
  else if (nthr <= 384) launch_passes<384>(plan, d_in, d_out, count, d_fb, st);
  else if (nthr <= 512) launch_passes<512>(plan, d_in, d_out, count, d_fb, st);
  else launch_passes<1024>(plan, d_in, d_out, count, d_fb, st);
  check(cudaGetLastError(), "kernel launch");
}

// ---------------------------------------------------------------- profiling
struct StageTimer {
  struct Mark {
    int stage;
    cudaEvent_t ev;
  };
  std::vector<Mark> marks;  // in record order; stage -1 = end marker
  float acc[kNumStages] = {};
  int launches[kNumStages] = {};
};

void stage_mark(Plan& plan, int stage, cudaStream_t st) {
  if (!plan.profile) return;
  if (!plan.timer) plan.timer = new StageTimer();
  cudaEvent_t e;
  check(cudaEventCreate(&e), "cudaEventCreate");
  check(cudaEventRecord(e, st), "cudaEventRecord");
  plan.timer->marks.push_back({stage, e});
}

void stage_end(Plan& plan, cudaStream_t st) { stage_mark(plan, -1, st); }

int stage_times(Plan& plan, float* ms, int max_stages) {
  StageTimer* t = plan.timer;
  if (t) {
    for (size_t i = 0; i + 1 < t->marks.size(); ++i) {
      if (t->marks[i].stage < 0) continue;
      check(cudaEventSynchronize(t->marks[i + 1].ev), "cudaEventSynchronize");
      float e = 0.f;
      check(cudaEventElapsedTime(&e, t->marks[i].ev, t->marks[i + 1].ev), "cudaEventElapsedTime");
      t->acc[t->marks[i].stage] += e;
      t->launches[t->marks[i].stage] += 1;
    }
    for (auto& m : t->marks) cudaEventDestroy(m.ev);
    t->marks.clear();
  }
  const int n = std::min(max_stages, static_cast<int>(kNumStages));
  for (int i = 0; i < n; ++i) ms[i] = t ? t->acc[i] : 0.f;
  return n;
}

int stage_marks(Plan& plan, cudaEvent_t ref, float* t_ms, int* stage, int max_marks) {
  StageTimer* t = plan.timer;
  if (!t) return 0;
  int n = 0;
  for (auto& m : t->marks) {
    if (n < max_marks) {
      check(cudaEventSynchronize(m.ev), "cudaEventSynchronize");
      float e = 0.f;
      check(cudaEventElapsedTime(&e, ref, m.ev), "cudaEventElapsedTime");
      t_ms[n] = e;
      stage[n] = m.stage;
      ++n;
    }
    cudaEventDestroy(m.ev);
  }
  t->marks.clear();
  return n;
}

void stage_reset(Plan& plan) {
  if (!plan.timer) return;
  for (auto& m : plan.timer->marks) cudaEventDestroy(m.ev);
  delete plan.timer;
  plan.timer = nullptr;
}

void launch_mean_f64(const double* d_in, long long n, int centering, double tc_fixed, double sigma_r,
                     double* partials, int blocks, double* scalars, cudaStream_t st) {
  k_mean_partial<double><<<dim3(blocks, 1), kMeanThreads, 0, st>>>(d_in, n, partials);
  k_mean_final<<<1, kMeanThreads, 0, st>>>(partials, blocks, n, centering, tc_fixed, 1.0 / sigma_r,
                                           kH32Limit, scalars, nullptr);
  check(cudaGetLastError(), "kernel launch (mean)");
}

void run_frames_f32(Plan& plan, const float* d_in, float* d_out, int count,
                    unsigned long long* d_fb, cudaStream_t st) {
  run_frames<float, float>(plan, d_in, d_out, count, d_fb, st);
}

void run_frames_f64(Plan& plan, const double* d_in, double* d_out, int count,
                    unsigned long long* d_fb, cudaStream_t st) {
  run_frames<double, double>(plan, d_in, d_out, count, d_fb, st);
}

}  // namespace gpfb
