// The direct (windowed) spatial backend in fp64: SpatialBackend::direct /
// GPF_BACKEND_DIRECT of the reference (direct_gaussian,
// proj/src/core/spatial.cpp:112-129; the two separable passes 71-108;
// boundary_index 48-66), for gpf_gaussian_direct and as apply_spatial
// (bilateral.cpp:58-62) of gpf_filter_gpf / gpf_filter_taylor.
//
// It is the reference's evaluation, tap for tap: 2W+1 taps per axis formed on
// the host by the same fp64 expression (glibc exp; kernel_scale rides on the
// row taps only), rows first into a temporary, then columns; every output is
// acc = 0; acc += tap[k] * src[m(k)] for k = -W..W in that order, with
// explicitly rounded multiplies and adds (no FMA contraction), skipping the
// taps the zero boundary drops. The outputs are bitwise the reference's.
//
// Not the hot path (its cost grows with W; north_star is the O(1) recursive
// backend): one thread per output sample, `planes` images per launch, lines
// staged through shared memory with their 2W-sample apron when the apron fits
// (W <= kMaxApron), read through L1/L2 otherwise.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "gpf_internal.h"

namespace gpfb {

namespace {

constexpr int kDirT = 256;       // threads per CTA = output samples per CTA line segment
constexpr int kMaxApron = 512;   // W up to this: row segments staged in shared memory with their apron
constexpr int kMaxTapW = 2048;   // W up to this: taps copied to shared memory (read through L1 above)
constexpr int kColTX = 32, kColTY = 32;  // column-pass tile (x, y)

// boundary_index (spatial.cpp:48-66): 0 replicate, 1 reflect (half-sample
// symmetric), 2 zero (-1 = tap dropped)
__device__ __forceinline__ int bidx(int i, int n, int boundary) {
  if (i >= 0 && i < n) return i;
  if (boundary == 0) return i < 0 ? 0 : n - 1;
  if (boundary == 1) {
    const long long period = 2LL * n;
    long long m = (long long)i % period;
    if (m < 0) m += period;
    return (int)(m < n ? m : period - 1 - m);
  }
  return -1;
}

// windowed_pass_rows (spatial.cpp:71-88): lines = planes * h rows of w samples.
// smem: the row segment with its apron [kDirT + 2W] holding src at the
// boundary-mapped positions (the zero boundary's dropped taps are skipped by
// index, as the reference does), then the taps [2W+1].
__global__ void __launch_bounds__(kDirT) k_direct_rows(const double* __restrict__ src,
                                                      double* __restrict__ dst,
                                                      const double* __restrict__ taps, int w,
                                                      long long lines, int W, int boundary,
                                                      int use_smem) {
  extern __shared__ double sm[];
  const double* st = taps;
  double* sx = sm;  // segment + apron (use_smem implies W <= kMaxTapW: taps follow it)
  if (W <= kMaxTapW) {
    double* stw = sm + (use_smem ? kDirT + 2 * W : 0);
    for (int k = threadIdx.x; k < 2 * W + 1; k += kDirT) stw[k] = taps[k];
    st = stw;
  }
  const int segs = (w + kDirT - 1) / kDirT;
  for (long long item = blockIdx.x; item < lines * segs; item += gridDim.x) {
    const long long line = item / segs;
    const int x0 = (int)(item % segs) * kDirT;
    const double* row = src + line * w;
    const int x = x0 + threadIdx.x;
    __syncthreads();  // taps visible; previous segment's readers done
    if (use_smem) {
      for (int j = threadIdx.x; j < kDirT + 2 * W; j += kDirT) {
        const int m = bidx(x0 - W + j, w, boundary);
        sx[j] = m >= 0 ? row[m] : 0.0;
      }
      __syncthreads();
      if (x < w) {
        double acc = 0.0;
        if (boundary == 2) {
          for (int k = -W; k <= W; ++k)
            if (x + k >= 0 && x + k < w) acc = __dadd_rn(acc, __dmul_rn(st[k + W], sx[threadIdx.x + k + W]));
        } else {
          for (int k = -W; k <= W; ++k) acc = __dadd_rn(acc, __dmul_rn(st[k + W], sx[threadIdx.x + k + W]));
        }
        dst[line * w + x] = acc;
      }
    } else if (x < w) {
      double acc = 0.0;
      for (int k = -W; k <= W; ++k) {
        const int m = bidx(x + k, w, boundary);
        if (m >= 0) acc = __dadd_rn(acc, __dmul_rn(st[k + W], __ldg(row + m)));
      }
      dst[line * w + x] = acc;
    }
  }
}

// windowed_pass_cols (spatial.cpp:90-108): one thread per (x, y) of a plane,
// threads of a warp on consecutive x (coalesced 256-B row segments; the 2W+1
// rows a CTA's tile touches are re-read through L1/L2 by its kColTY rows).
__global__ void __launch_bounds__(kColTX * 8) k_direct_cols(const double* __restrict__ src,
                                                           double* __restrict__ dst,
                                                           const double* __restrict__ taps, int w,
                                                           int h, int planes, int W, int boundary) {
  extern __shared__ double sm[];
  const double* st = taps;
  if (W <= kMaxTapW) {
    for (int k = threadIdx.y * kColTX + threadIdx.x; k < 2 * W + 1; k += kColTX * 8) sm[k] = taps[k];
    st = sm;
  }
  __syncthreads();
  const int tx = (w + kColTX - 1) / kColTX, ty = (h + kColTY - 1) / kColTY;
  const long long tiles = (long long)tx * ty * planes;
  for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int plane = (int)(t / ((long long)tx * ty));
    const int rem = (int)(t % ((long long)tx * ty));
    const int x = (rem % tx) * kColTX + threadIdx.x;
    const int y0 = (rem / tx) * kColTY;
    if (x >= w) continue;
    const double* sp = src + (size_t)plane * w * h;
    double* dp = dst + (size_t)plane * w * h;
    for (int y = y0 + threadIdx.y; y < min(y0 + kColTY, h); y += 8) {
      double acc = 0.0;
      for (int k = -W; k <= W; ++k) {
        const int m = bidx(y + k, h, boundary);
        if (m >= 0) acc = __dadd_rn(acc, __dmul_rn(st[k + W], __ldg(sp + (size_t)m * w + x)));
      }
      dp[(size_t)y * w + x] = acc;
    }
  }
}


// ---- register-tiled passes (W <= kMaxApron): one thread owns R consecutive
// outputs of a line and walks the R + 2W samples they touch once; sample j
// meets output r with tap j - r, so every output still accumulates its taps in
// the order k = -W..W (bitwise the simple kernels above, which stay as the
// path for wider windows). The last R taps live in registers (a rotating
// window, resolved statically by unrolling R samples per trip), so a
// multiply-add costs 2/R shared-memory loads instead of 2.
constexpr int kTileT = 128;  // threads per CTA of the tiled row pass

template <int R>
__global__ void __launch_bounds__(kTileT) k_direct_rows_tiled(const double* __restrict__ src,
                                                             double* __restrict__ dst,
                                                             const double* __restrict__ taps, int w,
                                                             long long lines, int W, int boundary) {
  extern __shared__ double sm[];
  const int nt = 2 * W + 1;
  const int span = kTileT * R;                  // outputs per segment
  const int P = kTileT + (2 * W + R - 1) / R + 1;  // pitch of the sample planes
  double* st = sm;                              // taps, padded to a multiple of R past nt
  double* sx = sm + ((nt + 2 * R) & ~1);        // samples, transposed: i -> (i % R) P + i / R
  for (int k = threadIdx.x; k < nt + R; k += kTileT) st[k] = k < nt ? taps[k] : 0.0;
  const int segs = (w + span - 1) / span;
  const int trips = (nt + R - 1 + R - 1) / R;   // ceil((2W + R) / R)
  for (long long item = blockIdx.x; item < lines * segs; item += gridDim.x) {
    const long long line = item / segs;
    const int x0 = (int)(item % segs) * span;
    const double* row = src + line * w;
    __syncthreads();
    for (int i = threadIdx.x; i < trips * R + span; i += kTileT) {
      const int m = bidx(x0 - W + i, w, boundary);
      sx[(i % R) * P + i / R] = m >= 0 ? row[m] : 0.0;
    }
    __syncthreads();
    const int xb = x0 + threadIdx.x * R;  // first output of this thread
    double acc[R], t[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0, t[r] = 0.0;
    for (int j0 = 0; j0 < trips * R; j0 += R) {
#pragma unroll
      for (int jj = 0; jj < R; ++jj) {
        const int j = j0 + jj;          // sample xb - W + j, tap index j - r for output r
        t[jj] = st[min(j, nt + R - 1)];
        const double s = sx[jj * P + threadIdx.x + j0 / R];
        const int pos = xb - W + j;
        const bool live = boundary != 2 || (pos >= 0 && pos < w);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int k = j - r;
          if (live && k >= 0 && k < nt) acc[r] = __dadd_rn(acc[r], __dmul_rn(t[(jj - r + R) % R], s));
        }
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (xb + r < w) dst[line * w + xb + r] = acc[r];
  }
}

template <int R>
__global__ void __launch_bounds__(kColTX * 8) k_direct_cols_tiled(const double* __restrict__ src,
                                                                 double* __restrict__ dst,
                                                                 const double* __restrict__ taps, int w,
                                                                 int h, int planes, int W, int boundary) {
  extern __shared__ double sm[];
  const int nt = 2 * W + 1;
  for (int k = threadIdx.y * kColTX + threadIdx.x; k < nt + R; k += kColTX * 8) sm[k] = k < nt ? taps[k] : 0.0;
  __syncthreads();
  const int TY = 8 * R;
  const int tx = (w + kColTX - 1) / kColTX, ty = (h + TY - 1) / TY;
  const long long tiles = (long long)tx * ty * planes;
  const int trips = (nt + R - 1 + R - 1) / R;
  for (long long tl = blockIdx.x; tl < tiles; tl += gridDim.x) {
    const int plane = (int)(tl / ((long long)tx * ty));
    const int rem = (int)(tl % ((long long)tx * ty));
    const int x = (rem % tx) * kColTX + threadIdx.x;
    const int yb = (rem / tx) * TY + threadIdx.y * R;
    if (x >= w || yb >= h) continue;
    const double* sp = src + (size_t)plane * w * h + x;
    double* dp = dst + (size_t)plane * w * h + x;
    double acc[R], t[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0, t[r] = 0.0;
    for (int j0 = 0; j0 < trips * R; j0 += R) {
#pragma unroll
      for (int jj = 0; jj < R; ++jj) {
        const int j = j0 + jj;
        t[jj] = sm[min(j, nt + R - 1)];
        const int m = bidx(yb - W + j, h, boundary);
        const double s = m >= 0 ? __ldg(sp + (size_t)m * w) : 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int k = j - r;
          if (m >= 0 && k >= 0 && k < nt) acc[r] = __dadd_rn(acc[r], __dmul_rn(t[(jj - r + R) % R], s));
        }
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (yb + r < h) dp[(size_t)(yb + r) * w] = acc[r];
  }
}

template <int R>
cudaError_t launch_tiled(const double* d_src, double* d_dst, double* d_tmp, const double* d_taps, int w,
                         int h, int planes, int W, int boundary, cudaStream_t st) {
  const int nt = 2 * W + 1;
  const long long lines = (long long)planes * h;
  const int span = kTileT * R;
  const int trips = (nt + 2 * R - 2) / R;
  const int P = kTileT + (2 * W + R - 1) / R + 1;
  const size_t smr = sizeof(double) * (((nt + 2 * R) & ~1) + (size_t)R * P + trips);
  const size_t smc = sizeof(double) * (nt + R);
  const long long segs = lines * ((w + span - 1) / span);
  k_direct_rows_tiled<R><<<(int)std::min<long long>(segs, 148 * 16), kTileT, smr, st>>>(
      d_src, d_tmp, d_taps, w, lines, W, boundary);
  const long long tiles = (long long)((w + kColTX - 1) / kColTX) * ((h + 8 * R - 1) / (8 * R)) * planes;
  k_direct_cols_tiled<R><<<(int)std::min<long long>(tiles, 148 * 32), dim3(kColTX, 8), smc, st>>>(
      d_tmp, d_dst, d_taps + nt, w, h, planes, W, boundary);
  return cudaGetLastError();
}

// GpfState::step's plane chain (bilateral.cpp:108-129): F_0, F_{n+1} = H F_n
__global__ void k_direct_gen_planes(const double* __restrict__ H, const double* __restrict__ F0,
                                    double* __restrict__ F, long long n, int planes) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double hv = H[i];
    double v = F0[i];
    for (int p = 0; p < planes; ++p) {
      F[(size_t)p * n + i] = v;
      v = __dmul_rn(hv, v);
    }
  }
}

// GPF_B200_DIRECT_SIMPLE=1: the one-output-per-thread kernels for every window
// (the cross-check of the tiled kernels in tests/test_gpu_direct.py)
bool direct_simple() {
  const char* e = std::getenv("GPF_B200_DIRECT_SIMPLE");
  return e != nullptr && e[0] != '\0' && e[0] != '0';
}

void chk_(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error{9, std::string(what) + ": " + cudaGetErrorString(e)};
  }
}

}  // namespace

void direct_gen_planes_f64(const double* H, const double* F0, double* F, long long n, int planes,
                           cudaStream_t st) {
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148 * 16);
  k_direct_gen_planes<<<blocks, 256, 0, st>>>(H, F0, F, n, planes);
  chk_(cudaGetLastError(), "kernel launch (direct planes)");
}

// `planes` images of w x h at d_src (plane stride w h) -> d_dst, through d_tmp
// (same shape; d_dst may alias d_src). Taps as direct_gaussian forms them.
void run_direct_gaussian_f64(const double* d_src, double* d_dst, double* d_tmp, int w, int h,
                             int planes, double sigma_s, double kernel_scale, int W, int boundary,
                             cudaStream_t st) {
  if (W < 1) throw Error{1, "SpatialParams: window_radius must be >= 1"};
  if (W > (1 << 20)) throw Error{1, "SpatialParams: window_radius must be <= 1048576 in the B200 library"};
  const int nt = 2 * W + 1;
  std::vector<double> taps(2 * (size_t)nt);
  for (int k = -W; k <= W; ++k) {
    // spatial.cpp:118-123
    const double g = std::exp(-(static_cast<double>(k) * k) / (2.0 * sigma_s * sigma_s));
    taps[k + W] = kernel_scale * g;
    taps[nt + k + W] = g;
  }
  double* d_taps = nullptr;
  chk_(cudaMallocAsync(&d_taps, sizeof(double) * taps.size(), st), "cudaMallocAsync (taps)");
  // pageable source: staged before the call returns, so `taps` may go out of scope
  cudaError_t e = cudaMemcpyAsync(d_taps, taps.data(), sizeof(double) * taps.size(),
                                  cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) {
    const long long lines = (long long)planes * h;
    if (W <= kMaxApron && !direct_simple()) {
      e = W <= 12 ? launch_tiled<4>(d_src, d_dst, d_tmp, d_taps, w, h, planes, W, boundary, st)
                  : launch_tiled<8>(d_src, d_dst, d_tmp, d_taps, w, h, planes, W, boundary, st);
      cudaFreeAsync(d_taps, st);
      chk_(e, "direct_gaussian launch");
      return;
    }
    const int use_smem = W <= kMaxApron;
    const size_t smc = sizeof(double) * (W <= kMaxTapW ? nt : 0);  // <= 32 KB
    const size_t smr = smc + sizeof(double) * (use_smem ? kDirT + 2 * W : 0);
    {
      const long long segs = lines * ((w + kDirT - 1) / kDirT);
      k_direct_rows<<<(int)std::min<long long>(segs, 148 * 32), kDirT, smr, st>>>(
          d_src, d_tmp, d_taps, w, lines, W, boundary, use_smem);
      const long long tiles =
          (long long)((w + kColTX - 1) / kColTX) * ((h + kColTY - 1) / kColTY) * planes;
      k_direct_cols<<<(int)std::min<long long>(tiles, 148 * 32), dim3(kColTX, 8), smc, st>>>(
          d_tmp, d_dst, d_taps + nt, w, h, planes, W, boundary);
      e = cudaGetLastError();
    }
  }
  cudaFreeAsync(d_taps, st);
  chk_(e, "direct_gaussian launch");
}

}  // namespace gpfb
