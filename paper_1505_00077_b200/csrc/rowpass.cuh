// K4: row pass (deriche_line over rows, spatial.cpp:235-239) on V, fused with
// the P/Q recombination and normalisation (bilateral.cpp:117-148).
// Included by gpf_kernels.cu.
//
// Warp-specialised TMA pipeline. A CTA owns kRowBand = 16 image rows and walks
// them strip by strip (32 columns):
//
//   aux warps (kAux)    : f tile (cp.async) + V tile of strip b+nbuf (one TMA
//                         box: 16 rows x 32 columns x all pairs) into ring slot
//                         b%nbuf; contraction + output of strip b.
//   sweep warps         : half-warp per plane pair, lane = row. Anticausal
//                         sweep from the K3 carry (outputs in registers), causal
//                         sweep (state carried across strips); Fbar in place.
//
//   full[s]  (tx bytes) : V tile in slot s has landed      aux -> sweep
//   swept[s] (warps)    : Fbar of slot s is complete        sweep -> aux
//
// An nbuf-deep ring (4 at N <= 22) lets the V stream of one SM run several
// strips ahead of the sweeps, so HBM reads overlap the FMA-bound sweeps and
// the contraction.
//
// Contraction, per pixel (row r, column c):
//   Q = sum_{n<=N} c_n Fbar_n,  P = sum_{n<=N} c_n Fbar_{n+1},  c_n = H^n/n!
// (weights and planes carry compensating 2^{-+s_n} scalings).
#pragma once

#include "sync.cuh"

namespace gpfb {

#ifndef GPF_ROW_AUX
#define GPF_ROW_AUX 4
#endif
constexpr int kAux = GPF_ROW_AUX;  // aux warps per CTA
constexpr int kRowBand = 16;    // image rows per CTA
constexpr int kRowBufsMax = 4;  // V ring depth bound (runtime nbuf <= this)

template <typename Tin, typename Tout>
__host__ __device__ constexpr size_t rowpass_smem_bytes(int pairs, int nbuf) {
  return (sizeof(float2) * (size_t)pairs * 32 * kRowBand + sizeof(Tin) * kRowBand * 33) * nbuf +
         sizeof(Tout) * kRowBand * 33 + 2 * kRowBufsMax * sizeof(uint64_t) + 16;
}

template <int MAXT, typename Tin, typename Tout>
__global__ void __launch_bounds__(MAXT, 1) k_rowpass(const Tin* __restrict__ in_all,
                                                     const double* __restrict__ scalars,
                                                     const float4* __restrict__ CH_all,
                                                     Tout* __restrict__ out_all,
                                                     unsigned long long* __restrict__ fb_all,
                                                     int w, int h, int nx, int pairs, int nbuf,
                                                     FilterConsts fc, RangeConsts rc,
                                                     const __grid_constant__ CUtensorMap vmap) {
  extern __shared__ float4 smem4[];
  const int f = blockIdx.y, lane = threadIdx.x, warp = threadIdx.y;
  const int nsweep = (pairs + 1) >> 1;  // sweep warps
  const int y0 = blockIdx.x * kRowBand;
  const int rows = min(kRowBand, h - y0);
  const size_t tile_elems = (size_t)pairs * 32 * kRowBand;  // float2 per slot: [g][c][16 rows]
  float2* T = reinterpret_cast<float2*>(smem4);
  Tin* F = reinterpret_cast<Tin*>(T + nbuf * tile_elems);       // [slot][16 rows][33]
  Tout* O = reinterpret_cast<Tout*>(F + nbuf * kRowBand * 33);  // [16 rows][33]
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(O + kRowBand * 33) + 15) & ~uintptr_t(15));
  uint64_t* full = bars;                  // [nbuf]
  uint64_t* swept = bars + kRowBufsMax;   // [nbuf]
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < nbuf; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&swept[s], nsweep);
    }
    mbar_fence_init();
  }
  __syncthreads();

  const Tin* in = in_all + (size_t)f * w * h;
  Tout* out = out_all + (size_t)f * w * h;

  if (warp < nsweep) {
    // ------------------------------------------------------------ sweep warps
    const int r = lane & (kRowBand - 1);
    const int g = 2 * warp + (lane >> 4);
    const bool live = g < pairs;
    const int gl = live ? g : pairs - 1;
    const int y = min(y0 + r, h - 1);
    const float4* CH = CH_all + (size_t)f * nx * pairs * h * 2 + (size_t)gl * h * 2 + (size_t)y * 2;
    const size_t ch_stride = (size_t)pairs * h * 2;
    float4 c0 = __ldg(CH), c1 = __ldg(CH + 1);
    PairState cs;
    ps_zero(cs);
    for (int b = 0; b < nx; ++b) {
      const int s = b % nbuf, cols = min(32, w - b * 32);
      PairState as;
      as.wr[0] = make_float2(c0.x, c0.y);
      as.wi[0] = make_float2(c0.z, c0.w);
      as.wr[1] = make_float2(c1.x, c1.y);
      as.wi[1] = make_float2(c1.z, c1.w);
      if (b + 1 < nx) {
        c0 = __ldg(CH + (size_t)(b + 1) * ch_stride);
        c1 = __ldg(CH + (size_t)(b + 1) * ch_stride + 1);
      }
      // element [g][c][r] of slot s at tl[c * kRowBand]
      float2* tl = T + (size_t)s * tile_elems + (size_t)gl * 32 * kRowBand + r;
      mbar_wait(&full[s], (b / nbuf) & 1);
      float2 ybuf[32];
      if (cols == 32) {
        // (an empty asm with a memory clobber every 4 columns stops the
        // compiler from hoisting all 32 smem loads into registers at once)
#pragma unroll
        for (int c = 31; c >= 0; --c) {
          if ((c & 3) == 3) asm volatile("" ::: "memory");
          ybuf[c] = ps_emit(as, fc.br2, fc.nbi2);
          ps_advance(as, tl[c * kRowBand], fc);
        }
        if (b == 0) ps_set_gain(cs, tl[0], fc);
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          if ((c & 3) == 0) asm volatile("" ::: "memory");
          ps_advance(cs, tl[c * kRowBand], fc);
          const float2 o = add2(ps_emit(cs, fc.ar2, fc.nai2), ybuf[c]);
          if (live) tl[c * kRowBand] = o;
        }
      } else {  // last, partial strip
#pragma unroll
        for (int c = 31; c >= 0; --c) {
          if (c < cols) {
            ybuf[c] = ps_emit(as, fc.br2, fc.nbi2);
            ps_advance(as, tl[c * kRowBand], fc);
          }
        }
        if (b == 0) ps_set_gain(cs, tl[0], fc);
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          if (c < cols) {
            ps_advance(cs, tl[c * kRowBand], fc);
            const float2 o = add2(ps_emit(cs, fc.ar2, fc.nai2), ybuf[c]);
            if (live) tl[c * kRowBand] = o;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&swept[s]);
    }
    return;
  }

  // -------------------------------------------------------------- aux warps
  const int atid = (warp - nsweep) * 32 + lane, nat = kAux * 32;
  const double t_c = scalars[2 * f];

  // V tile of strip b into slot s (one TMA box, completion on full[s]) and
  // its f tile (one cp.async group, waited before contracting strip b)
  auto load_strip = [&](int b, int s) {
    const int xs = b * 32, ncol = min(32, w - xs);
    if (atid == 0) {
      fence_proxy_async();
      mbar_arrive_expect_tx(&full[s], (uint32_t)(tile_elems * sizeof(float2)));
      tma_load_4d(T + (size_t)s * tile_elems, &vmap, 2 * y0, xs, 0, f, &full[s]);
    }
    Tin* Fs = F + s * kRowBand * 33;
    for (int p = atid; p < kRowBand * 32; p += nat) {
      const int r = p >> 5, c = p & 31;
      const bool ok = r < rows && c < ncol;
      cp_async_zfill<sizeof(Tin)>(Fs + r * 33 + c, ok ? in + (size_t)(y0 + r) * w + xs + c : in, ok);
    }
    cp_async_commit();
  };

  for (int s = 0; s < nbuf && s < nx; ++s) load_strip(s, s);
  unsigned my_fb = 0;
  const int full_pairs = (rc.degree + 1) >> 1;
  for (int b = 0; b < nx; ++b) {
    const int s = b % nbuf, xs = b * 32, cols = min(32, w - xs);
    // f tile of strip b: every cp.async group but the newer ones in flight done
    const int newer = min(nbuf, nx - b) - 1;
    if (newer >= 3) asm volatile("cp.async.wait_group 3;\n" ::: "memory");
    else if (newer == 2) asm volatile("cp.async.wait_group 2;\n" ::: "memory");
    else if (newer == 1) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    else asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    mbar_wait(&swept[s], (b / nbuf) & 1);
    named_bar(1, nat);  // every aux thread's share of the f tile has landed
    const float2* Ts = T + (size_t)s * tile_elems;
    const Tin* Fs = F + s * kRowBand * 33;
    // contraction: kPx pixels per thread with interleaved (independent) weight
    // chains; pixel p -> (row r = p & 15, col c = p >> 4); (Q, P) packed
    constexpr int kPx = 4;
    for (int p0 = atid; p0 < kRowBand * 32; p0 += nat * kPx) {
      double fv[kPx];
      float Hf[kPx], cc[kPx];
      float2 qp[kPx], cur2[kPx];
      const float2* col[kPx];
#pragma unroll
      for (int k = 0; k < kPx; ++k) {
        const int p = min(p0 + k * nat, kRowBand * 32 - 1);
        const int r = p & (kRowBand - 1), c = p >> 4;
        fv[k] = static_cast<double>(Fs[r * 33 + c]);
        Hf[k] = static_cast<float>((fv[k] - t_c) * rc.inv_sr);
        cc[k] = rc.c0;
        qp[k] = make_float2(0.f, 0.f);
        col[k] = Ts + (size_t)c * kRowBand + r;
        cur2[k] = col[k][0];
      }
      for (int gg = 0; gg < full_pairs; ++gg) {
        const float w0 = rc.w_step[2 * gg], w1 = rc.w_step[2 * gg + 1];
#pragma unroll
        for (int k = 0; k < kPx; ++k) {
          const float2 nxt = col[k][(size_t)(gg + 1) * 32 * kRowBand];
          qp[k] = fma2(f2(cc[k]), cur2[k], qp[k]);
          cc[k] = cc[k] * (Hf[k] * w0);
          qp[k] = fma2(f2(cc[k]), make_float2(cur2[k].y, nxt.x), qp[k]);
          cc[k] = cc[k] * (Hf[k] * w1);
          cur2[k] = nxt;
        }
      }
#pragma unroll
      for (int k = 0; k < kPx; ++k) {
        const int p = p0 + k * nat;
        const int r = p & (kRowBand - 1), c = p >> 4;
        if (p < kRowBand * 32 && r < rows && c < cols) {
          if (!(rc.degree & 1)) qp[k] = fma2(f2(cc[k]), cur2[k], qp[k]);  // n = N (even N)
          double o;
          if (!(fabsf(qp[k].x) > rc.q_thresh)) {
            o = fv[k];
            ++my_fb;
          } else {
            o = rc.sigma_r * ((static_cast<double>(qp[k].y) * rc.p_scale) /
                              static_cast<double>(qp[k].x)) + t_c;
          }
          O[r * 33 + c] = static_cast<Tout>(o);
        }
      }
    }
    named_bar(1, nat);
    for (int p = atid; p < kRowBand * 32; p += nat) {
      const int r = p >> 5, c = p & 31;
      if (r < rows && c < cols) out[(size_t)(y0 + r) * w + xs + c] = O[r * 33 + c];
    }
    named_bar(1, nat);  // slot s and O are free again
    if (b + nbuf < nx) load_strip(b + nbuf, s);
  }
  for (int o = 16; o; o >>= 1) my_fb += __shfl_xor_sync(0xffffffffu, my_fb, o);
  if (lane == 0 && my_fb) atomicAdd(fb_all + f, (unsigned long long)my_fb);
}

}  // namespace gpfb
