// K4: row pass (deriche_line over rows, spatial.cpp:235-239) on V, fused with
// the P/Q recombination and normalisation (bilateral.cpp:117-148).
// Included by gpf_kernels.cu.
//
// Two kernels: k_rowpass2 (N <= 22, the default path; further below) and the
// warp-specialised k_rowpass for larger N, described here. A k_rowpass CTA
// owns kRowBand = 16 image rows and walks them strip by strip (32 columns):
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
      ps_from_carry(as, c0, c1, fc);
      if (b + 1 < nx) {
        c0 = __ldg(CH + (size_t)(b + 1) * ch_stride);
        c1 = __ldg(CH + (size_t)(b + 1) * ch_stride + 1);
      }
      // element [g][c][r] of slot s at tl[c * kRowBand]
      float2* tl = T + (size_t)s * tile_elems + (size_t)gl * 32 * kRowBand + r;
      mbar_wait(&full[s], (b / nbuf) & 1);
      if (b == 0) ps_set_gain_sweep(cs, tl[0], fc);
      if (cols == 32) {
        // Both directions in one loop (two independent recurrences per step):
        // step t runs the anticausal section at column 31-t and the causal one
        // at column t. Outputs of the first half wait in registers; from
        // t = 16 on each column's other half is ready and the sum is written.
        float2 ya_hi[16], yc_lo[16];  // ya[16..31], yc[0..15]
#pragma unroll
        for (int t = 0; t < 32; ++t) {
          const int ca = 31 - t, cc = t;
          const float2 ya = ps_emit_a(as, fc);
          const float2 xa = tl[ca * kRowBand], xc = tl[cc * kRowBand];
          ps_advance_a(as, xa, fc);
          ps_advance_c(cs, xc, fc);
          const float2 yc = ps_emit_c(cs, fc);
          if (t < 16) {
            ya_hi[ca - 16] = ya;
            yc_lo[cc] = yc;
          } else {
            if (live) {
              tl[ca * kRowBand] = add2(ya, yc_lo[ca]);
              tl[cc * kRowBand] = add2(yc, ya_hi[cc - 16]);
            }
          }
        }
      } else {  // last, partial strip
        float2 ybuf[32];
#pragma unroll
        for (int c = 31; c >= 0; --c) {
          if (c < cols) {
            ybuf[c] = ps_emit_a(as, fc);
            ps_advance_a(as, tl[c * kRowBand], fc);
          }
        }
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          if (c < cols) {
            ps_advance_c(cs, tl[c * kRowBand], fc);
            const float2 o = add2(ps_emit_c(cs, fc), ybuf[c]);
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
      tma_load_5d(T + (size_t)s * tile_elems, &vmap, 0, xs, y0 / kRowBand, 0, f, &full[s]);
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
        Hf[k] = h_t<Tin>(Fs[r * 33 + c], t_c, static_cast<float>(t_c),
                         static_cast<float>(t_c - static_cast<float>(t_c)), rc);
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
            // sigma_r * (p / q) + t_c as the reference rounds it (bilateral.cpp:144): no FMA
            o = __dadd_rn(__dmul_rn(rc.sigma_r, __ddiv_rn(static_cast<double>(qp[k].y) * rc.p_scale,
                                                          static_cast<double>(qp[k].x))), t_c);
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

namespace gpfb {

// ----------------------------------------------------------------------------
// k_rowpass2 (pairs <= 12): no warp specialisation. A CTA of ceil(pairs/2)
// warps owns kRowBand rows; per 32-column strip it
//   1. waits for the strip's V box (TMA, 2-slot ring) and sweeps both
//      directions in one interleaved loop (half-warp per pair, lane = row),
//      Fbar in place;
//   2. contracts every pixel over all planes into an output tile;
//   3. writes the tile out coalesced and refills the slot with strip b+2.
// Two CTAs share an SM, so one's contraction / write-out / load phases
// overlap the other's FMA-bound sweeps.
// ----------------------------------------------------------------------------
#ifndef GPF_ROW_SLOTS
#define GPF_ROW_SLOTS 2
#endif
#ifndef GPF_ROW_CTAS
#define GPF_ROW_CTAS 2
#endif
constexpr int kRow2Slots = GPF_ROW_SLOTS;  // V slots per CTA (2: the next strip prefetched)
constexpr int kRow2MaxN = 22;  // pairs <= 12

// Band height RB: 16 rows (half-warp per pair, 2 CTAs/SM) or 8 rows (quarter-warp
// per pair, 4 CTAs/SM). The 8-row V box is 33 columns wide, so consecutive pairs
// sit 64 B apart in the bank space and a warp's four 64-B pair segments of one
// column are conflict-free (the 33rd column is loaded but unused).
template <int RB>
__host__ __device__ constexpr int row2_pair_cols() { return RB == 8 ? 33 : 32; }

template <typename Tin, typename Tout, int RB = kRowBand>
__host__ __device__ constexpr size_t rowpass2_smem_bytes(int pairs) {
  // V ring | f tiles | padded output tile | mbarriers | 1024-aligned swizzled
  // output tile | swizzled f tiles (TMA path)
  return (sizeof(float2) * (size_t)pairs * row2_pair_cols<RB>() * RB + 128) * kRow2Slots +
         sizeof(Tin) * RB * 33 * kRow2Slots + sizeof(Tout) * RB * 33 +
         kRow2Slots * sizeof(uint64_t) + 16 + 1024 + sizeof(float) * RB * 32 * (1 + kRow2Slots);
}

// Contraction of kPx pixels per thread (pixel p -> row p & 15, column p >> 4),
// their chains interleaved. Plane m adds c_m F_m to Q and c_{m-1} F_m to P;
// plane 0 is Q-only, plane N+1 P-only (bilateral.cpp:117-148). Returns the
// fallback count.
// f tile element (row r, column c): padded [16][33] (cp.async path) or the
// 128B-swizzled [16][32] box of the TMA path
template <bool SW>
__device__ __forceinline__ int f_at(int r, int c) {
  return SW ? r * 32 + ((((c >> 2) ^ (r & 7))) << 2) + (c & 3) : r * 33 + c;
}

// OSW: write into the 128B-swizzled [16][32] fp32 tile of the TMA output store
// (element (r, c) at r*32 + (((c/4) ^ (r%8)) * 4) + c%4) instead of the padded O.
template <int kPx, int NFIX, bool OSW, int RB, typename Tin, typename Tout>
__device__ __forceinline__ unsigned contract_px(const float2* Ts, const Tin* Fs, Tout* O, int p0,
                                                int nthr, int rows, int cols, const RangeConsts& rc,
                                                double t_c, float sr_f, float tc_hi, float tc_lo) {
  unsigned nfb = 0;
  const int nN = NFIX > 0 ? NFIX : rc.degree;  // planes 0..N+1
  float Hf[kPx];
  int off[kPx];
#pragma unroll
  for (int k = 0; k < kPx; ++k) {
    const int p = min(p0 + k * nthr, RB * 32 - 1);
    off[k] = p;  // [col][row]: column p / RB, row p % RB
    // H as the column pass formed it (pixel_terms): fp64 difference, fp32 H
    Hf[k] = h_t<Tin>(Fs[f_at<OSW>(p % RB, p / RB)], t_c, tc_hi, tc_lo, rc);
  }
  // Q = sum_{n<=N} c_n F_n and P = sum_{n<=N} c_n F_{n+1} with c_n = H^n k_n
  // share the coefficient polynomial: Horner in H over n = N..0 on the pair
  //   (Q, P) <- (Q, P) H + k_n (F_n, F_{n+1}),
  // one packed multiply and one packed FMA per plane. (F_n, F_{n+1}) is plane
  // pair n/2 for even n; for odd n it straddles two pairs (lo.y, hi.x). Every
  // partial sum is a tail of the same series in unscaled units (k_n F_n =
  // F_n-bar / n!), so no intermediate leaves the range the forward sum uses.
  // Unrolled to N (static build) or to kRow2MaxN with a guard, so smem
  // offsets and the k_n are immediates.
  constexpr int kTop = NFIX > 0 ? NFIX : kRow2MaxN;
  constexpr int kPS = row2_pair_cols<RB>() * RB;  // float2 per pair in a slot
  float2 qp[kPx];
  if constexpr (GPF_GSCALE) {
    // G units: plane n holds Gbar_n = Fbar_n 2^{s0-64} / n! (coeffs.cpp), so with T = 2^{s0-64}
    //   Q T = sum_{n<=N} H^n Gbar_n = b,   P T = sum_{n<=N} (n+1) H^n Gbar_{n+1} = d,
    // P being Q's derivative plus the top term: one joint Horner pass,
    //   d <- d H + b,  b <- b H + Gbar_n     (b = Gbar_N, d = (N+1) Gbar_{N+1} first),
    // taken two planes at a time from pair g = (Gbar_2g, Gbar_2g+1) = L:
    //   (d, b) <- (d, b) H^2 + (2 b H + L.y, H L.y + L.x).
    float2 db[kPx], h21[kPx];
    float hsq[kPx];
#pragma unroll
    for (int k = 0; k < kPx; ++k) {
      h21[k] = make_float2(2.f * Hf[k], Hf[k]);
      hsq[k] = Hf[k] * Hf[k];
      const float2 lo = Ts[off[k] + (nN >> 1) * kPS];
      if (!(nN & 1)) {
        db[k] = make_float2(static_cast<float>(nN + 1) * lo.y, lo.x);
      } else {  // N odd: Gbar_N = lo.y, Gbar_{N+1} in the next pair; then plane N-1 alone
        const float g1 = Ts[off[k] + ((nN + 1) >> 1) * kPS].x;
        float d = static_cast<float>(nN + 1) * g1, b = lo.y;
        d = fmaf(d, Hf[k], b);
        b = fmaf(b, Hf[k], lo.x);
        db[k] = make_float2(d, b);
      }
    }
    constexpr int kTopG = (kTop >> 1) - 1;  // highest pair taken two planes at a time
    const int gTop = (nN & 1) ? ((nN - 3) >> 1) : ((nN >> 1) - 1);
#pragma unroll
    for (int gq = kTopG; gq >= 0; --gq) {
      if (gq > gTop) continue;
#pragma unroll
      for (int k = 0; k < kPx; ++k) {
        const float2 L = Ts[off[k] + gq * kPS];
        const float2 u = fma2(make_float2(db[k].y, L.y), h21[k], make_float2(L.y, L.x));
        db[k] = fma2(db[k], f2(hsq[k]), u);
      }
    }
#pragma unroll
    for (int k = 0; k < kPx; ++k) qp[k] = make_float2(db[k].y, db[k].x);  // (Q, P) in G units
  } else {
  float2 acc[kPx], hi[kPx];
  {  // n = N
    const float kn = rc.k_coef[nN];
#pragma unroll
    for (int k = 0; k < kPx; ++k) {
      const float2 lo = Ts[off[k] + (nN >> 1) * kPS];
      float2 t = lo;
      if (nN & 1) t = make_float2(lo.y, Ts[off[k] + ((nN + 1) >> 1) * kPS].x);
      acc[k] = mul2(t, f2(kn));
      hi[k] = lo;
    }
  }
#pragma unroll
  for (int n = kTop - 1; n >= 0; --n) {
    if (n >= nN) continue;
    const float kn = rc.k_coef[n];
#pragma unroll
    for (int k = 0; k < kPx; ++k) {
      const float2 lo = Ts[off[k] + (n >> 1) * kPS];
      const float2 t = (n & 1) ? make_float2(lo.y, hi[k].x) : lo;
      acc[k] = fma2(acc[k], f2(Hf[k]), mul2(t, f2(kn)));
      hi[k] = lo;
    }
  }
#pragma unroll
  for (int k = 0; k < kPx; ++k) qp[k] = acc[k];
  }
  // G units: no P scale, the threshold in G units
  const float qth = GPF_GSCALE ? rc.q_thresh_g : rc.q_thresh;
  const float psc = GPF_GSCALE ? 1.f : rc.p_scale;
  // out = sr P/Q + t_c (bilateral.cpp:139-147); |Q| <= threshold -> input.
  // fp32 output: fp32 quotient (|error| <= sr |P/Q| 2^-22 < 1e-4 on [0, 255]);
  // fp64 output keeps the fp64 quotient.
#pragma unroll
  for (int k = 0; k < kPx; ++k) {
    const int p = p0 + k * nthr;
    const int pr = p % RB, pc = p / RB;
    if (p < RB * 32 && (OSW || (pr < rows && pc < cols))) {  // the TMA store clips
      Tout o;
      if (!(fabsf(qp[k].x) > qth)) {
        o = static_cast<Tout>(Fs[f_at<OSW>(pr, pc)]);
        if (pr < rows && pc < cols) ++nfb;
      } else if constexpr (sizeof(Tout) == sizeof(float)) {
        // fast quotient (2 ulp) inside its range; |Q| > threshold >> 2^-126 here
        const float num = qp[k].y * psc, den = qp[k].x;
        const float q = fabsf(den) < 1e37f ? __fdividef(num, den) : num / den;
        o = fmaf(sr_f, q, tc_hi) + tc_lo;
      } else {
        // sigma_r * (p / q) + t_c as the reference rounds it (bilateral.cpp:144): product, then
        // sum, no FMA -- so that the centred call equals the pre-shifted, uncentred one plus t_c
        // bit for bit (proj/tests/test_bilateral.cpp:234-258) in this mode too
        o = __dadd_rn(__dmul_rn(rc.sigma_r, __ddiv_rn(static_cast<double>(qp[k].y) * psc,
                                                      static_cast<double>(qp[k].x))), t_c);
      }
      if constexpr (OSW) O[pr * 32 + ((((pc >> 2) ^ (pr & 7))) << 2) + (pc & 3)] = o;
      else O[pr * 33 + pc] = o;
    }
  }
  return nfb;
}

// NFIX > 0: the degree N is a compile-time constant (the default N = 20 build);
// NFIX = 0: runtime N (<= kRow2MaxN).
// OTMA (fp32 output, width % 4 == 0): the contraction fills a 128B-swizzled
// [16][32] tile and one thread stores it with a TMA tensor store (`omap` =
// the caller's output), which drains under the next strip's sweeps; else the
// warps write the tile out row by row.
template <typename Tin, typename Tout, int NFIX, bool OTMA, int RB = kRowBand, bool AEV = true>
__global__ void __launch_bounds__(RB == 8 ? 96 : 192, RB == 8 ? 4 : GPF_ROW_CTAS) k_rowpass2(const Tin* __restrict__ in_all,
                                                      const double* __restrict__ scalars,
                                                      const float4* __restrict__ CH_all,
                                                      Tout* __restrict__ out_all,
                                                      unsigned long long* __restrict__ fb_all,
                                                      int w, int h, int nx, int pairs,
                                                      FilterConsts fc, RangeConsts rc,
                                                      const __grid_constant__ CUtensorMap vmap,
                                                      const __grid_constant__ CUtensorMap omap,
                                                      const __grid_constant__ CUtensorMap imap,
                                                      int band0) {
  extern __shared__ float4 smem4[];
  const int f = blockIdx.y, lane = threadIdx.x, warp = threadIdx.y;
  const int tid = warp * 32 + lane, nthr = blockDim.x * blockDim.y;
  constexpr int PC = row2_pair_cols<RB>();  // columns per pair in a slot
  const int y0 = (blockIdx.x + band0) * RB;  // band0: first band of this launch (row ranges)
  const int rows = min(RB, h - y0);
  const size_t tile_elems = (size_t)pairs * PC * RB;  // float2 per V box: [g][PC columns][RB rows]
  const size_t slot_elems = (tile_elems + 15) & ~size_t(15);  // slots 128-B aligned (TMA)
  float2* T = reinterpret_cast<float2*>(smem4);
  Tin* F = reinterpret_cast<Tin*>(T + kRow2Slots * slot_elems);  // [slot][RB rows][33]
  Tout* O = reinterpret_cast<Tout*>(F + kRow2Slots * RB * 33);   // [RB rows][33]
  uint64_t* full = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(O + RB * 33) + 15) & ~uintptr_t(15));
  // swizzled output tile, 1024-aligned in the shared window (offset from the base)
  float* O2;
  {
    char* base = reinterpret_cast<char*>(smem4);
    const uint32_t a = smem_u32(full + kRow2Slots);
    O2 = reinterpret_cast<float*>(base + (((a + 1023u) & ~1023u) - smem_u32(base)));
  }
  float* F2 = O2 + RB * 32;  // [slot][RB][32] swizzled f tiles (TMA path)
  const Tin* in = in_all + (size_t)f * w * h;
  Tout* out = out_all + (size_t)f * w * h;
  const double t_c = scalars[2 * f];

  // V box of strip b into slot s (TMA, completion on full[s]) and its f tile:
  // TMA path -- a swizzled tensor box completing on the same barrier; else
  // one cp.async group per thread, waited before the contraction
  auto load_strip = [&](int b, int s) {
    const int xs = b * 32, ncol = min(32, w - xs);
    if (tid == 0) {
      fence_proxy_async();
      mbar_arrive_expect_tx(&full[s], (uint32_t)(tile_elems * sizeof(float2) +
                                                 (OTMA ? sizeof(float) * RB * 32 : 0)));
      // V is band-major in 16-row bands: an 8-row band starts 0 or 16 floats into its band
#ifdef GPF_DIAG_L2V  // diagnostic: V boxes from a small L2-resident region
      tma_load_5d(T + (size_t)s * slot_elems, &vmap, 0, (b & 3) * 32, blockIdx.x & 1, 0, f, &full[s]);
#else
      if constexpr (GPF_L2HINT & 2)
        tma_load_5d_hint(T + (size_t)s * slot_elems, &vmap, (y0 & 15) * 2, xs, y0 >> 4, 0, f, &full[s], l2_evict_first());
      else tma_load_5d(T + (size_t)s * slot_elems, &vmap, (y0 & 15) * 2, xs, y0 >> 4, 0, f, &full[s]);
#endif
      if constexpr (OTMA) {
        if constexpr (GPF_L2HINT & 8) tma_load_3d_hint(F2 + s * RB * 32, &imap, xs, y0, f, &full[s], l2_evict_first());
        else tma_load_3d(F2 + s * RB * 32, &imap, xs, y0, f, &full[s]);
      }
    }
    if constexpr (!OTMA) {
      Tin* Fs = F + s * RB * 33;
      for (int p = tid; p < RB * 32; p += nthr) {
        const int r = p >> 5, c = p & 31;
        const bool ok = r < rows && c < ncol;
        cp_async_zfill<sizeof(Tin)>(Fs + r * 33 + c, ok ? in + (size_t)(y0 + r) * w + xs + c : in, ok);
      }
      cp_async_commit();
    }
  };

  if (tid == 0) {
    for (int s = 0; s < kRow2Slots; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  for (int s = 0; s < kRow2Slots && s < nx; ++s) load_strip(s, s);

  // sweep role: RB lanes per pair (half- or quarter-warp), lane = row
  const int r = lane & (RB - 1);
  const int g = (32 / RB) * warp + lane / RB;
  const bool live = g < pairs;
  const int gl = live ? g : pairs - 1;
  const int yr = min(y0 + r, h - 1);
  const float4* CH = CH_all + (size_t)f * nx * pairs * h * 2 + (size_t)gl * h * 2 + (size_t)yr * 2;
  const size_t ch_stride = (size_t)pairs * h * 2;
  float4 c0 = __ldg(CH), c1 = __ldg(CH + 1);
  PairState cs;
  ps_zero(cs);
  unsigned my_fb = 0;
  const float sr_f = static_cast<float>(rc.sigma_r);
  const float tc_hi = static_cast<float>(t_c), tc_lo = static_cast<float>(t_c - tc_hi);
#ifdef GPF_DIAG_CLOCKS
  long long tph[6] = {0, 0, 0, 0, 0, 0};  // wait V, sweep, f+bar, contract, bar+write, bar+load
  long long tq = clock64();
#define GPF_TICK(i) { const long long tn = clock64(); tph[i] += tn - tq; tq = tn; }
#else
#define GPF_TICK(i)
#endif

  for (int b = 0; b < nx; ++b) {
    const int s = b % kRow2Slots, xs = b * 32, cols = min(32, w - xs);
    PairState as;
    ps_from_carry(as, c0, c1, fc);
    if (b + 1 < nx) {
      c0 = __ldg(CH + (size_t)(b + 1) * ch_stride);
      c1 = __ldg(CH + (size_t)(b + 1) * ch_stride + 1);
    }
    // ---- 1. sweeps (element [g][c][r] of slot s at tl[c * RB])
    float2* tl = T + (size_t)s * slot_elems + (size_t)gl * PC * RB + r;
    GPF_TICK(5);
    mbar_wait(&full[s], (b / kRow2Slots) & 1);
    GPF_TICK(0);
    if (b == 0) ps_set_gain_sweep(cs, tl[0], fc);
#ifdef GPF_DIAG_NO_SWEEP
    constexpr bool kSweep = false;
#else
    constexpr bool kSweep = true;
#endif
    if (kSweep && live && cols == 32) {  // a dead half-warp (odd P) idles: same issue, less power
      // both directions in one loop: step t runs the anticausal sections at
      // column 31-t and the causal ones at column t; first-half outputs wait
      // in registers, second-half outputs add them and are written in place
      float2 ya_hi[16], yc_lo[16];  // ya[16..31], yc[0..15]
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        if ((t & 1) == 1) asm volatile("" ::: "memory");
        const int ca = 31 - t, cc = t;
        if (t < 16) {
          const float2 ya = ps_emit_a<AEV>(as, fc);
          const float2 xa = tl[ca * RB], xc = tl[cc * RB];
          ps_advance_a(as, xa, fc);
          ps_advance_c(cs, xc, fc);
          ya_hi[ca - 16] = ya;
          yc_lo[cc] = ps_emit_c(cs, fc);
        } else {  // the other direction's parked value seeds the emit
          const float2 ya = ps_emit_a_acc<AEV>(as, fc, yc_lo[ca]);
          const float2 xa = tl[ca * RB], xc = tl[cc * RB];
          ps_advance_a(as, xa, fc);
          ps_advance_c(cs, xc, fc);
          const float2 yc = ps_emit_c_acc(cs, fc, ya_hi[cc - 16]);
          if (live) {
            tl[ca * RB] = ya;
            tl[cc * RB] = yc;
          }
        }
      }
    } else if (kSweep && live) {  // last, partial strip
      float2 ybuf[32];
#pragma unroll
      for (int c = 31; c >= 0; --c) {
        if (c < cols) {
          ybuf[c] = ps_emit_a<AEV>(as, fc);
          ps_advance_a(as, tl[c * RB], fc);
        }
      }
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        if (c < cols) {
          ps_advance_c(cs, tl[c * RB], fc);
          const float2 o = add2(ps_emit_c(cs, fc), ybuf[c]);
          if (live) tl[c * RB] = o;
        }
      }
    }
    GPF_TICK(1);
    // this strip's f tile: the newer group (strip b+1) may stay in flight
    if constexpr (!OTMA) {
      if (kRow2Slots > 1 && b + 1 < nx) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
      else asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    if (OTMA && tid == 0) bulk_wait_read_all();  // the previous strip's store has left O2
    __syncthreads();
    GPF_TICK(2);
    // ---- 2. contraction: pixel p -> (row p & 15, col p >> 4); up to three
    // pixels per thread with interleaved (independent) Horner chains over the
    // plane pairs (contract_px).
    const float2* Ts = T + (size_t)s * slot_elems;
    const Tin* Fs = OTMA ? reinterpret_cast<const Tin*>(F2 + s * RB * 32) : F + s * RB * 33;
#ifdef GPF_DIAG_NO_CONTRACT
    for (int p0 = tid; p0 < 0; p0 += nthr * 3) {
#else
    for (int p0 = tid; p0 < RB * 32; p0 += nthr * 3) {
#endif
      // pixels per thread for this warp (warp-uniform: no work on pixels past the strip)
      const int wb = p0 - lane;
      Tout* Od = OTMA ? reinterpret_cast<Tout*>(O2) : O;
      if (wb + 2 * nthr + 31 < RB * 32)
        my_fb += contract_px<3, NFIX, OTMA, RB>(Ts, Fs, Od, p0, nthr, rows, cols, rc, t_c, sr_f, tc_hi, tc_lo);
      else if (wb + nthr < RB * 32)
        my_fb += contract_px<2, NFIX, OTMA, RB>(Ts, Fs, Od, p0, nthr, rows, cols, rc, t_c, sr_f, tc_hi, tc_lo);
      else
        my_fb += contract_px<1, NFIX, OTMA, RB>(Ts, Fs, Od, p0, nthr, rows, cols, rc, t_c, sr_f, tc_hi, tc_lo);
    }
    GPF_TICK(3);
    if constexpr (OTMA) {
      fence_proxy_async();  // O2 writes -> visible to the TMA store
      __syncthreads();      // slot s, its f tile are free; O2 is complete
      if (tid == 0) {
        if constexpr (GPF_L2HINT & 8) tma_store_3d_hint(&omap, xs, y0, f, O2, l2_evict_first());
        else tma_store_3d(&omap, xs, y0, f, O2);  // clipped to the image
        bulk_commit();
      }
      GPF_TICK(4);
    } else {
      __syncthreads();
      // ---- 3. write-out (row segments of 32, coalesced)
      for (int p = tid; p < RB * 32; p += nthr) {
        const int pr = p >> 5, pc = p & 31;
        if (pr < rows && pc < cols) out[(size_t)(y0 + pr) * w + xs + pc] = O[pr * 33 + pc];
      }
      GPF_TICK(4);
      __syncthreads();  // slot s, its f tile and O are free again
    }
    if (b + kRow2Slots < nx) load_strip(b + kRow2Slots, s);
  }
  if (OTMA && tid == 0) bulk_wait_all();  // the output is complete before the CTA retires
#ifdef GPF_DIAG_CLOCKS
  if ((blockIdx.x == 100 || blockIdx.x == 101 || blockIdx.x == 400) && (tid == 0 || tid == 160))
    printf("cta %d tid %d: waitV %lld sweep %lld fbar %lld contract %lld write %lld load %lld (per strip)\n",
           blockIdx.x, tid, tph[0] / nx, tph[1] / nx, tph[2] / nx, tph[3] / nx, tph[4] / nx,
           tph[5] / nx);
#endif
#undef GPF_TICK
  for (int o = 16; o; o >>= 1) my_fb += __shfl_xor_sync(0xffffffffu, my_fb, o);
  if (lane == 0 && my_fb) atomicAdd(fb_all + f, (unsigned long long)my_fb);
}

}  // namespace gpfb
