// K4: row pass (deriche_line over rows, spatial.cpp:235-239) on V, fused with
// the P/Q recombination and normalisation (bilateral.cpp:117-148).
// Included by gpf_kernels.cu (needs its cp.async helpers and issue_f_tile).
//
// Thread (row lane, pair g); a CTA covers 32 rows and walks them strip by
// strip (32 columns). Only ONE chunk-sized copy lives on chip: the strip's V
// inputs are streamed from global memory twice -- the anticausal sweep reads
// them from HBM, the causal sweep re-reads the same 256-byte rows from L2 a
// few microseconds later -- and smem holds only the anticausal outputs, which
// the causal sweep turns into Fbar in place. That keeps the CTA at ~100 KB of
// smem and few registers, so two CTAs share an SM and one CTA's sweeps
// overlap the other's contraction and stores.
//
// Per strip: anticausal sweep from the K3 carry, causal sweep (state carried
// across strips), then every pixel of the strip contracts its N+2 planes:
//   Q = sum_{n<=N} c_n Fbar_n,  P = sum_{n<=N} c_n Fbar_{n+1},  c_n = H^n/n!
// (weights and planes carry compensating 2^{-+s_n} scalings).
#pragma once

namespace gpfb {

constexpr int kRowPf = 4;  // prefetch depth of the streamed V columns

// Pulls the 256-byte V rows of a strip (and its f rows) into L2 ahead of use.
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes));
}

template <int MAXT, typename Tin, typename Tout>
__global__ void __launch_bounds__(MAXT, 2) k_rowpass(const Tin* __restrict__ in_all,
                                                     const double* __restrict__ scalars,
                                                     const float2* __restrict__ V_all,
                                                     const float4* __restrict__ CH_all,
                                                     Tout* __restrict__ out_all,
                                                     unsigned long long* __restrict__ fb_all,
                                                     int w, int h, int h_pad, int nx,
                                                     FilterConsts fc, RangeConsts rc) {
  extern __shared__ float4 smem4[];
  const int f = blockIdx.y, lane = threadIdx.x, g = threadIdx.y, pairs = blockDim.y;
  const int nthr = 32 * pairs, tid = g * 32 + lane;
  const int y0 = blockIdx.x * 32, y = y0 + lane;
  const int rows = min(32, h - y0);
  float2* tile = reinterpret_cast<float2*>(smem4);                                  // [g][x][32 rows]
  Tin* ftile = reinterpret_cast<Tin*>(tile + (size_t)pairs * 32 * 32);             // [32 rows][33]
  Tout* otile = reinterpret_cast<Tout*>(ftile + 32 * 33);                           // [32 rows][33]
  __shared__ unsigned fb_shared;
  if (tid == 0) fb_shared = 0;

  const Tin* in = in_all + (size_t)f * w * h;
  Tout* out = out_all + (size_t)f * w * h;
  // this thread's V column stream: V[g][x][y], consecutive x are h_pad apart
  const float2* vcol = V_all + (size_t)f * pairs * w * h_pad + (size_t)g * w * h_pad + y;
  const float4* CH = CH_all + (size_t)f * nx * pairs * h * 2 + (size_t)g * h * 2 + (size_t)y * 2;
  const size_t ch_stride = (size_t)pairs * h * 2;
  const double t_c = scalars[2 * f];
  float2* tl = tile + (size_t)g * 32 * 32 + lane;  // element [g][x][lane] = tl[x * 32]

  PairState cs;
  ps_zero(cs);
  unsigned my_fb = 0;
  for (int b = 0; b < nx; ++b) {
    const int xs = b * 32, cols = min(32, w - xs);
    issue_f_tile(ftile, in, w, h, xs, y0);
    cp_async_commit();
    if (b + 1 < nx) {  // next strip's V column (thread lane = column) into L2
      const int xn = xs + 32 + lane;
      if (xn < w)
        prefetch_l2(V_all + (size_t)f * pairs * w * h_pad + ((size_t)g * w + xn) * h_pad + y0, 256);
    }
    if (lane < rows) {
      const float2* src = vcol + (size_t)xs * h_pad;
      PairState as;
      ps_load(as, CH + (size_t)b * ch_stride);
      if (cols == 32) {
        // anticausal, right to left, HBM stream with a kRowPf-deep prefetch
        float2 q[kRowPf];
#pragma unroll
        for (int i = 0; i < kRowPf; ++i) q[i] = __ldg(src + (size_t)(31 - i) * h_pad);
#pragma unroll
        for (int c = 31; c >= 0; --c) {
          const float2 xv = q[(31 - c) % kRowPf];
          if (c - kRowPf >= 0) q[(31 - c) % kRowPf] = __ldg(src + (size_t)(c - kRowPf) * h_pad);
          tl[c * 32] = ps_emit(as, fc.br2, fc.nbi2);
          ps_advance(as, xv, fc);
        }
        // causal, left to right, the same rows again (L2 hits)
#pragma unroll
        for (int i = 0; i < kRowPf; ++i) q[i] = __ldg(src + (size_t)i * h_pad);
        if (b == 0) ps_set_gain(cs, q[0], fc);
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float2 xv = q[c % kRowPf];
          if (c + kRowPf < 32) q[c % kRowPf] = __ldg(src + (size_t)(c + kRowPf) * h_pad);
          ps_advance(cs, xv, fc);
          tl[c * 32] = add2(ps_emit(cs, fc.ar2, fc.nai2), tl[c * 32]);
        }
      } else {  // last, partial strip
        for (int c = cols - 1; c >= 0; --c) {
          tl[c * 32] = ps_emit(as, fc.br2, fc.nbi2);
          ps_advance(as, __ldg(src + (size_t)c * h_pad), fc);
        }
        if (b == 0) ps_set_gain(cs, __ldg(src), fc);
        for (int c = 0; c < cols; ++c) {
          ps_advance(cs, __ldg(src + (size_t)c * h_pad), fc);
          tl[c * 32] = add2(ps_emit(cs, fc.ar2, fc.nai2), tl[c * 32]);
        }
      }
    }
    cp_async_wait_all();
    __syncthreads();
    // contraction: pixel (row r = p & 31, col c = p >> 5); (Q, P) packed
    for (int p = tid; p < 1024; p += nthr) {
      const int r = p & 31, c = p >> 5;
      if (r < rows && c < cols) {
        const double fv = static_cast<double>(ftile[r * 33 + c]);
        const float Hf = static_cast<float>((fv - t_c) * rc.inv_sr);
        float cc = rc.c0;
        float2 qp = make_float2(0.f, 0.f);  // (Q, P)
        const float2* col = tile + (size_t)c * 32 + r;
        float2 cur2 = col[0];
        // pairs g with both n = 2g and 2g+1 <= N; pair `full` always exists
        const int full = (rc.degree + 1) >> 1;
#pragma unroll 4
        for (int gg = 0; gg < full; ++gg) {
          const float2 nxt = col[(size_t)(gg + 1) * 1024];
          qp = fma2(f2(cc), cur2, qp);
          cc = cc * (Hf * rc.w_step[2 * gg]);
          qp = fma2(f2(cc), make_float2(cur2.y, nxt.x), qp);
          cc = cc * (Hf * rc.w_step[2 * gg + 1]);
          cur2 = nxt;
        }
        if (!(rc.degree & 1)) qp = fma2(f2(cc), cur2, qp);  // n = N (even N)
        double o;
        if (!(fabsf(qp.x) > rc.q_thresh)) {
          o = fv;
          ++my_fb;
        } else {
          o = rc.sigma_r * ((static_cast<double>(qp.y) * rc.p_scale) / static_cast<double>(qp.x)) + t_c;
        }
        otile[r * 33 + c] = static_cast<Tout>(o);
      }
    }
    __syncthreads();
    for (int p = tid; p < 1024; p += nthr) {
      const int r = p >> 5, c = p & 31;
      if (r < rows && c < cols) out[(size_t)(y0 + r) * w + xs + c] = otile[r * 33 + c];
    }
    // the next strip's sweeps write `tile` and its f-tile load writes `ftile`:
    // both were last read above, before the barrier; otile is read here and
    // next written after the next strip's first barrier.
  }
  if (my_fb) atomicAdd(&fb_shared, my_fb);
  __syncthreads();
  if (tid == 0 && fb_shared) atomicAdd(fb_all + f, (unsigned long long)fb_shared);
}

}  // namespace gpfb
