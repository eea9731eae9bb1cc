// Device helpers shared by the GPF kernels.
#pragma once

#include <cuda_runtime.h>

#include "gpf_internal.h"

namespace gpfb {

// ---------------------------------------------------------------- prologue
// Per-pixel range terms (bilateral.cpp:92-101), fp64 like the reference:
//   h = f - t_c,  H = h/sr,  E = exp(-h^2 / 2 sr^2)
// packed for the fp32 plane chain: es = E 2^s0, m = H 2^-k, so that
// plane n (scaled by 2^{s0 - k n}) = es * m^n.
__device__ __forceinline__ float2 pixel_terms(double f, double t_c, const RangeConsts& rc) {
  const double h = f - t_c;
  float2 r;
  r.x = static_cast<float>(exp(-(h * h) * rc.inv2s2) * rc.e_scale);
  r.y = static_cast<float>(h * rc.inv_sr) * rc.h_step;
  return r;
}

// Planes (2g, 2g+1) of a pixel from its terms; g is warp-uniform.
__device__ __forceinline__ float2 pair_planes(float2 t, int g) {
  float base = t.y * t.y, acc = t.x;
  for (int e = g; e; e >>= 1) {
    if (e & 1) acc *= base;
    base *= base;
  }
  return make_float2(acc, acc * t.y);
}

// ------------------------------------------------------- IIR section state
// Two complex first-order sections (k) for the two planes (q) of a pair.
struct PairState {
  float wr[2][2], wi[2][2];  // [plane q][section k]
};

__device__ __forceinline__ void ps_set_gain(PairState& s, float2 x, const FilterConsts& fc) {
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    s.wr[0][k] = x.x * fc.gr[k];
    s.wi[0][k] = x.x * fc.gi[k];
    s.wr[1][k] = x.y * fc.gr[k];
    s.wi[1][k] = x.y * fc.gi[k];
  }
}

// w <- p w + x
__device__ __forceinline__ void ps_advance(PairState& s, float2 x, const FilterConsts& fc) {
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

// sum_k Re(c_k w_k)
__device__ __forceinline__ float2 ps_emit(const PairState& s, const float* cr, const float* ci) {
  float2 o;
  o.x = fmaf(cr[0], s.wr[0][0], fmaf(-ci[0], s.wi[0][0], fmaf(cr[1], s.wr[0][1], -ci[1] * s.wi[0][1])));
  o.y = fmaf(cr[0], s.wr[1][0], fmaf(-ci[0], s.wi[1][0], fmaf(cr[1], s.wr[1][1], -ci[1] * s.wi[1][1])));
  return o;
}

// Carry record: the 8 floats of a PairState, stored as two float4.
__device__ __forceinline__ void ps_store(float4* dst, const PairState& s) {
  dst[0] = make_float4(s.wr[0][0], s.wi[0][0], s.wr[0][1], s.wi[0][1]);
  dst[1] = make_float4(s.wr[1][0], s.wi[1][0], s.wr[1][1], s.wi[1][1]);
}

__device__ __forceinline__ void ps_load(PairState& s, const float4* src) {
  const float4 a = src[0], b = src[1];
  s.wr[0][0] = a.x; s.wi[0][0] = a.y; s.wr[0][1] = a.z; s.wi[0][1] = a.w;
  s.wr[1][0] = b.x; s.wi[1][0] = b.y; s.wr[1][1] = b.z; s.wi[1][1] = b.w;
}

// s <- agg + P s  with P = p^L per section (complex), applied to both planes.
__device__ __forceinline__ void ps_chain(PairState& s, const PairState& agg, const float* plr,
                                         const float* pli) {
#pragma unroll
  for (int k = 0; k < 2; ++k) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const float nr = fmaf(plr[k], s.wr[q][k], fmaf(-pli[k], s.wi[q][k], agg.wr[q][k]));
      const float ni = fmaf(plr[k], s.wi[q][k], fmaf(pli[k], s.wr[q][k], agg.wi[q][k]));
      s.wr[q][k] = nr;
      s.wi[q][k] = ni;
    }
  }
}

// agg += w_j x  (complex weight per section, real input per plane)
__device__ __forceinline__ void ps_accum(PairState& a, float2 x, float w0r, float w0i, float w1r,
                                         float w1i) {
  a.wr[0][0] = fmaf(w0r, x.x, a.wr[0][0]);
  a.wi[0][0] = fmaf(w0i, x.x, a.wi[0][0]);
  a.wr[1][0] = fmaf(w0r, x.y, a.wr[1][0]);
  a.wi[1][0] = fmaf(w0i, x.y, a.wi[1][0]);
  a.wr[0][1] = fmaf(w1r, x.x, a.wr[0][1]);
  a.wi[0][1] = fmaf(w1i, x.x, a.wi[0][1]);
  a.wr[1][1] = fmaf(w1r, x.y, a.wr[1][1]);
  a.wi[1][1] = fmaf(w1i, x.y, a.wi[1][1]);
}

__device__ __forceinline__ void ps_zero(PairState& s) {
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int k = 0; k < 2; ++k) s.wr[q][k] = s.wi[q][k] = 0.f;
}

}  // namespace gpfb
