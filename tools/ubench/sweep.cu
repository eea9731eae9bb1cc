// Sweep-loop microbenchmark: the column-pass recurrence (2 complex sections,
// plane pair in float2) in isolation, to find its achievable FFMA2 rate.
#include <cstdio>
#include <cuda_runtime.h>
struct PS { float2 wr[2], wi[2]; };
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
struct FC { float2 pr[2], pi[2], npi[2], ar[2], nai[2], br[2], nbi[2]; };
__device__ __forceinline__ void adv(PS& s, float2 x, const FC& c) {
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    float2 nr = fma2(c.pr[k], s.wr[k], fma2(c.npi[k], s.wi[k], x));
    float2 ni = fma2(c.pr[k], s.wi[k], mul2(c.pi[k], s.wr[k]));
    s.wr[k] = nr; s.wi[k] = ni;
  }
}
__device__ __forceinline__ float2 emit(const PS& s, const float2* cr, const float2* nci) {
  return fma2(cr[0], s.wr[0], fma2(nci[0], s.wi[0], fma2(cr[1], s.wr[1], mul2(nci[1], s.wi[1]))));
}
template <int MODE>
__global__ void k_sweep(float2* out, FC c, int chunks) {
  extern __shared__ float2 sm[];
  float2* mine = sm + (threadIdx.y * 32 + threadIdx.x) * 33;
  for (int j = 0; j < 32; ++j) mine[j] = make_float2(threadIdx.x * 0.01f + j, j * 0.5f);
  PS as, cs;
  for (int k = 0; k < 2; ++k) { as.wr[k] = as.wi[k] = cs.wr[k] = cs.wi[k] = make_float2(0.1f, 0.2f); }
  for (int it = 0; it < chunks; ++it) {
    float2 xr[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) xr[j] = mine[j];
#pragma unroll
    for (int j = 31; j >= 0; --j) {
      float2 y = emit(as, c.br, c.nbi);
      if (MODE >= 1) mine[j] = y; else xr[j] = add2(xr[j], y);
      adv(as, xr[j], c);
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      adv(cs, xr[j], c);
      float2 y = emit(cs, c.ar, c.nai);
      if (MODE >= 1) mine[j] = add2(y, mine[j]); else xr[j] = add2(xr[j], y);
    }
    if (MODE == 2) __syncthreads();
  }
  out[blockIdx.x * blockDim.x * blockDim.y + threadIdx.y * 32 + threadIdx.x] = add2(as.wr[0], cs.wi[1]);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  FC c;
  for (int k = 0; k < 2; ++k) { c.pr[k] = make_float2(0.7f, 0.7f); c.pi[k] = make_float2(0.1f, 0.1f); c.npi[k] = make_float2(-0.1f, -0.1f);
    c.ar[k] = make_float2(0.3f, 0.3f); c.nai[k] = make_float2(-0.2f, -0.2f); c.br[k] = make_float2(0.25f, 0.25f); c.nbi[k] = make_float2(0.1f, 0.1f); }
  float2* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int chunks = 256;
  for (int mode = 0; mode < 3; ++mode)
  for (int warps : {4, 8, 11, 16}) {
    for (int ctas_per_sm : {1, 2}) {
      dim3 blk(32, warps);
      size_t smem = warps * 32 * 33 * 8;
      auto k = mode == 0 ? k_sweep<0> : (mode == 1 ? k_sweep<1> : k_sweep<2>);
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
      k<<<sms * ctas_per_sm, blk, smem>>>(out, c, 4);
      cudaEventRecord(e0);
      k<<<sms * ctas_per_sm, blk, smem>>>(out, c, chunks);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ffma2 = (double)sms * ctas_per_sm * warps * chunks * 64 * 12;  // warp-FFMA2 (64 steps x 12)
      double clk = ms * 1e-3 * 1.965e9;
      printf("mode %d warps %2d ctas/sm %d: %.3f ms  FFMA2/clk/SM %.2f (peak 2.0)  err %s\n", mode, warps, ctas_per_sm, ms,
             ffma2 / clk / sms, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
