// Compares the packed and scalar contraction loops on identical inputs.
#include <cstdio>
#include <cmath>
struct RC { float c0; float w_step[64]; float2 w_pair[64]; };
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }
__global__ void k(const float2* T, const float* H, float4* out, RC rc) {
  const int t = threadIdx.x;
  const float Hf = H[t];
  const float2* col = T + t * 11;
  // packed
  float2 cur = col[0];
  float2 qp = make_float2(rc.c0 * cur.x, 0.f), W = make_float2(rc.c0 * (Hf * rc.w_step[0]), rc.c0);
#pragma unroll
  for (int m = 1; m <= 20; m += 2) {
    qp = fma2(W, f2(cur.y), qp);
    W = mul2(W, mul2(f2(Hf), rc.w_pair[m]));
    cur = col[(m + 1) >> 1];
    qp = fma2(W, f2(cur.x), qp);
    W = mul2(W, mul2(f2(Hf), rc.w_pair[m + 1]));
  }
  qp.y = fmaf(W.y, cur.y, qp.y);
  // scalar
  float2 cur2 = col[0];
  float2 qs = make_float2(rc.c0 * cur2.x, 0.f);
  float cq = rc.c0 * (Hf * rc.w_step[0]), cp = rc.c0;
#pragma unroll
  for (int m = 1; m <= 20; m += 2) {
    qs.x = fmaf(cq, cur2.y, qs.x);
    qs.y = fmaf(cp, cur2.y, qs.y);
    cp = cq;
    cq *= Hf * rc.w_step[m];
    cur2 = col[(m + 1) >> 1];
    qs.x = fmaf(cq, cur2.x, qs.x);
    qs.y = fmaf(cp, cur2.x, qs.y);
    cp = cq;
    cq *= Hf * rc.w_step[m + 1];
  }
  qs.y = fmaf(cp, cur2.y, qs.y);
  out[t] = make_float4(qp.x, qp.y, qs.x, qs.y);
}
int main() {
  RC rc; rc.c0 = 1.f;
  for (int n = 0; n < 64; ++n) rc.w_step[n] = 4.f / (n + 1);
  rc.w_pair[0] = make_float2(rc.w_step[0], 0.f);
  for (int n = 1; n < 64; ++n) rc.w_pair[n] = make_float2(rc.w_step[n], rc.w_step[n - 1]);
  const int N = 32;
  float2 hT[N * 11]; float hH[N];
  for (int i = 0; i < N * 11; ++i) hT[i] = make_float2(0.3f + 0.01f * i, 0.7f - 0.002f * i);
  for (int i = 0; i < N; ++i) hH[i] = -1.1f + 0.07f * i;
  float2* dT; float* dH; float4* dO;
  cudaMalloc(&dT, sizeof(hT)); cudaMalloc(&dH, sizeof(hH)); cudaMalloc(&dO, N * sizeof(float4));
  cudaMemcpy(dT, hT, sizeof(hT), cudaMemcpyHostToDevice); cudaMemcpy(dH, hH, sizeof(hH), cudaMemcpyHostToDevice);
  k<<<1, N>>>(dT, dH, dO, rc);
  float4 hO[N]; cudaMemcpy(hO, dO, sizeof(hO), cudaMemcpyDeviceToHost);
  for (int i = 0; i < 6; ++i) printf("H %6.3f packed Q %12.6g P %12.6g | scalar Q %12.6g P %12.6g\n", hH[i], hO[i].x, hO[i].y, hO[i].z, hO[i].w);
  return 0;
}
