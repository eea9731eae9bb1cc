// Microbenchmarks for design decisions: FP32 FFMA vs packed FFMA2 vs FP64 DFMA
// issue throughput, and HBM streaming bandwidth. Run on a B200 via gpurun.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CH>
__global__ void k_ffma(float* out, float a, float b, int iters) {
  float x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fmaf(x[c], a, b);
  }
  float s = 0; for (int c = 0; c < CH; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 3 distinct register operands (no constants) to probe the RF-bank limit
template <int CH>
__global__ void k_ffma_rrr(float* out, const float* ab, int iters) {
  float x[CH], y[CH];
  float a = ab[threadIdx.x & 1];
#pragma unroll
  for (int c = 0; c < CH; ++c) { x[c] = threadIdx.x * 1e-3f + c; y[c] = c * 0.5f; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fmaf(x[c], a, y[c]);
  }
  float s = 0; for (int c = 0; c < CH; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long pk(float lo, float hi) {
  return (unsigned long long)__float_as_uint(lo) | ((unsigned long long)__float_as_uint(hi) << 32);
}

template <int CH>
__global__ void k_ffma2(float* out, const float* ab, int iters) {
  unsigned long long x[CH], y[CH];
  unsigned long long a = pk(ab[threadIdx.x & 1], ab[(threadIdx.x + 1) & 1]);
#pragma unroll
  for (int c = 0; c < CH; ++c) { x[c] = pk(threadIdx.x * 1e-3f + c, c); y[c] = pk(c * 0.5f, c * 0.25f); }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = ffma2(x[c], a, y[c]);
  }
  float s = 0; for (int c = 0; c < CH; ++c) s += __uint_as_float((unsigned)x[c]) + __uint_as_float((unsigned)(x[c] >> 32));
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CH>
__global__ void k_dfma(double* out, const double* ab, int iters) {
  double x[CH], y[CH];
  double a = ab[threadIdx.x & 1];
#pragma unroll
  for (int c = 0; c < CH; ++c) { x[c] = threadIdx.x * 1e-3 + c; y[c] = c * 0.5; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, y[c]);
  }
  double s = 0; for (int c = 0; c < CH; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_copy(const float4* __restrict__ in, float4* __restrict__ out, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) out[i] = in[i];
}
__global__ void k_read(const float4* __restrict__ in, float* out, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  float s = 0;
  for (; i < n; i += stride) { float4 v = in[i]; s += v.x + v.y + v.z + v.w; }
  if (s == 123.f) out[0] = s;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int clk; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  printf("SMs %d clock %d kHz\n", sms, clk);
  float* fo; double* dout; float* fab; double* dab;
  CK(cudaMalloc(&fo, 1 << 24)); CK(cudaMalloc(&dout, 1 << 25));
  CK(cudaMalloc(&fab, 64)); CK(cudaMalloc(&dab, 64));
  float hab[2] = {0.999f, 0.5f}; double dhab[2] = {0.999, 0.5};
  CK(cudaMemcpy(fab, hab, 8, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dab, dhab, 16, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096; const int blocks = sms * 4, threads = 256;
  auto timeit = [&](auto launch, double ops_per_thread_iter, const char* name) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    double ops = ops_per_thread_iter * iters * (double)blocks * threads;
    printf("%-28s %8.3f ms  %8.2f Tops/s  (%.1f ops/clk/SM at nominal clk)\n", name, ms, ops / ms / 1e9,
           ops / (ms * 1e-3) / sms / (clk * 1e3));
  };
  timeit([&] { k_ffma<16><<<blocks, threads>>>(fo, 0.999f, 0.5f, iters); }, 16, "FFMA imm/const 16ch");
  timeit([&] { k_ffma_rrr<16><<<blocks, threads>>>(fo, fab, iters); }, 16, "FFMA reg 16ch");
  timeit([&] { k_ffma_rrr<32><<<blocks, threads>>>(fo, fab, iters); }, 32, "FFMA reg 32ch");
  timeit([&] { k_ffma2<8><<<blocks, threads>>>(fo, fab, iters); }, 16, "FFMA2 reg 8ch (x2 lanes)");
  timeit([&] { k_ffma2<16><<<blocks, threads>>>(fo, fab, iters); }, 32, "FFMA2 reg 16ch (x2 lanes)");
  timeit([&] { k_dfma<16><<<blocks, threads>>>(dout, dab, iters); }, 16, "DFMA reg 16ch");
  size_t n = (size_t)1 << 28;  // 1 GiB of floats per buffer
  float4 *a, *b; CK(cudaMalloc(&a, n * 4)); CK(cudaMalloc(&b, n * 4));
  cudaMemset(a, 0, n * 4);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); k_copy<<<sms * 8, 512>>>(a, b, n / 4); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy 1GiB: %.3f ms  %.1f GB/s (r+w)\n", ms, 2.0 * n * 4 / ms / 1e6);
    cudaEventRecord(e0); k_read<<<sms * 8, 512>>>(a, fo, n / 4); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("read 1GiB: %.3f ms  %.1f GB/s\n", ms, 1.0 * n * 4 / ms / 1e6);
  }
  CK(cudaGetLastError());
  return 0;
}
