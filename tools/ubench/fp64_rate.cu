// fp64 pipe on sm_100a: issue rate of DFMA / DMUL+DADD with independent chains
// and the latency of a dependent DADD chain (sizes the fp64 mode's floor).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_rate fp64_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE, int CH>
__global__ void k(double* out, int iters, double a, double b) {
  double v[CH];
  for (int i = 0; i < CH; ++i) v[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (MODE == 0) v[i] = __fma_rn(v[i], a, b);
      else if (MODE == 1) v[i] = __dadd_rn(__dmul_rn(v[i], a), b);
      else v[i] = __dadd_rn(v[i], b);
    }
  }
  double s = 0;
  for (int i = 0; i < CH; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE, int CH>
void run(const char* name, int threads, int ctas_per_sm, int ops_per_iter) {
  double* d;
  const int blocks = 148 * ctas_per_sm;
  cudaMalloc(&d, sizeof(double) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  k<MODE, CH><<<blocks, threads>>>(d, 100, 1.0000001, 1e-9);
  cudaEventRecord(e0);
  k<MODE, CH><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double instr = (double)blocks * threads / 32 * iters * CH * ops_per_iter;
  const double cyc = ms * 1e-3 * 1.9e9;
  printf("%-28s thr %4d x %d/SM chains %2d: %.3f ms, %.2f cycles per warp-instr per scheduler (at 1.9 GHz), %.2f T instr-lanes/s\n",
         name, threads, ctas_per_sm, CH, ms, cyc / (instr / (148.0 * 4)), instr * 32 / (ms * 1e-3) / 1e12);
  cudaFree(d);
}

int main() {
  run<0, 8>("DFMA independent", 256, 4, 1);
  run<1, 8>("DMUL+DADD independent", 256, 4, 2);
  run<2, 8>("DADD independent", 256, 4, 1);
  run<2, 1>("DADD dependent chain", 32, 1, 1);
  run<1, 1>("DMUL->DADD dependent", 32, 1, 2);
  run<1, 2>("DMUL+DADD 2 chains, 3 warps", 96, 3, 2);
  run<1, 2>("DMUL+DADD 2 chains, 4 warps", 128, 4, 2);
  // occupancy x ILP grid (independent dependent-chains per thread; warps per SM = thr/32 * CTAs)
  run<1, 1>("grid: 1 chain", 128, 1, 2);
  run<1, 2>("grid: 2 chains", 128, 1, 2);
  run<1, 4>("grid: 4 chains", 128, 1, 2);
  run<1, 8>("grid: 8 chains", 128, 1, 2);
  run<1, 1>("grid: 1 chain", 128, 2, 2);
  run<1, 2>("grid: 2 chains", 128, 2, 2);
  run<1, 4>("grid: 4 chains", 128, 2, 2);
  run<1, 8>("grid: 8 chains", 128, 2, 2);
  run<1, 1>("grid: 1 chain", 128, 4, 2);
  run<1, 4>("grid: 4 chains", 128, 4, 2);
  run<1, 1>("grid: 1 chain", 128, 8, 2);
  run<1, 2>("grid: 2 chains", 128, 8, 2);
  return 0;
}
