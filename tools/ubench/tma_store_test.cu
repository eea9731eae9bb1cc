// Checks a 5-D TMA tensor store with non-monotonic global strides and
// SWIZZLE_128B: smem [pair][half][col][32 floats] -> V[pair][col][2*h_pad]
// (rows y0..y0+31 of 32 columns), the layout the column pass stages.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_store(const __grid_constant__ CUtensorMap map, int x0, int y0, int pairs) {
  extern __shared__ __align__(1024) unsigned char raw[];
  float* st = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  // element (g, c, row j, plane e) -> value g*1e6 + (x0+c)*1e3 + (y0+j) + 0.5*e  (approx, exact in fp32 for small)
  for (int idx = threadIdx.x; idx < pairs * 32 * 32; idx += blockDim.x) {
    const int g = idx / 1024, c = (idx / 32) % 32, j = idx % 32;
    const int half = j >> 4, q = (j & 15) >> 1, sub = j & 1;
    const int R = (g * 2 + half) * 32 + c;          // 128-B row index in the box
    const int chunk = q ^ (R & 7);                  // 128B swizzle
    float* dst = st + R * 32 + chunk * 4 + sub * 2;
    dst[0] = g * 100000.f + c * 100.f + j;          // plane 2g
    dst[1] = -(g * 100000.f + c * 100.f + j);       // plane 2g+1
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile(
        "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];\n" ::"l"(&map),
        "r"(0), "r"(x0), "r"(y0 / 16), "r"(0), "r"(0), "r"(su32(st))
        : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  }
}

int main() {
  const int w = 96, h_pad = 64, pairs = 3, x0 = 32, y0 = 32;
  float* V;
  cudaMalloc(&V, sizeof(float) * pairs * w * 2 * h_pad);
  cudaMemset(V, 0, sizeof(float) * pairs * w * 2 * h_pad);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<decltype(&cuTensorMapEncodeTiled)>(fn);
  CUtensorMap map;
  cuuint64_t dims[5] = {32, (cuuint64_t)w, (cuuint64_t)(h_pad / 16), (cuuint64_t)pairs, 1};
  cuuint64_t strides[4] = {(cuuint64_t)2 * h_pad * 4, 128, (cuuint64_t)w * 2 * h_pad * 4,
                           (cuuint64_t)pairs * w * 2 * h_pad * 4};
  cuuint32_t box[5] = {32, 32, 2, (cuuint32_t)pairs, 1};
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, V, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)r);
  if (r != CUDA_SUCCESS) return 1;
  const int smem = pairs * 32 * 32 * 8 + 1024;
  cudaFuncSetAttribute(k_store, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_store<<<1, 256, smem>>>(map, x0, y0, pairs);
  printf("kernel: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  std::vector<float> hv((size_t)pairs * w * 2 * h_pad);
  cudaMemcpy(hv.data(), V, hv.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0, good = 0;
  for (int g = 0; g < pairs; ++g)
    for (int c = 0; c < w; ++c)
      for (int j = 0; j < h_pad; ++j) {
        const float* e = &hv[(((size_t)g * w + c) * h_pad + j) * 2];
        const bool inbox = c >= x0 && c < x0 + 32 && j >= y0 && j < y0 + 32;
        const float want = inbox ? g * 100000.f + (c - x0) * 100.f + (j - y0) : 0.f;
        if (e[0] != want || e[1] != (inbox ? -want : 0.f)) {
          if (bad < 5) printf("mismatch g%d c%d j%d: %f %f want %f\n", g, c, j, e[0], e[1], want);
          ++bad;
        } else if (inbox) ++good;
      }
  printf("bad %d good %d (expect %d)\n", bad, good, pairs * 32 * 32);
  return bad != 0;
}
