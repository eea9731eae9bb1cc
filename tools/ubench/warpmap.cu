// Which SM sub-partition (warpid % 4) do the warps of co-resident CTAs get?
#include <cstdio>
#include <vector>
#include <map>
__global__ void k(int* out, int iters) {
  unsigned smid, wid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
  if (threadIdx.x % 32 == 0) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
    out[2 * w] = smid;
    out[2 * w + 1] = wid;
  }
  // keep the CTA resident a while so the next ones co-reside
  long long t0 = clock64();
  while (clock64() - t0 < iters) {}
}
int main() {
  int* d; cudaMalloc(&d, 1 << 24);
  for (int wpc : {3, 4, 6}) {
    const int ctas = 148 * 4, nw = ctas * wpc;
    k<<<ctas, 32 * wpc>>>(d, 2000000);
    cudaDeviceSynchronize();
    std::vector<int> h(2 * nw);
    cudaMemcpy(h.data(), d, 8 * nw, cudaMemcpyDeviceToHost);
    // per SM: count warps per sub-partition among the first-wave warps
    std::map<int, std::vector<int>> per;
    for (int w = 0; w < nw; ++w) per[h[2 * w]].push_back(h[2 * w + 1]);
    int shown = 0;
    for (auto& [sm, ws] : per) {
      int cnt[4] = {0, 0, 0, 0};
      for (int x : ws) cnt[x % 4]++;
      if (shown++ < 4) {
        printf("wpc %d sm %3d: %zu warps, per-SMSP %d %d %d %d | ids", wpc, sm, ws.size(), cnt[0], cnt[1], cnt[2], cnt[3]);
        for (size_t i = 0; i < ws.size() && i < 24; ++i) printf(" %d", ws[i]);
        printf("\n");
      }
    }
  }
  return 0;
}
