// Which SMSP (hardware warp slot % 4) does warp w of each co-resident CTA land on?
#include <cstdio>
__global__ void __launch_bounds__(256, 2) k(int* out) {
  extern __shared__ double sm[];
  unsigned wid, smid;
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if ((threadIdx.x & 31) == 0) {
    int w = threadIdx.x >> 5;
    out[(blockIdx.x * 8 + w) * 2] = smid;
    out[(blockIdx.x * 8 + w) * 2 + 1] = wid;
  }
  long long t0 = clock64();
  while (clock64() - t0 < 2000000) {}
  sm[threadIdx.x] = 1.0;
}
int main() {
  int* o; cudaMallocManaged(&o, 4 * 2 * 8 * 296);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
  k<<<296, 256, 110 * 1024>>>(o); cudaDeviceSynchronize();
  int bad = 0, shown = 0;
  for (int b = 0; b < 296; ++b) {
    int ok = 1;
    for (int w = 0; w < 8; ++w) if (o[(b * 8 + w) * 2 + 1] % 4 != w % 4) ok = 0;
    if (!ok) { ++bad; if (shown++ < 4) { printf("cta %d sm %d slots:", b, o[b * 16]); for (int w = 0; w < 8; ++w) printf(" %d", o[(b * 8 + w) * 2 + 1]); printf("\n"); } }
  }
  printf("CTAs whose warp w is not on slot%%4 == w%%4: %d of 296 (%s)\n", bad, cudaGetErrorString(cudaGetLastError()));
  for (int b = 0; b < 4; ++b) { printf("cta %d sm %d slots:", b, o[b * 16]); for (int w = 0; w < 8; ++w) printf(" %d", o[(b * 8 + w) * 2 + 1]); printf("\n"); }
}
