// Single-warp FP64 issue/latency probes on B200 (what bounds a panel factorisation).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dep(double* out, long long* cyc, int n, double a, double b) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_indep(double* out, long long* cyc, int n, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (threadIdx.x == 0) cyc[1] = t1 - t0;
}
__global__ void k_sqrtdiv(double* out, long long* cyc, int n) {
  double x = 2.0 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = sqrt(x) + 1.0; x = 1.0 / x + 2.0; }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[2] = t1 - t0;
}
__global__ void k_shfl(double* out, long long* cyc, int n) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x += __shfl_xor_sync(0xffffffffu, x, 1); x += __shfl_xor_sync(0xffffffffu, x, 2); }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[3] = t1 - t0;
}
__global__ void k_smem_rt(double* out, long long* cyc, int n) {
  __shared__ double s[64];
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if ((threadIdx.x & 3) == 0) s[threadIdx.x >> 2] = x;
    __syncwarp();
    x += s[(threadIdx.x + 1) & 7];
    __syncwarp();
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[4] = t1 - t0;
}
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__global__ void k_dmma_dep(double* out, long long* cyc, int n) {
  double d[2] = {1.0, 2.0};
  double a = threadIdx.x * 1e-3, b = 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { dmma(d, a, b); dmma(d, a, b); dmma(d, a, b); dmma(d, a, b); }
  long long t1 = clock64();
  out[threadIdx.x] = d[0] + d[1];
  if (threadIdx.x == 0) cyc[5] = t1 - t0;
}
__global__ void k_dmma_ind(double* out, long long* cyc, int n) {
  double d[8][2] = {};
  double a = threadIdx.x * 1e-3, b = 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) dmma(d[k], a, b);
  }
  long long t1 = clock64();
  double s = 0; for (int k = 0; k < 8; ++k) s += d[k][0] + d[k][1];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[6] = t1 - t0;
}

int main() {
  double* out; long long* cyc; cudaMalloc(&out, 4096 * 8); cudaMallocManaged(&cyc, 64 * 8);
  const int n = 10000;
  for (int w = 0; w < 2; ++w) {
    k_dep<<<1, 32>>>(out, cyc, n, 0.9999, 1e-3);
    k_indep<<<1, 32>>>(out, cyc, n, 0.9999, 1e-3);
    k_sqrtdiv<<<1, 32>>>(out, cyc, n);
    k_shfl<<<1, 32>>>(out, cyc, n);
    k_smem_rt<<<1, 32>>>(out, cyc, n);
    k_dmma_dep<<<1, 32>>>(out, cyc, n);
    k_dmma_ind<<<1, 32>>>(out, cyc, n);
    cudaDeviceSynchronize();
  }
  printf("DFMA dependent latency      : %.2f cycles\n", cyc[0] / (4.0 * n));
  printf("DFMA independent issue (1 warp): %.2f cycles/instr\n", cyc[1] / (8.0 * n));
  printf("sqrt+div dependent pair     : %.2f cycles\n", cyc[2] / (1.0 * n));
  printf("shfl_xor(double)+add x2     : %.2f cycles per step\n", cyc[3] / (2.0 * n));
  printf("smem store/syncwarp/load rt : %.2f cycles\n", cyc[4] / (1.0 * n));
  printf("DMMA dependent latency      : %.2f cycles\n", cyc[5] / (4.0 * n));
  printf("DMMA independent issue (1 warp): %.2f cycles/instr\n", cyc[6] / (8.0 * n));
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
