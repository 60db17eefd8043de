// FP64 peak microbenchmark for B200 (sm_100a): DFMA (FP64 vector pipe) vs
// DMMA (mma.sync m8n8k4 f64, the FP64 tensor pipe). Used to obtain the FP64
// roofline denominator, which MEASURED_PEAKS.json does not carry.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void dmma_kernel(double* out, int iters, double a, double b) {
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) { c[t][0] = threadIdx.x + t; c[t][1] = 0; }
  double av = a + threadIdx.x * 1e-9, bv = b;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int t = 0; t < 8; ++t) dmma(c[t][0], c[t][1], av, bv);
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int threads : {256, 512, 1024}) {
    for (int bps : {1, 2}) {
      int grid = sms * bps, iters = 4000;
      dfma_kernel<<<grid, threads>>>(out, 10, 0.999999, 1e-7);
      cudaEventRecord(e0);
      dfma_kernel<<<grid, threads>>>(out, iters, 0.999999, 1e-7);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 128 * iters * (double)grid * threads;
      printf("DFMA threads=%d blocks/SM=%d : %.2f TFLOP/s\n", threads, bps, flops / ms / 1e9);
      dmma_kernel<<<grid, threads>>>(out, 10, 0.999999, 1e-7);
      cudaEventRecord(e0);
      dmma_kernel<<<grid, threads>>>(out, iters, 0.999999, 1e-7);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * 256 * 32 * iters * (double)grid * (threads / 32);
      printf("DMMA threads=%d blocks/SM=%d : %.2f TFLOP/s\n", threads, bps, flops / ms / 1e9);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("status: %s, SMs=%d\n", cudaGetErrorString(err), sms);
  return 0;
}
