// Latency floor of one Householder column step's dependency chain (8 warps).
#include <cstdio>
__device__ __forceinline__ double rcp_nr(double x) {
  double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0); r = fma(r, e, r); e = fma(-x, r, 1.0); return fma(r, e, r);
}
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double h = 0.5 * x; y = y * fma(-h * y, y, 1.5); return y * fma(-h * y, y, 1.5);
}
template <int MODE>
__global__ void k(double* out, long long* cyc, int reps) {
  __shared__ double P[2][8][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double v = 1.0 + lane * 1e-3 + warp * 1e-4;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    double d = v * v;
    if (MODE & 1) { d += __shfl_xor_sync(0xffffffffu, d, 1); d += __shfl_xor_sync(0xffffffffu, d, 2); }
    if (MODE & 2) {
      double* Pj = &P[r & 1][0][0];
      if (t == 0) Pj[warp * 8 + g] = d;
      __syncthreads();
      double s = 0; for (int w = 0; w < 8; ++w) s += Pj[w * 8 + g];
      d = s;
    }
    if (MODE & 4) {
      const double s2 = fma(v, v, d);
      const double rn = rsqrt_nr(s2);
      const double nrm = s2 * rn;
      const double sc = rcp_nr(v + nrm);
      d = fma(nrm, sc, rn);
    }
    v = fma(1e-9, d, v);
  }
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
}
template <int MODE>
void run(const char* nm) {
  double* o; long long* c; cudaMalloc(&o, 8192); cudaMallocManaged(&c, 64);
  k<MODE><<<1, 256>>>(o, c, 2000); cudaDeviceSynchronize();
  k<MODE><<<1, 256>>>(o, c, 2000); cudaDeviceSynchronize();
  printf("%-40s %lld cycles/step\n", nm, c[0]);
}
int main() {
  run<0>("fma only");
  run<1>("+ quad shuffle reduce");
  run<2>("+ smem partials + __syncthreads (8 warps)");
  run<3>("shuffles + barrier");
  run<4>("scalars only (rsqrt_nr + rcp_nr)");
  run<7>("full chain");
}
