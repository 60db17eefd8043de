// Cost of the per-row part of a Householder column step (single warp): x broadcast
// through smem + 2 FMA streams (dot, update) over V values per lane.
#include <cstdio>
template <int V>
__global__ void k(double* out, long long* cyc, int reps) {
  __shared__ __align__(16) double Xs[4 * V + 8];
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double cc[V], xv[V];
  for (int i = 0; i < V; ++i) cc[i] = 0.001 * (lane + i);
  long long t0 = clock64();
  double acc = 0;
  for (int r = 0; r < reps; ++r) {
    const int jj = r & 7;
    if (g == jj) {
#pragma unroll
      for (int it = 0; it < V / 2; ++it)
        *reinterpret_cast<double2*>(Xs + 8 * it + 2 * t) = make_double2(cc[2 * it], cc[2 * it + 1]);
    }
    __syncwarp();
    double dp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int it = 0; it < V / 2; ++it) {
      const double2 x2 = *reinterpret_cast<const double2*>(Xs + 8 * it + 2 * t);
      xv[2 * it] = x2.x; xv[2 * it + 1] = x2.y;
      dp[(2 * it) & 7] = fma(xv[2 * it], cc[2 * it], dp[(2 * it) & 7]);
      dp[(2 * it + 1) & 7] = fma(xv[2 * it + 1], cc[2 * it + 1], dp[(2 * it + 1) & 7]);
    }
    double d = ((dp[0] + dp[1]) + (dp[2] + dp[3])) + ((dp[4] + dp[5]) + (dp[6] + dp[7]));
    const double a = -1e-9 * d;
#pragma unroll
    for (int i = 0; i < V; ++i) cc[i] = fma(a, xv[i], cc[i]);
    __syncwarp();
  }
  long long t1 = clock64();
  for (int i = 0; i < V; ++i) acc += cc[i];
  out[lane] = acc;
  if (lane == 0) cyc[0] = (t1 - t0) / reps;
}
template <int V>
void run() {
  double* o; long long* c; cudaMalloc(&o, 1024); cudaMallocManaged(&c, 64);
  k<V><<<1, 32>>>(o, c, 1000); cudaDeviceSynchronize();
  k<V><<<1, 32>>>(o, c, 1000); cudaDeviceSynchronize();
  printf("V=%3d values/lane: %lld cycles per column step (%.2f per value)\n", V, c[0], c[0] / (double)V);
}
int main() { run<4>(); run<8>(); run<16>(); run<32>(); }
