// Accuracy of the MUFU f64 approximations (rcp.approx.ftz.f64, rsqrt.approx.ftz.f64)
// with 0/1/2 Newton steps: max relative error over a log-uniform sample.
#include <cstdio>
#include <cmath>
__global__ void k(double* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = exp2(-60.0 + 120.0 * ((i * 2654435761u) % 1000003) / 1000003.0) * (1.0 + (i % 977) / 977.0);
  double r, y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double r1 = fma(r, fma(-x, r, 1.0), r);
  double r2 = fma(r1, fma(-x, r1, 1.0), r1);
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double h = 0.5 * x;
  double y1 = y * fma(-h * y, y, 1.5);
  double y2 = y1 * fma(-h * y1, y1, 1.5);
  double er = 1.0 / x, ey = 1.0 / sqrt(x);
  // one cubic step: r (1 + e + e^2), y (1 + e/2 + 3e^2/8)
  double e = fma(-x, r, 1.0);
  double rc = fma(r, fma(e, e, e), r);
  double ey0 = fma(-x * y, y, 1.0);
  double yc = fma(y * ey0, fma(0.375, ey0, 0.5), y);
  out[6 * n + 2 * i + 0] = fabs(rc / er - 1);
  out[6 * n + 2 * i + 1] = fabs(yc / ey - 1);
  out[6 * i + 0] = fabs(r / er - 1); out[6 * i + 1] = fabs(r1 / er - 1); out[6 * i + 2] = fabs(r2 / er - 1);
  out[6 * i + 3] = fabs(y / ey - 1); out[6 * i + 4] = fabs(y1 / ey - 1); out[6 * i + 5] = fabs(y2 / ey - 1);
}
int main() {
  const int n = 1 << 20;
  double* d; cudaMallocManaged(&d, 8ull * n * 8);
  k<<<n / 256, 256>>>(d, n); cudaDeviceSynchronize();
  double m[6] = {0};
  for (int i = 0; i < n; ++i) for (int j = 0; j < 6; ++j) m[j] = fmax(m[j], d[6 * i + j]);
  printf("rcp  approx %.3e  +1 newton %.3e  +2 newton %.3e\n", m[0], m[1], m[2]);
  printf("rsqrt approx %.3e  +1 newton %.3e  +2 newton %.3e\n", m[3], m[4], m[5]);
  double c0 = 0, c1 = 0;
  for (int i = 0; i < n; ++i) { c0 = fmax(c0, d[6 * n + 2 * i]); c1 = fmax(c1, d[6 * n + 2 * i + 1]); }
  printf("one cubic step: rcp %.3e  rsqrt %.3e  (double eps 1.1e-16)\n", c0, c1);
}
