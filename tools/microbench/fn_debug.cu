// Debug harness: footnote-variant TSQR of tails (FigaroSrc with an empty A-part)
// vs the dense TSQR of the explicitly formed tail matrix.
#include "jq_internal.cuh"
#include <cstdio>
#include <vector>
#include <cmath>
using namespace jq;
int main(int argc, char** argv) {
  int m = argc > 1 ? atoi(argv[1]) : 200, n = argc > 2 ? atoi(argv[2]) : 64, other = argc > 3 ? atoi(argv[3]) : 205;
  jq_ctx* ctx; if (jq_ctx_create(0, &ctx)) { printf("ctx fail\n"); return 1; }
  std::vector<double> X(m * n), Tl((m - 1) * n);
  for (int i = 0; i < m * n; ++i) X[i] = splitmix_uniform(7, i);
  // explicit tails scaled by sqrt(other)
  std::vector<double> S(n, 0.0);
  for (int c = 0; c < n; ++c) S[c] = X[c];
  for (int r = 1; r < m; ++r)
    for (int c = 0; c < n; ++c) {
      double x = X[r * n + c];
      Tl[(r - 1) * n + c] = (sqrt((double)r) * x - S[c] / sqrt((double)r)) / sqrt(r + 1.0) * sqrt((double)other);
      S[c] += x;
    }
  begin_call(ctx);
  ws_reserve(ctx, size_t(1) << 30);
  double *dX, *dT, *r1, *r2;
  cudaMalloc(&dX, 8 * m * n); cudaMalloc(&dT, 8 * (m - 1) * n); cudaMalloc(&r1, 8 * n * n); cudaMalloc(&r2, 8 * n * n);
  cudaMemcpy(dX, X.data(), 8 * m * n, cudaMemcpyHostToDevice);
  cudaMemcpy(dT, Tl.data(), 8 * (m - 1) * n, cudaMemcpyHostToDevice);
  SegScan ss;
  int rc = segscan_dev(ctx, dX, m, n, nullptr, nullptr, nullptr, nullptr, 1, &ss);
  FigaroArgs fa{};
  fa.b = dX; fa.m2 = m; fa.n2 = n; fa.b_carry = ss.carry; fa.m1_global = other; fa.m2_global = m;
  rc |= figaro_tsqr_dev(ctx, fa, r1, true);
  rc |= tsqr_dense_dev(ctx, dT, m - 1, n, r2, true);
  cudaStreamSynchronize(ctx->stream);
  std::vector<double> h1(n * n), h2(n * n);
  cudaMemcpy(h1.data(), r1, 8 * n * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(h2.data(), r2, 8 * n * n, cudaMemcpyDeviceToHost);
  double num = 0, den = 0; int nans = 0;
  for (int i = 0; i < n * n; ++i) { num += (h1[i] - h2[i]) * (h1[i] - h2[i]); den += h2[i] * h2[i]; nans += std::isnan(h1[i]); }
  printf("m=%d n=%d rc=%d rel=%.3e nans=%d err=%s\n", m, n, rc, sqrt(num / den), nans, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
