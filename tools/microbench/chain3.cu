// Phase timing (clock64 stamps) inside the Cholesky panel factorisation, one warp alone.
#include "../../paper_2503_23385_b200/csrc/jq_tsqr.cu"
#include <cstdio>
namespace jq {
__device__ long long g_ph[16];
template <class C>
__global__ void __launch_bounds__(32, 1) chain3(double* sink, int reps) {
  extern __shared__ __align__(16) double smem_dyn[];
  double* Rs = smem_dyn + C::OFF_R;
  double* T = smem_dyn + C::OFF_T;
  double* Mg = smem_dyn + C::OFF_M;
  double* scr = smem_dyn + C::OFF_U;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, c0 = 2 * t, c1 = 2 * t + 1;
  for (int i = lane; i < C::SZ_R; i += 32) Rs[i] = 0.0;
  __syncwarp();
  for (int i = lane; i < 64; i += 32) { int r = i >> 3, c = i & 7; if (c >= r) Rs[rix<C>(r, c)] = (r == c ? 30.0 + r : 0.3 * (c - r)); }
  __syncwarp();
  double G[2];
  G[0] = (g == 2 * t ? 4.0 : 0.1) + 0.01 * lane;
  G[1] = (g == 2 * t + 1 ? 4.0 : 0.1) + 0.01 * lane;
  long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int j0 = 0;
  for (int rep = 0; rep < reps; ++rep) {
    long long c_0 = clock64();
    const double rp0 = (c0 >= g) ? Rs[rix<C>(j0 + g, j0 + c0)] : 0.0;
    const double rp1 = (c1 >= g) ? Rs[rix<C>(j0 + g, j0 + c1)] : 0.0;
    const double rt0 = (g >= c0) ? Rs[rix<C>(j0 + c0, j0 + g)] : 0.0;
    const double rt1 = (g >= c1) ? Rs[rix<C>(j0 + c1, j0 + g)] : 0.0;
    const double alpha = Rs[rix<C>(j0 + g, j0 + g)];
    const double dsg = alpha >= 0.0 ? -1.0 : 1.0;
    double S[2] = {G[0], G[1]};
    dmma(S, rt0, rt0);
    dmma(S, rt1, rt1);
    const double sdiag = diag_of(S, lane);
    double piv_g = 0.0, rs_g = 1.0, Rb[2] = {0.0, 0.0};
    long long c_1 = clock64();
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double e = (j & 1) ? S[1] : S[0];
      const double piv = __shfl_sync(FULL, e, 4 * j + (j >> 1));
      const double sgj = __shfl_sync(FULL, e, 4 * g + (j >> 1));
      const double sj0 = __shfl_sync(FULL, S[0], 4 * j + t);
      const double sj1 = __shfl_sync(FULL, S[1], 4 * j + t);
      const double inv = rcp_nr(piv);
      const double rs = rsqrt_nr(piv);
      if (g == j) { piv_g = piv; rs_g = rs; Rb[0] = c0 >= j ? dsg * sj0 * rs : 0.0; Rb[1] = c1 >= j ? dsg * sj1 * rs : 0.0; }
      const double f = sgj * inv;
      if (g > j && c0 > j) S[0] = fma(-f, sj0, S[0]);
      if (g > j && c1 > j) S[1] = fma(-f, sj1, S[1]);
    }
    long long c_2 = clock64();
    double* Wn = scr; double* Rn = scr + 8 * C::LDT; double* dg = scr + 16 * C::LDT;
    *reinterpret_cast<double2*>(Wn + g * C::LDT + c0) = make_double2(rp0 - Rb[0], rp1 - Rb[1]);
    *reinterpret_cast<double2*>(Rn + g * C::LDT + c0) = make_double2(Rb[0], Rb[1]);
    if (t == 0) { dg[g] = rcp_nr(alpha - dsg * piv_g * rs_g); dg[8 + g] = dsg * rs_g; }
    __syncwarp();
    long long c_3 = clock64();
    if (lane < 8) {
      const int c = lane;
      double acc[8], x[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = 0.0;
#pragma unroll
      for (int k = 7; k >= 0; --k) {
        x[k] = k > c ? 0.0 : (k == c ? dg[k] : -dg[k] * acc[k]);
#pragma unroll
        for (int i = 0; i < k; ++i) acc[i] = fma(Wn[i * C::LDT + k], x[k], acc[i]);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) Mg[i * C::LDT + c] = x[i];
    } else if (lane < 16) {
      const int i = lane - 8;
      double acc[8], y[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = j >= i ? -Wn[i * C::LDT + j] : 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        y[k] = k < i ? 0.0 : acc[k] * dg[8 + k];
#pragma unroll
        for (int j = k + 1; j < 8; ++j) acc[j] = fma(-y[k], Rn[k * C::LDT + j], acc[j]);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) T[i * C::LDT + j] = y[j];
    }
    __syncwarp();
    long long c_4 = clock64();
    const bool ok = __all_sync(FULL, piv_g >= 1e-2 * (sdiag + 1.0));
    long long c_5 = clock64();
    ph[0] += c_1 - c_0; ph[1] += c_2 - c_1; ph[2] += c_3 - c_2; ph[3] += c_4 - c_3; ph[4] += c_5 - c_4;
    G[0] += 1e-12 * (Rb[0] + T[(lane & 7) * C::LDT] + Mg[lane & 7] + ok);
  }
  sink[lane] = G[0];
  if (lane == 0) for (int k = 0; k < 5; ++k) g_ph[k] = ph[k] / reps;
}
}
int main() {
  using C = jq::Cfg<64>;
  double* sink; cudaMalloc(&sink, 4096);
  cudaFuncSetAttribute(jq::chain3<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  for (int w = 0; w < 2; ++w) jq::chain3<C><<<1, 32, C::SMEM>>>(sink, 200);
  cudaDeviceSynchronize();
  long long ph[16]; cudaMemcpyFromSymbol(ph, jq::g_ph, sizeof(ph));
  const char* nm[5] = {"S + loads", "cholesky 8 steps", "scratch stores + rcp", "two solves", "guard"};
  for (int k = 0; k < 5; ++k) printf("%-24s %6lld cycles\n", nm[k], ph[k]);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
