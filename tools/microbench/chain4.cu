// Phase timing of factor_panel_chol (built with -DJQ_CHOL_PHASES), one warp alone.
#include "../../paper_2503_23385_b200/csrc/jq_tsqr.cu"
#include <cstdio>
namespace jq {
template <class C>
__global__ void __launch_bounds__(32, 1) chain4(double* sink, int reps) {
  extern __shared__ __align__(16) double smem_dyn[];
  double* R = smem_dyn + C::OFF_R; double* T = smem_dyn + C::OFF_T; double* Mg = smem_dyn + C::OFF_M;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  for (int i = lane; i < C::SZ_R; i += 32) R[i] = 0.0;
  __syncwarp();
  for (int i = lane; i < 64; i += 32) { int r = i >> 3, c = i & 7; if (c >= r) R[rix<C>(r, c)] = (r == c ? 30.0 + r : 0.3 * (c - r)); }
  __syncwarp();
  double G[2] = {(g == 2 * t ? 4.0 : 0.1) + 0.01 * lane, (g == 2 * t + 1 ? 4.0 : 0.1) + 0.01 * lane};
  bool okall = true;
  for (int r = 0; r < reps; ++r) {
    double Gc[2] = {G[0], G[1]}, Rb[2];
    okall &= factor_panel_chol<C>(Gc, Rb, R, 0, T, Mg, smem_dyn + C::OFF_U, lane, diag_of(Gc, lane));
    __syncwarp();
    G[0] += 1e-12 * (Rb[0] + T[(lane & 7) * C::LDT] + Mg[lane & 7]);
  }
  sink[lane] = G[0] + okall;
}
}
int main() {
  using C = jq::Cfg<64>;
  double* sink; cudaMalloc(&sink, 4096);
  cudaFuncSetAttribute(jq::chain4<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  jq::chain4<C><<<1, 32, C::SMEM>>>(sink, 10);
  cudaDeviceSynchronize();
  long long z[8] = {0}; cudaMemcpyToSymbol(jq::g_chol_ph, z, sizeof(z));
  const int reps = 200;
  jq::chain4<C><<<1, 32, C::SMEM>>>(sink, reps);
  cudaDeviceSynchronize();
  long long ph[8]; cudaMemcpyFromSymbol(ph, jq::g_chol_ph, sizeof(ph));
  const char* nm[6] = {"S = G + Rp^T Rp, loads", "8 Cholesky steps", "R_new, W, scratch stores", "back substitutions", "T product", "guard"};
  for (int k = 0; k < 6; ++k) printf("%-28s %6lld cycles\n", nm[k], ph[k] / reps);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
