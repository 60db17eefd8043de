// Latency of factor_panel_gram (the 8-step Householder chain on the 8x8 Gram) + compute_T
// for one warp, in isolation.
#include "../../paper_2503_23385_b200/csrc/jq_tsqr.cu"
#include <cstdio>
namespace jq {
template <class C>
__global__ void __launch_bounds__(32, 1) gchain(long long* cyc, double* sink, int reps) {
  extern __shared__ __align__(16) double smem_dyn[];
  double* R = smem_dyn + C::OFF_R;
  double* T = smem_dyn + C::OFF_T; double* U = smem_dyn + C::OFF_U;
  double* taus = smem_dyn + C::OFF_TAU; double* scs = smem_dyn + C::OFF_SC;
  double* Mg = smem_dyn + C::OFF_M; double* Rst = smem_dyn + C::OFF_RST;
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  for (int i = lane; i < C::SZ_R; i += 32) R[i] = 0.0;
  __syncwarp();
  for (int i = lane; i < 8; i += 32) R[rix<C>(i, i)] = 3.0 + i;
  __syncwarp();
  double G[2];
  G[0] = (g == 2 * t ? 4.0 : 0.1) + 0.01 * lane;
  G[1] = (g == 2 * t + 1 ? 4.0 : 0.1) + 0.01 * lane;
  bool okall = true;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    double Gc[2] = {G[0], G[1]};
    okall &= factor_panel_gram<C>(Gc, R, 0, U, taus, scs, Mg, Rst, lane);
    __syncwarp();
    compute_T<C>(T, U, taus, scs, lane);
    __syncwarp();
    G[0] += 1e-9 * T[(lane & 7) * C::LDT];
  }
  long long t1 = clock64();
  sink[lane] = G[0] + okall;
  if (lane == 0) cyc[0] = (t1 - t0) / reps;
}
}
int main() {
  using C = jq::Cfg<64>;
  long long* cyc; double* sink;
  cudaMallocManaged(&cyc, 64); cudaMalloc(&sink, 4096);
  cudaFuncSetAttribute(jq::gchain<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  for (int w = 0; w < 2; ++w) jq::gchain<C><<<1, 32, C::SMEM>>>(cyc, sink, 100);
  cudaDeviceSynchronize();
  printf("gram chain + T (one warp): %lld cycles per panel (%.0f per column) %s\n", cyc[0], cyc[0] / 8.0,
         cudaGetErrorString(cudaGetLastError()));
}
