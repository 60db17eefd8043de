// Two co-resident CTAs per SM: each CTA picks its chain warp by %warpid % 4 == 0 and
// runs DMMA streams on the warps with %warpid % 4 != 0.  If %warpid % 4 is the SM
// sub-partition, both CTAs' chains run at the isolated speed.
#include "../../paper_2503_23385_b200/csrc/jq_tsqr.cu"
#include <cstdio>
namespace jq {
template <class C>
__global__ void __launch_bounds__(256, 2) gchain2(long long* cyc, double* sink, int reps, int mode) {
  extern __shared__ __align__(16) double smem_dyn[];
  __shared__ int role[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  unsigned wid;
  asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
  if (lane == 0) role[warp] = wid;
  __syncthreads();
  int chain_w = -1, chain_w2 = -1;
  for (int w = 0; w < 8; ++w) if ((role[w] & 3) == 0) { if (chain_w < 0) chain_w = (mode == 0) ? 0 : w; else if (chain_w2 < 0) chain_w2 = w; }
  if (mode != 3) chain_w2 = -1;
  const bool second = warp == chain_w2;
  if (warp != chain_w && !second) {
    const bool dm = mode == 2 ? true : (role[warp] & 3) != 0;  // mode 2: DMMA on every other warp
    if (!dm) return;
    double acc[8][2] = {};
    double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
    for (int r = 0; r < reps * 40; ++r) {
#pragma unroll
      for (int k = 0; k < 8; ++k) dmma(acc[k], a, b);
    }
    double s2 = 0; for (int k = 0; k < 8; ++k) s2 += acc[k][0] + acc[k][1];
    sink[blockIdx.x * 256 + threadIdx.x] = s2;
    return;
  }
  const int off = second ? 6000 : 0;  // private R / T / M' for the second chain (RAW area)
  double* R = smem_dyn + C::OFF_R + (second ? C::OFF_RAW : 0);
  double* T = smem_dyn + C::OFF_RAW + 3000 + off / 6; double* U = smem_dyn + C::OFF_RAW + 3200 + off / 6;
  double* taus = smem_dyn + C::OFF_RAW + 3400 + off / 6; double* scs = smem_dyn + C::OFF_RAW + 3500 + off / 6;
  double* Mg = smem_dyn + C::OFF_RAW + 3600 + off / 6;
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
    double Rb[2];
    okall &= factor_panel_gram<C>(Gc, Rb, R, 0, T, Mg, lane, jq::diag_of(Gc, lane));
    __syncwarp();
    G[0] += 1e-9 * T[(lane & 7) * C::LDT] + 1e-12 * Rb[0];
  }
  long long t1 = clock64();
  sink[blockIdx.x * 256 + threadIdx.x] = G[0] + okall;
  if (lane == 0 && !second) { cyc[2 * blockIdx.x] = (t1 - t0) / reps; cyc[2 * blockIdx.x + 1] = wid; }
}
}
int main() {
  using C = jq::Cfg<64>;
  long long* cyc; double* sink;
  const int n = 296;
  cudaMallocManaged(&cyc, 16 * n); cudaMalloc(&sink, 8 * 256 * n);
  cudaFuncSetAttribute(jq::gchain2<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  const char* names[4] = {"chain=warp 0, DMMA on %warpid%4!=0", "chain by %warpid, DMMA on %warpid%4!=0",
                          "chain by %warpid, DMMA on all other warps", "TWO chains on SMSP 0, DMMA elsewhere"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int w = 0; w < 2; ++w) jq::gchain2<C><<<n, 256, (int)C::SMEM>>>(cyc, sink, 100, mode);
    cudaDeviceSynchronize();
    double lo[2] = {0, 0}; int cnt[2] = {0, 0};
    for (int b = 0; b < n; ++b) { int second = cyc[2 * b + 1] >= 8; lo[second] += cyc[2 * b]; cnt[second]++; }
    printf("%-45s: chain cycles/panel first CTA %.0f (%d), second CTA %.0f (%d) %s\n", names[mode],
           cnt[0] ? lo[0] / cnt[0] : 0., cnt[0], cnt[1] ? lo[1] / cnt[1] : 0., cnt[1],
           cudaGetErrorString(cudaGetLastError()));
  }
}
