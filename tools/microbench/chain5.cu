// factor_panel_chol (one warp) alone and with DMMA / LDS traffic from other warps:
// does the chain's in-situ slowdown come from the data warps' DMMA on the other SMSPs?
#include "../../paper_2503_23385_b200/csrc/jq_tsqr.cu"
#include <cstdio>
namespace jq {
template <class C>
__global__ void __launch_bounds__(512, 1) chain5(long long* cyc, double* sink, int reps, int busy, int which) {
  extern __shared__ __align__(16) double smem_dyn[];
  double* R = smem_dyn + C::OFF_R; double* T = smem_dyn + C::OFF_T; double* Mg = smem_dyn + C::OFF_M;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3, warp = threadIdx.x >> 5;
  unsigned wid; asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
  if (warp != 0) {
    if (busy == 0) return;
    if ((wid & 3) == 0 && busy != 3) return;  // keep SMSP 0 free (except busy 3)
    double acc[8][2] = {};
    double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
    double* sm = smem_dyn + C::OFF_RAW + warp * 512;
    for (int r = 0; r < reps * 60; ++r) {
      if (busy == 4) {  // ~40 % duty: 8 DMMA then a pause
#pragma unroll
        for (int k = 0; k < 8; ++k) dmma(acc[k], a, b);
        __nanosleep(200);
      } else if (busy == 2) {
#pragma unroll
        for (int k = 0; k < 8; ++k) { acc[k][0] += sm[(lane * 2 + k * 17) & 511]; sm[(lane * 3 + k * 5) & 511] = acc[k][1]; }
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) dmma(acc[k], a, b);
      }
    }
    double s2 = 0; for (int k = 0; k < 8; ++k) s2 += acc[k][0] + acc[k][1];
    sink[threadIdx.x] = s2;
    return;
  }
  for (int i = lane; i < C::SZ_R; i += 32) R[i] = 0.0;
  __syncwarp();
  for (int i = lane; i < 64; i += 32) { int r = i >> 3, c = i & 7; if (c >= r) R[rix<C>(r, c)] = (r == c ? 30.0 + r : 0.3 * (c - r)); }
  __syncwarp();
  double G[2] = {(g == 2 * t ? 4.0 : 0.1) + 0.01 * lane, (g == 2 * t + 1 ? 4.0 : 0.1) + 0.01 * lane};
  bool okall = true;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    double Gc[2] = {G[0], G[1]}, Rb[2];
    if (which == 0) okall &= factor_panel_chol<C>(Gc, Rb, R, 0, T, Mg, smem_dyn + C::OFF_U, lane, diag_of(Gc, lane));
    else if (which == 1) okall &= factor_panel_gram<C>(Gc, Rb, R, 0, T, Mg, lane, diag_of(Gc, lane));
    else if (which == 2) { double z[2] = {Gc[0], Gc[1]}; for (int k = 0; k < 4; ++k) dmma(z, z[0], z[1]); Rb[0] = z[0]; Rb[1] = z[1]; }
    else { double z0 = Gc[0], z1 = Gc[1]; for (int k = 0; k < 32; ++k) { z0 = fma(z0, z1, 0.5); } Rb[0] = z0; Rb[1] = z1; }
    __syncwarp();
    G[0] += 1e-12 * (Rb[0] + T[(lane & 7) * C::LDT] + Mg[lane & 7]);
  }
  long long t1 = clock64();
  sink[lane] = G[0] + okall;
  if (lane == 0) cyc[0] = (t1 - t0) / reps;
}
}
int main() {
  using C = jq::Cfg<64>;
  long long* cyc; double* sink;
  cudaMallocManaged(&cyc, 64); cudaMalloc(&sink, 65536);
  cudaFuncSetAttribute(jq::chain5<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  const char* nm[5] = {"alone", "+12 warps DMMA on SMSP 1-3", "+12 warps LDS/STS on SMSP 1-3", "+15 warps DMMA incl. SMSP 0",
                       "+12 warps DMMA ~40% duty"};
  const char* wn[4] = {"cholesky panel", "reflector chain", "4 dependent DMMA", "32 dependent DFMA"};
  for (int which = 0; which < 4; ++which)
    for (int busy = 0; busy < 5; ++busy) {
      if (busy == 2 || busy == 3) continue;
      for (int w = 0; w < 2; ++w) jq::chain5<C><<<1, 512, C::SMEM>>>(cyc, sink, 100, busy, which);
      cudaDeviceSynchronize();
      printf("%-18s %-32s %6lld cycles  %s\n", wn[which], nm[busy], cyc[0], cudaGetErrorString(cudaGetLastError()));
    }
}
