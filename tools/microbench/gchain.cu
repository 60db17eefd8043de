// Latency of factor_panel_gram (the 8-step Householder chain on the 8x8 Gram) + compute_T
// for one warp, in isolation.
#include "../../paper_2503_23385_b200/csrc/jq_tsqr.cu"
#include <cstdio>
namespace jq {
template <class C>
__global__ void __launch_bounds__(256, 1) gchain(long long* cyc, double* sink, int reps, int busy) {
  extern __shared__ __align__(16) double smem_dyn[];
  double* R = smem_dyn + C::OFF_R + (threadIdx.x >= 32 ? 8192 : 0);
  const int off2 = threadIdx.x >= 32 ? 4096 : 0;
  double* T = smem_dyn + C::OFF_T + off2; double* U = smem_dyn + C::OFF_U + off2;
  double* taus = smem_dyn + C::OFF_TAU; double* scs = smem_dyn + C::OFF_SC;
  double* Mg = smem_dyn + C::OFF_M + off2;
  (void)U; (void)taus; (void)scs;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const bool second_chain = busy == 6 && (threadIdx.x >> 5) == 4;
  if (threadIdx.x >= 32 && !second_chain) {  // other warps: DMMA (busy=1) or DFMA (busy=2) streams on the same SM
    if (busy == 0 || busy == 6) return;
    if (busy >= 3 && (threadIdx.x >> 5) % 4 == 0) return;  // keep the chain warp's SMSP free of DMMA
    double acc[8][2] = {};
    double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
    for (int r = 0; r < reps * 40; ++r) {
      if (busy == 4) {  // shared-memory traffic (LDS.64 / STS.64) like the data warps' update
        double* sm = smem_dyn + C::OFF_RAW + (threadIdx.x >> 5) * 256;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          acc[k][0] += sm[(lane * 2 + k * 17) & 255];
          sm[(lane * 3 + k * 5) & 255] = acc[k][1];
          acc[k][1] += sm[(lane + k * 9) & 255];
        }
      } else if (busy == 5) {  // shuffles
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k][0] += __shfl_sync(0xffffffffu, acc[k][1], (lane + k) & 31);
      } else if (busy == 1 || busy == 3) {
#pragma unroll
        for (int k = 0; k < 8; ++k) dmma(acc[k], a, b);
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) { acc[k][0] = fma(a, acc[k][0], b); acc[k][1] = fma(b, acc[k][1], a); }
      }
    }
    double s2 = 0; for (int k = 0; k < 8; ++k) s2 += acc[k][0] + acc[k][1];
    sink[threadIdx.x] = s2;
    return;
  }
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
    double Rb[2] = {R[rix<C>(g, 2 * t)], R[rix<C>(g, 2 * t + 1)]};
    okall &= factor_panel_gram<C>(Gc, Rb, R, 0, T, Mg, lane, jq::diag_of(Gc, lane));
    __syncwarp();
    __syncwarp();
    G[0] += 1e-9 * T[(lane & 7) * C::LDT];
  }
  long long t1 = clock64();
  sink[lane] = G[0] + okall;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
}
}
int main() {
  using C = jq::Cfg<64>;
  long long* cyc; double* sink;
  cudaMallocManaged(&cyc, 64); cudaMalloc(&sink, 4096);
  cudaFuncSetAttribute(jq::gchain<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  const char* names[7] = {"alone", "+7 warps DMMA", "+7 warps DFMA", "+6 warps DMMA on SMSP 1-3",
                          "+6 warps LDS/STS on SMSP 1-3", "+6 warps SHFL on SMSP 1-3", "+ a 2nd chain on SMSP 0"};
  for (int busy = 0; busy < 7; ++busy) {
    for (int w = 0; w < 2; ++w) jq::gchain<C><<<1, 256, C::SMEM>>>(cyc, sink, 100, busy);
    cudaDeviceSynchronize();
    printf("gram chain (one warp, %s): %lld cycles per panel (%.0f per column) %s\n", names[busy], cyc[0],
           cyc[0] / 8.0, cudaGetErrorString(cudaGetLastError()));
  }
}
