// Warp-independent TSQR (tsqr_wkernel) compute in isolation: each active warp runs
// the panel loop of one KW-row chunk (factor_panel_warp + trailing tile updates)
// `reps` times on register-resident data; reports cycles per chunk per warp and the
// SM-level rows/cycle for 1..8 active warps (no loads).
#include "../../paper_2503_23385_b200/csrc/jq_tsqr.cu"
#include <cstdio>

namespace jq {
template <class C, bool UPDATE>
__global__ void __launch_bounds__(C::THREADS, 1) wbench(long long* cyc, double* sink, int reps, int active) {
  extern __shared__ __align__(16) double smem_dyn[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  double* R = smem_dyn + C::OFF_R + warp * C::SZ_R;
  double* Ytw = smem_dyn + C::OFF_YT + warp * C::SZ_YT;
  double* T = smem_dyn + C::OFF_T + warp * 8 * C::LDT;
  double* U = smem_dyn + C::OFF_U + warp * 64;
  double* taus = smem_dyn + C::OFF_TAU + warp * 8;
  double* scs = smem_dyn + C::OFF_SC + warp * 8;
  for (int i = lane; i < C::SZ_R; i += 32) R[i] = 0.0;
  __syncwarp();
  if (warp >= active) return;
  double c[C::NLT][C::KWT][2];
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int q = 0; q < C::NLT; ++q)
#pragma unroll
      for (int it = 0; it < C::KWT; ++it) {
        c[q][it][0] = 0.001 * (lane + it + q + r) + 0.5;
        c[q][it][1] = 0.002 * (lane - it + q) + 0.25;
      }
#pragma unroll 1
    for (int p = 0; p < C::NLT; ++p) {
      const int j0 = 8 * p;
      double cp[C::KWT][2];
#pragma unroll
      for (int q = 0; q < C::NLT; ++q)
        if (q == p)
#pragma unroll
          for (int it = 0; it < C::KWT; ++it) { cp[it][0] = c[q][it][0]; cp[it][1] = c[q][it][1]; }
      factor_panel_warp<C>(cp, R, j0, Ytw, T, U, taus, scs, lane);
      if (UPDATE) {
#pragma unroll
        for (int q = 0; q < C::NLT; ++q) {
          if (q > p) {
            const int r0i = rix<C>(j0 + 2 * t, 8 * q + g), r1i = rix<C>(j0 + 2 * t + 1, 8 * q + g);
            double z[2] = {R[r0i], R[r1i]}, z2[2] = {0.0, 0.0};
#pragma unroll
            for (int it = 0; it < C::KWT; ++it) {
              dmma(z, c[q][it][0], cp[it][0]);
              dmma(z2, c[q][it][1], cp[it][1]);
            }
            double wv[2] = {0.0, 0.0};
            dmma(wv, z[0] + z2[0], T[(2 * t) * C::LDT + g]);
            dmma(wv, z[1] + z2[1], T[(2 * t + 1) * C::LDT + g]);
            R[r0i] -= wv[0];
            R[r1i] -= wv[1];
#pragma unroll
            for (int it = 0; it < C::KWT; ++it) {
              dmma(c[q][it], -wv[0], Ytw[(2 * t) * C::LDYT + 8 * it + g]);
              dmma(c[q][it], -wv[1], Ytw[(2 * t + 1) * C::LDYT + 8 * it + g]);
            }
          }
        }
      }
      __syncwarp();
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int q = 0; q < C::NLT; ++q)
#pragma unroll
    for (int it = 0; it < C::KWT; ++it) s += c[q][it][0] + c[q][it][1];
  sink[tid] = s;
  if (lane == 0) cyc[warp] = (t1 - t0) / reps;
}
}  // namespace jq

template <class C, bool UPDATE>
void run() {
  long long* cyc; double* sink;
  cudaMallocManaged(&cyc, 64 * 8); cudaMalloc(&sink, 8 * 4096);
  cudaFuncSetAttribute(jq::wbench<C, UPDATE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  for (int active : {1, 2, 4, 8}) {
    for (int w = 0; w < 2; ++w) jq::wbench<C, UPDATE><<<1, C::THREADS, C::SMEM>>>(cyc, sink, 20, active);
    cudaDeviceSynchronize();
    long long mx = 0;
    for (int i = 0; i < active; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
    printf("NP=%d KW=%d update=%d warps=%d: %lld cycles/chunk/warp = %.0f per column; SM %.3f rows/cycle (%s)\n",
           C::NP, C::KW, UPDATE, active, mx, mx / (double)C::NP, active * C::KW / (double)mx,
           cudaGetErrorString(cudaGetLastError()));
  }
}
int main() {
  run<jq::CfgW<64>, false>();
  run<jq::CfgW<64>, true>();
  run<jq::CfgW<32>, true>();
}
