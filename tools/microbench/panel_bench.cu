// Times factor_panel<Cfg<NP>> (one 8-column Householder panel, owner warp) in
// isolation: one CTA, clock64 per call, optional per-phase breakdown.
#define JQ_PANEL_TIMING 1
#include "../../paper_2503_23385_b200/csrc/jq_tsqr.cu"
#include <cstdio>

namespace jq {
template <class C>
__global__ void __launch_bounds__(C::THREADS, 1) panel_bench(long long* cyc, double* sink, int reps) {
  extern __shared__ __align__(16) double smem_dyn[];
  double* R = smem_dyn + C::OFF_R;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < C::SZ_R; i += C::THREADS) R[i] = 0.0;
  for (int i = 0; i < 8; ++i) if (tid == 0) R[rix<C>(i, i)] = 1.0;
  __syncthreads();
  double c[C::KWT][2];
  for (int it = 0; it < C::KWT; ++it) { c[it][0] = 0.001 * (tid + it); c[it][1] = 0.002 * (tid - it); }
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    factor_panel_all<C>(c, R, 0, smem_dyn + C::OFF_YT + warp * C::SZ_YT, smem_dyn + C::OFF_T, smem_dyn + C::OFF_U,
                        smem_dyn + C::OFF_TAU, smem_dyn + C::OFF_SC, smem_dyn + C::OFF_X + warp * C::KW,
                        smem_dyn + C::OFF_P, warp, lane);
    __syncthreads();
  }
  long long t1 = clock64();
  double s = 0;
  for (int it = 0; it < C::KWT; ++it) s += c[it][0] + c[it][1];
  sink[tid] = s;
  if (tid == 0) cyc[0] = (t1 - t0) / reps;
}
}  // namespace jq

template <class C>
void run(const char* name) {
  long long* cyc; double* sink;
  cudaMallocManaged(&cyc, 64); cudaMalloc(&sink, 8 * 4096);
  cudaFuncSetAttribute(jq::panel_bench<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  const int reps = 200;
  long long zero[16] = {};
  for (int w = 0; w < 2; ++w) {
    cudaMemcpyToSymbol(jq::g_ptime, zero, sizeof(zero));
    jq::panel_bench<C><<<1, C::THREADS, C::SMEM>>>(cyc, sink, reps);
    cudaDeviceSynchronize();
  }
  long long pt[16]; cudaMemcpyFromSymbol(pt, jq::g_ptime, sizeof(pt));
  const char* nm[6] = {"publish + dots + quad reduce", "CTA barrier + partial sums", "-", "scalars", "update + writes", "Y + T tail (per panel)"};
  for (int i = 0; i < 6; ++i) if (i != 2) printf("  %-32s %8.1f cycles\n", nm[i], pt[i] / (double)reps / (i == 5 ? 1 : 8));
  printf("%s: %lld cycles per panel (%.0f per column) status %s\n", name, cyc[0], cyc[0] / 8.0,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<jq::Cfg<128>>("NP=128 K=128 (8 warps x 16 rows)");
  run<jq::Cfg<64>>("NP=64  K=128 (8 warps x 16 rows)");
}
