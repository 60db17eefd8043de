// Latency of the panel factorisations (one warp, alone on its SM): factor_panel_gram
// (8-step reflector chain) vs factor_panel_chol (Cholesky + back substitutions), and
// the Cholesky variant's phases (STOP = 1: S only, 2: + Cholesky, 3: + inverses).
#include "../../paper_2503_23385_b200/csrc/jq_tsqr.cu"
#include <cstdio>
namespace jq {
__device__ __forceinline__ double* smem_dyn_scr() { extern __shared__ __align__(16) double smem_dyn[]; return smem_dyn + Cfg<64>::OFF_U; }
template <class C, int STOP>
__device__ __forceinline__ bool chol_phases(const double (&G)[2], double (&Rb)[2], const double* Rs, const int j0,
                                            double* T, double* Mg, const int lane, const double Pg) {
  const int g = lane >> 2, t = lane & 3, c0 = 2 * t, c1 = 2 * t + 1;
  const double rp0 = (c0 >= g) ? Rs[rix<C>(j0 + g, j0 + c0)] : 0.0;
  const double rp1 = (c1 >= g) ? Rs[rix<C>(j0 + g, j0 + c1)] : 0.0;
  const double rt0 = (g >= c0) ? Rs[rix<C>(j0 + c0, j0 + g)] : 0.0;
  const double rt1 = (g >= c1) ? Rs[rix<C>(j0 + c1, j0 + g)] : 0.0;
  const double alpha = Rs[rix<C>(j0 + g, j0 + g)];
  const double dsg = alpha >= 0.0 ? -1.0 : 1.0;
  double S[2] = {G[0], G[1]};
  dmma(S, rt0, rt0);
  dmma(S, rt1, rt1);
  if (STOP == 1) { Rb[0] = S[0]; Rb[1] = S[1]; return true; }
  double piv_g = 0.0, rs_g = 1.0;
  Rb[0] = 0.0; Rb[1] = 0.0;
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
  if (STOP == 2) return true;
  double* scr = smem_dyn_scr();
  double* Wn = scr; double* Rn = scr + 8 * C::LDT; double* dg = scr + 16 * C::LDT;
  *reinterpret_cast<double2*>(Wn + g * C::LDT + c0) = make_double2(rp0 - Rb[0], rp1 - Rb[1]);
  *reinterpret_cast<double2*>(Rn + g * C::LDT + c0) = make_double2(Rb[0], Rb[1]);
  if (t == 0) { dg[g] = rcp_nr(alpha - dsg * piv_g * rs_g); dg[8 + g] = dsg * rs_g; }
  __syncwarp();
  if (STOP == 3) return true;
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
  } else if (lane < 16 && STOP != 4) {
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
  return __all_sync(FULL, piv_g >= 1e-2 * Pg);
}

template <class C, int MODE>
__global__ void __launch_bounds__(32, 1) chainb(long long* cyc, double* sink, int reps) {
  extern __shared__ __align__(16) double smem_dyn[];
  double* R = smem_dyn + C::OFF_R;
  double* T = smem_dyn + C::OFF_T;
  double* Mg = smem_dyn + C::OFF_M;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  for (int i = lane; i < C::SZ_R; i += 32) R[i] = 0.0;
  __syncwarp();
  for (int i = lane; i < 64; i += 32) { int r = i >> 3, c = i & 7; if (c >= r) R[rix<C>(r, c)] = (r == c ? 30.0 + r : 0.3 * (c - r)); }
  __syncwarp();
  double G[2];
  G[0] = (g == 2 * t ? 4.0 : 0.1) + 0.01 * lane;
  G[1] = (g == 2 * t + 1 ? 4.0 : 0.1) + 0.01 * lane;
  bool okall = true;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    double Gc[2] = {G[0], G[1]};
    double Rb[2];
    if (MODE == 0) okall &= factor_panel_gram<C>(Gc, Rb, R, 0, T, Mg, lane, diag_of(Gc, lane));
    else if (MODE == 10) okall &= factor_panel_chol<C>(Gc, Rb, R, 0, T, Mg, smem_dyn + C::OFF_U, lane, diag_of(Gc, lane));
    else okall &= chol_phases<C, MODE>(Gc, Rb, R, 0, T, Mg, lane, diag_of(Gc, lane));
    __syncwarp();
    G[0] += 1e-12 * (Rb[0] + T[(lane & 7) * C::LDT] + Mg[lane & 7]);
  }
  long long t1 = clock64();
  sink[lane] = G[0] + okall;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
}
}
template <int MODE>
void run(const char* name, long long* cyc, double* sink) {
  using C = jq::Cfg<64>;
  cudaFuncSetAttribute(jq::chainb<C, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  for (int w = 0; w < 2; ++w) jq::chainb<C, MODE><<<1, 32, C::SMEM>>>(cyc, sink, 200);
  cudaDeviceSynchronize();
  printf("%-40s %6lld cycles per panel  %s\n", name, cyc[0], cudaGetErrorString(cudaGetLastError()));
}
int main() {
  long long* cyc; double* sink;
  cudaMallocManaged(&cyc, 64); cudaMalloc(&sink, 4096);
  run<0>("reflector chain (factor_panel_gram)", cyc, sink);
  run<10>("cholesky panel (factor_panel_chol)", cyc, sink);
  run<1>("  chol: S = G + Rp^T Rp only", cyc, sink);
  run<2>("  chol: + 8 Cholesky steps", cyc, sink);
  run<3>("  chol: + scratch stores", cyc, sink);
  run<4>("  chol: + M' solve only", cyc, sink);
  run<5>("  chol: + both solves (no T product)", cyc, sink);
}
