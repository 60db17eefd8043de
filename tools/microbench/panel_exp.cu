// Knock-out experiments on the all-warp panel factorisation (copy of factor_panel_all).
#include "../../paper_2503_23385_b200/csrc/jq_tsqr.cu"
#include <cstdio>
namespace jq {
template <class C, int F>
__device__ __forceinline__ void factor_panel_x(double (&cp)[C::KWT][2], double* R, const int j0, double* Ytw,
                                                 double* T, double* U, double* taus, double* scs, double* Xw,
                                                 double* P, const int warp, const int lane) {
  const int g = lane >> 2, t = lane & 3;
#ifdef JQ_PANEL_TIMING
  long long pt_last = clock64(), pt_acc[6] = {0, 0, 0, 0, 0, 0};
#endif
  double alpha_n = (F & 1) ? 1.0 : R[rix<C>(j0, j0)], rg_n = (F & 1) ? 0.5 : R[rix<C>(j0, j0 + g)];
  double tau_r = 0.0, scale_r = 0.0;  // warp 0, lane r < 8: tau / scale of column r
  double scale_g = 0.0;                // every lane: scale of its own column g
#pragma unroll 1
  for (int jj = 0; jj < 8; ++jj) {
    const double alpha = alpha_n, rgj = rg_n;
    if (!(F & 1) && jj < 7) {  // panel R rows are final at panel start; prefetch the next column's entries
      alpha_n = R[rix<C>(j0 + jj + 1, j0 + jj + 1)];
      rg_n = R[rix<C>(j0 + jj + 1, j0 + g)];
    }
    if (!(F & 4)) {
    if (g == jj) {
#pragma unroll
      for (int it = 0; it < C::KWT; ++it)
        *reinterpret_cast<double2*>(Xw + 8 * it + 2 * t) = make_double2(cp[it][0], cp[it][1]);
    }
    __syncwarp();
    }
    double xv[C::KWT][2];
    double dp0 = 0.0, dp1 = 0.0;
#pragma unroll
    for (int it = 0; it < C::KWT; ++it) {
      const double2 x2 = (F & 4) ? make_double2(cp[it][0], cp[it][1]) : *reinterpret_cast<const double2*>(Xw + 8 * it + 2 * t);
      xv[it][0] = x2.x;
      xv[it][1] = x2.y;
      dp0 = fma(xv[it][0], cp[it][0], dp0);
      dp1 = fma(xv[it][1], cp[it][1], dp1);
    }
    double d = dp0 + dp1;
    d += __shfl_xor_sync(FULL, d, 1);
    d += __shfl_xor_sync(FULL, d, 2);
    double* Pj = P + (jj & 1) * (C::WARPS * 8);
    if (t == 0) Pj[warp * 8 + g] = d;
    PT(0);
    __syncthreads();
    d = 0.0;
    double sj = 0.0;
#pragma unroll
    for (int w = 0; w < C::WARPS; ++w) {  // fixed order: bit-identical in every warp
      d += Pj[w * 8 + g];
      sj += Pj[w * 8 + jj];
    }
    PT(1);
    double tau = 0.0, beta = alpha, scale = 0.0;
    if (sj != 0.0) {
      const double s2 = fma(alpha, alpha, sj);
      if (s2 > 1e-280 && s2 < 1e280) {                 // uniform branch: MUFU + Newton fast path
        const double rn = rsqrt_nr(s2);                // 1 / |[alpha; x]|
        const double nrm = s2 * rn;
        beta = alpha >= 0.0 ? -nrm : nrm;
        tau = fma(fabs(alpha), rn, 1.0);               // (beta - alpha) / beta
        scale = rcp_nr(alpha - beta);                  // 1 / (alpha - beta), no cancellation
      } else {                                         // IEEE path (ftz approximations would flush)
        const double nrm = sqrt(alpha * alpha + sj);
        beta = alpha >= 0.0 ? -nrm : nrm;
        tau = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
    }
    PT(3);
    // g > jj: c_g <- c_g - tau (R[j][g] + y_j . c_g) y_j,  y_j = scale x_j
    const double tw = tau * fma(scale, d, rgj);
    const double a = g > jj ? -tw * scale : 0.0;
#pragma unroll
    for (int it = 0; it < C::KWT; ++it)
#pragma unroll
      for (int b = 0; b < 2; ++b) cp[it][b] = fma(a, xv[it][b], cp[it][b]);
    if (!(F & 2) && warp == 0) {
      if (t == 0) {
        if (g > jj) R[rix<C>(j0 + jj, j0 + g)] = rgj - tw;
        else if (g < jj) U[g * 8 + jj] = d;  // x_g . x_jj  (scaled in T below)
        else R[rix<C>(j0 + jj, j0 + jj)] = beta;
      }
      if (lane == jj) { tau_r = tau; scale_r = scale; }
    }
    if (g == jj) scale_g = scale;
    PT(4);
  }
  // Y = X diag(scale): registers (B operand of Z) and this warp's rows of Y^T
#pragma unroll
  for (int it = 0; it < C::KWT; ++it) {
    cp[it][0] *= scale_g;
    cp[it][1] *= scale_g;
    *reinterpret_cast<double2*>(Ytw + g * C::LDYT + 8 * it + 2 * t) = make_double2(cp[it][0], cp[it][1]);
  }
  if (!(F & 8) && warp == 0) {
    if (lane < 8) { taus[lane] = tau_r; scs[lane] = scale_r; }
    __syncwarp();
    // T (8 x 8 upper triangular): T[r][r] = tau_r,
    // T[r][j] = -tau_j sum_{m=r}^{j-1} T[r][m] (y_m . y_j); lane r builds row r.
    if (lane < 8) {
      const int r = lane;
      double trow[8], sc[8], tu[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) { sc[m] = scs[m]; tu[m] = taus[m]; }
#pragma unroll
      for (int m = 0; m < 8; ++m) trow[m] = (m == r) ? tu[m] : 0.0;
#pragma unroll
      for (int j = 1; j < 8; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int m = 0; m < j; ++m) acc = fma(trow[m], (U[m * 8 + j] * sc[m]) * sc[j], acc);  // trow[m] = 0 for m < r
        if (j > r) trow[j] = -tu[j] * acc;
      }
#pragma unroll
      for (int m = 0; m < 8; ++m) T[r * C::LDT + m] = trow[m];
    }
  }
  PT(5);
#ifdef JQ_PANEL_TIMING
  if (lane == 0 && warp == 0)
    for (int i = 0; i < 6; ++i) g_ptime[i] += pt_acc[i];
#endif
}


template <class C, int F>
__global__ void __launch_bounds__(C::THREADS, 1) pexp(long long* cyc, double* sink, int reps) {
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
    factor_panel_x<C, F>(c, R, 0, smem_dyn + C::OFF_YT + warp * C::SZ_YT, smem_dyn + C::OFF_T, smem_dyn + C::OFF_U,
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
}
template <int F>
void run(const char* nm) {
  using C = jq::Cfg<128>;
  long long* cyc; double* sink; cudaMallocManaged(&cyc, 64); cudaMalloc(&sink, 8 * 4096);
  cudaFuncSetAttribute(jq::pexp<C, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  for (int w = 0; w < 2; ++w) { jq::pexp<C, F><<<1, C::THREADS, C::SMEM>>>(cyc, sink, 200); cudaDeviceSynchronize(); }
  printf("%-36s %6lld cycles/panel %6.0f /column  %s\n", nm, cyc[0], cyc[0] / 8.0, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<0>("baseline");
  run<1>("no R loads");
  run<2>("no warp-0 writes");
  run<4>("no publish");
  run<8>("no T tail");
  run<15>("none of the above");
}
