// jq_svd.cu — singular values and right singular vectors of R by one-sided
// Jacobi (replaces the paper's cusolverDnXgesvd).
//
// Rule: rotate column pairs until every |a_p . a_q| /
// (|a_p| |a_q|) < 1e-14, at most 64 sweeps, else error (JQ_E_NOCONV).  A column
// with |a|^2 <= (n eps |R|_F)^2 is numerically zero and never rotated (the same
// guard as oracle/svd.py; without it rank-deficient R never meets the bar).
// Parallel order: the SPEC's cyclic-by-rows order is inherently sequential, so the
// GPU uses the round-robin (circle) tournament — n-1 rounds of n/2 disjoint
// pairs per sweep, every pair once per sweep.  Same rotation formula and
// stopping rule; results agree with the oracle to rounding.
#include <algorithm>
#include <cmath>

#include <cooperative_groups.h>

#include "jq_internal.cuh"

namespace jq {

constexpr int SVD_THREADS = 1024;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// player at position k in round r of the circle method over n (even) players
__device__ __forceinline__ int rr_player(int k, int r, int n) {
  return k == 0 ? 0 : ((k - 1 + r) % (n - 1)) + 1;
}

// A (column-major n x n, column j = R[:, j]) and V (column-major) in global memory.
__global__ void __launch_bounds__(SVD_THREADS, 1)
jacobi_kernel(double* __restrict__ A, double* __restrict__ V, int n, int want_v, double tol,
              int max_sweeps, int* flags, double* __restrict__ values, double* __restrict__ vout, int n_out) {
  __shared__ int rotated;
  __shared__ double red[SVD_THREADS / 32];
  __shared__ double sig[256];
  __shared__ int perm[256];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = SVD_THREADS / 32;

  // |R|_F^2 -> negligible-column threshold
  double f = 0.0;
  for (int i = tid; i < n * n; i += SVD_THREADS) f = fma(A[i], A[i], f);
  f = warp_sum(f);
  if (lane == 0) red[warp] = f;
  __syncthreads();
  if (warp == 0) {
    double v = lane < nw ? red[lane] : 0.0;
    v = warp_sum(v);
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  const double eps = 2.220446049250313e-16;
  const double tiny = (double(n) * eps) * (double(n) * eps) * red[0];
  const int npairs = n / 2;

  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int r = 0; r < n - 1; ++r) {
      for (int pi = warp; pi < npairs; pi += nw) {
        int p = rr_player(pi, r, n), q = rr_player(n - 1 - pi, r, n);
        if (p > q) { int tmp = p; p = q; q = tmp; }
        double* ap = A + (size_t)p * n;
        double* aq = A + (size_t)q * n;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < n; i += 32) {
          const double x = ap[i], y = aq[i];
          al = fma(x, x, al);
          be = fma(y, y, be);
          ga = fma(x, y, ga);
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (al <= tiny || be <= tiny) continue;
        if (ga == 0.0 || fabs(ga) < tol * (sqrt(al) * sqrt(be))) continue;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = zeta >= 0.0 ? 1.0 / (zeta + sqrt(1.0 + zeta * zeta))
                                     : -1.0 / (-zeta + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int i = lane; i < n; i += 32) {
          const double x = ap[i], y = aq[i];
          ap[i] = c * x - s * y;
          aq[i] = s * x + c * y;
        }
        if (want_v) {
          double* vp = V + (size_t)p * n;
          double* vq = V + (size_t)q * n;
          for (int i = lane; i < n; i += 32) {
            const double x = vp[i], y = vq[i];
            vp[i] = c * x - s * y;
            vq[i] = s * x + c * y;
          }
        }
        if (lane == 0) rotated = 1;
      }
      __syncthreads();
    }
    if (!rotated) break;
    __syncthreads();
  }
  if (sweep == max_sweeps && tid == 0) atomicOr(flags, FLAG_NOCONV);

  // sigma = column norms, sorted descending (stable on index)
  for (int j = warp; j < n; j += nw) {
    double s = 0.0;
    for (int i = lane; i < n; i += 32) s = fma(A[(size_t)j * n + i], A[(size_t)j * n + i], s);
    s = warp_sum(s);
    if (lane == 0) sig[j] = sqrt(s);
  }
  __syncthreads();
  for (int j = tid; j < n; j += SVD_THREADS) {
    int rank = 0;
    const double sj = sig[j];
    for (int k = 0; k < n; ++k) rank += (sig[k] > sj) || (sig[k] == sj && k < j);
    perm[rank] = j;
  }
  __syncthreads();
  for (int k = tid; k < n_out; k += SVD_THREADS) values[k] = sig[perm[k]];
  if (want_v && vout) {
    // V row-major n_out x n_out: vout[i][k] = V[:, perm[k]][i]
    for (int idx = tid; idx < n_out * n_out; idx += SVD_THREADS) {
      const int i = idx / n_out, k = idx - i * n_out;
      vout[idx] = V[(size_t)perm[k] * n + i];
    }
  }
}

// Multi-CTA variant: one CTA per column pair and round (np/2 CTAs, cooperative
// launch, one grid-wide barrier per round).  Same pairs, rotation formula and
// stopping rule as jacobi_kernel; the block reductions and the norm partials are
// summed in a fixed order, so results are deterministic.  Thread i owns row i.
constexpr int SVDC_THREADS = 256;

__device__ __forceinline__ void block_sum3(double& a, double& b, double& c, double* red) {
  a = warp_sum(a); b = warp_sum(b); c = warp_sum(c);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) { red[warp] = a; red[32 + warp] = b; red[64 + warp] = c; }
  __syncthreads();
  a = b = c = 0.0;
  for (int w = 0; w < nw; ++w) { a += red[w]; b += red[32 + w]; c += red[64 + w]; }
}

__global__ void __launch_bounds__(SVDC_THREADS)
jacobi_coop_kernel(double* __restrict__ A, double* __restrict__ V, int n, int want_v, double tol, int max_sweeps,
                   int* flags, double* __restrict__ part, int* __restrict__ rotated_sweep, double* __restrict__ values,
                   double* __restrict__ vout, int n_out) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[96];
  __shared__ double sig[256];
  __shared__ int perm[256];
  const int pi = blockIdx.x, i = threadIdx.x;
  // |R|_F^2 (fixed-order two-level sum) -> negligible-column threshold
  {
    double f = 0.0;
    for (int j = pi; j < n; j += gridDim.x)
      if (i < n) f = fma(A[(size_t)j * n + i], A[(size_t)j * n + i], f);
    double z1 = 0.0, z2 = 0.0;
    block_sum3(f, z1, z2, red);
    if (i == 0) part[pi] = f;
  }
  grid.sync();
  double fro = 0.0;
  for (int b = 0; b < (int)gridDim.x; ++b) fro += part[b];
  const double eps = 2.220446049250313e-16;
  const double tiny = (double(n) * eps) * (double(n) * eps) * fro;
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    for (int r = 0; r < n - 1; ++r) {
      int p = rr_player(pi, r, n), q = rr_player(n - 1 - pi, r, n);
      if (p > q) { const int tmp = p; p = q; q = tmp; }
      double* ap = A + (size_t)p * n;
      double* aq = A + (size_t)q * n;
      const double x = i < n ? ap[i] : 0.0, y = i < n ? aq[i] : 0.0;
      double al = x * x, be = y * y, ga = x * y;
      block_sum3(al, be, ga, red);
      const bool rot = !(al <= tiny || be <= tiny || ga == 0.0 || fabs(ga) < tol * (sqrt(al) * sqrt(be)));
      if (rot) {
        const double zeta = (be - al) / (2.0 * ga);
        const double t = zeta >= 0.0 ? 1.0 / (zeta + sqrt(1.0 + zeta * zeta))
                                     : -1.0 / (-zeta + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        if (i < n) {
          ap[i] = c * x - s * y;
          aq[i] = s * x + c * y;
          if (want_v) {
            double* vp = V + (size_t)p * n;
            double* vq = V + (size_t)q * n;
            const double u = vp[i], w = vq[i];
            vp[i] = c * u - s * w;
            vq[i] = s * u + c * w;
          }
        }
        if (i == 0) rotated_sweep[sweep] = 1;  // benign race: every writer stores 1
      }
      grid.sync();
    }
    if (!*(volatile int*)&rotated_sweep[sweep]) break;
  }
  if (sweep == max_sweeps && pi == 0 && i == 0) atomicOr(flags, FLAG_NOCONV);
  // sigma = column norms (CTA pi: columns pi, pi + grid, ...), then CTA 0 sorts
  for (int j = pi; j < n; j += gridDim.x) {
    double s = (i < n) ? A[(size_t)j * n + i] * A[(size_t)j * n + i] : 0.0, z1 = 0.0, z2 = 0.0;
    block_sum3(s, z1, z2, red);
    if (i == 0) part[j] = sqrt(s);
  }
  grid.sync();
  if (pi != 0) return;
  for (int j = i; j < n; j += blockDim.x) sig[j] = part[j];
  __syncthreads();
  for (int j = i; j < n; j += blockDim.x) {
    int rank = 0;
    const double sj = sig[j];
    for (int k = 0; k < n; ++k) rank += (sig[k] > sj) || (sig[k] == sj && k < j);
    perm[rank] = j;
  }
  __syncthreads();
  for (int k = i; k < n_out; k += blockDim.x) values[k] = sig[perm[k]];
  if (want_v && vout)
    for (int idx = i; idx < n_out * n_out; idx += blockDim.x) {
      const int r = idx / n_out, k = idx - r * n_out;
      vout[idx] = V[(size_t)perm[k] * n + r];
    }
}

// A_cm[j*np + i] = R[i*n + j] (zero padded to np), V = I
__global__ void svd_init_kernel(const double* __restrict__ r, int n, int np, double* __restrict__ A,
                                double* __restrict__ V) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < np * np; idx += gridDim.x * blockDim.x) {
    const int j = idx / np, i = idx - j * np;
    A[idx] = (i < n && j < n) ? r[i * n + j] : 0.0;
    if (V) V[idx] = (i == j) ? 1.0 : 0.0;
  }
}

size_t svd_ws_bytes(int64_t n) {
  const int64_t np = n + (n & 1);
  return 2 * ws_bytes(size_t(np) * np, 8) + ws_bytes(512, 8) + ws_bytes(128, 4);
}

int svd_dev(jq_ctx* ctx, const double* r, int64_t n, int want_v, double* values, double* v) {
  if (n > 256) return fail(JQ_E_INVALID, "svd_of_r supports n <= 256");
  if (n == 0) return JQ_OK;
  const int np = (int)(n + (n & 1));  // the tournament needs an even count; pad a zero column
  double* A = ws_alloc<double>(ctx, size_t(np) * np);
  double* V = ws_alloc<double>(ctx, size_t(np) * np);
  if (!A || !V) return fail(JQ_E_OOM, "workspace exhausted (svd)");
  svd_init_kernel<<<(unsigned)cdiv(int64_t(np) * np, 256), 256, 0, ctx->stream>>>(r, (int)n, np, A, V);
  JQ_CHECK_LAUNCH(ctx);
  if (np >= 32) {
    // cooperative multi-CTA sweep: np/2 CTAs (<= 128, co-resident on 148 SMs)
    double* part = ws_alloc<double>(ctx, 512);
    int* rot = ws_alloc<int>(ctx, 128);
    if (!part || !rot) return fail(JQ_E_OOM, "workspace exhausted (svd)");
    JQ_CUDA(cudaMemsetAsync(rot, 0, 128 * sizeof(int), ctx->stream));
    int npi = np, wv = want_v, ms = 64, nout = (int)n;
    double tol = 1e-14;
    double* vo = want_v ? v : nullptr;
    int* fl = ctx->d_flags;
    void* args[] = {&A, &V, &npi, &wv, &tol, &ms, &fl, &part, &rot, &values, &vo, &nout};
    JQ_CUDA(cudaLaunchCooperativeKernel((const void*)jacobi_coop_kernel, dim3(np / 2), dim3(SVDC_THREADS), args, 0,
                                        ctx->stream));
    JQ_CHECK_LAUNCH(ctx);
    return JQ_OK;
  }
  jacobi_kernel<<<1, SVD_THREADS, 0, ctx->stream>>>(A, V, np, want_v, 1e-14, 64, ctx->d_flags, values,
                                                    want_v ? v : nullptr, (int)n);
  JQ_CHECK_LAUNCH(ctx);
  return JQ_OK;
}

}  // namespace jq

using namespace jq;

extern "C" int jq_svd_of_r(jq_ctx* ctx, const double* r, int64_t n, int want_v, double* values, double* v) {
  if (!ctx) return fail(JQ_E_INVALID, "null context");
  if (n < 0) return fail(JQ_E_INVALID, "negative size");
  if (n == 0) return JQ_OK;
  JQ_TRY(begin_call(ctx));
  JQ_TRY(ws_reserve(ctx, stage_bytes(r, n * n) + stage_bytes((const double*)values, n) +
                             stage_bytes((const double*)v, n * n) + svd_ws_bytes(n)));
  const double* dr;
  double *dval, *dv = nullptr;
  JQ_TRY(stage_in(ctx, r, n * n, &dr));
  JQ_TRY(stage_out(ctx, values, n, &dval));
  if (want_v) JQ_TRY(stage_out(ctx, v, n * n, &dv));
  JQ_TRY(svd_dev(ctx, dr, n, want_v, dval, dv));
  JQ_TRY(copy_out(ctx, values, (const double*)dval, n));
  if (want_v) JQ_TRY(copy_out(ctx, v, (const double*)dv, n * n));
  return sync_and_check_flags(ctx);
}
