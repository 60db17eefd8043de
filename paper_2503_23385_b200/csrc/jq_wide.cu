// jq_wide.cu — Householder QR for WIDE matrices (256 < n <= 512 columns): the
// path householder_r / figaro_r / reduce take where the register-resident streaming
// TSQR leaves (jq_tsqr.cu, NP <= 256) do not fit.  SPEC.md:250-258 (Householder R,
// zero-row padding :296), :356 ("n <= a few hundred").
//
// TSQR with dense leaves in global memory: the rows are cut into blocks of B >= n rows,
// each block is copied (zero padded) into a workspace slab and factored in place by
// one CTA with blocked Householder (panels of P = 8 columns: explicit reflectors for
// the panel, compact WY T, then ONE two-pass update of the trailing columns,
// Z = V^T W, Z' = T^T Z, W -= V Z', threads over columns so every row access is
// coalesced); the n x n R factors are then combined by a fixed binary tree of the
// same kernel on [R_a; R_b] slabs.  Reductions run in a fixed order (deterministic).
// The slabs stay in L2 for moderate sizes; this path trades the leaves' tensor-core
// throughput for generality (the narrow path is the performance path).
#include <algorithm>
#include <cmath>

#include "jq_internal.cuh"

namespace jq {

constexpr int WQ_THREADS = 256;
constexpr int WQ_P = 8;        // panel width
constexpr int WQ_MAXN = 512;   // columns
constexpr int WQ_CPT = WQ_MAXN / WQ_THREADS;  // trailing columns per thread

__device__ __forceinline__ double wq_warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum K per-thread partials across the CTA (fixed order); result in every thread.
template <int K>
__device__ __forceinline__ void wq_block_sum(double (&v)[K], double* red /* [8][K] */) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = wq_warp_sum(v[k]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) red[warp * K + k] = v[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < WQ_THREADS / 32; ++w) s += red[w * K + k];
    v[k] = s;
  }
}

// Factor the slab W (B x n, row-major, ld n) in place: on exit its upper n x n
// triangle is R (not sign-canonical).  Dynamic shared memory: the panel V (B x P).
__device__ void wq_factor(double* __restrict__ W, int B, int n, double* __restrict__ Vs, double* red) {
  __shared__ double T[WQ_P][WQ_P];
  __shared__ double tau_s[WQ_P];
  const int tid = threadIdx.x;
  for (int j0 = 0; j0 < n; j0 += WQ_P) {
    const int pw = min(WQ_P, n - j0);
    // ---- panel: explicit Householder column by column on rows j0.., columns j0..j0+pw-1
    for (int jj = 0; jj < pw; ++jj) {
      const int j = j0 + jj;
      double s[1] = {0.0};
      for (int r = j + 1 + tid; r < B; r += WQ_THREADS) s[0] = fma(W[(size_t)r * n + j], W[(size_t)r * n + j], s[0]);
      wq_block_sum<1>(s, red);
      const double alpha = W[(size_t)j * n + j];
      double tau = 0.0, beta = alpha, scale = 0.0;
      if (s[0] > 0.0) {
        const double nrm = sqrt(fma(alpha, alpha, s[0]));
        beta = alpha >= 0.0 ? -nrm : nrm;
        tau = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      // y_j = scale x_j (below the diagonal), kept in W and in the panel copy V
      for (int r = j0 + tid; r < B; r += WQ_THREADS) {
        double v;
        if (r < j) v = 0.0;
        else if (r == j) v = 1.0;
        else {
          v = W[(size_t)r * n + j] * scale;
          W[(size_t)r * n + j] = v;
        }
        Vs[(size_t)(r - j0) * WQ_P + jj] = v;
      }
      if (tid == 0) {
        W[(size_t)j * n + j] = beta;
        tau_s[jj] = tau;
      }
      __syncthreads();
      // apply H_j to the remaining panel columns j+1 .. j0+pw-1
      const int rem = pw - jj - 1;
      if (rem > 0) {
        double d[WQ_P - 1];
#pragma unroll
        for (int k = 0; k < WQ_P - 1; ++k) d[k] = 0.0;
        for (int r = j + tid; r < B; r += WQ_THREADS) {
          const double v = Vs[(size_t)(r - j0) * WQ_P + jj];
#pragma unroll
          for (int k = 0; k < WQ_P - 1; ++k)
            if (k < rem) d[k] = fma(v, W[(size_t)r * n + j + 1 + k], d[k]);
        }
        wq_block_sum<WQ_P - 1>(d, red);
        for (int r = j + tid; r < B; r += WQ_THREADS) {
          const double v = Vs[(size_t)(r - j0) * WQ_P + jj];
#pragma unroll
          for (int k = 0; k < WQ_P - 1; ++k)
            if (k < rem) W[(size_t)r * n + j + 1 + k] = fma(-tau * d[k], v, W[(size_t)r * n + j + 1 + k]);
        }
        __syncthreads();
      }
    }
    if (j0 + pw >= n) break;
    // ---- T (pw x pw, upper): T[k][k] = tau_k, T[0:k, k] = -tau_k T[0:k, 0:k] (V^T v_k)
    {
      double g[WQ_P * (WQ_P - 1) / 2];
#pragma unroll
      for (int k = 0; k < WQ_P * (WQ_P - 1) / 2; ++k) g[k] = 0.0;
      for (int r = j0 + tid; r < B; r += WQ_THREADS) {
        const double* vr = Vs + (size_t)(r - j0) * WQ_P;
#pragma unroll
        for (int a = 0; a < WQ_P; ++a)
#pragma unroll
          for (int b = a + 1; b < WQ_P; ++b) {
            const int e = a * WQ_P - a * (a + 1) / 2 + (b - a - 1);
            g[e] = fma(vr[a], vr[b], g[e]);
          }
      }
      wq_block_sum<WQ_P * (WQ_P - 1) / 2>(g, red);
      if (tid == 0) {
        double G[WQ_P][WQ_P];
        for (int a = 0; a < WQ_P; ++a)
          for (int b = a + 1; b < WQ_P; ++b) G[a][b] = g[a * WQ_P - a * (a + 1) / 2 + (b - a - 1)];
        for (int k = 0; k < pw; ++k) {
          T[k][k] = tau_s[k];
          for (int a = 0; a < k; ++a) {
            double acc = 0.0;
            for (int m = a; m < k; ++m) acc = fma(T[a][m], G[m][k], acc);
            T[a][k] = -tau_s[k] * acc;
          }
          for (int a = k + 1; a < WQ_P; ++a) T[a][k] = 0.0;
        }
      }
      __syncthreads();
    }
    // ---- trailing update of columns c >= j0 + pw: Z = V^T W, Z' = T^T Z, W -= V Z'
    double z[WQ_CPT][WQ_P];
#pragma unroll
    for (int u = 0; u < WQ_CPT; ++u)
#pragma unroll
      for (int k = 0; k < WQ_P; ++k) z[u][k] = 0.0;
    const int c0 = j0 + pw;
    for (int r = j0; r < B; ++r) {
      const double* vr = Vs + (size_t)(r - j0) * WQ_P;
      double v[WQ_P];
#pragma unroll
      for (int k = 0; k < WQ_P; ++k) v[k] = vr[k];
#pragma unroll
      for (int u = 0; u < WQ_CPT; ++u) {
        const int c = c0 + tid + u * WQ_THREADS;
        if (c < n) {
          const double w = W[(size_t)r * n + c];
#pragma unroll
          for (int k = 0; k < WQ_P; ++k) z[u][k] = fma(v[k], w, z[u][k]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < WQ_CPT; ++u) {
      double zz[WQ_P];
#pragma unroll
      for (int k = 0; k < WQ_P; ++k) {
        double acc = 0.0;
#pragma unroll
        for (int m = 0; m < WQ_P; ++m) acc = fma(T[m][k], z[u][m], acc);  // (T^T z)[k]
        zz[k] = acc;
      }
#pragma unroll
      for (int k = 0; k < WQ_P; ++k) z[u][k] = zz[k];
    }
    for (int r = j0; r < B; ++r) {
      const double* vr = Vs + (size_t)(r - j0) * WQ_P;
      double v[WQ_P];
#pragma unroll
      for (int k = 0; k < WQ_P; ++k) v[k] = vr[k];
#pragma unroll
      for (int u = 0; u < WQ_CPT; ++u) {
        const int c = c0 + tid + u * WQ_THREADS;
        if (c < n) {
          double w = W[(size_t)r * n + c];
#pragma unroll
          for (int k = 0; k < WQ_P; ++k) w = fma(-v[k], z[u][k], w);
          W[(size_t)r * n + c] = w;
        }
      }
    }
    __syncthreads();
  }
}

// Leaves: block b copies rows [b B, b B + B) of M (zero padded) into slab b, factors it
// and writes R_b (n x n upper) to out[b].
__global__ void __launch_bounds__(WQ_THREADS, 1) wq_leaf_kernel(const double* __restrict__ M, int64_t rows, int n,
                                                                int B, double* __restrict__ slabs,
                                                                double* __restrict__ out) {
  extern __shared__ __align__(16) double Vs[];
  __shared__ double red[8 * 28];
  const int64_t b = blockIdx.x;
  double* W = slabs + (size_t)b * B * n;
  for (int64_t e = threadIdx.x; e < (int64_t)B * n; e += WQ_THREADS) {
    const int64_t r = b * B + e / n;
    W[e] = r < rows ? M[r * n + e % n] : 0.0;
  }
  __syncthreads();
  wq_factor(W, B, n, Vs, red);
  double* R = out + (size_t)b * n * n;
  for (int e = threadIdx.x; e < n * n; e += WQ_THREADS) {
    const int r = e / n, c = e % n;
    R[e] = c >= r ? W[(size_t)r * n + c] : 0.0;
  }
}

// Tree level: pair c = (R[2c], R[2c + 1]) -> out[c] (an odd last factor is copied).
__global__ void __launch_bounds__(WQ_THREADS, 1) wq_combine_kernel(const double* __restrict__ in, int64_t count,
                                                                   int n, double* __restrict__ slabs,
                                                                   double* __restrict__ out) {
  extern __shared__ __align__(16) double Vs[];
  __shared__ double red[8 * 28];
  const int64_t c = blockIdx.x;
  const double* a = in + (size_t)(2 * c) * n * n;
  double* R = out + (size_t)c * n * n;
  if (2 * c + 1 >= count) {
    for (int e = threadIdx.x; e < n * n; e += WQ_THREADS) R[e] = a[e];
    return;
  }
  const double* bb = a + (size_t)n * n;
  double* W = slabs + (size_t)c * 2 * n * n;
  for (int e = threadIdx.x; e < 2 * n * n; e += WQ_THREADS) W[e] = e < n * n ? a[e] : bb[e - n * n];
  __syncthreads();
  wq_factor(W, 2 * n, n, Vs, red);
  for (int e = threadIdx.x; e < n * n; e += WQ_THREADS) {
    const int r = e / n, cc = e % n;
    R[e] = cc >= r ? W[(size_t)r * n + cc] : 0.0;
  }
}

static int64_t wq_block_rows(int64_t rows, int n, int sms) {
  // >= n rows per leaf (R needs them), about one leaf per SM, at most 4 n rows
  const int64_t per = cdiv(std::max<int64_t>(rows, 1), sms);
  return std::max<int64_t>(n, std::min<int64_t>(4 * (int64_t)n, cdiv(per, 8) * 8));
}

size_t wide_tsqr_ws_bytes(int64_t rows, int64_t n, int sms) {
  const int64_t B = wq_block_rows(rows, (int)n, sms);
  const int64_t leaves = std::max<int64_t>(1, cdiv(rows, B));
  return ws_bytes(size_t(leaves) * B * n, 8) + 2 * ws_bytes(size_t(leaves) * n * n, 8) + 4096;
}

// R (n x n, canonical when asked) of the row-major rows x n matrix m (device).
int wide_tsqr_dev(jq_ctx* ctx, const double* m, int64_t rows, int64_t n, double* r_out, bool canonical) {
  if (n > WQ_MAXN) return fail(JQ_E_INVALID, "more than 512 columns");
  const int64_t B = wq_block_rows(rows, (int)n, ctx->sms);
  const int64_t leaves = std::max<int64_t>(1, cdiv(rows, B));
  double* slabs = ws_alloc<double>(ctx, size_t(leaves) * B * n);
  double* ra = ws_alloc<double>(ctx, size_t(leaves) * n * n);
  double* rb = ws_alloc<double>(ctx, size_t(leaves) * n * n);
  if (!slabs || !ra || !rb) return fail(JQ_E_OOM, "workspace exhausted (wide TSQR)");
  const size_t smem_leaf = size_t(B) * WQ_P * 8;
  const size_t smem_comb = size_t(2 * n) * WQ_P * 8;
  const size_t smem = std::max(smem_leaf, smem_comb);
  JQ_CUDA(cudaFuncSetAttribute(wq_leaf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  JQ_CUDA(cudaFuncSetAttribute(wq_combine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  stage_event(ctx, 3);
  wq_leaf_kernel<<<(unsigned)leaves, WQ_THREADS, smem_leaf, ctx->stream>>>(m, rows, (int)n, (int)B, slabs, ra);
  JQ_CHECK_LAUNCH(ctx);
  stage_event(ctx, 4);
  int64_t count = leaves;
  double* cur = ra;
  double* nxt = rb;
  while (count > 1) {
    const int64_t half = (count + 1) / 2;
    wq_combine_kernel<<<(unsigned)half, WQ_THREADS, smem_comb, ctx->stream>>>(cur, count, (int)n, slabs, nxt);
    JQ_CHECK_LAUNCH(ctx);
    std::swap(cur, nxt);
    count = half;
  }
  if (canonical) return canonicalize_dev(ctx, cur, n, r_out);
  JQ_CUDA(cudaMemcpyAsync(r_out, cur, size_t(n) * n * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  return JQ_OK;
}

}  // namespace jq
