// jq_tsqr.cu — tall-skinny Householder QR (TSQR) on the FP64 tensor pipe (DMMA).
//
// Replaces the paper's cusolverDnXgeqrf finishing step (SPEC.md
// householder_r :250-258, figaro_r :278-286).  Design:
//
//  * Streaming leaves.  Each CTA owns a contiguous range of rows of the (virtual)
//    reduced matrix and keeps a running upper-triangular R (NP x NP, in shared
//    memory for NP <= 128, in its L2-resident global slab for NP = 256).  It
//    absorbs the range K rows at a time: R <- qr([R; C]).  Every reflector of
//    [R; C] is v = [e_j ; y_j] (it touches one row of R and all K chunk rows), so
//    the block reflector of a panel is V = [I; Y] and the compact-WY trailing
//    update is
//        Z = R[panel rows, trail] + Y^T C[:, trail];  W = T^T Z;
//        R[panel rows, trail] -= W;                     C[:, trail] -= Y W.
//  * Register-resident chunk.  C lives in registers in the DMMA (m8n8k4 f64)
//    accumulator layout, transposed: warp w owns column tiles w and NLT-1-w
//    (balanced triangular work) and holds C^T[l][i] for all K rows.  Both GEMMs
//    of the trailing update take their A operand straight from those registers by
//    permuting the reduction index of each DMMA (k = t  <->  i = 8*it + 2*t + b),
//    so the only shared-memory operands are Y, Y^T and T.
//  * Panels of 8 columns (one column tile) are factored by the warp that owns the
//    tile, from registers, with 4-lane (quad) reductions; the owner of the next
//    panel updates that tile first, so panel factorisation overlaps the other
//    warps' trailing updates (one __syncthreads per panel).
//  * Tree.  The P leaf R's are combined by a fixed binary tree of the same kernel
//    (R_init = R_a, rows = R_b), so results are deterministic for a given P.
//
// The Figaro source generates the reduced rows of Claim 1 on the fly (PAPER.md
// :53-58): top rows [sqrt(m2g) A_i | head(B_g)], bottom rows
// [0 | sqrt(m1g) tail(B_g)_r] with the prefix sum carried from the head/tail pass
// (jq_headtail.cu), so the reduced matrix never exists in HBM.
#include <algorithm>
#include <cmath>

#include "jq_internal.cuh"

namespace jq {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

template <int NP_>
struct Cfg {
  static constexpr int NP = NP_;
  static constexpr int WARPS = NP / 16;     // 2 column tiles per warp
  static constexpr int THREADS = WARPS * 32;
  static constexpr int NLT = NP / 8;        // column tiles
  static constexpr int K = NP >= 256 ? 32 : 64;  // chunk rows
  static constexpr int KT = K / 8;          // row tiles per chunk
  static constexpr bool R_SMEM = NP <= 128;
  static constexpr int LDS = NP + 2;        // stage row stride   (== 2 mod 16: conflict-free)
  static constexpr int LDR = R_SMEM ? NP + 2 : NP;
  static constexpr int LDY = 10;            // Ys  (K x 8)
  static constexpr int LDYT = K + 2;        // Yt  (8 x K)
  static constexpr int LDT = 10;            // T   (8 x 8)
  // shared memory carve-up (doubles)
  static constexpr int OFF_STAGE = 0;
  static constexpr int SZ_STAGE = K * LDS;
  static constexpr int OFF_R = OFF_STAGE + SZ_STAGE;
  static constexpr int SZ_R = R_SMEM ? NP * LDR : 0;
  static constexpr int OFF_YS = OFF_R + SZ_R;
  static constexpr int SZ_YS = K * LDY;
  static constexpr int OFF_YT = OFF_YS + 2 * SZ_YS;
  static constexpr int SZ_YT = 8 * LDYT;
  static constexpr int OFF_T = OFF_YT + 2 * SZ_YT;
  static constexpr int SZ_T = 8 * LDT;
  static constexpr int OFF_U = OFF_T + 2 * SZ_T;
  static constexpr int OFF_TAU = OFF_U + 64;
  static constexpr int OFF_S = OFF_TAU + 8;   // running prefix sums (Figaro source, <= NP)
  static constexpr int TOTAL = OFF_S + NP;
  static constexpr size_t SMEM = size_t(TOTAL) * sizeof(double);
};

// ------------------------------------------------------------------ row sources
// A source fills stage[i * LDS + c] for i < K, c < NP with rows row0 .. row0+K-1
// of its virtual matrix (zero beyond its rows / columns).

struct DenseSrc {
  const double* m;
  int64_t rows, cols, ld;
  template <class C>
  __device__ void begin(double*, int64_t) const {}
  template <class C>
  __device__ void load(double* stage, double*, int64_t row0) const {
    for (int idx = threadIdx.x; idx < C::K * C::NP; idx += C::THREADS) {
      int i = idx / C::NP, c = idx - i * C::NP;
      int64_t r = row0 + i;
      stage[i * C::LDS + c] = (r < rows && c < cols) ? __ldg(m + r * ld + c) : 0.0;
    }
  }
};

struct FigaroSrc {
  FigaroArgs fa;
  int64_t m1pad;  // A-part padded to a TILE_ROWS multiple; B-part starts here
  int n;          // n1 + n2

  // Running prefix S (per B column) at the first B-part row of this CTA.
  template <class C>
  __device__ void begin(double* S, int64_t row0) const {
    if (row0 < m1pad) row0 = m1pad;  // prefix is first used at the B-part start
    int64_t brow = row0 - m1pad;
    if (brow >= fa.m2) return;
    int64_t tile = brow / TILE_ROWS;
    for (int c = threadIdx.x; c < fa.n2; c += C::THREADS) {
      double s = fa.b_carry ? fa.b_carry[tile * fa.n2 + c] : 0.0;
      if (fa.b_prefix0) s += fa.b_prefix0[c];
      S[c] = s;
    }
  }

  template <class C>
  __device__ void load(double* stage, double* S, int64_t row0) const {
    const int n1 = (int)fa.n1, n2 = (int)fa.n2;
    if (row0 < m1pad) {
      // ---- top block rows: [sqrt(m2g) A_i | head(B_g)]
      for (int idx = threadIdx.x; idx < C::K * C::NP; idx += C::THREADS) {
        int i = idx / C::NP, c = idx - i * C::NP;
        int64_t r = row0 + i;
        double v = 0.0;
        if (r < fa.m1 && c < n) {
          int g = fa.gid_a ? fa.gid_a[r] : 0;
          if (g >= 0) {
            double m2g = fa.gid_a ? (double)fa.b_count[g] : (double)fa.m2_global;
            if (c < n1) v = __ldg(fa.a + r * n1 + c) * sqrt(m2g);
            else        v = fa.b_totals[(int64_t)g * n2 + (c - n1)] / sqrt(m2g);
          }
        }
        stage[i * C::LDS + c] = v;
      }
      return;
    }
    // ---- bottom block rows: [0 | sqrt(m1g) tail(B_g)]
    const int64_t b0 = row0 - m1pad;
    for (int idx = threadIdx.x; idx < C::K * C::NP; idx += C::THREADS) {
      int i = idx / C::NP, c = idx - i * C::NP;
      if (c < n1 || c >= n) stage[i * C::LDS + c] = 0.0;
    }
    for (int c = threadIdx.x; c < n2; c += C::THREADS) {
      double s = S[c];
#pragma unroll 8
      for (int i = 0; i < C::K; ++i) {
        int64_t br = b0 + i;
        double out = 0.0;
        if (br < fa.m2) {
          double x = __ldg(fa.b + br * n2 + c);
          int64_t rr;       // index of this row inside its key group
          double m1g;
          bool valid = true;
          if (fa.gid_b) {
            int g = fa.gid_b[br];
            valid = g >= 0;
            rr = valid ? br - fa.b_start[g] : 0;
            m1g = valid ? (double)fa.a_count[g] : 0.0;
          } else {
            rr = fa.b_row0 + br;
            m1g = (double)fa.m1_global;
          }
          if (valid) {
            if (rr == 0) {
              s = x;  // group's first row: it only feeds the head
            } else {
              double si = sqrt((double)rr);
              out = (si * x - s / si) / sqrt((double)rr + 1.0) * sqrt(m1g);
              s += x;
            }
          }
        }
        stage[i * C::LDS + n1 + c] = out;
      }
      S[c] = s;
    }
  }
};

// Householder factorisation of one 8-column panel held in registers by its owner
// warp (LAPACK dlarfg convention: beta = -sign(alpha) |x|, tau = (beta-alpha)/beta,
// v = [1; x2 / (alpha - beta)]).  Lane (g, t) holds column j0+g, rows 8*it+2*t+b.
// Writes Y (both layouts), T (forward accumulation) and the panel's R rows.
template <class C>
__device__ __forceinline__ void factor_panel(double (&cc)[C::KT][2], double* R, const int LDR, const int j0,
                                             double* Ys, double* Yt, double* T, double* U, double* taus,
                                             const int lane) {
  const int g = lane >> 2, t = lane & 3;
#pragma unroll 1
  for (int jj = 0; jj < 8; ++jj) {
    double sq = 0.0;
#pragma unroll
    for (int it = 0; it < C::KT; ++it)
#pragma unroll
      for (int b = 0; b < 2; ++b) sq = fma(cc[it][b], cc[it][b], sq);
    sq += __shfl_xor_sync(FULL, sq, 1);
    sq += __shfl_xor_sync(FULL, sq, 2);
    const double sj = __shfl_sync(FULL, sq, jj * 4);
    const double alpha = R[(j0 + jj) * LDR + j0 + jj];
    double tau = 0.0, beta = alpha, scale = 0.0;
    if (sj != 0.0) {
      const double nrm = sqrt(fma(alpha, alpha, sj));
      beta = alpha >= 0.0 ? -nrm : nrm;
      tau = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    if (g == jj) {
#pragma unroll
      for (int it = 0; it < C::KT; ++it)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const double y = cc[it][b] * scale;
          cc[it][b] = y;
          const int i = 8 * it + 2 * t + b;
          Ys[i * C::LDY + jj] = y;
          Yt[jj * C::LDYT + i] = y;
        }
    }
    // R row entries of the panel, read before lane (g,0) rewrites them
    const double rjg = R[(j0 + jj) * LDR + j0 + g];
    __syncwarp();
    if (lane == 0) {
      R[(j0 + jj) * LDR + j0 + jj] = beta;
      taus[jj] = tau;
    }
    double d = 0.0;
    double yv[C::KT][2];
#pragma unroll
    for (int it = 0; it < C::KT; ++it)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        yv[it][b] = Ys[(8 * it + 2 * t + b) * C::LDY + jj];
        d = fma(cc[it][b], yv[it][b], d);
      }
    d += __shfl_xor_sync(FULL, d, 1);
    d += __shfl_xor_sync(FULL, d, 2);
    if (g > jj) {
      const double tw = tau * (rjg + d);
#pragma unroll
      for (int it = 0; it < C::KT; ++it)
#pragma unroll
        for (int b = 0; b < 2; ++b) cc[it][b] = fma(-tw, yv[it][b], cc[it][b]);
      if (t == 0) R[(j0 + jj) * LDR + j0 + g] = rjg - tw;
    } else if (g < jj) {
      if (t == 0) U[g * 8 + jj] = d;  // y_g . y_jj  (for T)
    }
    __syncwarp();
  }
  // T (8 x 8 upper triangular): T[r][r] = tau_r,
  // T[r][j] = -tau_j sum_{m=r}^{j-1} T[r][m] (y_m . y_j); lane r builds row r.
  if (lane < 8) {
    const int r = lane;
    double trow[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) trow[m] = (m == r) ? taus[m] : 0.0;
#pragma unroll
    for (int j = 1; j < 8; ++j) {
      double acc = 0.0;
#pragma unroll
      for (int m = 0; m < j; ++m) acc = fma(trow[m], U[m * 8 + j], acc);  // trow[m] = 0 for m < r
      if (j > r) trow[j] = -taus[j] * acc;
    }
#pragma unroll
    for (int m = 0; m < 8; ++m) T[r * C::LDT + m] = trow[m];
  }
}

// ------------------------------------------------------------------ the kernel
// Each CTA: R (init zero, or R_init[cta]) absorbs its rows [row_begin, row_end)
// of `src`, then writes R (NP x NP, row-major, zeros below the diagonal) to
// r_out + cta * NP * NP.  For the combine step, CTA c absorbs rows of stack
// element 2c+1 into R = element 2c.
template <class C, class Src, bool COMBINE>
__global__ void __launch_bounds__(C::THREADS, 1)
tsqr_kernel(Src src, int64_t rows_per_cta, int64_t total_rows, const double* __restrict__ r_init,
            int64_t init_count, double* __restrict__ r_out) {
  extern __shared__ double smem_dyn[];
  double* stage = smem_dyn + C::OFF_STAGE;
  double* Ys0 = smem_dyn + C::OFF_YS;
  double* Yt0 = smem_dyn + C::OFF_YT;
  double* T0 = smem_dyn + C::OFF_T;
  double* U = smem_dyn + C::OFF_U;
  double* taus = smem_dyn + C::OFF_TAU;
  double* S = smem_dyn + C::OFF_S;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int64_t cta = blockIdx.x;

  double* R;
  constexpr int LDR = C::LDR;
  if constexpr (C::R_SMEM) R = smem_dyn + C::OFF_R;
  else R = r_out + cta * C::NP * C::NP;

  // ---- R init
  const double* rinit = nullptr;
  Src s = src;
  int64_t row_begin, row_end;
  if constexpr (COMBINE) {
    // stack element 2c is R_init, element 2c+1 supplies the rows
    rinit = r_init + (2 * cta) * C::NP * C::NP;
    if (2 * cta + 1 < init_count) {
      s.m = r_init + (2 * cta + 1) * C::NP * C::NP;
      row_begin = 0; row_end = C::NP;
    } else {
      row_begin = row_end = 0;
    }
  } else {
    row_begin = cta * rows_per_cta;
    row_end = min(total_rows, row_begin + rows_per_cta);
  }
  for (int idx = tid; idx < C::NP * C::NP; idx += C::THREADS) {
    int r = idx / C::NP, c = idx - r * C::NP;
    R[r * LDR + c] = rinit ? rinit[idx] : 0.0;
  }
  s.template begin<C>(S, row_begin);
  __syncthreads();

  // balanced column-tile ownership: warp w owns tiles w and NLT-1-w
  const int lt_idx[2] = {warp, C::NLT - 1 - warp};
  double c[2][C::KT][2];

  for (int64_t row0 = row_begin; row0 < row_end; row0 += C::K) {
    s.template load<C>(stage, S, row0);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int l0 = lt_idx[q] * 8;
#pragma unroll
      for (int it = 0; it < C::KT; ++it)
#pragma unroll
        for (int b = 0; b < 2; ++b) c[q][it][b] = stage[(8 * it + 2 * t + b) * C::LDS + l0 + g];
    }

    for (int p = 0; p < C::NLT; ++p) {
      const int j0 = 8 * p;
      const int buf = p & 1;
      double* Ys = Ys0 + buf * C::SZ_YS;
      double* Yt = Yt0 + buf * C::SZ_YT;
      double* T = T0 + buf * C::SZ_T;
      const int owner = p < C::WARPS ? p : C::NLT - 1 - p;
      if (warp == owner) {
        if (p < C::WARPS) factor_panel<C>(c[0], R, LDR, j0, Ys, Yt, T, U, taus, lane);
        else              factor_panel<C>(c[1], R, LDR, j0, Ys, Yt, T, U, taus, lane);
      }
      __syncthreads();

      // ---------------- trailing update of my column tiles right of the panel
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int lt = lt_idx[q];
        if (lt <= p) continue;
        const int l0 = lt * 8;
        double z[2];
        z[0] = R[(j0 + 2 * t) * LDR + l0 + g];
        z[1] = R[(j0 + 2 * t + 1) * LDR + l0 + g];
#pragma unroll
        for (int it = 0; it < C::KT; ++it) {
          dmma(z, c[q][it][0], Ys[(8 * it + 2 * t) * C::LDY + g]);
          dmma(z, c[q][it][1], Ys[(8 * it + 2 * t + 1) * C::LDY + g]);
        }
        double w[2] = {0.0, 0.0};
        dmma(w, z[0], T[(2 * t) * C::LDT + g]);
        dmma(w, z[1], T[(2 * t + 1) * C::LDT + g]);
        R[(j0 + 2 * t) * LDR + l0 + g] -= w[0];
        R[(j0 + 2 * t + 1) * LDR + l0 + g] -= w[1];
        const double nw0 = -w[0], nw1 = -w[1];
#pragma unroll
        for (int it = 0; it < C::KT; ++it) {
          dmma(c[q][it], nw0, Yt[(2 * t) * C::LDYT + 8 * it + g]);
          dmma(c[q][it], nw1, Yt[(2 * t + 1) * C::LDYT + 8 * it + g]);
        }
      }
    }
    __syncthreads();
  }

  // ---- write R (zeros strictly below the diagonal)
  if constexpr (C::R_SMEM) {
    double* out = r_out + cta * C::NP * C::NP;
    for (int idx = tid; idx < C::NP * C::NP; idx += C::THREADS) {
      int r = idx / C::NP, c2 = idx - r * C::NP;
      out[idx] = c2 >= r ? R[r * LDR + c2] : 0.0;
    }
  } else {
    for (int idx = tid; idx < C::NP * C::NP; idx += C::THREADS) {
      int r = idx / C::NP, c2 = idx - r * C::NP;
      if (c2 < r) R[idx] = 0.0;
    }
  }
}

// crop NP x NP -> n x n, optional canonical signs
__global__ void finalize_r_kernel(const double* __restrict__ rnp, int np, int n, bool canonical,
                                  double* __restrict__ out) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n * n; idx += gridDim.x * blockDim.x) {
    int r = idx / n, c = idx - r * n;
    double v = c >= r ? rnp[r * np + c] : 0.0;
    if (canonical && rnp[r * np + r] < 0.0) v = -v;
    out[idx] = (c >= r) ? v : 0.0;
  }
}

__global__ void canonicalize_kernel(const double* __restrict__ r, int n, double* __restrict__ out) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n * n; idx += gridDim.x * blockDim.x) {
    int row = idx / n;
    double v = r[idx];
    out[idx] = r[row * n + row] < 0.0 ? -v : v;
  }
}

// ------------------------------------------------------------------ host side
static int np_for(int64_t n) {
  if (n <= 16) return 16;
  if (n <= 32) return 32;
  if (n <= 64) return 64;
  if (n <= 128) return 128;
  if (n <= 256) return 256;
  return -1;
}

template <class C>
static int ctas_per_sm() {
  return C::R_SMEM ? std::max(1, int((227 * 1024) / (C::SMEM + 1024))) : 1;
}

template <class C, class Src, bool COMBINE>
static int launch_tsqr(jq_ctx* ctx, int grid, const Src& src, int64_t rows_per_cta,
                       int64_t total_rows, const double* r_init, int64_t init_count, double* r_out) {
  auto kern = tsqr_kernel<C, Src, COMBINE>;
  JQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
  kern<<<grid, C::THREADS, C::SMEM, ctx->stream>>>(src, rows_per_cta, total_rows, r_init,
                                                   init_count, r_out);
  JQ_CHECK_LAUNCH(ctx);
  return JQ_OK;
}

// Binary-tree combine of `count` NP x NP factors in `a` (ping-pong with `b`);
// returns a pointer to the final factor.
template <class C>
static int tree_combine(jq_ctx* ctx, double* a, double* b, int64_t count, double** result) {
  while (count > 1) {
    int64_t half = (count + 1) / 2;
    DenseSrc ds{nullptr, C::NP, C::NP, C::NP};
    JQ_TRY((launch_tsqr<C, DenseSrc, true>(ctx, (int)half, ds, 0, 0, a, count, b)));
    std::swap(a, b);
    count = half;
  }
  *result = a;
  return JQ_OK;
}

size_t tsqr_ws_bytes(int64_t rows, int64_t n, int sms) {
  int np = np_for(n);
  if (np < 0) return 0;
  int64_t leaves = std::max<int64_t>(1, std::min<int64_t>(int64_t(sms) * 32, cdiv(rows, 64)));
  return 2 * ws_bytes(size_t(leaves) * np * np, sizeof(double)) + ws_bytes(size_t(np) * np, 8);
}

size_t figaro_tsqr_ws_bytes(int64_t m1, int64_t m2, int64_t n, int sms) {
  return tsqr_ws_bytes(m1 + m2 + TILE_ROWS, n, sms);
}

template <class C, class Src>
static int run_stream(jq_ctx* ctx, const Src& src, int64_t vrows, int64_t align, int n,
                      bool canonical, double* r_out) {
  int64_t max_leaves = int64_t(ctx->sms) * ctas_per_sm<C>();
  int64_t units = std::max<int64_t>(1, cdiv(vrows, align));
  int64_t leaves = std::min(max_leaves, units);
  int64_t rows_per_cta = cdiv(units, leaves) * align;
  leaves = std::max<int64_t>(1, cdiv(vrows, rows_per_cta));
  double* a = ws_alloc<double>(ctx, size_t(leaves) * C::NP * C::NP);
  double* b = ws_alloc<double>(ctx, size_t((leaves + 1) / 2) * C::NP * C::NP + 1);
  if (!a || !b) return fail(JQ_E_OOM, "workspace exhausted (TSQR leaves)");
  ctx->timing.tsqr_ctas = leaves;
  ctx->timing.reduced_rows = vrows;
  cudaEventRecord(ctx->ev[3], ctx->stream);
  JQ_TRY((launch_tsqr<C, Src, false>(ctx, (int)leaves, src, rows_per_cta, vrows, nullptr, 0, a)));
  cudaEventRecord(ctx->ev[4], ctx->stream);
  double* fin = nullptr;
  JQ_TRY(tree_combine<C>(ctx, a, b, leaves, &fin));
  finalize_r_kernel<<<(int)cdiv(int64_t(n) * n, 256), 256, 0, ctx->stream>>>(fin, C::NP, n, canonical, r_out);
  JQ_CHECK_LAUNCH(ctx);
  cudaEventRecord(ctx->ev[5], ctx->stream);
  return JQ_OK;
}

template <class Src>
static int dispatch_stream(jq_ctx* ctx, const Src& src, int64_t vrows, int64_t align, int n,
                           bool canonical, double* r_out) {
  switch (np_for(n)) {
    case 16: return run_stream<Cfg<16>>(ctx, src, vrows, align, n, canonical, r_out);
    case 32: return run_stream<Cfg<32>>(ctx, src, vrows, align, n, canonical, r_out);
    case 64: return run_stream<Cfg<64>>(ctx, src, vrows, align, n, canonical, r_out);
    case 128: return run_stream<Cfg<128>>(ctx, src, vrows, align, n, canonical, r_out);
    case 256: return run_stream<Cfg<256>>(ctx, src, vrows, align, n, canonical, r_out);
  }
  return fail(JQ_E_INVALID, "column count above 256 is not supported by the TSQR kernels");
}

int tsqr_dense_dev(jq_ctx* ctx, const double* m, int64_t rows, int64_t cols, double* r_out,
                   bool canonical) {
  DenseSrc src{m, rows, cols, cols};
  return dispatch_stream(ctx, src, std::max<int64_t>(rows, 1), 64, (int)cols, canonical, r_out);
}

__global__ void pad_stack_kernel(const double* __restrict__ rs, int64_t count, int n, int np,
                                 double* __restrict__ out) {
  int64_t total = count * np * np;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t k = idx / (np * np);
    int rem = (int)(idx - k * np * np), r = rem / np, c = rem - r * np;
    out[idx] = (r < n && c < n) ? rs[(k * n + r) * n + c] : 0.0;
  }
}

template <class C>
static int stack_impl(jq_ctx* ctx, const double* rs, int64_t count, int64_t n, double* r_out,
                      bool canonical) {
  double* a = ws_alloc<double>(ctx, size_t(count) * C::NP * C::NP);
  double* b = ws_alloc<double>(ctx, size_t((count + 1) / 2) * C::NP * C::NP + 1);
  if (!a || !b) return fail(JQ_E_OOM, "workspace exhausted (R stack)");
  int64_t total = count * C::NP * C::NP;
  pad_stack_kernel<<<(int)std::min<int64_t>(cdiv(total, 256), 4096), 256, 0, ctx->stream>>>(
      rs, count, (int)n, C::NP, a);
  JQ_CHECK_LAUNCH(ctx);
  double* fin = nullptr;
  JQ_TRY(tree_combine<C>(ctx, a, b, count, &fin));
  finalize_r_kernel<<<(int)cdiv(n * n, 256), 256, 0, ctx->stream>>>(fin, C::NP, (int)n, canonical, r_out);
  JQ_CHECK_LAUNCH(ctx);
  return JQ_OK;
}

int tsqr_stack_dev(jq_ctx* ctx, const double* rs, int64_t count, int64_t n, double* r_out,
                   bool canonical) {
  switch (np_for(n)) {
    case 16: return stack_impl<Cfg<16>>(ctx, rs, count, n, r_out, canonical);
    case 32: return stack_impl<Cfg<32>>(ctx, rs, count, n, r_out, canonical);
    case 64: return stack_impl<Cfg<64>>(ctx, rs, count, n, r_out, canonical);
    case 128: return stack_impl<Cfg<128>>(ctx, rs, count, n, r_out, canonical);
    case 256: return stack_impl<Cfg<256>>(ctx, rs, count, n, r_out, canonical);
  }
  return fail(JQ_E_INVALID, "column count above 256 is not supported by the TSQR kernels");
}

int figaro_tsqr_dev(jq_ctx* ctx, const FigaroArgs& fa, double* r_out, bool canonical) {
  FigaroSrc src;
  src.fa = fa;
  src.m1pad = cdiv(fa.m1, TILE_ROWS) * TILE_ROWS;
  src.n = (int)(fa.n1 + fa.n2);
  int64_t vrows = src.m1pad + fa.m2;
  return dispatch_stream(ctx, src, std::max<int64_t>(vrows, 1), TILE_ROWS, src.n, canonical, r_out);
}

int canonicalize_dev(jq_ctx* ctx, const double* r, int64_t n, double* out) {
  canonicalize_kernel<<<(int)cdiv(n * n, 256), 256, 0, ctx->stream>>>(r, (int)n, out);
  JQ_CHECK_LAUNCH(ctx);
  return JQ_OK;
}

}  // namespace jq
