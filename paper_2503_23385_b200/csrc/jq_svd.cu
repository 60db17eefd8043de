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
#include <cstdlib>
#include <cstring>

#include <cooperative_groups.h>

#include "jq_internal.cuh"

namespace jq {

constexpr int SVD_THREADS = 1024;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
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
  // thread i owns rows i and i + SVDC_THREADS (n <= 2 SVDC_THREADS = 512)
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  constexpr int RPT = 2;
  __shared__ double red[96];
  __shared__ double sig[RPT * SVDC_THREADS];
  __shared__ int perm[RPT * SVDC_THREADS];
  const int pi = blockIdx.x, i = threadIdx.x;
  // |R|_F^2 (fixed-order two-level sum) -> negligible-column threshold
  {
    double f = 0.0;
    for (int j = pi; j < n; j += gridDim.x)
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int row = i + u * SVDC_THREADS;
        if (row < n) f = fma(A[(size_t)j * n + row], A[(size_t)j * n + row], f);
      }
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
      double x[RPT], y[RPT];
      double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int row = i + u * SVDC_THREADS;
        x[u] = row < n ? ap[row] : 0.0;
        y[u] = row < n ? aq[row] : 0.0;
        al = fma(x[u], x[u], al);
        be = fma(y[u], y[u], be);
        ga = fma(x[u], y[u], ga);
      }
      block_sum3(al, be, ga, red);
      const bool rot = !(al <= tiny || be <= tiny || ga == 0.0 || fabs(ga) < tol * (sqrt(al) * sqrt(be)));
      if (rot) {
        const double zeta = (be - al) / (2.0 * ga);
        const double t = zeta >= 0.0 ? 1.0 / (zeta + sqrt(1.0 + zeta * zeta))
                                     : -1.0 / (-zeta + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          const int row = i + u * SVDC_THREADS;
          if (row < n) {
            ap[row] = c * x[u] - s * y[u];
            aq[row] = s * x[u] + c * y[u];
            if (want_v) {
              double* vp = V + (size_t)p * n;
              double* vq = V + (size_t)q * n;
              const double uu = vp[row], w = vq[row];
              vp[row] = c * uu - s * w;
              vq[row] = s * uu + c * w;
            }
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
    double s = 0.0, z1 = 0.0, z2 = 0.0;
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
      const int row = i + u * SVDC_THREADS;
      if (row < n) s = fma(A[(size_t)j * n + row], A[(size_t)j * n + row], s);
    }
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

// Cluster variant (the default for n >= 31): one thread-block cluster of np/(2 WPC) CTAs
// (<= 16; 8 warps each), one warp per column pair, A resident in the cluster's shared
// memory for the whole solve.  Columns are stored by tournament POSITION: CTA c owns
// the positions of pairs WPC c .. WPC c + WPC-1 (k and np-1-k), and between rounds
// every player moves from position k to k-1 (1 -> np-1, 0 fixed), so a warp reads its
// pair from local shared memory and writes the rotated columns to their next positions
// -- local except at the band edges (two columns per CTA per round over distributed
// shared memory), double-buffered by round parity.  One cluster barrier per round.
// V is not carried: every rotation (c, s) is logged and jacobi_v_kernel replays the
// log on the rows of V afterwards (rows of V are independent).  Same pairs and stopping
// rule as jacobi_coop_kernel; the rotation is computed with the MUFU reciprocal /
// reciprocal square root plus one cubic correction (<= 2.2e-16 relative, like the
// TSQR chain), the acceptance test as ga^2 < tol^2 al be; lane l owns rows l, l + 32,
// ... and the dot products are warp-tree sums (deterministic).  A round is
// issue-bound (~300 instructions per pair), hence few warps per SM.
constexpr int SVD_MAX_SWEEPS = 64;

template <int WPC>
__device__ __forceinline__ void pos_home(int k, int np, int& cta, int& slot) {
  const int half = np >> 1;
  const int pi = k < half ? k : np - 1 - k;
  cta = pi / WPC;
  slot = (k < half ? 0 : WPC) + pi % WPC;
}

#ifndef JQ_SVD_ZETA_ROT
constexpr bool kFastRot = true;  // the two-MUFU rotation scalars (-DJQ_SVD_ZETA_ROT: the zeta form, A/B)
#else
constexpr bool kFastRot = false;
#endif
template <int WPC, int NKC = 0>  // NKC > 0: np = 32 NKC at compile time (the row bounds fold away)
__global__ void __launch_bounds__(WPC * 32, 1)
jacobi_cluster_kernel(const double* __restrict__ A, int np, double tol, int max_sweeps, int* flags,
                      double* __restrict__ sig, double2* __restrict__ rlog, int* __restrict__ nsweeps,
                      int* __restrict__ progress, double* __restrict__ values, int n_out) {
  namespace cg = cooperative_groups;
  constexpr int COLS = 2 * WPC, THREADS = WPC * 32;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double cols[];  // [2 buffers][COLS][np], by position; then the
  // sweep's rotation log of this CTA's pairs [np - 1][WPC] (global stores inside the round
  // loop would make every cluster barrier wait for them)
  double2* slog = reinterpret_cast<double2*>(cols + 2 * COLS * np);
  __shared__ int rotf[3];
  __shared__ double red[WPC];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rank = (int)cluster.block_rank(), nct = (int)cluster.num_blocks();
  const int half = np >> 1;
  for (int idx = tid; idx < COLS * np; idx += THREADS) {
    const int sl = idx / np, i = idx - sl * np;
    const int pi = rank * WPC + (sl % WPC);
    const int k = sl < WPC ? pi : np - 1 - pi;  // round 0: player k at position k
    cols[idx] = A[(size_t)k * np + i];
  }
  // |R|_F^2, the same fixed-order sum in every CTA -> negligible-column threshold
  double f = 0.0;
  for (int idx = tid; idx < np * np; idx += THREADS) f = fma(A[idx], A[idx], f);
  f = warp_sum(f);
  if (lane == 0) red[warp] = f;
  if (tid < 3) rotf[tid] = 0;
  __syncthreads();
  double fro = 0.0;
  for (int w = 0; w < WPC; ++w) fro += red[w];
  const double eps = 2.220446049250313e-16;
  const double tiny = (double(np) * eps) * (double(np) * eps) * fro;
  const double tol2 = tol * tol;
  const int pi = rank * WPC + warp;
  const int klo = pi, khi = np - 1 - pi;
  // next positions of the two players and where they live
  int dlo_c, dlo_s, dhi_c, dhi_s;
  pos_home<WPC>(klo == 0 ? 0 : (klo == 1 ? np - 1 : klo - 1), np, dlo_c, dlo_s);
  pos_home<WPC>(khi - 1, np, dhi_c, dhi_s);
  double* const wlo0 = dlo_c == rank ? cols + dlo_s * np : cluster.map_shared_rank(cols + dlo_s * np, dlo_c);
  double* const whi0 = dhi_c == rank ? cols + dhi_s * np : cluster.map_shared_rank(cols + dhi_s * np, dhi_c);
  const size_t bufsz = size_t(COLS) * np;
  constexpr int RPL = 256 / 32;  // rows per lane (np <= 256, a multiple of 32: warp-uniform bounds)
  const int nk = NKC > 0 ? NKC : np >> 5;
  cluster.sync();

  int sweep = 0, cur = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (tid == 0) rotf[(sweep + 1) % 3] = 0;  // read two sweeps ago, before this sweep's barriers
    bool rotated = false;
    int plo = klo, phi = khi;  // players at the two positions (round 0: identity)
    for (int r = 0; r < np - 1; ++r, cur ^= 1) {
      const bool lo_is_p = plo < phi;
      const double* src = cols + cur * bufsz;
      const double* cp = src + (lo_is_p ? warp : WPC + warp) * np;
      const double* cq = src + (lo_is_p ? WPC + warp : warp) * np;
      double x[RPL], y[RPL];
#pragma unroll
      for (int k = 0; k < RPL; ++k) {
        x[k] = k < nk ? cp[lane + 32 * k] : 0.0;
        y[k] = k < nk ? cq[lane + 32 * k] : 0.0;
      }
      double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
      for (int k = 0; k < RPL; ++k) {
        al = fma(x[k], x[k], al);
        be = fma(y[k], y[k], be);
        ga = fma(x[k], y[k], ga);
      }
      al = warp_sum(al);
      be = warp_sum(be);
      ga = warp_sum(ga);
      const bool rot = !(al <= tiny || be <= tiny || ga == 0.0 || ga * ga < tol2 * (al * be));
      double c = 1.0, sn = 0.0;
      if (rot) {
        // t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), zeta = d / e (d = be - al, e = 2 ga),
        // as sign(d) e / (|d| + sqrt(d^2 + e^2)): one reciprocal square root and one
        // reciprocal on the chain instead of two of each (the warp-uniform branch keeps
        // the zeta form where d^2 + e^2 could leave the double range)
        const double d = be - al, e = 2.0 * ga;
        const double ad = fabs(d), ae = fabs(e);
        double t;
        if (!(kFastRot && ad < 1e150 && ae < 1e150 && ae > 1e-150)) {
          const double zeta = d * rcp_nr(e);
          const double az = fabs(zeta);
          if (az < 1e100) {
            const double q = fma(az, az, 1.0);
            t = rcp_nr(fma(q, rsqrt_nr(q), az));  // 1 / (|zeta| + sqrt(1 + zeta^2))
          } else {
            t = 0.5 * rcp_nr(az);
          }
          t = zeta >= 0.0 ? t : -t;
        } else {
          const double h = fma(d, d, e * e);
          t = e * rcp_nr(fma(h, rsqrt_nr(h), ad));  // e / (|d| + sqrt(d^2 + e^2))
          t = (d >= 0.0) == (e >= 0.0) ? fabs(t) : -fabs(t);  // the sign of zeta = d / e
        }
        c = rsqrt_nr(fma(t, t, 1.0));
        sn = c * t;
#pragma unroll
        for (int k = 0; k < RPL; ++k) {
          const double xk = x[k], yk = y[k];
          x[k] = c * xk - sn * yk;
          y[k] = sn * xk + c * yk;
        }
        rotated = true;
      }
      if (lane == 0) slog[r * WPC + warp] = make_double2(c, sn);
      // players to their next positions (buffer cur ^ 1)
      double* wlo = wlo0 + (cur ^ 1) * bufsz;
      double* whi = whi0 + (cur ^ 1) * bufsz;
      double* wp = lo_is_p ? wlo : whi;
      double* wq = lo_is_p ? whi : wlo;
#pragma unroll
      for (int k = 0; k < RPL; ++k) {
        if (k < nk) {
          wp[lane + 32 * k] = x[k];
          wq[lane + 32 * k] = y[k];
        }
      }
      plo = plo == 0 ? 0 : (plo == np - 1 ? 1 : plo + 1);
      phi = phi == np - 1 ? 1 : phi + 1;
      cluster.sync();
    }
    if (rotated && lane == 0) rotf[sweep % 3] = 1;
    __syncthreads();
    for (int e = tid; e < (np - 1) * WPC; e += THREADS) {  // this sweep's log out
      const int r = e / WPC, w = e - r * WPC;
      rlog[((size_t)sweep * (np - 1) + r) * half + rank * WPC + w] = slog[e];
    }
    __threadfence();  // the log is read by jacobi_v_kernel while the sweeps go on
    cluster.sync();
    if (rank == 0 && tid == 0) st_release_gpu(progress, sweep + 1);
    int any = 0;
    for (int b = 0; b < nct; ++b) any |= *cluster.map_shared_rank(&rotf[sweep % 3], b);
    if (!any) break;
  }
  if (rank == 0 && tid == 0) {
    if (sweep == max_sweeps) atomicOr(flags, FLAG_NOCONV);
    *nsweeps = sweep;  // sweeps with rotations (the last, clean one is not replayed)
  }
  int* const done = progress + 1;
  // after whole sweeps every player is back at its own position: sigma_j = |column j|
  const double* fin = cols + cur * bufsz;
  for (int sl = warp; sl < COLS; sl += WPC) {
    const int pj = rank * WPC + (sl % WPC);
    const int j = sl < WPC ? pj : np - 1 - pj;
    double sq = 0.0;
    for (int i = lane; i < np; i += 32) sq = fma(fin[sl * np + i], fin[sl * np + i], sq);
    sq = warp_sum(sq);
    if (lane == 0) sig[j] = sqrt(sq);
  }
  cluster.sync();
  for (int sl = warp; sl < COLS; sl += WPC) {
    const int pj = rank * WPC + (sl % WPC);
    const int j = sl < WPC ? pj : np - 1 - pj;
    const double sj = sig[j];
    int rk = 0;
    for (int k = lane; k < np; k += 32) {
      const double sk = sig[k];
      rk += (sk > sj) || (sk == sj && k < j);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rk += __shfl_xor_sync(0xffffffffu, rk, o);
    if (rk < n_out && lane == 0) values[rk] = sj;
  }
  // sigma (global) and nsweeps published: the V replay may rank and finish
  if (rank == 0 && tid == 0) {
    __threadfence();
    st_release_gpu(done, 1);
  }
}

// Row i of V (one warp per row): replay the logged rotations of jacobi_cluster_kernel
// on V[i, :] (V = I at the start), rounds in order, lane l doing pairs l, l + 32, ...
// (the same element arithmetic as a carried V); then vout[i][rank(j)] = V[i][j] for the
// n_out largest sigma.  By default it runs after the cluster kernel on the same stream;
// with JQ_SVD_V_OVERLAP=1 it runs on a second stream WHILE the sweeps go on: a sweep is
// replayed once progress[0] says its log is out, and the kernel ends when progress[1]
// (done) is set and nsweeps sweeps are replayed (the final, clean sweep is skipped).
constexpr int SVDV_WARPS = 2, SVDV_BATCH = 4;  // 2 warps per CTA: n = 256 rows on 128 SMs

__global__ void __launch_bounds__(SVDV_WARPS * 32)
jacobi_v_kernel(const double2* __restrict__ rlog, const int* nsweeps, const int* progress, int np,
                const double* sig, double* __restrict__ vout, int n_out) {
  __shared__ double rows[SVDV_WARPS][256];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, half = np >> 1;
  const int i = blockIdx.x * SVDV_WARPS + warp;
  if (i >= n_out) return;
  double* row = rows[warp];
  for (int j = lane; j < np; j += 32) row[j] = i == j ? 1.0 : 0.0;
  __syncwarp();
  int plo[4], phi[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    plo[k] = lane + 32 * k;
    phi[k] = np - 1 - (lane + 32 * k);
  }
  const int rps = np - 1;  // rounds per sweep
  for (int s = 0;; ++s) {
    // wait for sweep s's log, or for the end (then nsweeps says whether s is replayed)
    int ready;
    for (;;) {
      ready = ld_acquire_gpu(progress);
      if (ready > s || ld_acquire_gpu(progress + 1)) break;
      __nanosleep(2000);
    }
    if (ld_acquire_gpu(progress + 1) && s >= *(volatile const int*)nsweeps) break;
    const int r0s = s * rps, r1s = r0s + rps;
    double2 nx[SVDV_BATCH][4];  // the next batch of (c, s), loaded one batch ahead
    auto load = [&](int r0) {
#pragma unroll
      for (int b = 0; b < SVDV_BATCH; ++b)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int pi = lane + 32 * k;
          nx[b][k] = (pi < half && r0 + b < r1s) ? __ldcg(rlog + (size_t)(r0 + b) * half + pi)
                                                 : make_double2(1.0, 0.0);
        }
    };
    load(r0s);
    for (int r0 = r0s; r0 < r1s; r0 += SVDV_BATCH) {
      double2 cs[SVDV_BATCH][4];
#pragma unroll
      for (int b = 0; b < SVDV_BATCH; ++b)
#pragma unroll
        for (int k = 0; k < 4; ++k) cs[b][k] = nx[b][k];
      if (r0 + SVDV_BATCH < r1s) load(r0 + SVDV_BATCH);
#pragma unroll
      for (int b = 0; b < SVDV_BATCH; ++b) {
        if (r0 + b >= r1s) break;
        // the lane's (up to 4) disjoint pairs: every load first, then the rotations and
        // the stores (one shared-memory round trip per round instead of one per pair)
        double u[4], w[4];
        int pp[4], qq[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          pp[k] = min(plo[k], phi[k]);
          qq[k] = max(plo[k], phi[k]);
          const bool act = lane + 32 * k < half;
          u[k] = act ? row[pp[k]] : 0.0;
          w[k] = act ? row[qq[k]] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (lane + 32 * k < half) {
            const double c = cs[b][k].x, sn = cs[b][k].y;
            row[pp[k]] = c * u[k] - sn * w[k];
            row[qq[k]] = sn * u[k] + c * w[k];
            plo[k] = plo[k] == 0 ? 0 : (plo[k] == np - 1 ? 1 : plo[k] + 1);
            phi[k] = phi[k] == np - 1 ? 1 : phi[k] + 1;
          }
        }
        __syncwarp();
      }
    }
  }
  for (int j = lane; j < np; j += 32) {
    const double sj = __ldcg(sig + j);
    int rk = 0;
    for (int k = 0; k < np; ++k) {
      const double sk = __ldcg(sig + k);
      rk += (sk > sj) || (sk == sj && k < j);
    }
    if (rk < n_out) vout[(size_t)i * n_out + rk] = row[j];
  }
}

// The default (after-sweeps) V replay: FOUR warps per row of V, lane l of warp k doing
// pair 32 k + l of every round, a 128-thread named barrier between rounds.  A round is
// then one load / rotate / store per lane (the one-warp replay above does four pairs per
// lane and is bound by that serial chain: ~400 cycles per round).  The log is read
// SVDV4_D rounds ahead into registers.  Same element arithmetic, in the same order, as
// jacobi_v_kernel (every pair's rotation is independent of the others in its round).
constexpr int SVDV4_ROWS = 2, SVDV4_D = 8;

__global__ void __launch_bounds__(SVDV4_ROWS * 128)
jacobi_v4_kernel(const double2* __restrict__ rlog, const int* nsweeps, int np, const double* sig,
                 double* __restrict__ vout, int n_out) {
  __shared__ double rows[SVDV4_ROWS][256];
  const int grp = threadIdx.x >> 7, k = (threadIdx.x >> 5) & 3, lane = threadIdx.x & 31, gt = threadIdx.x & 127;
  const int i = blockIdx.x * SVDV4_ROWS + grp, half = np >> 1, pi = lane + 32 * k;
  const bool act = pi < half;
  const int total = __ldcg(nsweeps) * (np - 1);  // the final, clean sweep is not replayed
  double* row = rows[grp];
  for (int j = gt; j < np; j += 128) row[j] = i == j ? 1.0 : 0.0;
  asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory");
  int plo = pi, phi = np - 1 - pi;
  double2 nx[SVDV4_D];
  auto load = [&](int r0) {
#pragma unroll
    for (int b = 0; b < SVDV4_D; ++b)
      nx[b] = (act && r0 + b < total) ? __ldcg(rlog + (size_t)(r0 + b) * half + pi) : make_double2(1.0, 0.0);
  };
  load(0);
  for (int r0 = 0; r0 < total; r0 += SVDV4_D) {
    double2 cs[SVDV4_D];
#pragma unroll
    for (int b = 0; b < SVDV4_D; ++b) cs[b] = nx[b];
    if (r0 + SVDV4_D < total) load(r0 + SVDV4_D);
#pragma unroll
    for (int b = 0; b < SVDV4_D; ++b) {
      if (r0 + b >= total) break;
      if (act) {
        const int p = min(plo, phi), q = max(plo, phi);
        const double u = row[p], w = row[q];
        row[p] = cs[b].x * u - cs[b].y * w;
        row[q] = cs[b].y * u + cs[b].x * w;
        plo = plo == 0 ? 0 : (plo == np - 1 ? 1 : plo + 1);
        phi = phi == np - 1 ? 1 : phi + 1;
      }
      asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory");
    }
  }
  if (i >= n_out) return;
  for (int j = gt; j < np; j += 128) {
    const double sj = __ldcg(sig + j);
    int rk = 0;
    for (int kk = 0; kk < np; ++kk) {
      const double sk = __ldcg(sig + kk);
      rk += (sk > sj) || (sk == sj && kk < j);
    }
    if (rk < n_out) vout[(size_t)i * n_out + rk] = row[j];
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
  const int64_t np = (n + 31) / 32 * 32;  // covers both paths' padding
  return 2 * ws_bytes(size_t(np) * np, 8) + ws_bytes(512, 8) + ws_bytes(128, 4) + ws_bytes(256, 8) +
         ws_bytes(4, 4) + ws_bytes(size_t(SVD_MAX_SWEEPS) * std::max<int64_t>(np - 1, 1) * (np / 2), 16);
}

// one cluster over the np/2 pairs: 8 warps per CTA (a 16-CTA cluster at np = 256, opt-in
// non-portable size), else 16 warps per CTA when the device refuses clusters above 8
static bool svd_generic() {  // JQ_SVD_GENERIC=1: the runtime-np cluster kernel only (A/B)
  static const bool g = [] {
    const char* e = getenv("JQ_SVD_GENERIC");
    return e && e[0] == '1';
  }();
  return g;
}

template <int WPC>
static int launch_cluster_wpc(jq_ctx* ctx, const double* A, int np, double* sig, double2* rlog, int* nsw,
                              double* values, int n_out) {
  // np = 256 (n in 225..256, C5's 128 + 128) gets the compile-time row count
  auto kern = np == 256 && !svd_generic() ? jacobi_cluster_kernel<WPC, 8> : jacobi_cluster_kernel<WPC>;
  const int nct = (np / 2 + WPC - 1) / WPC;
  const size_t smem = size_t(2) * 2 * WPC * np * sizeof(double) + size_t(np - 1) * WPC * sizeof(double2);
  JQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (nct > 8) JQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nct);
  cfg.blockDim = dim3(WPC * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = nct;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) != cudaSuccess || ncl < 1) {
    cudaGetLastError();
    return -1;  // not launchable with this shape
  }
  const double tol = 1e-14;
  JQ_CUDA(cudaLaunchKernelEx(&cfg, kern, A, np, tol, SVD_MAX_SWEEPS, ctx->d_flags, sig, rlog, nsw, nsw + 1, values,
                             n_out));
  JQ_CHECK_LAUNCH(ctx);
  return JQ_OK;
}

static int launch_jacobi_cluster(jq_ctx* ctx, const double* A, int np, double* sig, double2* rlog, int* nsw,
                                 double* values, int n_out) {
  int rc = launch_cluster_wpc<8>(ctx, A, np, sig, rlog, nsw, values, n_out);
  if (rc == -1) rc = launch_cluster_wpc<16>(ctx, A, np, sig, rlog, nsw, values, n_out);
  if (rc == -1) return fail(JQ_E_CUDA, "no cluster shape is launchable for the Jacobi SVD");
  return rc;
}

int svd_dev(jq_ctx* ctx, const double* r, int64_t n, int want_v, double* values, double* v) {
  if (n > 512) return fail(JQ_E_INVALID, "svd_of_r supports n <= 512");
  if (n == 0) return JQ_OK;
  static const bool coop = [] {  // JQ_SVD_IMPL=coop: the grid-barrier kernel (A/B tests)
    const char* e = getenv("JQ_SVD_IMPL");
    return e && strcmp(e, "coop") == 0;
  }();
  if (n >= 31 && n <= 256 && !coop) {
    // cluster path: zero columns pad the tournament to a multiple of 32 (never rotated,
    // sigma 0, ranked after every real column)
    const int npc = (int)((n + 31) / 32 * 32);
    double* A = ws_alloc<double>(ctx, size_t(npc) * npc);
    double* sig = ws_alloc<double>(ctx, 256);
    int* nsw = ws_alloc<int>(ctx, 4);
    double2* rlog = ws_alloc<double2>(ctx, size_t(SVD_MAX_SWEEPS) * (npc - 1) * (npc / 2));
    if (!A || !sig || !nsw || !rlog) return fail(JQ_E_OOM, "workspace exhausted (svd)");
    svd_init_kernel<<<(unsigned)cdiv(int64_t(npc) * npc, 256), 256, 0, ctx->stream>>>(r, (int)n, npc, A, nullptr);
    JQ_CHECK_LAUNCH(ctx);
    // nsw = {nsweeps, sweeps whose log is out, done}
    JQ_CUDA(cudaMemsetAsync(nsw, 0, 4 * sizeof(int), ctx->stream));
    // V replay: by default on the same stream AFTER the sweeps (it then finds every
    // sweep published and never waits).  JQ_SVD_V_OVERLAP=1 runs it on a second stream
    // concurrently with the sweeps (it spins on the cluster kernel's progress flags:
    // ~0.5 ms faster at n = 256, but it relies on both kernels being co-scheduled, which
    // CUDA does not guarantee -- MPS partitions, serialising tools -- so it is opt-in).
    static const bool overlap_v = [] {
      const char* e = getenv("JQ_SVD_V_OVERLAP");
      return e && strcmp(e, "1") == 0;
    }();
    if (want_v && overlap_v && !ctx->aux_stream) {
      JQ_CUDA(cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking));
      for (auto& e : ctx->aev) JQ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    if (want_v && overlap_v) JQ_CUDA(cudaEventRecord(ctx->aev[0], ctx->stream));
    JQ_TRY(launch_jacobi_cluster(ctx, A, npc, sig, rlog, nsw, values, (int)n));
    if (want_v && overlap_v) {
      JQ_CUDA(cudaStreamWaitEvent(ctx->aux_stream, ctx->aev[0], 0));
      jacobi_v_kernel<<<(unsigned)cdiv(n, SVDV_WARPS), SVDV_WARPS * 32, 0, ctx->aux_stream>>>(rlog, nsw, nsw + 1,
                                                                                           npc, sig, v, (int)n);
      JQ_CHECK_LAUNCH(ctx);
      JQ_CUDA(cudaEventRecord(ctx->aev[1], ctx->aux_stream));
      JQ_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->aev[1], 0));
    } else if (want_v) {
      // four warps per row (a shared-memory ring of TMA-fetched log stages for the one-warp
      // replay was measured slower: 0.70 vs 0.60 ms at n = 256 -- the replay is bound by
      // its per-round chain, not by the log's L2 reads).  JQ_SVD_V1=1: the one-warp replay.
      static const bool v1 = [] {
        const char* e = getenv("JQ_SVD_V1");
        return e && e[0] == '1';
      }();
      if (v1)
        jacobi_v_kernel<<<(unsigned)cdiv(n, SVDV_WARPS), SVDV_WARPS * 32, 0, ctx->stream>>>(rlog, nsw, nsw + 1, npc,
                                                                                          sig, v, (int)n);
      else
        jacobi_v4_kernel<<<(unsigned)cdiv(n, SVDV4_ROWS), SVDV4_ROWS * 128, 0, ctx->stream>>>(rlog, nsw, npc, sig, v,
                                                                                             (int)n);
      JQ_CHECK_LAUNCH(ctx);
    }
    return JQ_OK;
  }
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
  JQ_NVTX("jq_svd_of_r");
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
