// jq_tsqr.cu — tall-skinny Householder QR (TSQR) on the FP64 tensor pipe (DMMA).
//
// Replaces the paper's cusolverDnXgeqrf finishing step (SPEC.md
// householder_r :250-258, figaro_r :278-286).  Design:
//
//  * Streaming leaves.  Each CTA owns a contiguous range of rows of the (virtual)
//    reduced matrix and keeps a running upper-triangular R (NP x NP: packed by
//    8-row panels in shared memory for NP <= 128, in its L2-resident global slab
//    for NP = 256).  It absorbs the range K rows at a time: R <- qr([R; C]).  Every
//    reflector of [R; C] is v = [e_j ; y_j] (it touches one row of R and all K
//    chunk rows), so the block reflector of a panel is V = [I; Y] and the
//    compact-WY trailing update is
//        Z = R[panel rows, trail] + Y^T C[:, trail];  W = T^T Z;
//        R[panel rows, trail] -= W;                     C[:, trail] -= Y W.
//  * Asynchronous input.  The raw input rows of the NEXT chunk (A or B rows of the
//    join, or dense rows) are fetched by one TMA bulk copy (cp.async.bulk + an
//    mbarrier) into a shared-memory buffer while the current chunk is being
//    factored; the Claim-1 rows are then formed in place from shared memory.
//  * Register-resident chunk.  C (K = 128 rows for NP <= 128) lives in registers
//    in the DMMA (m8n8k4 f64) accumulator layout, transposed: warp w owns column
//    tiles w and NLT-1-w (balanced triangular work) and holds C^T[l][i] for all K
//    rows.  Both GEMMs of the trailing update take their A operand straight from
//    those registers by permuting the reduction index of each DMMA
//    (k = t  <->  i = 8*it + 2*t + b), so the only shared-memory operands are Y,
//    Y^T and T.
//  * Panels of 8 columns (one column tile) are factored by the warp that owns the
//    tile, from registers, with ONE quad reduction per column (the raw column x is
//    broadcast through shared memory and every quad forms x . c_g at once: for
//    g = j that is |x|^2, for g > j the reflector dot product, for g < j the T
//    entries); reflector scaling is deferred to the end of the panel.  The owner
//    of the next panel updates that tile first, so panel factorisation overlaps
//    the other warps' trailing updates (one __syncthreads per panel).
//  * Tree.  The P leaf R's are combined by a fixed binary tree of the same kernel
//    (R_init = R_a, rows = R_b), so results are deterministic for a given P.
//
// The Figaro source generates the reduced rows of Claim 1 on the fly (PAPER.md
// :53-58): top rows [sqrt(m2g) A_i | head(B_g)], bottom rows
// [0 | sqrt(m1g) tail(B_g)_r] with the prefix sum carried from the head/tail pass
// (jq_headtail.cu), so the reduced matrix never exists in HBM.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "jq_internal.cuh"
#include "jq_segscan.cuh"

namespace jq {

constexpr unsigned FULL = 0xffffffffu;

template <int V>
struct IntC {
  static constexpr int value = V;
};
// f(IntC<P>), ..., f(IntC<N-1>): a loop whose index is a compile-time constant in the body
template <int P, int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (P < N) {
    f(IntC<P>{});
    static_for<P + 1, N>(f);
  }
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int NP_>
struct Cfg {
  static constexpr int NP = NP_;
  static constexpr int NLT = NP / 8;        // column tiles of 8
  static constexpr int WARPS = 8;           // row-split: warp w holds rows [w*KW, (w+1)*KW) of every tile
  static constexpr int THREADS = WARPS * 32;
  static constexpr int K = NP >= 256 ? 64 : 128;  // chunk rows held in registers
  static constexpr int KW = K / WARPS;      // rows per warp
  static constexpr int KWT = KW / 8;        // row tiles per warp
  static constexpr bool R_SMEM = NP <= 128;
  // one CTA per SM (255 registers): this kernel is the tree combine of every leaf width
  // (and the JQ_TSQR_IMPL=cta leaf); at 2 CTAs per SM its N <= 64 instantiations spilled
  // in the panel loop (192-224 bytes of stack)
  static constexpr int MIN_CTAS = 1;
  // R packed by 8-row panels: panel p holds rows 8p..8p+7, columns 8p..NP-1,
  // row stride NP - 8p + 2 (== 2 or 10 mod 16: conflict-free DMMA fragment access)
  __host__ __device__ static constexpr int rp_off(int p) { return 8 * (p * (NP + 2) - 4 * p * (p - 1)); }
  static constexpr int LDT = 10;            // T   (8 x 8)
  static constexpr int LDYT = KW + 2;       // per-warp Y^T (8 x KW), == 2 mod 16
  static constexpr int RAW = NP >= 256 ? NP * 32 : NP * 64;  // raw-row buffer
  // shared memory carve-up (doubles; every offset even -> 16-byte aligned)
  static constexpr int OFF_R = 0;
  static constexpr int SZ_R = R_SMEM ? rp_off(NLT) : 0;
  static constexpr int OFF_RAW = OFF_R + SZ_R;
  static constexpr int OFF_YT = OFF_RAW + RAW;            // [WARPS][8][LDYT]
  static constexpr int SZ_YT = 8 * LDYT;
  static constexpr int OFF_ZP = OFF_YT + WARPS * SZ_YT;   // partial Z^T [WARPS][NLT][64]
  static constexpr int OFF_WS = OFF_ZP + WARPS * NLT * 64;  // W^T [NLT][64]
  static constexpr int OFF_T = OFF_WS + NLT * 64;
  static constexpr int OFF_U = OFF_T + 8 * LDT;
  static constexpr int OFF_TAU = OFF_U + 64;
  static constexpr int OFF_SC = OFF_TAU + 8;  // reflector scales of the panel
  static constexpr int OFF_P = OFF_SC + 8;    // column dot partials [2 parity][WARPS][8]
  static constexpr int OFF_S = OFF_P + 2 * WARPS * 8;  // running prefix sums (Figaro source, <= NP)
  static constexpr int OFF_LD = OFF_S + NP;   // loader scratch: 3 per-row coefficients + 2 per thread
  static constexpr int SZ_LD = 3 * K + 2 * THREADS;
  static constexpr int OFF_M = OFF_LD + SZ_LD;    // M' (8 x LDT): Y = X M' of the Gram panel
  static constexpr int OFF_FLAG = OFF_M + 8 * LDT; // Gram panel accepted (1) / explicit fallback (0)
  static constexpr int OFF_BAR = OFF_FLAG + 2;    // mbarrier (8 bytes)
  static constexpr int TOTAL = OFF_BAR + 2;
  static constexpr size_t SMEM = size_t(TOTAL) * sizeof(double);
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
  static_assert(KW % 8 == 0, "whole row tiles per warp");
  static_assert(OFF_S - OFF_U >= 16 * LDT + 16 + 32, "factor_panel_chol scratch (U .. P)");
};

// R element (r, c), c >= 8 * (r / 8), in the packed (smem) or dense (global) layout
template <class C>
__device__ __forceinline__ int rix(int r, int c) {
  if constexpr (C::R_SMEM) {
    const int p = r >> 3;
    return C::rp_off(p) + (r & 7) * (C::NP - 8 * p + 2) + (c - 8 * p);
  } else {
    return r * C::NP + c;
  }
}

// ------------------------------------------------------------------ row sources
// A source describes, for the pass starting at virtual row v0, the contiguous raw
// rows to fetch (ptr, raw columns rc, rows available), turns the fetched raw rows
// into Claim-1 rows in place (prep) and yields C[i][l] for the register load.

// sub-segments per loader warp in the multi-loader tail transform (independent
// recurrences in flight per lane; FigaroSrc::seg_pass1 / seg_pass2)
constexpr int SEG_SUB = 4;

// bar.sync id, n: a barrier among the n threads (whole warps) that execute it
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// the same barrier, returning the AND of `v` over the n threads
__device__ __forceinline__ bool named_bar_and(int id, int n, bool v) {
  int r;
  asm volatile(
      "{\n .reg .pred p, q;\n setp.ne.s32 p, %1, 0;\n bar.red.and.pred q, %2, %3, p;\n selp.s32 %0, 1, 0, q;\n}\n"
      : "=r"(r)
      : "r"(v ? 1 : 0), "r"(id), "r"(n)
      : "memory");
  return r != 0;
}
// the barrier among the NW row warps of a direct chunk load: __syncthreads (BAR 0, the
// CTA-wide leaf) or named barrier BAR (the data warps of the warp-specialised leaf)
template <int NW, int BAR>
struct RowBar {
  static constexpr int NW_ = NW;
  __device__ static void sync() {
    if constexpr (BAR == 0) __syncthreads();
    else named_bar(BAR, NW * 32);
  }
  __device__ static bool sync_and(bool v) {
    if constexpr (BAR == 0) return __syncthreads_and(v);
    else return named_bar_and(BAR, NW * 32, v);
  }
};

// chunk row held in register slot (it, b) of lane quad t of `warp` by the direct-load
// leaves: 2 KWT consecutive rows per thread (the staged path: row 8 it + 2 t + b)
template <class C>
__device__ __forceinline__ int direct_row(int warp, int t, int it, int b) {
  return warp * C::KW + t * (2 * C::KWT) + 2 * it + b;
}

struct DenseSrc {
  const double* m;
  int64_t rows, cols;
  template <class C>
  __device__ void begin(double*, int64_t) const {}
  __device__ int rc(int64_t) const { return (int)cols; }
  __device__ const double* ptr(int64_t v0) const { return m + v0 * cols; }
  __device__ int64_t avail(int64_t v0) const { return rows - v0; }
  template <class C>
  __device__ void prep(double*, double*, double*, int64_t, int) const {}
  template <class C>
  __device__ double value(const double* raw, const double*, int64_t, int i, int l, int nrows, int rcols) const {
    return (i < nrows && l < rcols) ? raw[i * rcols + l] : 0.0;
  }
  // direct chunk load (load_direct): global -> the C^T registers of the NW row warps
  // (Bar::NW_), no shared-memory staging; the rows v0 .. v0 + nr - 1 (the rest zero).
  // Early form (warp-specialised leaf, the next chunk while this one is factored):
  // early_ok / early_coefs / load_tile per tile as its registers free up / load_finish.
  static constexpr bool DIRECT = true;
  __device__ bool early_ok(int64_t) const { return true; }
  template <class C, int NW>
  __device__ bool early_coefs(int64_t, int, double*, int, int) const { return true; }
  template <class C>
  __device__ void load_tile(double (&ct)[C::KWT][2], int64_t v0, int nr, int q, int warp, int lane) const {
    const int g = lane >> 2, t = lane & 3, l = 8 * q + g;
    const double* base = m + v0 * cols;
#pragma unroll
    for (int it = 0; it < C::KWT; ++it)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int i = direct_row<C>(warp, t, it, b);
        ct[it][b] = (i < nr && l < (int)cols) ? __ldg(base + (int64_t)i * cols + l) : 0.0;
      }
  }
  template <class C, class Bar, class Mark>
  __device__ void load_finish(double (&)[C::NLT][C::KWT][2], int64_t, int, double*, double*, double*, double*, int,
                              int, bool, Mark) const {}
  template <class C, class Bar, class Mark>
  __device__ void load_direct(double (&c)[C::NLT][C::KWT][2], int64_t v0, int nr, double*, double*, double*,
                              double*, int warp, int lane, Mark) const {
    const int g = lane >> 2, t = lane & 3, nc = (int)cols;
    const double* base = m + v0 * cols;
#pragma unroll
    for (int q = 0; q < C::NLT; ++q)
#pragma unroll
      for (int it = 0; it < C::KWT; ++it)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const int i = direct_row<C>(warp, t, it, b), l = 8 * q + g;
          c[q][it][b] = (i < nr && l < nc) ? __ldg(base + (int64_t)i * cols + l) : 0.0;
        }
  }
  // warp-specialised loader (tsqr_ws_kernel): chunk rows never cross limit(v0)
  __device__ int64_t limit(int64_t) const { return INT64_MAX; }
  template <class C>
  __device__ void prep_warp(double*, double*, double*, int64_t, int, int) const {}
  template <class C>
  __device__ void seg_coeffs(double*, int64_t, int, int, int, int) const {}
  template <class C>
  __device__ void seg_pass1(const double*, const double*, double*, int64_t, int, int, int, int,
                            double (&)[SEG_SUB][2], bool (&)[SEG_SUB][2]) const {}
  template <class C>
  __device__ void seg_pass2(double*, double*, const double*, const double*, double, double, int64_t, int, int, int,
                            int, int, int, const double (&)[SEG_SUB][2], const bool (&)[SEG_SUB][2]) const {}
  SideScan side_job() const { return SideScan{}; }
  __device__ void side_scan(int, int, int) const {}
  // after the leaf's last chunk: S holds the running prefix (carry-free leaves export it)
  __device__ void finish(const double*, int, int) const {}
};

// Rows of the join matrix generated from A and B in every data warp (brute force; no
// raw rows, no loader work: rc() = 0)
struct JoinSrc : DenseSrc {
  JoinArgs ja;
  static constexpr bool DIRECT = false;  // rows generated in value()
  __device__ int rc(int64_t) const { return 0; }
  __device__ const double* ptr(int64_t) const { return nullptr; }
  __device__ int64_t avail(int64_t v0) const { return ja.rows - v0; }
  template <class C>
  __device__ double value(const double*, const double*, int64_t v0, int i, int l, int nrows, int) const {
    const int n1 = (int)ja.n1;
    if (i >= nrows || l >= n1 + (int)ja.n2) return 0.0;
    int64_t ia, ib;
    join_row(ja, v0 + i, ia, ib);
    return l < n1 ? __ldg(ja.a + ia * n1 + l) : __ldg(ja.b + ib * ja.n2 + (l - n1));
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
      double s = 0.0;
      if (!fa.blk_rows) {  // carry-free leaves start from 0
        if (fa.b_carry) s = fa.b_carry[tile * fa.n2 + c];
        if (fa.b_prefix0) s += fa.b_prefix0[c];
      }
      S[c] = s;
    }
  }
  // Cartesian row index within the group: the global one, or within the leaf's block
  __device__ int64_t cart_row(int64_t br) const { return fa.blk_rows ? br % fa.blk_rows : fa.b_row0 + br; }
  __device__ void finish(const double* S, int i0, int stride) const {
    if (!fa.blk_sums) return;
    for (int c = i0; c < fa.n2; c += stride) fa.blk_sums[blockIdx.x * fa.n2 + c] = S[c];
  }
  // the tile pass of another segmented scan (fa.side), run by the leaf's spare warps:
  // spare warp si of nsp per CTA takes tiles blockIdx.x * nsp + si, strided by the grid
  SideScan side_job() const { return fa.side; }
  __device__ void side_scan(int si, int nsp, int lane) const {
    const SideScan& sd = fa.side;
    if (!sd.x) return;
    for (int64_t t = (int64_t)blockIdx.x * nsp + si; t < sd.ntiles; t += (int64_t)gridDim.x * nsp)
      segscan_tile(sd.x, sd.rows, sd.cols, sd.gid, t, sd.agg, sd.flag, sd.totals, lane);
  }
  __device__ int rc(int64_t v0) const { return v0 < m1pad ? (int)fa.n1 : (int)fa.n2; }
  __device__ const double* ptr(int64_t v0) const {
    return v0 < m1pad ? fa.a + v0 * fa.n1 : fa.b + (v0 - m1pad) * fa.n2;
  }
  __device__ int64_t avail(int64_t v0) const { return v0 < m1pad ? fa.m1 - v0 : fa.m2 - (v0 - m1pad); }

  // Per-row scalars once per row into scratch; B-part: in-place tail transform of
  // the raw rows by a segmented scan over (segment, column) threads.
  template <class C>
  __device__ void prep(double* raw, double* S, double* scratch, int64_t v0, int nrows) const {
    const int n2 = (int)fa.n2;
    double* c1 = scratch;                // K
    double* c2 = scratch + C::K;         // K
    double* mode = scratch + 2 * C::K;   // K: B-part 0 zero row / 1 group start / 2 tail row; A-part gid
    double* ls = scratch + 3 * C::K;     // THREADS
    double* rs = ls + C::THREADS;        // THREADS
    if (v0 < m1pad) {
      // ---- top block rows: [sqrt(m2g) A_i | head(B_g)]
      for (int i = threadIdx.x; i < C::K; i += C::THREADS) {
        int g = -1;
        double m2g = 0.0;
        if (i < nrows) {
          const int64_t r = v0 + i;
          g = fa.gid_a ? fa.gid_a[r] : 0;
          if (g >= 0) m2g = fa.gid_a ? (double)fa.b_count[g] : (double)fa.m2_global;
        }
        const double rs2 = g >= 0 && m2g > 0.0 ? rsqrt_nr(m2g) : 0.0;
        c1[i] = m2g * rs2;  // sqrt(m2g)
        c2[i] = rs2;
        mode[i] = (double)g;
      }
      return;
    }
    // ---- bottom block rows: [0 | sqrt(m1g) tail(B_g)]
    //   tail_r = (sqrt(r) x - S / sqrt(r)) / sqrt(r+1) * sqrt(m1g) = c1 x - c2 S
    const int64_t b0 = v0 - m1pad;
    for (int i = threadIdx.x; i < C::K; i += C::THREADS) {
      double md = 0.0, a1 = 0.0, a2 = 0.0;
      if (i < nrows) {
        const int64_t br = b0 + i;
        int64_t rr = 0;
        double m1g = 0.0;
        bool valid = true;
        if (fa.gid_b) {
          const int g = fa.gid_b[br];
          valid = g >= 0;
          if (valid) { rr = br - fa.b_start[g]; m1g = (double)fa.a_count[g]; }
        } else {
          rr = cart_row(br);
          m1g = (double)fa.m1_global;
        }
        if (valid) {
          if (rr == 0) {
            md = 1.0;
          } else {
            // sqrt(r)/sqrt(r+1) sqrt(m1g) = r a2,  a2 = sqrt(m1g) / sqrt(r (r+1))  (MUFU + Newton)
            const double rd = (double)rr;
            md = 2.0;
            a2 = (m1g * rsqrt_nr(m1g)) * rsqrt_nr(rd * (rd + 1.0));
            a1 = rd * a2;
          }
        }
      }
      c1[i] = a1; c2[i] = a2; mode[i] = md;
    }
    __syncthreads();
    if (n2 == 0) return;
    constexpr int MAXSEG = 8;
    const int nseg = min(MAXSEG, max(1, C::THREADS / n2));
    const int rps = (nrows + nseg - 1) / nseg;
    const int c = threadIdx.x % n2, seg = threadIdx.x / n2;
    const bool active = threadIdx.x < nseg * n2;
    // rows are processed in batches of 4 (loads issued together, then the short
    // sequential recurrence in registers)
    double loc = 0.0, reset = 0.0;
    const int i0 = seg * rps, i1 = min(nrows, i0 + rps);
    if (active) {
      for (int ib = i0; ib < i1; ib += 4) {
        double xv[4], md[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const bool in = ib + k < i1;
          xv[k] = in ? raw[(ib + k) * n2 + c] : 0.0;
          md[k] = in ? mode[ib + k] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (md[k] == 1.0) { loc = xv[k]; reset = 1.0; }
          else if (md[k] == 2.0) loc += xv[k];
        }
      }
      ls[seg * n2 + c] = loc;
      rs[seg * n2 + c] = reset;
    }
    __syncthreads();
    double sv = 0.0;
    if (active) {
      sv = S[c];
      for (int k = 0; k < seg; ++k) sv = rs[k * n2 + c] != 0.0 ? ls[k * n2 + c] : sv + ls[k * n2 + c];
    }
    __syncthreads();  // every thread of a column has read S before the last segment rewrites it
    if (active) {
      for (int ib = i0; ib < i1; ib += 4) {
        double xv[4], md[4], a1[4], a2[4], out[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const bool in = ib + k < i1;
          xv[k] = in ? raw[(ib + k) * n2 + c] : 0.0;
          md[k] = in ? mode[ib + k] : 0.0;
          a1[k] = in ? c1[ib + k] : 0.0;
          a2[k] = in ? c2[ib + k] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          out[k] = 0.0;
          if (md[k] == 1.0) sv = xv[k];
          else if (md[k] == 2.0) { out[k] = fma(a1[k], xv[k], -a2[k] * sv); sv += xv[k]; }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (ib + k < i1) raw[(ib + k) * n2 + c] = out[k];
      }
      if (seg == nseg - 1) S[c] = sv;
    }
  }

  __device__ int64_t limit(int64_t v0) const { return v0 < m1pad ? m1pad : INT64_MAX; }

  // ---- direct chunk load (load_direct) by the NW row warps (Bar::NW_; `warp` = the
  // caller's row-warp index).  A part: [c1 A_i | c2 totals(B_g)] per row.  B part: the tail
  // transform out_r = c1_r x_r - c2_r S_r, S_{r+1} = keep_r S_r + w_r x_r (keep 0 at a
  // group start, w 0 for a row without a group) is a scan of affine maps S -> K S + A along
  // the chunk rows, done in the DMMA register layout.  The chunk's rows are assigned to the
  // register slots so that a thread holds 2 KWT CONSECUTIVE rows (direct_row; R is
  // invariant under a row permutation of the chunk): the thread folds its rows into one
  // map, the maps are scanned across the 4 lanes t of the column by shuffles, and the
  // warps' totals over the warps (one column per thread) from the running prefix S.  Fast
  // path (only tail rows in the chunk): plain prefix sums.  lo: [NLT][NW*32] (the
  // thread's offsets), wt: [NW][NP] double2, coef: c1 | c2 | mode per chunk row (3 K); all
  // three idle between chunks.  Chunks never cross m1pad (limit()).
  static constexpr bool DIRECT = true;
  // the early form covers B-part chunks (the A part's values need the coefficients first)
  __device__ bool early_ok(int64_t v0) const { return v0 >= m1pad; }
  // B part: per-row coefficients, one thread per chunk row: c1, c2 -> coef, the row mode
  // -> coef + 2K (int); returns this thread's "only tail rows" flag
  template <class C, int NW>
  __device__ bool early_coefs(int64_t v0, int nr, double* coef, int warp, int lane) const {
    const int rt = warp * 32 + lane;
    const int64_t b0 = v0 - m1pad;
    int* cmode = reinterpret_cast<int*>(coef + 2 * C::K);
    bool tails = true;  // every row a tail row (or past the chunk)
    for (int i = rt; i < C::K; i += NW * 32) {
      int md = 0;
      double c1v = 0.0, c2v = 0.0;
      if (i < nr) {
        const int64_t br = b0 + i;
        int64_t rr = 0;
        double m1g = 0.0;
        bool valid = true;
        if (fa.gid_b) {
          const int gg = __ldg(fa.gid_b + br);
          valid = gg >= 0;
          if (valid) { rr = br - __ldg(fa.b_start + gg); m1g = (double)__ldg(fa.a_count + gg); }
        } else {
          rr = cart_row(br);
          m1g = (double)fa.m1_global;
        }
        if (valid) {
          if (rr == 0) {
            md = 1;
          } else {
            const double rd = (double)rr;
            md = 2;
            c2v = (m1g * rsqrt_nr(m1g)) * rsqrt_nr(rd * (rd + 1.0));
            c1v = rd * c2v;
          }
        }
        tails = tails && md == 2;
      }
      coef[i] = c1v;
      coef[C::K + i] = c2v;
      cmode[i] = md;
    }
    return tails;
  }
  // B part: the raw rows of tile q (columns 8q .. 8q+7) into this thread's slots
  template <class C>
  __device__ void load_tile(double (&ct)[C::KWT][2], int64_t v0, int nr, int q, int warp, int lane) const {
    const int g = lane >> 2, t = lane & 3, l = 8 * q + g;
    const int n1 = (int)fa.n1, n2 = (int)fa.n2;
    const double* bb = fa.b + (v0 - m1pad) * fa.n2 - n1;
#pragma unroll
    for (int it = 0; it < C::KWT; ++it)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int i = direct_row<C>(warp, t, it, b);
        ct[it][b] = (i < nr && l >= n1 && l < n) ? __ldg(bb + (int64_t)i * n2 + l) : 0.0;
      }
  }
  // B part, raw rows and coefficients in place: the scan and the transform
  template <class C, class Bar, class Mark>
  __device__ void load_finish(double (&c)[C::NLT][C::KWT][2], int64_t v0, int nr, double* S, double* lo, double* wt,
                              double* coef, int warp, int lane, bool tails, Mark mark) const {
    static_assert(C::NLT <= 32, "one keep bit per tile");
    constexpr int NW = Bar::NW_, NT = NW * 32;
    const int g = lane >> 2, t = lane & 3, rt = warp * 32 + lane;
    const int n1 = (int)fa.n1;
    const int* cmode = reinterpret_cast<const int*>(coef + 2 * C::K);
    (void)v0;
    (void)nr;
    const bool fast = Bar::sync_and(tails);
    unsigned kb = 0, wb = 0;  // bit 2 it + b: keep S / add x
#pragma unroll
    for (int it = 0; it < C::KWT; ++it)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int md = cmode[direct_row<C>(warp, t, it, b)];
        if (md != 1) kb |= 1u << (2 * it + b);
        if (md != 0) wb |= 1u << (2 * it + b);
      }
    mark(7);
    // phase 1: per tile, the thread's map from the warp's first row (K bit, A -> lo) and
    // the warp's total map (-> wt)
    unsigned kx = 0;
    if (fast) {
#pragma unroll
      for (int q = 0; q < C::NLT; ++q) {
        double A = 0.0;
#pragma unroll
        for (int it = 0; it < C::KWT; ++it) A += c[q][it][0] + c[q][it][1];
#pragma unroll
        for (int d = 1; d < 4; d <<= 1) {
          const double Ae = __shfl_up_sync(0xffffffffu, A, d, 4);
          if (t >= d) A += Ae;
        }
        const double Ax = __shfl_up_sync(0xffffffffu, A, 1, 4);
        const double At = __shfl_sync(0xffffffffu, A, 3, 4);
        lo[q * NT + rt] = t == 0 ? 0.0 : Ax;
        if (t == 0) *reinterpret_cast<double2*>(wt + 2 * (warp * C::NP + 8 * q + g)) = make_double2(1.0, At);
      }
      kx = ~0u;
    } else {
#pragma unroll
      for (int q = 0; q < C::NLT; ++q) {
        double K = 1.0, A = 0.0;
#pragma unroll
        for (int it = 0; it < C::KWT; ++it)
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const bool kk = (kb >> (2 * it + b)) & 1, ww = (wb >> (2 * it + b)) & 1;
            A = (kk ? A : 0.0) + (ww ? c[q][it][b] : 0.0);
            K = kk ? K : 0.0;
          }
#pragma unroll
        for (int d = 1; d < 4; d <<= 1) {
          const double Ke = __shfl_up_sync(0xffffffffu, K, d, 4), Ae = __shfl_up_sync(0xffffffffu, A, d, 4);
          if (t >= d) { A = fma(K, Ae, A); K *= Ke; }
        }
        const double Kx = __shfl_up_sync(0xffffffffu, K, 1, 4), Ax = __shfl_up_sync(0xffffffffu, A, 1, 4);
        const double Kt = __shfl_sync(0xffffffffu, K, 3, 4), At = __shfl_sync(0xffffffffu, A, 3, 4);
        lo[q * NT + rt] = t == 0 ? 0.0 : Ax;
        if (t == 0 || Kx != 0.0) kx |= 1u << q;
        if (t == 0) *reinterpret_cast<double2*>(wt + 2 * (warp * C::NP + 8 * q + g)) = make_double2(Kt, At);
      }
    }
    Bar::sync();
    mark(8);
    // the warps' carry-ins per column from the running prefix S; S <- the chunk's carry-out
    for (int l = rt; l < C::NP; l += NT) {
      if (l >= n1 && l < n) {
        double sv = S[l - n1];
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const double2 mp = *reinterpret_cast<const double2*>(wt + 2 * (w * C::NP + l));
          wt[2 * (w * C::NP + l)] = sv;
          sv = fma(mp.x, sv, mp.y);
        }
        S[l - n1] = sv;
      }
    }
    Bar::sync();
    mark(9);
    // phase 2: the transform
    double c1r[C::KWT][2], c2r[C::KWT][2];
#pragma unroll
    for (int it = 0; it < C::KWT; ++it)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int i = direct_row<C>(warp, t, it, b);
        c1r[it][b] = coef[i];
        c2r[it][b] = coef[C::K + i];
      }
    if (fast) {
#pragma unroll
      for (int q = 0; q < C::NLT; ++q) {
        const int l = 8 * q + g;
        if (l >= n1 && l < n) {
          double sv = wt[2 * (warp * C::NP + l)] + lo[q * NT + rt];
#pragma unroll
          for (int it = 0; it < C::KWT; ++it)
#pragma unroll
            for (int b = 0; b < 2; ++b) {
              const double x = c[q][it][b];
              c[q][it][b] = fma(c1r[it][b], x, -c2r[it][b] * sv);
              sv += x;
            }
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < C::NLT; ++q) {
        const int l = 8 * q + g;
        if (l >= n1 && l < n) {
          double sv = (((kx >> q) & 1) ? wt[2 * (warp * C::NP + l)] : 0.0) + lo[q * NT + rt];
#pragma unroll
          for (int it = 0; it < C::KWT; ++it)
#pragma unroll
            for (int b = 0; b < 2; ++b) {
              const double x = c[q][it][b];
              c[q][it][b] = fma(c1r[it][b], x, -c2r[it][b] * sv);
              sv = (((kb >> (2 * it + b)) & 1) ? sv : 0.0) + (((wb >> (2 * it + b)) & 1) ? x : 0.0);
            }
        }
      }
    }
    Bar::sync();  // wt / lo / coef read before the caller reuses them
  }
  template <class C, class Bar, class Mark>
  __device__ void load_direct(double (&c)[C::NLT][C::KWT][2], int64_t v0, int nr, double* S, double* lo, double* wt,
                              double* coef, int warp, int lane, Mark mark) const {
    constexpr int NW = Bar::NW_, NT = NW * 32;
    const int g = lane >> 2, t = lane & 3, rt = warp * 32 + lane;
    const int n1 = (int)fa.n1, n2 = (int)fa.n2;
    int* cmode = reinterpret_cast<int*>(coef + 2 * C::K);
    if (v0 < m1pad) {
      // ---- top block rows: [sqrt(m2g) A_i | head(B_g)]; no scan
      for (int i = rt; i < C::K; i += NT) {
        int gg = -1;
        double m2g = 0.0;
        if (i < nr) {
          const int64_t r = v0 + i;
          gg = fa.gid_a ? __ldg(fa.gid_a + r) : 0;
          if (gg >= 0) m2g = fa.gid_a ? (double)__ldg(fa.b_count + gg) : (double)fa.m2_global;
        }
        const double rs2 = gg >= 0 && m2g > 0.0 ? rsqrt_nr(m2g) : 0.0;
        coef[i] = m2g * rs2;
        coef[C::K + i] = rs2;
        cmode[i] = gg;
      }
      Bar::sync();
      const double* ab = fa.a + v0 * fa.n1;
#pragma unroll
      for (int it = 0; it < C::KWT; ++it)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const int i = direct_row<C>(warp, t, it, b);
          const int gg = cmode[i];
          const double c1v = coef[i], c2v = coef[C::K + i];
#pragma unroll
          for (int q = 0; q < C::NLT; ++q) {
            const int l = 8 * q + g;
            double v = 0.0;
            if (i < nr && gg >= 0) {
              if (l < n1) v = __ldg(ab + (int64_t)i * n1 + l) * c1v;
              else if (l < n) v = __ldg(fa.b_totals + (int64_t)gg * n2 + (l - n1)) * c2v;
            }
            c[q][it][b] = v;
          }
        }
      Bar::sync();  // coef / cmode read before the next chunk rewrites them
      return;
    }
    const bool tails = early_coefs<C, NW>(v0, nr, coef, warp, lane);
    mark(5);
#pragma unroll
    for (int q = 0; q < C::NLT; ++q) load_tile<C>(c[q], v0, nr, q, warp, lane);
    load_finish<C, Bar>(c, v0, nr, S, lo, wt, coef, warp, lane, tails, mark);
  }

  // prep by ONE warp (the loader warp of tsqr_ws_kernel): per-row scalars, then the
  // B-part tail transform in place, lane = column (sequential over the chunk rows,
  // loads batched by 4); S is the running prefix of the loader.
  template <class C>
  __device__ void prep_warp(double* raw, double* S, double* scratch, int64_t v0, int nrows, int lane) const {
    double* c1 = scratch;
    double* c2 = scratch + C::K;
    double* mode = scratch + 2 * C::K;
    if (v0 < m1pad) {
#pragma unroll
      for (int ii = 0; ii < (C::K + 31) / 32; ++ii) {  // independent rows: all in flight
        const int i = lane + 32 * ii;
        if (i >= C::K) break;
        int g = -1;
        double m2g = 0.0;
        if (i < nrows) {
          const int64_t r = v0 + i;
          g = fa.gid_a ? fa.gid_a[r] : 0;
          if (g >= 0) m2g = fa.gid_a ? (double)fa.b_count[g] : (double)fa.m2_global;
        }
        const double rs2 = g >= 0 && m2g > 0.0 ? rsqrt_nr(m2g) : 0.0;
        c1[i] = m2g * rs2;
        c2[i] = rs2;
        mode[i] = (double)g;
      }
      __syncwarp();
      return;
    }
    const int64_t b0 = v0 - m1pad;
    int* imode = reinterpret_cast<int*>(mode);  // B part: 0 no row / 1 group start / 2 tail row
#pragma unroll
    for (int ii = 0; ii < (C::K + 31) / 32; ++ii) {
      const int i = lane + 32 * ii;
      if (i >= C::K) break;
      int md = 0;
      double a1 = 0.0, a2 = 0.0;
      if (i < nrows) {
        const int64_t br = b0 + i;
        int64_t rr = 0;
        double m1g = 0.0;
        bool valid = true;
        if (fa.gid_b) {
          const int g = fa.gid_b[br];
          valid = g >= 0;
          if (valid) { rr = br - fa.b_start[g]; m1g = (double)fa.a_count[g]; }
        } else {
          rr = cart_row(br);
          m1g = (double)fa.m1_global;
        }
        if (valid) {
          if (rr == 0) {
            md = 1;
          } else {
            const double rd = (double)rr;
            md = 2;
            a2 = (m1g * rsqrt_nr(m1g)) * rsqrt_nr(rd * (rd + 1.0));
            a1 = rd * a2;
          }
        }
      }
      c1[i] = a1; c2[i] = a2; imode[i] = md;
    }
    __syncwarp();
    // lane = columns lane + 32 j (n2 <= 32 CPL), one pass over the rows in batches of
    // 4 (vector loads of the row scalars; a select-free path when the 4 rows are all
    // tail rows, the Cartesian case), the next batch's loads issued first
    constexpr int CPL = C::NP <= 32 ? 1 : C::NP / 32;
    const int n2 = (int)fa.n2;
    bool h[CPL];
    double sc[CPL];
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      h[j] = lane + 32 * j < n2;
      sc[j] = h[j] ? S[lane + 32 * j] : 0.0;
    }
    const int nfull = nrows & ~3;
    double x[CPL][4];
    double2 q1[2], q2[2];
    int4 qm;
    auto load = [&](int ib) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int j = 0; j < CPL; ++j) x[j][k] = h[j] ? raw[(ib + k) * n2 + lane + 32 * j] : 0.0;
      q1[0] = *reinterpret_cast<const double2*>(c1 + ib);
      q1[1] = *reinterpret_cast<const double2*>(c1 + ib + 2);
      q2[0] = *reinterpret_cast<const double2*>(c2 + ib);
      q2[1] = *reinterpret_cast<const double2*>(c2 + ib + 2);
      qm = *reinterpret_cast<const int4*>(imode + ib);
    };
    if (nfull > 0) load(0);
    for (int ib = 0; ib < nfull; ib += 4) {
      double y[CPL][4];
#pragma unroll
      for (int j = 0; j < CPL; ++j)
#pragma unroll
        for (int k = 0; k < 4; ++k) y[j][k] = x[j][k];
      const double b1[4] = {q1[0].x, q1[0].y, q1[1].x, q1[1].y}, b2[4] = {q2[0].x, q2[0].y, q2[1].x, q2[1].y};
      const int mk[4] = {qm.x, qm.y, qm.z, qm.w};
      if (ib + 4 < nfull) load(ib + 4);
      double o[CPL][4];
      if ((mk[0] & mk[1] & mk[2] & mk[3]) == 2) {  // all tail rows
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int j = 0; j < CPL; ++j) {
            o[j][k] = fma(b1[k], y[j][k], -b2[k] * sc[j]);
            sc[j] += y[j][k];
          }
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int j = 0; j < CPL; ++j) {
            o[j][k] = mk[k] == 2 ? fma(b1[k], y[j][k], -b2[k] * sc[j]) : 0.0;
            sc[j] = mk[k] == 1 ? y[j][k] : (mk[k] == 2 ? sc[j] + y[j][k] : sc[j]);
          }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int j = 0; j < CPL; ++j)
          if (h[j]) raw[(ib + k) * n2 + lane + 32 * j] = o[j][k];
    }
    for (int i = nfull; i < nrows; ++i) {  // tail of a partial chunk
      const int mk = imode[i];
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        const double xv = h[j] ? raw[i * n2 + lane + 32 * j] : 0.0;
        const double ov = mk == 2 ? fma(c1[i], xv, -c2[i] * sc[j]) : 0.0;
        sc[j] = mk == 1 ? xv : (mk == 2 ? sc[j] + xv : sc[j]);
        if (h[j]) raw[i * n2 + lane + 32 * j] = ov;
      }
    }
#pragma unroll
    for (int j = 0; j < CPL; ++j)
      if (h[j]) S[lane + 32 * j] = sc[j];
    __syncwarp();
  }

  // ---- the same transform split over several loader warps (row segments [i0, i1)):
  // per-row scalars, then per-column (sum since the last group start, group start seen)
  // of each segment, then each segment's carry-in from S and the earlier segments and
  // the in-place transform.  lsr: [segment][2][64].
  template <class C>
  __device__ void seg_coeffs(double* scratch, int64_t v0, int nrows, int lane, int i0, int i1) const {
    double* c1 = scratch;
    double* c2 = scratch + C::K;
    double* mode = scratch + 2 * C::K;
    if (v0 < m1pad) {
      for (int i = i0 + lane; i < i1; i += 32) {
        int g = -1;
        double m2g = 0.0;
        if (i < nrows) {
          const int64_t r = v0 + i;
          g = fa.gid_a ? fa.gid_a[r] : 0;
          if (g >= 0) m2g = fa.gid_a ? (double)fa.b_count[g] : (double)fa.m2_global;
        }
        const double rs2 = g >= 0 && m2g > 0.0 ? rsqrt_nr(m2g) : 0.0;
        c1[i] = m2g * rs2;
        c2[i] = rs2;
        mode[i] = (double)g;
      }
      return;
    }
    const int64_t b0 = v0 - m1pad;
    int* imode = reinterpret_cast<int*>(mode);
    // all row gathers of the segment first (group id, then the group's start and the
    // other side's count): two dependent rounds of global loads instead of 2 per row
    constexpr int IT = (C::K / (C::NLOAD > 0 ? C::NLOAD : 1) + 31) / 32;
    const int e = min(i1, nrows);
    int gg[IT];
    int64_t st[IT], cnt[IT];
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int i = i0 + lane + 32 * it;
      gg[it] = (i < e && fa.gid_b) ? __ldg(fa.gid_b + b0 + i) : 0;
    }
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int i = i0 + lane + 32 * it;
      st[it] = 0;
      cnt[it] = fa.m1_global;
      if (fa.gid_b && i < e && gg[it] >= 0) {
        st[it] = __ldg(fa.b_start + gg[it]);
        cnt[it] = __ldg(fa.a_count + gg[it]);
      }
    }
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int i = i0 + lane + 32 * it;
      if (i >= i1) break;
      int md = 0;
      double a1 = 0.0, a2 = 0.0;
      if (i < nrows && gg[it] >= 0) {
        const int64_t br = b0 + i;
        const int64_t rr = fa.gid_b ? br - st[it] : cart_row(br);
        const double m1g = (double)cnt[it];
        if (rr == 0) {
          md = 1;
        } else {
          const double rd = (double)rr;
          md = 2;
          a2 = (m1g * rsqrt_nr(m1g)) * rsqrt_nr(rd * (rd + 1.0));
          a1 = rd * a2;
        }
      }
      // packed per-row coefficients of the branch-free passes: out = c1 x - c2 S and
      // S <- keep S + w x (group start: keep 0, w 1; tail row: 1, 1; no row: 1, 0) --
      // exactly the selects of the row mode (multiplications by 0 / 1 are exact)
      *reinterpret_cast<double4*>(scratch + 4 * i) =
          make_double4(a1, a2, md == 1 ? 0.0 : 1.0, md == 0 ? 0.0 : 1.0);
      (void)imode;
    }
  }
  // Segment [i0, i1) in SEG_SUB sub-segments processed in lockstep (independent
  // recurrences: the per-row latency is paid once per SEG_SUB rows).  pass1: each
  // sub-segment's (sum since its last group start, group start seen) per column, kept
  // in registers, and their combination -> lsr (the segment's aggregate).
  template <class C>
  __device__ void seg_pass1(const double* raw, const double* scratch, double* lsr, int64_t v0, int nrows, int lane,
                            int i0, int i1, double (&sl)[SEG_SUB][2], bool (&sr)[SEG_SUB][2]) const {
    if (v0 < m1pad) return;
    const int n2 = (int)fa.n2;
    const int e = min(i1, nrows);
    const int L = (i1 - i0 + SEG_SUB - 1) / SEG_SUB;
    const double4* cf = reinterpret_cast<const double4*>(scratch);
    int cnt[SEG_SUB];
#pragma unroll
    for (int u = 0; u < SEG_SUB; ++u) cnt[u] = max(0, min(L, e - (i0 + u * L)));
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = lane + 32 * h;
#pragma unroll
      for (int u = 0; u < SEG_SUB; ++u) { sl[u][h] = 0.0; sr[u][h] = false; }
      if (c >= n2) continue;
      // sub-segment cursors (strength-reduced addressing); rows r < cnt[SEG_SUB-1] exist in
      // every sub-segment (cnt is non-increasing), the few others are predicated
      const double* xp[SEG_SUB];
      const double4* cp[SEG_SUB];
#pragma unroll
      for (int u = 0; u < SEG_SUB; ++u) {
        xp[u] = raw + (i0 + u * L) * n2 + c;
        cp[u] = cf + i0 + u * L;
      }
      const int rfull = cnt[SEG_SUB - 1];
      for (int r = 0; r < rfull; ++r) {
        double xv[SEG_SUB];
        double4 q[SEG_SUB];
#pragma unroll
        for (int u = 0; u < SEG_SUB; ++u) {
          xv[u] = *xp[u];
          q[u] = *cp[u];
          xp[u] += n2;
          ++cp[u];
        }
#pragma unroll
        for (int u = 0; u < SEG_SUB; ++u) {
          sl[u][h] = fma(q[u].z, sl[u][h], q[u].w * xv[u]);
          sr[u][h] = sr[u][h] || q[u].z == 0.0;
        }
      }
      for (int r = rfull; r < L; ++r) {
#pragma unroll
        for (int u = 0; u < SEG_SUB; ++u) {
          if (r < cnt[u]) {
            const double xv = *xp[u];
            const double4 q = *cp[u];
            xp[u] += n2;
            ++cp[u];
            sl[u][h] = fma(q.z, sl[u][h], q.w * xv);
            sr[u][h] = sr[u][h] || q.z == 0.0;
          }
        }
      }
      double loc = 0.0;
      bool rst = false;
#pragma unroll
      for (int u = 0; u < SEG_SUB; ++u) {
        loc = sr[u][h] ? sl[u][h] : loc + sl[u][h];
        rst = rst || sr[u][h];
      }
      lsr[c] = loc;
      lsr[64 + c] = rst ? 1.0 : 0.0;
    }
  }
  // pass2: carry-in of the segment (S and the earlier segments), of each sub-segment,
  // then the in-place transform of the sub-segments in lockstep.  s_in0 / s_in1: S of
  // this lane's columns read before the barrier that precedes this pass (the last
  // segment rewrites S at its end).
  template <class C>
  __device__ void seg_pass2(double* raw, double* S, const double* scratch, const double* lsr_all, double s_in0,
                            double s_in1, int64_t v0, int nrows, int lane, int i0, int i1, int seg, int nseg,
                            const double (&sl)[SEG_SUB][2], const bool (&sr)[SEG_SUB][2]) const {
    if (v0 < m1pad) return;
    const int n2 = (int)fa.n2;
    const int e = min(i1, nrows);
    const int L = (i1 - i0 + SEG_SUB - 1) / SEG_SUB;
    const double4* cf = reinterpret_cast<const double4*>(scratch);
    int cnt[SEG_SUB];
#pragma unroll
    for (int u = 0; u < SEG_SUB; ++u) cnt[u] = max(0, min(L, e - (i0 + u * L)));
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = lane + 32 * h;
      if (c >= n2) continue;
      double sv = h == 0 ? s_in0 : s_in1;
      for (int k = 0; k < seg; ++k) {
        const double l = lsr_all[k * 128 + c], r = lsr_all[k * 128 + 64 + c];
        sv = r != 0.0 ? l : sv + l;
      }
      double su[SEG_SUB];
#pragma unroll
      for (int u = 0; u < SEG_SUB; ++u) {
        su[u] = sv;
        sv = sr[u][h] ? sl[u][h] : sv + sl[u][h];
      }
      if (seg == nseg - 1) S[c] = sv;  // the chunk's carry-out (all reads of S happened before)
      double* xp[SEG_SUB];
      const double4* cp[SEG_SUB];
#pragma unroll
      for (int u = 0; u < SEG_SUB; ++u) {
        xp[u] = raw + (i0 + u * L) * n2 + c;
        cp[u] = cf + i0 + u * L;
      }
      const int rfull = cnt[SEG_SUB - 1];
      // tail rows: c1 x - c2 S; group starts and empty rows have c1 = c2 = 0 -> 0
      for (int r = 0; r < rfull; ++r) {
        double xv[SEG_SUB];
        double4 q[SEG_SUB];
#pragma unroll
        for (int u = 0; u < SEG_SUB; ++u) {
          xv[u] = *xp[u];
          q[u] = *cp[u];
        }
#pragma unroll
        for (int u = 0; u < SEG_SUB; ++u) {
          const double out = fma(q[u].x, xv[u], -q[u].y * su[u]);
          su[u] = fma(q[u].z, su[u], q[u].w * xv[u]);
          *xp[u] = out;
          xp[u] += n2;
          ++cp[u];
        }
      }
      for (int r = rfull; r < L; ++r) {
#pragma unroll
        for (int u = 0; u < SEG_SUB; ++u) {
          if (r < cnt[u]) {
            const double xv = *xp[u];
            const double4 q = *cp[u];
            const double out = fma(q.x, xv, -q.y * su[u]);
            su[u] = fma(q.z, su[u], q.w * xv);
            *xp[u] = out;
            xp[u] += n2;
            ++cp[u];
          }
        }
      }
    }
  }

  template <class C>
  __device__ double value(const double* raw, const double* scratch, int64_t v0, int i, int l, int nrows,
                          int rcols) const {
    if (i >= nrows || l >= n) return 0.0;
    const int n1 = (int)fa.n1;
    if (v0 < m1pad) {
      const int g = (int)scratch[2 * C::K + i];
      if (g < 0) return 0.0;
      return l < n1 ? raw[i * rcols + l] * scratch[i]
                    : fa.b_totals[(int64_t)g * fa.n2 + (l - n1)] * scratch[C::K + i];
    }
    return l < n1 ? 0.0 : raw[i * rcols + (l - n1)];
  }
};

// ------------------------------------------------------------------ TMA bulk copy + mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// Bounded wait: a lost transaction traps (launch error) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  for (uint32_t spin = 0;; ++spin) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    if (ok) return;
    if (spin > (1u << 26)) __trap();
  }
}
// Wait for a long phase (a whole chunk) without spinning: the waiting warp shares its
// SM sub-partition with the latency-bound chain warp, so it backs off with nanosleep.
__device__ __forceinline__ void mbar_wait_idle(uint64_t* bar, uint32_t phase) {
  for (uint32_t spin = 0;; ++spin) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
    if (ok) return;
    __nanosleep(256);
    if (spin > (1u << 24)) __trap();
  }
}
// thread 0: fetch `bytes16` (multiple of 16) bytes, or just complete the phase
__device__ __forceinline__ void bulk_fetch(uint64_t* bar, void* dst, const void* src, uint32_t bytes16) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (bytes16) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes16)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(__cvta_generic_to_global(src)), "r"(bytes16), "r"(smem_u32(bar))
        : "memory");
  } else {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
  }
}

// thread 0: pull the next chunk's rows into L2 (the direct-load leaf reads them from there)
__device__ __forceinline__ void l2_prefetch(const void* src, uint32_t bytes16) {
  if (bytes16)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(__cvta_generic_to_global(src)), "r"(bytes16)
                 : "memory");
}

// ------------------------------------------------------------------ panel factorisation
#ifdef JQ_PANEL_TIMING
__device__ long long g_ptime[16];
#define PT(i)                                                   \
  do {                                                          \
    long long now_ = clock64();                                 \
    pt_acc[i] += now_ - pt_last;                                \
    pt_last = now_;                                             \
  } while (0)
#else
#define PT(i) do {} while (0)
#endif

// Householder factorisation of one 8-column panel by ALL warps of the CTA.  Warp w
// holds rows [w*KW, (w+1)*KW) of the panel tile in `cp` (lane (g,t): column j0+g,
// local rows 8*it + 2*t + b).  LAPACK dlarfg convention: beta = -sign(alpha)|x|,
// tau = (beta - alpha)/beta = 1 + |alpha|/|x|, v = [1; x2/(alpha - beta)].  Columns keep
// their UNscaled values during the panel (y_g = scale_g x_g).  Per column: the owner
// quad publishes its rows of x inside the warp, every quad forms its partial
// x . c_g, one quad reduction, and a CTA-wide fixed-order sum of the WARPS partials
// gives d_g (g = j: |x|^2; g > j: reflector dot product; g < j: T entries).
// On return cp holds Y (scaled) and Yt (this warp's rows) / T / R rows are written.
// NW = warps holding rows (partials summed in warp order), BAR = 0: __syncthreads,
// else named barrier BAR over those NW warps; `warp` = the caller's row-warp index.
template <class C, int NW = C::WARPS, int BAR = 0>
__device__ __forceinline__ void factor_panel_all(double (&cp)[C::KWT][2], double* R, const int j0, double* Ytw,
                                                 double* T, double* U, double* taus, double* scs,
                                                 double* P, const int warp, const int lane) {
  const int g = lane >> 2, t = lane & 3;
  // The panel's R rows are final at panel start (reflector jj rewrites only row
  // j0+jj): the next column's entries are prefetched one column ahead.
  double alpha_n = R[rix<C>(j0, j0)], rg_n = R[rix<C>(j0, j0 + g)];
  double scale_g = 0.0;  // scale of my own column g
#pragma unroll
  for (int jj = 0; jj < 8; ++jj) {
    const double alpha = alpha_n, rgj = rg_n;
    if (jj < 7) {
      alpha_n = R[rix<C>(j0 + jj + 1, j0 + jj + 1)];
      rg_n = R[rix<C>(j0 + jj + 1, j0 + g)];
    }
    // x_jj broadcast inside the warp: lane (g,t) needs rows (it, t, b) held by lane (jj, t)
    double xv[C::KWT][2];
#pragma unroll
    for (int it = 0; it < C::KWT; ++it) {
      xv[it][0] = __shfl_sync(FULL, cp[it][0], jj * 4 + t);
      xv[it][1] = __shfl_sync(FULL, cp[it][1], jj * 4 + t);
    }
    double dp0 = 0.0, dp1 = 0.0;
#pragma unroll
    for (int it = 0; it < C::KWT; ++it) {
      dp0 = fma(xv[it][0], cp[it][0], dp0);
      dp1 = fma(xv[it][1], cp[it][1], dp1);
    }
    double d = dp0 + dp1;
    d += __shfl_xor_sync(FULL, d, 1);
    d += __shfl_xor_sync(FULL, d, 2);
    double* Pj = P + (jj & 1) * (NW * 8);
    if (t == 0) Pj[warp * 8 + g] = d;
    if (BAR == 0) __syncthreads();
    else named_bar(BAR, NW * 32);
    d = 0.0;
    double sj = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {  // fixed order: bit-identical in every warp
      d += Pj[w * 8 + g];
      sj += Pj[w * 8 + jj];
    }
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
    // g > jj: c_g <- c_g - tau (R[j][g] + y_j . c_g) y_j,  y_j = scale x_j
    const double tw = tau * fma(scale, d, rgj);
    const double a = g > jj ? -tw * scale : 0.0;
#pragma unroll
    for (int it = 0; it < C::KWT; ++it)
#pragma unroll
      for (int b = 0; b < 2; ++b) cp[it][b] = fma(a, xv[it][b], cp[it][b]);
    if (g == jj) scale_g = scale;
    if (warp == 0 && t == 0) {  // off the chain: plain predicated stores
      if (g >= jj) R[rix<C>(j0 + jj, j0 + g)] = g > jj ? rgj - tw : beta;
      else U[g * 8 + jj] = d;   // x_g . x_jj  (scaled in T below)
      if (g == jj) { taus[jj] = tau; scs[jj] = scale; }
    }
  }
  // Y = X diag(scale): registers (B operand of Z) and this warp's rows of Y^T
#pragma unroll
  for (int it = 0; it < C::KWT; ++it) {
    cp[it][0] *= scale_g;
    cp[it][1] *= scale_g;
    *reinterpret_cast<double2*>(Ytw + g * C::LDYT + 8 * it + 2 * t) = make_double2(cp[it][0], cp[it][1]);
  }
  if (warp == 0) {
    __syncwarp();
    // T (8 x 8 upper triangular): T[r][r] = tau_r,
    // T[r][j] = -tau_j sum_{m=r}^{j-1} T[r][m] (y_m . y_j),  y_m . y_j = sc_m sc_j x_m . x_j
    if (lane < 8) {
      const int r = lane;
      double sc[8], tu[8], trow[8];
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
}

// T (8 x 8 upper triangular) of the compact WY form from U[m][j] = x_m . x_j (m < j),
// taus and scales: T[r][r] = tau_r, T[r][j] = -tau_j sum_{m=r}^{j-1} T[r][m] (y_m . y_j).
// Lanes 0..7 of the calling warp (U / taus / scs visible to them).
template <class C>
__device__ __forceinline__ void compute_T(double* T, const double* U, const double* taus, const double* scs,
                                          const int lane) {
  if (lane < 8) {
    const int r = lane;
    double sc[8], tu[8], trow[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) { sc[m] = scs[m]; tu[m] = taus[m]; }
#pragma unroll
    for (int m = 0; m < 8; ++m) trow[m] = (m == r) ? tu[m] : 0.0;
#pragma unroll
    for (int j = 1; j < 8; ++j) {
      double acc = 0.0;
#pragma unroll
      for (int m = 0; m < j; ++m) acc = fma(trow[m], (U[m * 8 + j] * sc[m]) * sc[j], acc);
      if (j > r) trow[j] = -tu[j] * acc;
    }
#pragma unroll
    for (int m = 0; m < 8; ++m) T[r * C::LDT + m] = trow[m];
  }
}

// ------------------------------------------------------------------ Gram panel
// X[g][g] of an 8 x 8 matrix held in accumulator layout, in every lane of quad g
__device__ __forceinline__ double diag_of(const double (&X)[2], const int lane) {
  const int g = lane >> 2;
  return __shfl_sync(FULL, (g & 1) ? X[1] : X[0], 4 * g + (g >> 1));
}
#ifdef JQ_KTIME
__device__ unsigned long long g_gram_fail[16];
#endif
// Householder factorisation of the stacked panel [R_p; X] (R_p: the panel's 8 R rows,
// X: the chunk's K rows of the panel columns, CTA-wide) computed from the 8 x 8 Gram
// G = X^T X alone.  Reflector i (alpha = R[i][i], |x_i'|^2 = G[i][i]) only needs inner
// products of the current columns, and applying it is the rank-2 update
//   x_c <- x_c + a_c x_i  =>  G[g][c] += a_g G[i][c] + a_c G[g][i] + a_g a_c G[i][i],
// so the 8-step chain runs on registers (two Gram entries per lane, accumulator
// layout) with no row data, no CTA barrier and a latency independent of K.  The
// columns are tracked as x' = X M; the trailing update uses Y = X M' (M' = M diag(scale))
// through 8 x 8 products.  Cancellation guard (checked once, after the 8 steps): every
// step i must have  alpha_i^2 + G[i][i] >= 1e-2 (alpha_i^2 + P_i)  with
// P_i = sum_k M[k][i]^2 G0[k][k] (x_i' = X M[:, i]: the scale of the rounding error of
// |x_i'|^2), which bounds the relative error of |[alpha; x_i']|^2 by ~1e-13; otherwise
// the panel is redone by factor_panel_all (explicit row data).
template <class C>
__device__ __forceinline__ bool factor_panel_gram(double (&G)[2], double (&Rb)[2], const double* Rs,
                                                  const int j0, double* T, double* Mg, const int lane,
                                                  const double Pg) {
  // Rs/j0: R in shared memory (read only); Rb: on return the panel's new 8 x 8 R block
  // in accumulator layout (lane (g,t): R[g][c0], R[g][c1]), committed by the caller.
  const int g = lane >> 2, t = lane & 3, c0 = 2 * t, c1 = 2 * t + 1;
  double M0 = (g == c0) ? 1.0 : 0.0, M1 = (g == c1) ? 1.0 : 0.0;
  // cancellation guard, evaluated after the 8 steps: per step s2_i = alpha_i^2 + |x_i'|^2
  // and alpha_i are kept; P_i = sum_k M[k][i]^2 Pg_k bounds the scale of the rounding
  // error of |x_i'|^2 (x_i' = X M[:, i], Pg_k = G0[k][k] or a larger bound)
  double s2r[8], alr[8];
  unsigned reflm = 0;
  double T0 = 0.0, T1 = 0.0;  // T[g][c0], T[g][c1], built one column per step
  double sc0 = 0.0, sc1 = 0.0;
  bool ok = true;
  // row i of the R block (alpha = R[i][i], rg = R[i][g], r0/r1 = R[i][c0/c1]) from shared
  // memory, one step ahead (row i is only rewritten at step i, in registers)
  auto rrow = [&](int i, double& al, double& rg_, double& r0_, double& r1_) {
    al = Rs[rix<C>(j0 + i, j0 + i)];
    rg_ = Rs[rix<C>(j0 + i, j0 + g)];
    r0_ = Rs[rix<C>(j0 + i, j0 + c0)];
    r1_ = Rs[rix<C>(j0 + i, j0 + c1)];
  };
  double alpha_n, rg_n, r0_n, r1_n;
  rrow(0, alpha_n, rg_n, r0_n, r1_n);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const double alpha = alpha_n, rg = rg_n, r0 = r0_n, r1 = r1_n;
    if (i < 7) rrow(i + 1, alpha_n, rg_n, r0_n, r1_n);
    const double e = (i & 1) ? G[1] : G[0];
    const double d0 = __shfl_sync(FULL, G[0], 4 * i + t);        // G[i][c0]
    const double d1 = __shfl_sync(FULL, G[1], 4 * i + t);        // G[i][c1]
    const double dg = __shfl_sync(FULL, e, 4 * g + (i >> 1));    // G[g][i]
    const double sj = __shfl_sync(FULL, e, 4 * i + (i >> 1));    // G[i][i]
    const double mgi = __shfl_sync(FULL, (i & 1) ? M1 : M0, 4 * g + (i >> 1));  // M[g][i]
    const double s2 = fma(alpha, alpha, sj);
    // branch-free scalars; |[alpha; x]|^2 outside the safe range of the MUFU
    // approximations rejects the panel (the explicit path has an IEEE branch)
    const bool refl = sj > 0.0;
    s2r[i] = s2;
    alr[i] = alpha;
    reflm |= refl ? (1u << i) : 0u;
    const double rn = rsqrt_nr(refl ? s2 : 1.0);
    const double nrm = s2 * rn;
    const double beta = refl ? (alpha >= 0.0 ? -nrm : nrm) : alpha;
    const double tau = refl ? fma(fabs(alpha), rn, 1.0) : 0.0;
    const double scale = refl ? rcp_nr(alpha - beta) : 0.0;
    const double twg = tau * fma(scale, dg, rg), tw0 = tau * fma(scale, d0, r0), tw1 = tau * fma(scale, d1, r1);
    const double ag = g > i ? -twg * scale : 0.0;
    const double a0 = c0 > i ? -tw0 * scale : 0.0;
    const double a1 = c1 > i ? -tw1 * scale : 0.0;
    if (g == i) {  // new row i of R
      Rb[0] = c0 > i ? r0 - tw0 : (c0 == i ? beta : 0.0);
      Rb[1] = c1 > i ? r1 - tw1 : (c1 == i ? beta : 0.0);
    }
    // T column i: T[g][i] = -tau_i sum_m T[g][m] (y_m . y_i),  y_m . y_i = sc_m sc_i G[m][i]
    // (entries of T for columns >= i and scales of columns > i are still zero)
    double tp = fma(T1 * sc1, d1, T0 * sc0 * d0);
    tp += __shfl_xor_sync(FULL, tp, 1);
    tp += __shfl_xor_sync(FULL, tp, 2);
    const double tgi = g < i ? -tau * scale * tp : (g == i ? tau : 0.0);
    if (c0 == i) { sc0 = scale; T0 = tgi; }
    if (c1 == i) { sc1 = scale; T1 = tgi; }
    G[0] = fma(ag * a0, sj, fma(a0, dg, fma(ag, d0, G[0])));
    G[1] = fma(ag * a1, sj, fma(a1, dg, fma(ag, d1, G[1])));
    M0 = fma(a0, mgi, M0);
    M1 = fma(a1, mgi, M1);
  }
  // guard: P_c for this lane's columns c0, c1 (sum over the 8 rows g of the quad column)
  double p0 = M0 * M0 * Pg, p1 = M1 * M1 * Pg;
#pragma unroll
  for (int off = 4; off < 32; off <<= 1) {
    p0 += __shfl_xor_sync(FULL, p0, off);
    p1 += __shfl_xor_sync(FULL, p1, off);
  }
  double s2a = 0.0, ala = 0.0, s2b = 0.0, alb = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (c0 == i) { s2a = s2r[i]; ala = alr[i]; }
    if (c1 == i) { s2b = s2r[i]; alb = alr[i]; }
  }
  const bool ra = (reflm >> c0) & 1u, rb = (reflm >> c1) & 1u;
  const bool good = (s2a >= 1e-2 * fma(ala, ala, p0)) && (!ra || (s2a > 1e-280 && s2a < 1e280)) &&
                    (s2b >= 1e-2 * fma(alb, alb, p1)) && (!rb || (s2b > 1e-280 && s2b < 1e280));
  ok = __all_sync(FULL, good);
#ifdef JQ_KTIME
  if (!ok && lane == 0) atomicAdd(&g_gram_fail[0], 1ull);
#endif
  *reinterpret_cast<double2*>(Mg + g * C::LDT + c0) = make_double2(M0 * sc0, M1 * sc1);
  *reinterpret_cast<double2*>(T + g * C::LDT + c0) = make_double2(T0, T1);
  return ok;
}

// ------------------------------------------------------------------ Cholesky panel
// The same panel factorisation as factor_panel_gram (identical outputs: R rows, M', T,
// the guard), derived in closed form from S = R_p^T R_p + G instead of the 8-step
// reflector chain.  For the stacked panel [R_p; X] (R_p: the panel's 8 x 8 upper R
// block, X: the chunk rows) the Householder QR with reflectors v = [e_j; y_j] is
//   R_new = D chol(S)^T,  D_jj = -sign(R_p[j][j])   (beta = -sign(alpha) |.|: no
//                                                   cancellation in W = R_p - R_new)
//   Y = X W^{-1}  (M' = W^{-1}),    T = -W R_new^{-1}
// (Q^T [R_p; X] = [R_new; 0] with Q = I - V T V^T, V = [I; Y], fixes Y and T given
// R_new; T^{-1} + T^{-T} = I + Y^T Y follows from R_new^T R_new = R_p^T R_p + X^T X).
// The critical path is the 8 Cholesky steps, each ONE reciprocal (MUFU + one cubic
// correction) between two shuffles -- versus rsqrt then rcp plus the T column in the
// reflector chain -- then W^{-1} and R_new^{-1} by back substitution (one lane per
// column, operands in shared memory `scr`: >= 16 LDT + 16 doubles, the explicit path's
// U / taus / scales / partials, idle while the chain runs) and one 8 x 8 DMMA product.
// Guard (the reflector chain's, made slightly stricter): pivot_c (= R_new[c][c]^2 =
// alpha_c^2 + |x_c'|^2) >= 1e-2 (S[c][c] + P_c), with P_c = sum_k M[k][c]^2 Pg_k bounding the
// rounding error of |x_c'|^2 from the (derived) Gram's -- M = M' diag(W) read off the
// back substitution -- and S[c][c] >= alpha_c^2 that of the elimination itself.  Otherwise
// the panel goes to the reflector chain, then the explicit path.
#ifdef JQ_CHOL_PHASES
__device__ long long g_chol_ph[8];
#define CHOL_PH(k) do { if (lane == 0) { const long long t_ = clock64(); atomicAdd((unsigned long long*)&g_chol_ph[k], (unsigned long long)(t_ - ph_t)); ph_t = t_; } } while (0)
#else
#define CHOL_PH(k) do {} while (0)
#endif
template <class C>
__device__ __forceinline__ bool factor_panel_chol(const double (&G)[2], double (&Rb)[2], const double* Rs,
                                                  const int j0, double* T, double* Mg, double* scr,
                                                  const int lane, const double Pg) {
  const int g = lane >> 2, t = lane & 3, c0 = 2 * t, c1 = 2 * t + 1;
#ifdef JQ_CHOL_PHASES
  long long ph_t = clock64();
#endif
  // R_p in accumulator layout, and the fragments R_p[2t+b][g] of R_p^T R_p
  const double rp0 = (c0 >= g) ? Rs[rix<C>(j0 + g, j0 + c0)] : 0.0;
  const double rp1 = (c1 >= g) ? Rs[rix<C>(j0 + g, j0 + c1)] : 0.0;
  const double rt0 = (g >= c0) ? Rs[rix<C>(j0 + c0, j0 + g)] : 0.0;
  const double rt1 = (g >= c1) ? Rs[rix<C>(j0 + c1, j0 + g)] : 0.0;
  const double alpha = Rs[rix<C>(j0 + g, j0 + g)];
  const double dsg = alpha >= 0.0 ? -1.0 : 1.0;  // D_gg
  double S[2] = {G[0], G[1]};
  dmma(S, rt0, rt0);
  dmma(S, rt1, rt1);
  const double sdiag = diag_of(S, lane);
  CHOL_PH(0);
  // 8 Cholesky steps; lanes of quad j keep row j of S^{(j)} (R_new row j up to the
  // 1 / sqrt(pivot) applied after the loop: no rsqrt on the critical path).  Every lane
  // also forms the NEXT pivot itself, with exactly the owner lane's operations
  // (S[j+1][j+1] - (S[j+1][j] / S[j][j]) S[j][j+1]), from values shuffled at the start of
  // the step, so the critical path per step is one reciprocal + one multiply + one FMA
  // (no shuffle between consecutive reciprocals).
  double piv_g = 1.0, sv0 = 0.0, sv1 = 0.0;
  bool rng_ok = true;
  double piv = __shfl_sync(FULL, S[0], 0);  // S[0][0]
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double e = (j & 1) ? S[1] : S[0];
    const double sgj = __shfl_sync(FULL, e, 4 * g + (j >> 1));  // S[g][j]
    const double sj0 = __shfl_sync(FULL, S[0], 4 * j + t);      // S[j][c0]
    const double sj1 = __shfl_sync(FULL, S[1], 4 * j + t);      // S[j][c1]
    double a_lo = 0.0, a_up = 0.0, b_nx = 0.0;
    if (j < 7) {
      const int jn = j + 1;
      a_lo = __shfl_sync(FULL, e, 4 * jn + (j >> 1));                        // S[j+1][j]
      a_up = __shfl_sync(FULL, (jn & 1) ? S[1] : S[0], 4 * j + (jn >> 1));   // S[j][j+1]
      b_nx = __shfl_sync(FULL, (jn & 1) ? S[1] : S[0], 4 * jn + (jn >> 1));  // S[j+1][j+1]
    }
    const bool in = piv > 1e-280 && piv < 1e280;  // MUFU approximations' safe range
    rng_ok = rng_ok && in;
    const double inv = rcp_nr(in ? piv : 1.0);
    const double f = sgj * inv;  // S[g][c] -= S[g][j] S[j][c] / S[j][j]  (g, c > j)
    if (g == j) {
      piv_g = piv;
      sv0 = c0 >= j ? sj0 : 0.0;
      sv1 = c1 >= j ? sj1 : 0.0;
    }
    if (g > j && c0 > j) S[0] = fma(-f, sj0, S[0]);
    if (g > j && c1 > j) S[1] = fma(-f, sj1, S[1]);
    if (j < 7) piv = fma(-(a_lo * inv), a_up, b_nx);  // = the owner lane's S[j+1][j+1]
  }
  CHOL_PH(1);
  const double rs_g = rsqrt_nr(rng_ok ? piv_g : 1.0);
  Rb[0] = dsg * sv0 * rs_g;  // R_new[g][:] = D_g S^{(g)}[g][:] / sqrt(pivot_g)
  Rb[1] = dsg * sv1 * rs_g;
  const double w0 = rp0 - Rb[0], w1 = rp1 - Rb[1];
  // W and R_new in natural layout (scratch), their diagonals' reciprocals
  double* Un = scr;                 // [2][8][LDT]: W, R_new
  double* dg = scr + 16 * C::LDT;   // [2][8]: 1 / W[i][i], 1 / R_new[i][i]
  *reinterpret_cast<double2*>(Un + g * C::LDT + c0) = make_double2(w0, w1);
  *reinterpret_cast<double2*>(Un + (8 + g) * C::LDT + c0) = make_double2(Rb[0], Rb[1]);
  double* gq = scr + 16 * C::LDT + 16;  // [4][8]: pivot, W[g][g]^2, S[g][g], Pg of row g (guard)
  if (t == 0) {
    const double wgg = alpha - dsg * piv_g * rs_g;  // W[g][g] = alpha - R_new[g][g]
    dg[g] = rcp_nr(wgg);
    dg[8 + g] = dsg * rs_g;                      // 1 / R_new[g][g]
    gq[g] = piv_g;
    gq[8 + g] = wgg * wgg;
    gq[16 + g] = sdiag;
    gq[24 + g] = Pg;
  }
  __syncwarp();
  CHOL_PH(2);
  // Inverses of the two upper-triangular matrices by back substitution, one lane per
  // column (lanes 0..7: W^{-1} = M', lanes 8..15: R_new^{-1}), the same code on every
  // lane (no divergence), right-looking: per step one multiply + one FMA on the path.
  bool good_c = true;
  {
    const int m = (lane >> 3) & 1, c = lane & 7;
    const double* U = Un + m * 8 * C::LDT;
    const double* d = dg + 8 * m;
    double acc[8], x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.0;
#pragma unroll
    for (int k = 7; k >= 0; --k) {
      const double xk = -d[k] * acc[k];
      x[k] = k > c ? 0.0 : (k == c ? d[k] : xk);
#pragma unroll
      for (int i = 0; i < k; ++i) acc[i] = fma(U[i * C::LDT + k], x[k], acc[i]);
    }
    __syncwarp();
    if (lane < 16) {
      double* out = m ? T : Mg;  // R_new^{-1} parks in T's buffer
#pragma unroll
      for (int i = 0; i < 8; ++i) out[i * C::LDT + c] = x[i];
    }
    // Guard, tracking nothing in the elimination: the chunk columns' combination of
    // eliminated column c is x_c' = X M[:, c] with M = M' diag(W) (y_c = x_c' / W[c][c]),
    // so the rounding error of |x_c'|^2 from the Gram's is bounded by
    // P_c = W[c][c]^2 sum_k M'[k][c]^2 Pg_k (lane c < 8 holds column c of M').
    if (lane < 8) {
      double pa = 0.0, pb = 0.0;  // two short chains (the chain warp is latency-bound)
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        pa = fma(x[k] * x[k], gq[24 + k], pa);
        pb = fma(x[k + 1] * x[k + 1], gq[24 + k + 1], pb);
      }
      // pivot >= 1e-2 (S[c][c] + P_c): S[c][c] >= alpha_c^2 covers both conditions
      good_c = gq[c] >= 1e-2 * fma(pa + pb, gq[8 + c], gq[16 + c]);
    }
  }
  __syncwarp();
  CHOL_PH(3);
  // T = -W R_new^{-1}  (B fragments R_new^{-1}[2t+b][g] from the parked copy)
  const double b0 = T[c0 * C::LDT + g], b1 = T[c1 * C::LDT + g];
  double P[2] = {0.0, 0.0};
  dmma(P, w0, b0);
  dmma(P, w1, b1);
  __syncwarp();
  *reinterpret_cast<double2*>(T + g * C::LDT + c0) = make_double2(-P[0], -P[1]);
  CHOL_PH(4);
  const bool good = rng_ok && good_c;
  const bool ok = __all_sync(FULL, good);
#ifdef JQ_KTIME
  if (!ok && lane == 0) atomicAdd(&g_gram_fail[0], 1ull);
#endif
  CHOL_PH(5);
  return ok;
}

// ------------------------------------------------------------------ the kernel
// Each CTA: R (init zero, or R_init[cta]) absorbs its rows [row_begin, row_end)
// of `src`, then writes R (NP x NP, row-major, zeros below the diagonal) to
// r_out + cta * NP * NP.  For the combine step, CTA c absorbs rows of stack
// element 2c+1 into R = element 2c.
#ifndef JQ_PROBE
#define JQ_PROBE 0
#endif
#ifdef JQ_KTIME
__device__ unsigned long long g_ktime[16];
#define KT_DECL long long kt_acc[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0}; long long kt_t = clock64();
#define KT_MARK(i) do { long long n_ = clock64(); kt_acc[i] += n_ - kt_t; kt_t = n_; } while (0)
#define KT_FLUSH() do { if (lane == 0) for (int i_ = 0; i_ < 10; ++i_) atomicAdd(&g_ktime[i_], (unsigned long long)kt_acc[i_]); \
                        if (tid == 0) atomicAdd(&g_ktime[15], 1ull); } while (0)
#else
#define KT_DECL
#define KT_MARK(i) do {} while (0)
#define KT_FLUSH() do {} while (0)
#endif
template <class C>
__device__ __forceinline__ int pass_rows(int rcol) {
  return rcol > 0 ? min(C::K, (C::RAW / rcol) & ~7) : C::K;
}

template <class C, class Src, bool COMBINE>
__global__ void __launch_bounds__(C::THREADS, C::MIN_CTAS)
tsqr_kernel(Src src, int64_t rows_per_cta, int64_t total_rows, const double* __restrict__ r_init,
            int64_t init_count, double* __restrict__ r_out, int use_tma) {
  extern __shared__ __align__(16) double smem_dyn[];
  double* raw = smem_dyn + C::OFF_RAW;
  double* T = smem_dyn + C::OFF_T;
  double* U = smem_dyn + C::OFF_U;
  double* taus = smem_dyn + C::OFF_TAU;
  double* scs = smem_dyn + C::OFF_SC;
  double* P = smem_dyn + C::OFF_P;
  double* Zp = smem_dyn + C::OFF_ZP;
  double* Ws = smem_dyn + C::OFF_WS;
  double* S = smem_dyn + C::OFF_S;
  double* scratch = smem_dyn + C::OFF_LD;
  double* Mg = smem_dyn + C::OFF_M;
  volatile int* flag = reinterpret_cast<volatile int*>(smem_dyn + C::OFF_FLAG);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_dyn + C::OFF_BAR);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int64_t cta = blockIdx.x;
  double* Ytw = smem_dyn + C::OFF_YT + warp * C::SZ_YT;

  double* R;
  if constexpr (C::R_SMEM) R = smem_dyn + C::OFF_R;
  else R = r_out + cta * C::NP * C::NP;

  // ---- R init
  const double* rinit = nullptr;
  Src s = src;
  int64_t row_begin, row_end;
  if constexpr (COMBINE) {
    // one stack (init_count elements), or -- rows_per_cta = k > 0 -- two stacks of k
    // elements each, the first at r_init and the second at src.m, combined side by side
    // (CTA c < ceil(k/2) works on the first; outputs stay contiguous)
    const double* base = r_init;
    int64_t j = cta, cnt = init_count;
    if (rows_per_cta > 0) {
      const int64_t half = (rows_per_cta + 1) / 2;
      cnt = rows_per_cta;
      if (cta >= half) { base = src.m; j = cta - half; }
    }
    rinit = base + (2 * j) * C::NP * C::NP;
    if (2 * j + 1 < cnt) {
      s.m = base + (2 * j + 1) * C::NP * C::NP;
      row_begin = 0; row_end = C::NP;
    } else {
      row_begin = row_end = 0;
    }
  } else {
    row_begin = cta * rows_per_cta;
    row_end = min(total_rows, row_begin + rows_per_cta);
  }
  for (int idx = tid; idx < C::NP * C::NP; idx += C::THREADS) {
    const int r = idx / C::NP, c = idx - r * C::NP;
    if (c >= 8 * (r >> 3)) R[rix<C>(r, c)] = rinit ? rinit[idx] : 0.0;
  }
  s.template begin<C>(S, row_begin);
  if (tid == 0) mbar_init(bar);
  __syncthreads();

  // rows of the pass starting at v0: never past its chunk (the prefix state S must
  // not run ahead), the CTA range or the source
  auto pass_nrows = [&](int64_t v0, int rb, int64_t chunk0) -> int {
    int64_t lim = chunk0 + C::K < row_end ? chunk0 + C::K : row_end;
    int64_t nr = lim - v0 < (int64_t)rb ? lim - v0 : (int64_t)rb;
    const int64_t av = s.avail(v0);
    nr = av < nr ? av : nr;
    return nr > 0 ? (int)nr : 0;
  };
  auto issue = [&](int64_t v0, int64_t chunk0) {  // thread 0 only
    const int rcol = s.rc(v0);
    const int nr = pass_nrows(v0, pass_rows<C>(rcol), chunk0);
    const uint32_t bytes = uint32_t(nr) * uint32_t(rcol) * 8u;
    bulk_fetch(bar, raw, s.ptr(v0), bytes & ~15u);
  };
  // direct chunk loads (flag 256 off: JQ_TSQR_STAGED=1) for sources that have them
  const bool direct = Src::DIRECT && !(use_tma & 256);
  auto prefetch = [&](int64_t v0) {  // thread 0, direct mode: the chunk at v0 into L2
    if (!(use_tma & 1) || v0 >= row_end) return;
    const int64_t lim = v0 + C::K < row_end ? v0 + C::K : row_end;
    int64_t nr = lim - v0;
    const int64_t av = s.avail(v0);
    nr = av < nr ? av : nr;
    if (nr > 0) l2_prefetch(s.ptr(v0), uint32_t(nr * s.rc(v0) * 8) & ~15u);
  };
  if (tid == 0 && row_begin < row_end) {
    if (direct) prefetch(row_begin);
    else if (use_tma & 1) issue(row_begin, row_begin);
  }

  double c[C::NLT][C::KWT][2];  // this warp's rows of every column tile (C^T accumulator layout)
  uint32_t phase = 0;
  KT_DECL

  for (int64_t row0 = row_begin; row0 < row_end; row0 += C::K) {
    if (direct) {
      if (tid == 0) prefetch(row0 + C::K);
      const int64_t lim = row0 + C::K < row_end ? row0 + C::K : row_end;
      int64_t nr = lim - row0;
      const int64_t av = s.avail(row0);
      nr = av < nr ? av : nr;
      s.template load_direct<C, RowBar<C::WARPS, 0>>(c, row0, nr > 0 ? (int)nr : 0, S, raw, Zp, scratch, warp, lane,
                                                    [&](int i) { KT_MARK(i); });
      KT_MARK(6);
    }
    const int rcol = s.rc(row0);
    const int rb = pass_rows<C>(rcol);
    const int npass = (C::K + rb - 1) / rb;
    if (!direct) {
#pragma unroll
      for (int q = 0; q < C::NLT; ++q)
#pragma unroll
        for (int it = 0; it < C::KWT; ++it) c[q][it][0] = c[q][it][1] = 0.0;  // rows past the range stay zero
    }
    for (int h = 0; !direct && h < npass && row0 + (int64_t)h * rb < row_end; ++h) {
      const int64_t pv0 = row0 + (int64_t)h * rb;
      const int nr = pass_nrows(pv0, rb, row0);
      const int nel = nr * rcol;
      if (use_tma & 1) {
        mbar_wait(bar, phase);
        phase ^= 1;
        if ((nel & 1) && tid == 0) raw[nel - 1] = __ldg(s.ptr(pv0) + nel - 1);  // 8-byte tail
      } else {
        const double* src_rows = s.ptr(pv0);
        for (int e = tid; e < nel; e += C::THREADS) raw[e] = __ldg(src_rows + e);
      }
      __syncthreads();
      KT_MARK(0);
      s.template prep<C>(raw, S, scratch, pv0, nr);
      __syncthreads();
      KT_MARK(5);
#pragma unroll
      for (int q = 0; q < C::NLT; ++q) {
        const int l = q * 8 + g;
#pragma unroll
        for (int it = 0; it < C::KWT; ++it)
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const int li = warp * C::KW + 8 * it + 2 * t + b - h * rb;
            if (li >= 0 && li < rb) c[q][it][b] = s.template value<C>(raw, scratch, pv0, li, l, nr, rcol);
          }
      }
      __syncthreads();  // raw consumed: prefetch the next pass / chunk behind the panel loop
      if ((use_tma & 1) && tid == 0) {
        const bool same = h + 1 < npass && pv0 + rb < row_end;
        const int64_t nv0 = same ? pv0 + rb : row0 + C::K;
        if (nv0 < row_end) issue(nv0, same ? row0 : nv0);
      }
      KT_MARK(6);
    }

#pragma unroll 1
    for (int p = 0; p < C::NLT; ++p) {
      const int j0 = 8 * p;
      double cp[C::KWT][2];  // panel tile X (this warp's rows)
#pragma unroll
      for (int q = 0; q < C::NLT; ++q)
        if (q == p)
#pragma unroll
          for (int it = 0; it < C::KWT; ++it) { cp[it][0] = c[q][it][0]; cp[it][1] = c[q][it][1]; }
      // ---------------- (1) partial Gram X^T X (slot p) and partial (X^T C_q)^T of the
      // trailing tiles, X^T rows of this warp for the apply step
      {
        double z[2] = {0.0, 0.0}, z2[2] = {0.0, 0.0};
#pragma unroll
        for (int it = 0; it < C::KWT; ++it) {
          dmma(z, cp[it][0], cp[it][0]);
          dmma(z2, cp[it][1], cp[it][1]);
        }
        *reinterpret_cast<double2*>(Zp + (warp * C::NLT + p) * 64 + 2 * lane) = make_double2(z[0] + z2[0], z[1] + z2[1]);
      }
#pragma unroll
      for (int q = 0; q < C::NLT; ++q) {
        if (q > p) {
          double z[2] = {0.0, 0.0}, z2[2] = {0.0, 0.0};
#pragma unroll
          for (int it = 0; it < C::KWT; ++it) {
            dmma(z, c[q][it][0], cp[it][0]);
            dmma(z2, c[q][it][1], cp[it][1]);
          }
          *reinterpret_cast<double2*>(Zp + (warp * C::NLT + q) * 64 + 2 * lane) = make_double2(z[0] + z2[0], z[1] + z2[1]);
        }
      }
#pragma unroll
      for (int it = 0; it < C::KWT; ++it)
        *reinterpret_cast<double2*>(Ytw + g * C::LDYT + 8 * it + 2 * t) = make_double2(cp[it][0], cp[it][1]);
      __syncthreads();
      KT_MARK(1);
      // ---------------- (2) the 8-column Householder chain on the summed Gram (warp 0)
      if (warp == 0) {
        double G[2] = {0.0, 0.0};
#pragma unroll
        for (int w = 0; w < C::WARPS; ++w) {  // fixed order
          const double2 gg = *reinterpret_cast<const double2*>(Zp + (w * C::NLT + p) * 64 + 2 * lane);
          G[0] += gg.x;
          G[1] += gg.y;
        }
        double Rb[2];
        const double pg = diag_of(G, lane);
        bool ok = !(use_tma & 16) && factor_panel_chol<C>(G, Rb, R, j0, T, Mg, U, lane, pg);
        if (!ok) ok = factor_panel_gram<C>(G, Rb, R, j0, T, Mg, lane, pg);  // looser guard
        ok = ok && !(use_tma & 2);
        if (ok) {  // commit the panel's R rows
          if (2 * t >= g) R[rix<C>(j0 + g, j0 + 2 * t)] = Rb[0];
          if (2 * t + 1 >= g) R[rix<C>(j0 + g, j0 + 2 * t + 1)] = Rb[1];
        }
        if (lane == 0) flag[0] = ok ? 1 : 0;
      }
      __syncthreads();
      if (flag[0] == 0) {
        // cancellation: explicit factorisation from the row data (rare; CTA-uniform)
        factor_panel_all<C>(cp, R, j0, Ytw, T, U, taus, scs, P, warp, lane);  // cp <- Y, Ytw <- Y^T
        if (warp == 0) {
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const int e = 2 * lane + k, r = e >> 3, cc = e & 7;
            Mg[r * C::LDT + cc] = r == cc ? 1.0 : 0.0;
          }
        }
#pragma unroll
        for (int q = 0; q < C::NLT; ++q) {
          if (q > p) {
            double z[2] = {0.0, 0.0};
#pragma unroll
            for (int it = 0; it < C::KWT; ++it) {
              dmma(z, c[q][it][0], cp[it][0]);
              dmma(z, c[q][it][1], cp[it][1]);
            }
            *reinterpret_cast<double2*>(Zp + (warp * C::NLT + q) * 64 + 2 * lane) = make_double2(z[0], z[1]);
          }
        }
        __syncthreads();
      }
      KT_MARK(2);
      // ---------------- (3) tile q by warp q % WARPS:  Z^T = R_rows^T + S M',  W^T = Z^T T,
      // R_rows -= W,  V^T = W^T M'^T  (S = sum of the partials, fixed order)
      if (JQ_PROBE != 1 && JQ_PROBE != 3) {
        for (int q = p + 1 + ((warp - (p + 1)) % C::WARPS + C::WARPS) % C::WARPS; q < C::NLT; q += C::WARPS) {
          const int l0 = q * 8;
          const int r0i = rix<C>(j0 + 2 * t, l0 + g), r1i = rix<C>(j0 + 2 * t + 1, l0 + g);
          double s0 = 0.0, s1 = 0.0;
#pragma unroll
          for (int w = 0; w < C::WARPS; ++w) {
            const double2 zz = *reinterpret_cast<const double2*>(Zp + (w * C::NLT + q) * 64 + 2 * lane);
            s0 += zz.x;
            s1 += zz.y;
          }
          double zt[2] = {R[r0i], R[r1i]};
          dmma(zt, s0, Mg[(2 * t) * C::LDT + g]);
          dmma(zt, s1, Mg[(2 * t + 1) * C::LDT + g]);
          double wv[2] = {0.0, 0.0};
          dmma(wv, zt[0], T[(2 * t) * C::LDT + g]);
          dmma(wv, zt[1], T[(2 * t + 1) * C::LDT + g]);
          R[r0i] -= wv[0];
          R[r1i] -= wv[1];
          double vv[2] = {0.0, 0.0};
          dmma(vv, wv[0], Mg[g * C::LDT + 2 * t]);
          dmma(vv, wv[1], Mg[g * C::LDT + 2 * t + 1]);
          *reinterpret_cast<double2*>(Ws + q * 64 + 2 * lane) = make_double2(-vv[0], -vv[1]);
        }
      }
      __syncthreads();
      // ---------------- (4) C_q -= X V on this warp's rows (A = -V^T from smem, B = X^T rows)
      if (JQ_PROBE != 1 && JQ_PROBE != 3) {
#pragma unroll
        for (int q = 0; q < C::NLT; ++q) {
          if (q > p) {
            const double2 nw = *reinterpret_cast<const double2*>(Ws + q * 64 + 2 * lane);
#pragma unroll
            for (int it = 0; it < C::KWT; ++it) {
              dmma(c[q][it], nw.x, Ytw[(2 * t) * C::LDYT + 8 * it + g]);
              dmma(c[q][it], nw.y, Ytw[(2 * t + 1) * C::LDYT + 8 * it + g]);
            }
          }
        }
      }
      __syncwarp();  // Ytw read by the whole warp before the next panel rewrites it
      KT_MARK(3);
    }
    __syncthreads();
    KT_MARK(4);
  }
  KT_FLUSH();
  s.finish(S, tid, C::THREADS);

  // ---- write R (zeros strictly below the diagonal)
  double* out = r_out + cta * C::NP * C::NP;
  if constexpr (C::R_SMEM) {
    for (int idx = tid; idx < C::NP * C::NP; idx += C::THREADS) {
      const int r = idx / C::NP, c2 = idx - r * C::NP;
      out[idx] = c2 >= r ? R[rix<C>(r, c2)] : 0.0;
    }
  } else {
    for (int idx = tid; idx < C::NP * C::NP; idx += C::THREADS) {
      const int r = idx / C::NP, c2 = idx - r * C::NP;
      if (c2 < r) out[idx] = 0.0;
    }
  }
}

#include "jq_tsqr_ws.cuh"

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

template <class C, class Src>
static int ctas_per_sm() {
  int n = 0;
  cudaFuncSetAttribute(tsqr_kernel<C, Src, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, tsqr_kernel<C, Src, false>, C::THREADS, C::SMEM) !=
      cudaSuccess) {
    cudaGetLastError();
    n = 1;
  }
  if (const char* e = getenv("JQ_TSQR_CTAS_PER_SM")) n = std::min(n, atoi(e));  // experiments
  return std::max(1, n);
}

// JQ_TSQR_CHAIN=householder: the reflector chain (factor_panel_gram) instead of the
// Cholesky panel (factor_panel_chol, the default); kernel flag 16.  A/B and parity only.
static int chain_flag() {
  static const int f = [] {
    const char* e = getenv("JQ_TSQR_CHAIN");
    return (e && strcmp(e, "householder") == 0) ? 16 : 0;
  }();
  return f;
}

// Kernel flag 32 (opt-in, JQ_TSQR_REDUCERS=1): the ws2 leaf's spare warps reduce the
// trailing tiles (reducer warps) when they have no side scan to run.  Measured slower at
// C4 (175.1 vs 169.5 ms): the reducers sit on SM sub-partition 0 with the chain, whose
// lookahead then publishes V later, and the data warps wait on two V barriers per panel.
// JQ_TSQR_PROBE_NOPREP=1 (flag 128): the loader skips its transform -- WRONG results,
// a timing probe of how much the loader's work slows the chain on its sub-partition.
static int probe_flag() {
  static const int f = [] {
    const char* e = getenv("JQ_TSQR_PROBE_NOPREP");
    return (e && e[0] == '1') ? 128 : 0;
  }();
  return f;
}
// JQ_TSQR_REDUCERS=chain (flag 64): the chain warp reduces every trailing tile itself.
static int reducer_flag(int nspare, const SideScan& side) {
  static const int mode = [] {
    const char* e = getenv("JQ_TSQR_REDUCERS");
    if (!e) return 0;
    if (strcmp(e, "chain") == 0) return 64;
    return e[0] == '1' ? 32 : 0;
  }();
  if (mode == 64) return 64;
  return (mode == 32 && nspare > 0 && side.x == nullptr) ? 32 : 0;
}

template <class C, class Src, bool COMBINE>
static int launch_tsqr(jq_ctx* ctx, int grid, const Src& src, int64_t rows_per_cta,
                       int64_t total_rows, const double* r_init, int64_t init_count, double* r_out,
                       int use_tma) {
  auto kern = tsqr_kernel<C, Src, COMBINE>;
  JQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
  // JQ_TSQR_EXPLICIT=1: every panel takes the explicit (row data) path (tests / A-B timing)
  static const bool explicit_panels = [] {
    const char* e = getenv("JQ_TSQR_EXPLICIT");
    return e && e[0] == '1';
  }();
  if (explicit_panels) use_tma |= 2;
  // JQ_TSQR_STAGED=1: chunks staged through shared memory (TMA + in-place transform) also
  // where the direct register load applies (A/B timing and tests)
  static const bool staged = [] {
    const char* e = getenv("JQ_TSQR_STAGED");
    return e && e[0] == '1';
  }();
  if (staged) use_tma |= 256;
  use_tma |= chain_flag();
  kern<<<grid, C::THREADS, C::SMEM, ctx->stream>>>(src, rows_per_cta, total_rows, r_init,
                                                   init_count, r_out, use_tma);
  JQ_CHECK_LAUNCH(ctx);
  return JQ_OK;
}

// Binary-tree combine of `count` NP x NP factors in `a` (ping-pong with `b`);
// returns a pointer to the final factor.
template <class C>
static int tree_combine(jq_ctx* ctx, double* a, double* b, int64_t count, double** result) {
  while (count > 1) {
    int64_t half = (count + 1) / 2;
    DenseSrc ds{nullptr, C::NP, C::NP};
    JQ_TRY((launch_tsqr<C, DenseSrc, true>(ctx, (int)half, ds, 0, 0, a, count, b, 1)));
    std::swap(a, b);
    count = half;
  }
  *result = a;
  return JQ_OK;
}

// Both sides' trees in the same launches (footnote variant): stacks a0 and a1 of k
// elements each (one level = one launch of 2 ceil(k/2) CTAs); tmp holds
// 2 * 2 * ceil(k/2) factors.  Same pairing per stack as tree_combine, so the same bits.
template <class C>
static int tree_combine_pair(jq_ctx* ctx, const double* a0, const double* a1, int64_t k, double* tmp,
                             const double** r0, const double** r1) {
  const size_t nn = size_t(C::NP) * C::NP;
  double* t[2] = {tmp, tmp + 2 * size_t((k + 1) / 2) * nn};
  int w = 0;
  while (k > 1) {
    const int64_t half = (k + 1) / 2;
    DenseSrc ds{a1, C::NP, C::NP};
    JQ_TRY((launch_tsqr<C, DenseSrc, true>(ctx, (int)(2 * half), ds, k, 0, a0, 0, t[w], 1)));
    a0 = t[w];
    a1 = t[w] + half * nn;
    w ^= 1;
    k = half;
  }
  *r0 = a0;
  *r1 = a1;
  return JQ_OK;
}

size_t tsqr_pair_ws_bytes(int64_t n, int sms) {
  const int64_t np = n <= 16 ? 16 : n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : 256;
  return 2 * ws_bytes(size_t(2 * (2 * sms + 1)) * np * np, 8);
}

size_t tsqr_ws_bytes(int64_t rows, int64_t n, int sms) {
  if (n > 256) return wide_tsqr_ws_bytes(rows, n, sms);
  int np = np_for(n);
  if (np < 0) return 0;
  int64_t leaves = std::max<int64_t>(1, std::min<int64_t>(int64_t(sms) * 32, cdiv(rows, 32) + 16));
  return 2 * ws_bytes(size_t(leaves) * np * np, sizeof(double)) + ws_bytes(size_t(np) * np, 8);
}

size_t figaro_tsqr_ws_bytes(int64_t m1, int64_t m2, int64_t n, int sms) {
  return tsqr_ws_bytes(m1 + m2 + TILE_ROWS, n, sms);
}

// carry-free leaves: the leaf's row block size goes into the source (FigaroSrc only)
template <class Src>
static Src with_block(const Src& s, int64_t) { return s; }
static FigaroSrc with_block(const FigaroSrc& s, int64_t rows_per_cta) {
  FigaroSrc t = s;
  if (t.fa.blk_sums) t.fa.blk_rows = rows_per_cta;
  return t;
}

// room behind the leaves for the between-block row elements (block_stack_layout)
template <class Src>
static int64_t block_extra(const Src&, int64_t, int) { return 0; }
static int64_t block_extra(const FigaroSrc& s, int64_t leaves, int np) {
  return s.fa.blk_sums ? 2 * cdiv(leaves, np) + 2 : 0;
}

template <class C, class Src>
static int run_stream(jq_ctx* ctx, const Src& src_in, int64_t vrows, int64_t align, int n,
                      bool canonical, double* r_out, int use_tma, LeafSet* defer = nullptr) {
  align = std::max<int64_t>(align, C::K);
  if (align % C::K) return fail(JQ_E_INVALID, "row alignment must be a multiple of the TSQR chunk");
  int64_t max_leaves = int64_t(ctx->sms) * ctas_per_sm<C, Src>();
  int64_t units = std::max<int64_t>(1, cdiv(vrows, align));
  int64_t leaves = std::min(max_leaves, units);
  int64_t rows_per_cta = cdiv(units, leaves) * align;
  leaves = std::max<int64_t>(1, cdiv(vrows, rows_per_cta));
  const Src src = with_block(src_in, rows_per_cta);
  const int64_t cap = leaves + block_extra(src, leaves, C::NP);
  double* a = ws_alloc<double>(ctx, size_t(cap) * C::NP * C::NP);
  double* b = ws_alloc<double>(ctx, size_t((cap + 1) / 2) * C::NP * C::NP + 1);
  if (!a || !b) return fail(JQ_E_OOM, "workspace exhausted (TSQR leaves)");
  ctx->timing.tsqr_ctas += leaves;
  ctx->timing.reduced_rows += vrows;
  if (ctx->record_tsqr_events) stage_event(ctx, 3);
  JQ_TRY(segscan_tiles(ctx, src.side_job()));  // this leaf has no spare warps for it
  JQ_TRY((launch_tsqr<C, Src, false>(ctx, (int)leaves, src, rows_per_cta, vrows, nullptr, 0, a, use_tma)));
  if (defer) {
    *defer = LeafSet{a, b, leaves, C::NP, n, rows_per_cta};
    return JQ_OK;
  }
  if (ctx->record_tsqr_events) stage_event(ctx, 4);
  double* fin = nullptr;
  JQ_TRY(tree_combine<C>(ctx, a, b, leaves, &fin));
  finalize_r_kernel<<<(int)cdiv(int64_t(n) * n, 256), 256, 0, ctx->stream>>>(fin, C::NP, n, canonical, r_out);
  JQ_CHECK_LAUNCH(ctx);
  if (ctx->record_tsqr_events) stage_event(ctx, 5);
  return JQ_OK;
}

// Leaf kernel for NP <= 128: warp-specialised tsqr_ws2_kernel (default; direct loads for
// NP = 64 / 128, a staged loader warp for NP <= 32) or the CTA-wide
// tsqr_kernel (JQ_TSQR_IMPL=cta, for A/B timing and tests); NP = 256 always CTA-wide.
static int leaf_impl() {
  static const int w = [] {
    const char* e = getenv("JQ_TSQR_IMPL");
    return (e && e[0] == 'c') ? 2 : 0;
  }();
  return w;
}

template <class CS, class Src>
static int run_stream_ws(jq_ctx* ctx, const Src& src_in, int64_t vrows, int64_t align, int n,
                         bool canonical, double* r_out, int use_tma, LeafSet* defer = nullptr) {
  using C = Cfg<CS::NP>;  // tree combine
  static int occ = [] {
    int o = 0;
    auto k = tsqr_ws2_kernel<CS, Src>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CS::SMEM);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k, CS::THREADS, CS::SMEM) != cudaSuccess) {
      cudaGetLastError();
      o = 1;
    }
    if (const char* e = getenv("JQ_TSQR_CTAS_PER_SM")) o = std::min(o, atoi(e));
    return std::max(1, o);
  }();
  static const bool explicit_panels = [] {
    const char* e = getenv("JQ_TSQR_EXPLICIT");
    return e && e[0] == '1';
  }();
  static const int debug_flags = [] {  // JQ_TSQR_DEBUG=8: ignore %warpid (fallback role layout; tests)
    const char* e = getenv("JQ_TSQR_DEBUG");
    int f = e ? atoi(e) & 8 : 0;
    // JQ_TSQR_PREFETCH=none | whole: the direct-load leaf's L2 prefetch of the next chunk
    // off / as one bulk prefetch (default: 32 pieces)
    const char* pf = getenv("JQ_TSQR_PREFETCH");
    if (pf && strcmp(pf, "none") == 0) f |= 1024;
    if (pf && strcmp(pf, "whole") == 0) f |= 2048;
    return f;
  }();
  align = std::max<int64_t>(align, 8);
  int64_t max_ctas = int64_t(ctx->sms) * occ;
  int64_t units = std::max<int64_t>(1, cdiv(vrows, align));
  int64_t ctas = std::min(max_ctas, units);
  int64_t rows_per_cta = cdiv(units, ctas) * align;
  ctas = std::max<int64_t>(1, cdiv(vrows, rows_per_cta));
  const Src src = with_block(src_in, rows_per_cta);
  const int64_t cap = ctas + block_extra(src, ctas, C::NP);
  double* a = ws_alloc<double>(ctx, size_t(cap) * C::NP * C::NP);
  double* b = ws_alloc<double>(ctx, size_t((cap + 1) / 2) * C::NP * C::NP + 1);
  if (!a || !b) return fail(JQ_E_OOM, "workspace exhausted (TSQR leaves)");
  ctx->timing.tsqr_ctas += ctas;
  ctx->timing.reduced_rows += vrows;
  if (ctx->record_tsqr_events) stage_event(ctx, 3);
  if (CS::NSPARE == 0) JQ_TRY(segscan_tiles(ctx, src.side_job()));  // else the spare warps run it
  auto kern = tsqr_ws2_kernel<CS, Src>;
  JQ_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CS::SMEM));
  kern<<<(int)ctas, CS::THREADS, CS::SMEM, ctx->stream>>>(src, rows_per_cta, vrows, a,
                                                          (use_tma ? 1 : 0) | (explicit_panels ? 2 : 0) | debug_flags |
                                                              chain_flag() | reducer_flag(CS::NSPARE, src.side_job()) |
                                                              probe_flag());
  JQ_CHECK_LAUNCH(ctx);
  if (defer) {
    *defer = LeafSet{a, b, ctas, C::NP, n, rows_per_cta};
    return JQ_OK;
  }
  if (ctx->record_tsqr_events) stage_event(ctx, 4);
  double* fin = nullptr;
  JQ_TRY(tree_combine<C>(ctx, a, b, ctas, &fin));
  finalize_r_kernel<<<(int)cdiv(int64_t(n) * n, 256), 256, 0, ctx->stream>>>(fin, C::NP, n, canonical, r_out);
  JQ_CHECK_LAUNCH(ctx);
  if (ctx->record_tsqr_events) stage_event(ctx, 5);
  return JQ_OK;
}

// NP = 128 warp-specialised leaf: 12 warps (168 registers), 9 data warps x 16 rows (144-row
// chunks, three data warps per SM sub-partition: C5 TSQR 5.86 ms, dense C4 642 ms) by default;
// JQ_TSQR_WS128=kw24: 8 warps, 6 data warps x 24 rows (5.93 / 691 ms); =kw16: 8 warps, 6 x 16
// rows (6.93 / 828 ms: the chain's per-panel cost over fewer rows).  (16 warps with 12 data
// warps x 8 rows at 128 registers: 7.02 ms.)
static int ws128_cfg() {
  static const int c = [] {
    const char* e = getenv("JQ_TSQR_WS128");
    return (e && strcmp(e, "kw16") == 0) ? 1 : (e && strcmp(e, "kw24") == 0) ? 2 : 0;
  }();
  return c;
}

// N = 32 warp-specialised leaf: 12 data warps x 40 rows (480-row chunks; C3 TSQR 5.46 vs
// 5.82 ms for 384-row chunks, the chain's per-panel cost over more rows) by default;
// JQ_TSQR_WS32=kw32: x 32 rows (A/B).
static int ws32_cfg() {
  static const int c = [] {
    const char* e = getenv("JQ_TSQR_WS32");
    return (e && strcmp(e, "kw32") == 0) ? 1 : 0;
  }();
  return c;
}

// N = 64: JQ_TSQR_WS64=w8 -- direct loads with 8 warps, 6 data warps x 48 rows (A/B)
static bool ws64_w8() {
  static const bool on = [] {
    const char* e = getenv("JQ_TSQR_WS64");
    return e && strcmp(e, "w8") == 0;
  }();
  return on;
}
// N = 64: JQ_TSQR_WS64=staged -- the 16-warp leaf with a loader warp (A/B, tests)
static bool ws64_staged() {
  static const bool on = [] {
    const char* e = getenv("JQ_TSQR_WS64");
    return e && strcmp(e, "staged") == 0;
  }();
  return on;
}

template <class Src>
static int dispatch_stream(jq_ctx* ctx, const Src& src, int64_t vrows, int64_t align, int n,
                           bool canonical, double* r_out, int use_tma, LeafSet* defer = nullptr) {
  switch (np_for(n)) {
    case 16:
      // (12 x 64-row data warps measured the same at C2: 0.638 ms either way)
      if (leaf_impl() == 0)
        return run_stream_ws<CfgS<16, 16, 12, 1, 32>>(ctx, src, vrows, align, n, canonical, r_out, use_tma, defer);
      return run_stream<Cfg<16>>(ctx, src, vrows, align, n, canonical, r_out, use_tma, defer);
    case 32:
      if (leaf_impl() == 0) {
        if (ws32_cfg() == 1)
          return run_stream_ws<CfgS<32, 16, 12, 1, 32>>(ctx, src, vrows, align, n, canonical, r_out, use_tma, defer);
        return run_stream_ws<CfgS<32, 16, 12, 1, 40>>(ctx, src, vrows, align, n, canonical, r_out, use_tma, defer);
      }
      return run_stream<Cfg<32>>(ctx, src, vrows, align, n, canonical, r_out, use_tma, defer);
    case 64:
      // default: warp-specialised with direct loads, 16 warps (128 registers), 12 data warps x
      // 24 rows (288-row chunks; C4 127.4 ms vs 144.3 for the staged 16-warp leaf -- the chain
      // alone on SMSP 0 and 1.5x the rows per panel chain -- and 131.9 for 8 warps with 6 x 48
      // rows, JQ_TSQR_WS64=w8: four data warps per SMSP hide the DMMA latency better).
      // JQ_TSQR_WS64=staged: the staged leaf with the loader warp (12 data warps x 16 rows).
      // (A staged 8-warp leaf with 6 x 40 rows was slower: 155.9 ms.)
      if constexpr (Src::DIRECT) {
        if (leaf_impl() == 0 && ws64_w8())
          return run_stream_ws<CfgS<64, 8, 6, 1, 48, true>>(ctx, src, vrows, align, n, canonical, r_out, use_tma,
                                                            defer);
        if (leaf_impl() == 0 && !ws64_staged())
          return run_stream_ws<CfgS<64, 16, 12, 1, 24, true>>(ctx, src, vrows, align, n, canonical, r_out, use_tma,
                                                              defer);
      }
      if (leaf_impl() == 0) return run_stream_ws<CfgS<64>>(ctx, src, vrows, align, n, canonical, r_out, use_tma, defer);
      return run_stream<Cfg<64>>(ctx, src, vrows, align, n, canonical, r_out, use_tma, defer);
    case 128:
      // warp-specialised with direct loads: 12 data warps x 8 rows (96-row chunks) off the
      // chain's SM sub-partition; the staged variant (loader warp + raw-row buffer beside the
      // 70 KB R) only fitted 64-row chunks and was slower than the CTA-wide kernel
      if constexpr (Src::DIRECT) {
        if (leaf_impl() == 0) {
          if (ws128_cfg() == 1)
            return run_stream_ws<CfgS<128, 8, 6, 1, 16, true>>(ctx, src, vrows, align, n, canonical, r_out, use_tma,
                                                               defer);
          if (ws128_cfg() == 2)
            return run_stream_ws<CfgS<128, 8, 6, 1, 24, true>>(ctx, src, vrows, align, n, canonical, r_out, use_tma,
                                                               defer);
          return run_stream_ws<CfgS<128, 12, 9, 1, 16, true>>(ctx, src, vrows, align, n, canonical, r_out, use_tma,
                                                              defer);
        }
      }
      return run_stream<Cfg<128>>(ctx, src, vrows, align, n, canonical, r_out, use_tma, defer);
    case 256: return run_stream<Cfg<256>>(ctx, src, vrows, align, n, canonical, r_out, use_tma, defer);
  }
  return fail(JQ_E_INVALID, "column count above 256 is not supported by the TSQR kernels");
}

// the tree + finalize of deferred leaf sets: both in shared launches when they have the
// same width and leaf count, else one after the other
template <class C>
static int finish_pair_np(jq_ctx* ctx, const LeafSet& x, const LeafSet& y, double* tmp, double* rx, double* ry) {
  const double *fx = nullptr, *fy = nullptr;
  if (x.count == y.count && tmp) {
    JQ_TRY(tree_combine_pair<C>(ctx, x.leaves, y.leaves, x.count, tmp, &fx, &fy));
  } else {
    double* f = nullptr;
    JQ_TRY(tree_combine<C>(ctx, x.leaves, x.tmp, x.count, &f));
    fx = f;
    JQ_TRY(tree_combine<C>(ctx, y.leaves, y.tmp, y.count, &f));
    fy = f;
  }
  finalize_r_kernel<<<(int)cdiv(int64_t(x.n) * x.n, 256), 256, 0, ctx->stream>>>(fx, C::NP, x.n, false, rx);
  JQ_CHECK_LAUNCH(ctx);
  finalize_r_kernel<<<(int)cdiv(int64_t(y.n) * y.n, 256), 256, 0, ctx->stream>>>(fy, C::NP, y.n, false, ry);
  JQ_CHECK_LAUNCH(ctx);
  return JQ_OK;
}

template <class C>
static int finish_one(jq_ctx* ctx, const LeafSet& x, double* rx) {
  double* f = nullptr;
  JQ_TRY(tree_combine<C>(ctx, x.leaves, x.tmp, x.count, &f));
  finalize_r_kernel<<<(int)cdiv(int64_t(x.n) * x.n, 256), 256, 0, ctx->stream>>>(f, C::NP, x.n, false, rx);
  JQ_CHECK_LAUNCH(ctx);
  return JQ_OK;
}

static int finish_np(jq_ctx* ctx, const LeafSet& x, double* rx) {
  switch (x.np) {
    case 16: return finish_one<Cfg<16>>(ctx, x, rx);
    case 32: return finish_one<Cfg<32>>(ctx, x, rx);
    case 64: return finish_one<Cfg<64>>(ctx, x, rx);
    case 128: return finish_one<Cfg<128>>(ctx, x, rx);
    case 256: return finish_one<Cfg<256>>(ctx, x, rx);
  }
  return fail(JQ_E_INVALID, "bad leaf width");
}

int figaro_tsqr_leaves(jq_ctx* ctx, const FigaroArgs& fa, LeafSet* out) {
  FigaroSrc src;
  src.fa = fa;
  src.m1pad = cdiv(fa.m1, TILE_ROWS) * TILE_ROWS;
  src.n = (int)(fa.n1 + fa.n2);
  int64_t vrows = src.m1pad + fa.m2;
  const int tma = ((reinterpret_cast<uintptr_t>(fa.a) | reinterpret_cast<uintptr_t>(fa.b)) & 15) == 0;
  // carry-free leaves (blk_sums) start their prefix from zero, so a leaf's row block need
  // not begin on a scan tile: finer blocks balance the grid (C5: 140 -> 148 leaves)
  const int64_t align = (fa.blk_sums && fa.m1 == 0 && !getenv("JQ_LEAF_TILE_ALIGN")) ? 8 : TILE_ROWS;
  return dispatch_stream(ctx, src, std::max<int64_t>(vrows, 1), align, src.n, false, nullptr, tma, out);
}

int tsqr_finish_pair(jq_ctx* ctx, const LeafSet& x, const LeafSet& y, double* rx, double* ry) {
  if (x.np != y.np) {
    JQ_TRY(finish_np(ctx, x, rx));
    return finish_np(ctx, y, ry);
  }
  double* tmp = x.count == y.count ? ws_alloc<double>(ctx, 4 * size_t((x.count + 1) / 2) * x.np * x.np) : nullptr;
  switch (x.np) {
    case 16: return finish_pair_np<Cfg<16>>(ctx, x, y, tmp, rx, ry);
    case 32: return finish_pair_np<Cfg<32>>(ctx, x, y, tmp, rx, ry);
    case 64: return finish_pair_np<Cfg<64>>(ctx, x, y, tmp, rx, ry);
    case 128: return finish_pair_np<Cfg<128>>(ctx, x, y, tmp, rx, ry);
    case 256: return finish_pair_np<Cfg<256>>(ctx, x, y, tmp, rx, ry);
  }
  return fail(JQ_E_INVALID, "bad leaf width");
}

int tsqr_dense_dev(jq_ctx* ctx, const double* m, int64_t rows, int64_t cols, double* r_out,
                   bool canonical) {
  if (cols > 256) return wide_tsqr_dev(ctx, m, rows, cols, r_out, canonical);  // jq_wide.cu
  DenseSrc src{m, rows, cols};
  const int tma = (reinterpret_cast<uintptr_t>(m) & 15) == 0;
  return dispatch_stream(ctx, src, std::max<int64_t>(rows, 1), 64, (int)cols, canonical, r_out, tma);
}

int join_tsqr_dev(jq_ctx* ctx, const JoinArgs& ja, double* r_out, bool canonical) {
  JoinSrc src;
  src.m = nullptr;
  src.rows = ja.rows;
  src.cols = ja.n1 + ja.n2;
  src.ja = ja;
  return dispatch_stream(ctx, src, std::max<int64_t>(ja.rows, 1), 64, (int)(ja.n1 + ja.n2), canonical, r_out, 0);
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
  if (n <= 512) return wide_tsqr_dev(ctx, rs, count * n, n, r_out, canonical);  // the stack as rows
  return fail(JQ_E_INVALID, "column count above 512 is not supported by the TSQR kernels");
}

int figaro_tsqr_dev(jq_ctx* ctx, const FigaroArgs& fa, double* r_out, bool canonical) {
  FigaroSrc src;
  src.fa = fa;
  src.m1pad = cdiv(fa.m1, TILE_ROWS) * TILE_ROWS;
  src.n = (int)(fa.n1 + fa.n2);
  int64_t vrows = src.m1pad + fa.m2;
  const int tma = ((reinterpret_cast<uintptr_t>(fa.a) | reinterpret_cast<uintptr_t>(fa.b)) & 15) == 0;
  return dispatch_stream(ctx, src, std::max<int64_t>(vrows, 1), TILE_ROWS, src.n, canonical, r_out, tma);
}

int canonicalize_dev(jq_ctx* ctx, const double* r, int64_t n, double* out) {
  canonicalize_kernel<<<(int)cdiv(n * n, 256), 256, 0, ctx->stream>>>(r, (int)n, out);
  JQ_CHECK_LAUNCH(ctx);
  return JQ_OK;
}

}  // namespace jq

#ifdef JQ_KTIME
extern "C" JQ_API int jq_debug_trace(long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, jq::g_trace, sizeof(long long) * 4096);
  if (reset) {
    static long long z[4096];
    cudaMemcpyToSymbol(jq::g_trace, z, sizeof(z));
  }
  return 0;
}
extern "C" JQ_API int jq_debug_gram_fail(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, jq::g_gram_fail, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(jq::g_gram_fail, z, sizeof(z));
  }
  return 0;
}
extern "C" JQ_API int jq_debug_ktime(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, jq::g_ktime, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(jq::g_ktime, z, sizeof(z));
  }
  return 0;
}
#endif
