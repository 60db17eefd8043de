// Warp-specialised streaming-TSQR leaf (NP <= 128), included by jq_tsqr.cu.
//
// Measured on B200 (tools/microbench/gchain.cu): the 8-step Householder chain of a
// panel takes ~3.5k cycles alone but ~8.6k when other warps issue DMMA on the SAME
// SM sub-partition (the FP64 datapath is shared per SMSP), and is unaffected by DMMA
// on the other three.  A co-resident second CTA has its warps rotated by one SMSP
// (tools/microbench/warpid.cu).  So the CTA (16 warps, one per SM) reads %warpid and
// gives two of its warps on SMSP 0 the latency-bound roles:
//   * the CHAIN warp: the Gram-panel chain (factor_panel_gram: T, M', R rows), then
//     the update of the next tile (the lookahead tile) and its Gram, derived from
//     partials -- the whole critical path;
//   * the LOADER warp(s): TMA of the next chunk's raw rows and the Claim-1 / tail
//     transform in place (prep_warp; for NP <= 32 three loader warps split the rows:
//     segment sums, carries, transform), one chunk ahead of the data warps;
// and the twelve warps on SMSPs 1-3 hold the chunk (DW x KW rows in registers) and
// do all bulk DMMA work: partials, the reduces of the other tiles and the applies.
// The role assignment only moves work between warps: results do not depend on it
// (row ownership and every reduction order follow the data-warp index).
//
// Synchronisation: named barrier BAR_ALL (chain + data warps) once per panel (plus F / D
// after an explicit-fallback panel), BAR_DATA (data warps) inside the update, mbarriers
// READY (loader -> data) and FREE (data -> loader) once per chunk, VREADY
// (chain -> data) once per panel, and the loader's TMA mbarrier.

// WARPS_ warps per CTA, DW_ of them data warps (the warps off SM sub-partition 0),
// MINB_ CTAs per SM.  <NP, 16, 12, 1>: one CTA per SM, 12 data warps (K = 192 rows
// per chain), two spare SMSP-0 warps.  (Two CTAs of 8 warps, 6 data warps each, were
// measured 5% slower: their chains share SMSP 0 and the lookahead DMMAs of one CTA
// queue behind the other's bulk update.)
// DIRECT_: the data warps load their rows straight from global memory (load_direct; no
// loader warp, no raw-row buffer) -- the NP = 128 leaf, whose R leaves no room for a
// staged chunk beside the partials.
template <int NP_, int WARPS_ = 16, int DW_ = 12, int MINB_ = 1, int KW_ = 16, bool DIRECT_ = false>
struct CfgS {
  static constexpr bool DIRECT = DIRECT_;
  static constexpr int NP = NP_;
  static constexpr int NLT = NP / 8;
  static constexpr int WARPS = WARPS_;
  static constexpr int THREADS = WARPS * 32;
  static constexpr int DW = DW_;             // data warps
  static constexpr int KW = KW_;             // rows per data warp
  static constexpr int KWT = KW / 8;
  static constexpr int K = DW * KW;          // chunk rows
  static constexpr bool R_SMEM = true;
  static constexpr int MIN_CTAS = MINB_;
  __host__ __device__ static constexpr int rp_off(int p) { return 8 * (p * (NP + 2) - 4 * p * (p - 1)); }
  static constexpr int LDT = 10;
  static constexpr int LDYT = KW + 2;
  static constexpr int RAW = DIRECT ? 0 : K * NP;  // one whole chunk of raw rows
  static constexpr int OFF_R = 0;
  static constexpr int SZ_R = rp_off(NLT);
  static constexpr int OFF_RAW = OFF_R + SZ_R;
  static constexpr int OFF_YT = OFF_RAW + RAW;            // [DW][8][LDYT]  X^T (or Y^T) of the panel
  static constexpr int SZ_YT = 8 * LDYT;
  static constexpr int OFF_ZP = OFF_YT + DW * SZ_YT;      // [DW][NLT][64]  Gram / Z partials
  static constexpr int OFF_WS = OFF_ZP + DW * NLT * 64;   // [NLT][64]      -V^T per tile
  static constexpr int OFF_T = OFF_WS + NLT * 64;         // [2][8 x LDT]   T by panel parity
  static constexpr int OFF_M = OFF_T + 16 * LDT;          // [2][8 x LDT]   M' by panel parity
  static constexpr int OFF_U = OFF_M + 16 * LDT;          // explicit fallback: U, taus, scales, partials
  static constexpr int OFF_TAU = OFF_U + 64;
  static constexpr int OFF_SC = OFF_TAU + 8;
  static constexpr int OFF_P = OFF_SC + 8;                // [2][DW][8]
  static constexpr int OFF_LD = OFF_U + (80 + 2 * DW * 8 > 16 * LDT + 48 ? 80 + 2 * DW * 8 : 16 * LDT + 48);
  // ^ loader per-row scalars (past the partials [2][DW][8] and factor_panel_chol's scratch): c1, c2, mode [3][K], then
  // the multi-loader transform's packed {c1, c2, keep, w} per row [K][4] (B-part chunks; it
  // aliases the scalars, which only A-part chunks use)
  static constexpr int OFF_S = OFF_LD + (NP <= 32 ? 4 : 3) * K;  // loader running prefix (the packed
  // coefficients are only used by the multi-loader transform, NP <= 32)
  static constexpr int OFF_FLAG = OFF_S + NP;             // [2] chain accepted, by parity
  static constexpr int OFF_GP = OFF_FLAG + 2;             // [DW][64] C^T C partials of the next tile (ws2)
  static constexpr int OFF_GD = OFF_GP + DW * 64;         // [DW][64] direct Gram partials (ws2)
  static constexpr int NLOAD = DIRECT ? 0 : NP <= 32 ? 3 : 1;  // loader warps: narrow leaves are loader-bound; at
  // NP = 64 two extra active warps on SMSP 0 slow the chain more than they help (4.62 vs 4.47 ms)
  static constexpr int NSPARE = WARPS - 1 - NLOAD - DW;  // spare warps: the side scan (FigaroSrc::side_scan)
  static constexpr int OFF_LSR = OFF_GD + DW * 64;        // [NLOAD][2][64] loader segment sums
  static constexpr int OFF_ROLE = OFF_LSR + NLOAD * 128;  // WARPS ints: SMSP of each warp
  static constexpr int OFF_BAR = OFF_ROLE + WARPS / 2;    // mbarriers: TMA, READY, FREE, VREADY, VREADY2
  static constexpr int TOTAL = OFF_BAR + 5;
  static constexpr size_t SMEM = size_t(TOTAL) * sizeof(double);
  static_assert(SMEM <= (MIN_CTAS == 1 ? 227 : 113) * 1024, "shared memory per CTA");
  static_assert(NP <= 128, "loader transform assumes <= 128 columns per side");
  static_assert(OFF_LD - OFF_U >= 16 * LDT + 16 + 32, "factor_panel_chol scratch (U .. P)");
  static_assert(OFF_LD % 2 == 0, "16-byte aligned packed loader coefficients");
  static_assert(NP <= 32 || NLOAD <= 1, "the packed loader coefficients need the 4 K scratch");
  static_assert(NLT * DW * 32 + 2 * DW * NP <= DW * NLT * 64, "direct load: lo and wt inside the partials");
};

__device__ __forceinline__ void mbar_init_n(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}


#ifdef JQ_KTIME
__device__ long long g_trace[4096];
// (who, event) timestamps of CTA 0, lane 0, per-warp slots (no atomics on the path)
#define TR(who, ev) do { if (blockIdx.x == 0 && lane == 0 && tr_k < 600) { \
                           g_trace[(who) * 1365 + 2 * tr_k] = (ev); g_trace[(who) * 1365 + 2 * tr_k + 1] = clock64(); ++tr_k; } } while (0)
#else
#define TR(who, ev) do {} while (0)
#endif

constexpr int BAR_ALL = 1;   // chain + data warps
constexpr int BAR_DATA = 2;  // data warps
constexpr int BAR_LOAD = 3;  // loader warps
constexpr int BAR_GD = 4;    // chain + data warps: direct Gram after an explicit panel

// ------------------------------------------------------------------ the kernel (ws2)
// The chain warp also performs, right after B_p,
// the update of tile p+1 by panel p (S = sum of the (X^T C)^T partials, Z, W = T^T Z,
// R rows, V = M' W) and derives the Gram of the updated tile without touching its
// rows:  (C - X V)^T (C - X V) = C^T C - V^T S - S^T V + V^T (X^T X) V,  from the
// data warps' C^T C partials (computed one panel ahead), S, V and the panel's own
// Gram X^T X -- eight 8 x 8 DMMA products on SM sub-partition 0.  The data warps
// are then off the critical path: they apply V to tile p+1 when the chain signals it
// (mbarrier VREADY) and finish panel p's other tiles while the chain runs panel p+1.
// The cancellation guard starts from P = diag(C^T C) + diag(V^T X^T X V) (the scale of
// the rounding error of the derived Gram).  After an explicit-fallback panel the next
// Gram is taken directly from the updated rows (barrier D).
template <class C, class Src>
__global__ void __launch_bounds__(C::THREADS, C::MIN_CTAS)
tsqr_ws2_kernel(Src src, int64_t rows_per_cta, int64_t total_rows, double* __restrict__ r_out, int flags) {
  extern __shared__ __align__(16) double smem_dyn[];
  double* R = smem_dyn + C::OFF_R;
  double* raw = smem_dyn + C::OFF_RAW;
  double* Zp = smem_dyn + C::OFF_ZP;
  double* Ws = smem_dyn + C::OFF_WS;
  double* Gp = smem_dyn + C::OFF_GP;
  double* Gd = smem_dyn + C::OFF_GD;
  double* S = smem_dyn + C::OFF_S;
  double* scratch = smem_dyn + C::OFF_LD;
  volatile int* flag = reinterpret_cast<volatile int*>(smem_dyn + C::OFF_FLAG);  // integer compares: the
  // data warps' FP64 datapath is busy with DMMA
  int* role = reinterpret_cast<int*>(smem_dyn + C::OFF_ROLE);
  uint64_t* bar_tma = reinterpret_cast<uint64_t*>(smem_dyn + C::OFF_BAR);
  uint64_t* bar_ready = bar_tma + 1;
  uint64_t* bar_free = bar_tma + 2;
  uint64_t* bar_v = bar_tma + 3;
  uint64_t* bar_v2 = bar_tma + 4;  // reducer warps -> data warps (tiles q > p + 1)

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int64_t cta = blockIdx.x;
  const int64_t row_begin = cta * rows_per_cta;
  const int64_t row_end = min(total_rows, row_begin + rows_per_cta);
  constexpr int NALL = (C::DW + 1) * 32;  // chain + data warps
  // REDUCER warps (flags & 32: the spare warps have no side scan to run): they reduce the
  // tiles q > p + 1 of panel p (Z^T = R^T + S M', W^T = Z^T T, V^T = W^T M'^T) while the
  // chain does the lookahead tile p + 1 and the next panel, so the data warps only apply
  const bool red_warps = C::NSPARE > 0 && (flags & 32) && !(flags & 64);
  // flag 64: the CHAIN warp itself reduces the tiles q > p + 1 right after its lookahead
  const bool chain_red = (flags & 64) != 0;
  const bool use_red = red_warps || chain_red;  // data warps: apply-only protocol (VREADY2)
  const int NB = NALL + (red_warps ? C::NSPARE * 32 : 0);  // BAR_ALL: chain + data (+ reducer warps)
  int tr_k = 0;
  (void)tr_k;

  if (lane == 0) {
    unsigned wid;
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
    role[warp] = (int)(wid & 3);
  }
  for (int idx = tid; idx < C::SZ_R; idx += C::THREADS) R[idx] = 0.0;
  src.template begin<C>(S, row_begin);
  if (tid == 0) {
    mbar_init_n(bar_tma, 1);
    mbar_init_n(bar_ready, 1);
    mbar_init_n(bar_free, C::DW);
    mbar_init_n(bar_v, 1);
    mbar_init_n(bar_v2, (C::NSPARE > 0 && (flags & 32) && !(flags & 64)) ? C::NSPARE : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  // chain: the first warp on SMSP 0; loaders: the next NLOAD warps on SMSP 0; data
  // warps: the first DW warps elsewhere (any other layout falls back to chain 0, loaders
  // 1..NLOAD, data warps after them)
  int chain_w = -1, li = -1, nz = 0, ndata = 0;
  for (int w = 0; w < C::WARPS; ++w) {
    if (role[w] == 0) {
      if (nz == 0) chain_w = w;
      else if (nz <= C::NLOAD && w == warp) li = nz - 1;
      ++nz;
    } else {
      ++ndata;
    }
  }
  const bool mapped = !(flags & 8) && nz >= 1 + C::NLOAD && ndata >= C::DW;
  if (!mapped) {
    chain_w = 0;
    li = (warp >= 1 && warp <= C::NLOAD) ? warp - 1 : -1;
  }
  int d = -1;  // data-warp index
  {
    int k = 0;
    for (int w = 0; w < C::WARPS; ++w) {
      const bool data = mapped ? role[w] != 0 : (w >= 1 + C::NLOAD && w < 1 + C::NLOAD + C::DW);
      if (!data || k == C::DW) continue;
      if (w == warp) d = k;
      ++k;
    }
  }
  int red_i = -1;  // reducer index (spare warps when use_red)
  if (warp != chain_w && li < 0 && d < 0) {
    // spare warp: the tile pass of the other side's scan, if the host attached one
    int si = 0, zc = 0, dk = 0;
    for (int w = 0; w < warp; ++w) {
      bool busy;
      if (mapped) {
        busy = role[w] == 0 ? zc <= C::NLOAD : dk < C::DW;
        if (role[w] == 0) ++zc; else ++dk;
      } else {
        busy = w < 1 + C::NLOAD + C::DW;
      }
      si += busy ? 0 : 1;
    }
    if (!red_warps) {
      src.side_scan(si, C::NSPARE, lane);
      return;
    }
    red_i = si;
  }

  auto chunk_end = [&](int64_t r0) -> int64_t {
    int64_t e = r0 + C::K < row_end ? r0 + C::K : row_end;
    const int64_t lim = src.limit(r0);
    return e < lim ? e : lim;
  };
  auto chunk_rows = [&](int64_t r0, int64_t r1) -> int {
    const int64_t av = src.avail(r0);
    const int64_t nr = r1 - r0 < av ? r1 - r0 : av;
    return nr > 0 ? (int)nr : 0;
  };
  // sum of the DW partials of an 8 x 8 accumulator-layout matrix: all loads first, then a
  // fixed pairwise tree (deterministic, dependent depth log2(DW) instead of DW)
  auto sum_partials = [&](const double* base, int stride, double (&out)[2]) {
    double2 v[C::DW];
#pragma unroll
    for (int w = 0; w < C::DW; ++w) v[w] = *reinterpret_cast<const double2*>(base + w * stride + 2 * lane);
#pragma unroll
    for (int h = 1; h < C::DW; h <<= 1)
#pragma unroll
      for (int w = 0; w + h < C::DW; w += 2 * h) {
        v[w].x += v[w + h].x;
        v[w].y += v[w + h].y;
      }
    out[0] = v[0].x;
    out[1] = v[0].y;
  };

  if (red_i >= 0) {
    const int si = red_i;
    // ================= reducer warp si: tiles q = p + 2 + si, p + 2 + si + NSPARE, ...
    for (int64_t r0 = row_begin; r0 < row_end; r0 = chunk_end(r0)) {
      named_bar(BAR_ALL, NB);  // direct Gram partials of tile 0
#pragma unroll 1
      for (int p = 0; p < C::NLT; ++p) {
        const int par = p & 1, j0 = 8 * p;
        named_bar(BAR_ALL, NB);  // B_p
        if (flag[par] == 0) named_bar(BAR_ALL, NB);  // F_p: explicit T / M' of the panel
        if (p + 1 < C::NLT) {
          const double* Tc = smem_dyn + C::OFF_T + par * 8 * C::LDT;
          const double* Mc = smem_dyn + C::OFF_M + par * 8 * C::LDT;
          for (int q = p + 2 + si; q < C::NLT; q += C::NSPARE) {
            const int l0 = 8 * q;
            const int r0i = rix<C>(j0 + 2 * t, l0 + g), r1i = rix<C>(j0 + 2 * t + 1, l0 + g);
            double st[2];
            sum_partials(Zp + q * 64, C::NLT * 64, st);
            double zt[2] = {R[r0i], R[r1i]};
            dmma(zt, st[0], Mc[(2 * t) * C::LDT + g]);
            dmma(zt, st[1], Mc[(2 * t + 1) * C::LDT + g]);
            double wv[2] = {0.0, 0.0};
            dmma(wv, zt[0], Tc[(2 * t) * C::LDT + g]);
            dmma(wv, zt[1], Tc[(2 * t + 1) * C::LDT + g]);
            R[r0i] -= wv[0];
            R[r1i] -= wv[1];
            double vt[2] = {0.0, 0.0};
            dmma(vt, wv[0], Mc[g * C::LDT + 2 * t]);
            dmma(vt, wv[1], Mc[g * C::LDT + 2 * t + 1]);
            *reinterpret_cast<double2*>(Ws + q * 64 + 2 * lane) = make_double2(-vt[0], -vt[1]);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_v2);  // tiles q > p + 1 may be updated
        }
      }
    }
    named_bar(BAR_ALL, NB);  // R final
    return;
  }

  if (li >= 0) {
    // ================= loader warp(s): li == 0 fetches; all transform a row segment
    uint32_t ph_tma = 0, ph_free = 0;
    int64_t nchunk = 0;
    double* lsr = smem_dyn + C::OFF_LSR;
    for (int64_t r0 = row_begin; r0 < row_end; r0 = chunk_end(r0), ++nchunk) {
      const int64_t r1 = chunk_end(r0);
      const int nr = chunk_rows(r0, r1);
      const int rcol = src.rc(r0);
      const int nel = nr * rcol;
      if (li == 0) {
        if (nchunk > 0) {
          mbar_wait_idle(bar_free, ph_free);  // the loader sits next to the chain warp on SMSP 0
          ph_free ^= 1;
        }
        TR(2, 1);
        if (flags & 1) {
          if (lane == 0) bulk_fetch(bar_tma, raw, src.ptr(r0), uint32_t(nel) * 8u & ~15u);
          mbar_wait(bar_tma, ph_tma);
          ph_tma ^= 1;
          if ((nel & 1) && lane == 0) raw[nel - 1] = __ldg(src.ptr(r0) + nel - 1);
        } else {
          const double* p = src.ptr(r0);
          for (int e = lane; e < nel; e += 32) raw[e] = __ldg(p + e);
        }
        __syncwarp();
        TR(2, 2);
      }
      if (C::NLOAD == 1) {
        if (!(flags & 128)) src.template prep_warp<C>(raw, S, scratch, r0, nr, lane);  // 128: timing probe only
      } else {
        named_bar(BAR_LOAD, C::NLOAD * 32);  // raw rows of the chunk in shared memory
        if (li == 0) TR(2, 4);
        constexpr int NLD = C::NLOAD > 0 ? C::NLOAD : 1;
        const int i0 = li * C::K / NLD, i1 = (li + 1) * C::K / NLD;
        src.template seg_coeffs<C>(scratch, r0, nr, lane, i0, i1);
        __syncwarp();
        if (li == 0) TR(2, 5);
        double sub_l[SEG_SUB][2];
        bool sub_r[SEG_SUB][2];
        src.template seg_pass1<C>(raw, scratch, lsr + li * 128, r0, nr, lane, i0, i1, sub_l, sub_r);
        const double s_in0 = lane < C::NP ? S[lane] : 0.0, s_in1 = lane + 32 < C::NP ? S[lane + 32] : 0.0;
        if (li == 0) TR(2, 6);
        named_bar(BAR_LOAD, C::NLOAD * 32);  // segment sums published, S read by every segment
        if (li == 0) TR(2, 7);
        src.template seg_pass2<C>(raw, S, scratch, lsr, s_in0, s_in1, r0, nr, lane, i0, i1, li, C::NLOAD, sub_l,
                                  sub_r);
        named_bar(BAR_LOAD, C::NLOAD * 32);  // chunk transformed
      }
      TR(2, 3);
      if (li == 0 && lane == 0) mbar_arrive(bar_ready);
    }
    if (li == 0) src.finish(S, lane, 32);  // S final: prep_warp's __syncwarp / the last BAR_LOAD
    return;
  }

  if (warp == chain_w) {
    // ================= chain warp: the whole critical path
    for (int64_t r0 = row_begin; r0 < row_end; r0 = chunk_end(r0)) {
      named_bar(BAR_ALL, NB);  // direct Gram partials of tile 0
      double G[2];
      sum_partials(Gd, 64, G);
      double Pg = diag_of(G, lane);
#pragma unroll 1
      for (int p = 0; p < C::NLT; ++p) {
        const int par = p & 1, j0 = 8 * p;
        double* Tc = smem_dyn + C::OFF_T + par * 8 * C::LDT;
        double* Mc = smem_dyn + C::OFF_M + par * 8 * C::LDT;
        const double G0[2] = {G[0], G[1]};  // X^T X of panel p (before the chain)
        TR(0, 1);
        double Rb[2];
        // Cholesky panel; where its guard rejects (pivot cancellation) the reflector chain,
        // whose guard is looser (it never forms R_p^T R_p); then the explicit path
        bool ok = !(flags & 16) && factor_panel_chol<C>(G, Rb, R, j0, Tc, Mc, smem_dyn + C::OFF_U, lane, Pg);
        if (!ok) ok = factor_panel_gram<C>(G, Rb, R, j0, Tc, Mc, lane, Pg);
        ok = ok && !(flags & 2);
        if (ok) {
          if (2 * t >= g) R[rix<C>(j0 + g, j0 + 2 * t)] = Rb[0];
          if (2 * t + 1 >= g) R[rix<C>(j0 + g, j0 + 2 * t + 1)] = Rb[1];
        }
        if (lane == 0) flag[par] = ok ? 1 : 0;
        TR(0, 2);
        named_bar(BAR_ALL, NB);  // B_p: chain results out, data partials in
        TR(0, 3);
        if (!ok) named_bar(BAR_ALL, NB);  // F_p: explicit panel done by the data warps
        if (p + 1 < C::NLT) {
          const int q = p + 1, l0 = 8 * q;
          double cc[2] = {0.0, 0.0};
          if (ok) sum_partials(Gp, 64, cc);  // C^T C of tile q (read before VREADY frees Gp)
          double st[2];
          sum_partials(Zp + q * 64, C::NLT * 64, st);  // (X^T C_q)^T
          const int r0i = rix<C>(j0 + 2 * t, l0 + g), r1i = rix<C>(j0 + 2 * t + 1, l0 + g);
          double zt[2] = {R[r0i], R[r1i]};
          dmma(zt, st[0], Mc[(2 * t) * C::LDT + g]);
          dmma(zt, st[1], Mc[(2 * t + 1) * C::LDT + g]);
          double wv[2] = {0.0, 0.0};
          dmma(wv, zt[0], Tc[(2 * t) * C::LDT + g]);
          dmma(wv, zt[1], Tc[(2 * t + 1) * C::LDT + g]);
          R[r0i] -= wv[0];
          R[r1i] -= wv[1];
          double vt[2] = {0.0, 0.0};  // V^T = W^T M'^T
          dmma(vt, wv[0], Mc[g * C::LDT + 2 * t]);
          dmma(vt, wv[1], Mc[g * C::LDT + 2 * t + 1]);
          *reinterpret_cast<double2*>(Ws + q * 64 + 2 * lane) = make_double2(-vt[0], -vt[1]);
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_v);  // tile q may be updated
          TR(0, 4);
          if (chain_red) {
            // the other trailing tiles' reduces with panel p (independent: their DMMA
            // chains interleave), then VREADY2 -- before the Gram of the next panel, whose
            // explicit-path barrier the data warps only reach after these applies
            for (int q2 = q + 1; q2 < C::NLT; ++q2) {
              const int m0 = 8 * q2;
              const int s0i = rix<C>(j0 + 2 * t, m0 + g), s1i = rix<C>(j0 + 2 * t + 1, m0 + g);
              double st2[2];
              sum_partials(Zp + q2 * 64, C::NLT * 64, st2);
              double z2[2] = {R[s0i], R[s1i]};
              dmma(z2, st2[0], Mc[(2 * t) * C::LDT + g]);
              dmma(z2, st2[1], Mc[(2 * t + 1) * C::LDT + g]);
              double w2[2] = {0.0, 0.0};
              dmma(w2, z2[0], Tc[(2 * t) * C::LDT + g]);
              dmma(w2, z2[1], Tc[(2 * t + 1) * C::LDT + g]);
              R[s0i] -= w2[0];
              R[s1i] -= w2[1];
              double v2[2] = {0.0, 0.0};
              dmma(v2, w2[0], Mc[g * C::LDT + 2 * t]);
              dmma(v2, w2[1], Mc[g * C::LDT + 2 * t + 1]);
              *reinterpret_cast<double2*>(Ws + q2 * 64 + 2 * lane) = make_double2(-v2[0], -v2[1]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_v2);
          }
          if (ok) {
            // Gram of the updated tile: C^T C - V^T S - S^T V + (V^T G0) V   (all ^T as stored)
            double gn[2] = {cc[0], cc[1]};
            dmma(gn, -vt[0], st[0]);  // - V^T S   : A = V^T (k-perm), B = S^T rows
            dmma(gn, -vt[1], st[1]);
            dmma(gn, -st[0], vt[0]);  // - S^T V
            dmma(gn, -st[1], vt[1]);
            double e2[2] = {0.0, 0.0};  // V^T G0
            dmma(e2, vt[0], G0[0]);
            dmma(e2, vt[1], G0[1]);
            double e3[2] = {0.0, 0.0};  // (V^T G0) V
            dmma(e3, e2[0], vt[0]);
            dmma(e3, e2[1], vt[1]);
            G[0] = gn[0] + e3[0];
            G[1] = gn[1] + e3[1];
            const double dcc = diag_of(cc, lane), de3 = diag_of(e3, lane);
            Pg = dcc + de3;
            TR(0, 5);
          } else {
            named_bar(BAR_GD, NALL);  // D_q: direct Gram partials of the updated tile
            sum_partials(Gd, 64, G);
            Pg = diag_of(G, lane);
          }
        }
      }
    }
    named_bar(BAR_ALL, NB);  // R final
  } else {
    // ================= data warps
    double* Ytw = smem_dyn + C::OFF_YT + d * C::SZ_YT;
    double* U = smem_dyn + C::OFF_U;
    double* taus = smem_dyn + C::OFF_TAU;
    double* scs = smem_dyn + C::OFF_SC;
    double* P = smem_dyn + C::OFF_P;
    double c[C::NLT][C::KWT][2];
    uint32_t ph_ready = 0, ph_v = 0, ph_v2 = 0;

    // (single DMMA accumulation chains: a final DADD would queue behind the other warps'
    // DMMAs in this SM sub-partition's FP64 datapath)
    auto gram_partial = [&](int q, double* dst) {  // (C_q^T C_q) partial of this warp's rows
#pragma unroll
      for (int qq = 0; qq < C::NLT; ++qq) {
        if (qq == q) {
          double z[2] = {0.0, 0.0};
#pragma unroll
          for (int it = 0; it < C::KWT; ++it) {
            dmma(z, c[qq][it][0], c[qq][it][0]);
            dmma(z, c[qq][it][1], c[qq][it][1]);
          }
          *reinterpret_cast<double2*>(dst + d * 64 + 2 * lane) = make_double2(z[0], z[1]);
        }
      }
    };

    for (int64_t r0 = row_begin; r0 < row_end; r0 = chunk_end(r0)) {
      const int64_t r1 = chunk_end(r0);
      const int nr = chunk_rows(r0, r1);
      const int rcol = src.rc(r0);
      if constexpr (C::DIRECT) {
        // the partials' buffer holds the load's scan state: free since B of the last panel
        // the next chunk into L2 meanwhile: by default 32 bulk prefetches (one per lane of
        // data warp 0); flag 2048: one bulk prefetch of the whole chunk; 1024: none
        if (d == 0 && (flags & 1) && !(flags & 1024) && r1 < row_end) {
          const int64_t r2 = chunk_end(r1);
          const int nr2 = chunk_rows(r1, r2);
          const uint32_t bytes = uint32_t(nr2) * uint32_t(src.rc(r1)) * 8u & ~15u;
          const char* base = reinterpret_cast<const char*>(src.ptr(r1));
          if (flags & 2048) {
            if (lane == 0) l2_prefetch(base, bytes);
          } else {
            const uint32_t piece = ((bytes + 31u) / 32u + 15u) & ~15u, off = uint32_t(lane) * piece;
            if (off < bytes) l2_prefetch(base + off, min(piece, bytes - off));
          }
        }
        if (d == 0) TR(1, 7);
        src.template load_direct<C, RowBar<C::DW, BAR_DATA>>(c, r0, nr, S, Zp, Zp + C::NLT * C::DW * 32, scratch,
                                                             d, lane, [&](int i) {
                                                               if (d == 0) TR(1, 10 + i);
                                                             });
        if (d == 0) TR(1, 8);
      } else {
        if (d == 0) TR(1, 7);
        mbar_wait(bar_ready, ph_ready);
        ph_ready ^= 1;
        if (d == 0) TR(1, 8);
#pragma unroll
        for (int q = 0; q < C::NLT; ++q) {
          const int l = q * 8 + g;
#pragma unroll
          for (int it = 0; it < C::KWT; ++it)
#pragma unroll
            for (int b = 0; b < 2; ++b)
              c[q][it][b] = src.template value<C>(raw, scratch, r0, d * C::KW + 8 * it + 2 * t + b, l, nr, rcol);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_free);
      }
      gram_partial(0, Gd);
      named_bar(BAR_ALL, NB);

      // fully unrolled over the panels: every "tile q > p" test becomes compile time, so
      // the applies / partials of different tiles are straight-line independent DMMA
      // chains the scheduler can interleave (C4 leaf 172.8 -> 138.7 ms; the runtime-p
      // loop left one predicated block per tile).  The chain warp's loop stays rolled
      // (unrolled it is slower: 190 ms, instruction-cache pressure on SMSP 0).
      // (static_for: at NP = 128 the compiler declines the 16-panel `#pragma unroll` and
      // issues every tile's DMMAs predicated, so each panel cost as much as the first)
      static_for<0, C::NLT>([&](auto pc) {
        constexpr int p = decltype(pc)::value;
        const int j0 = 8 * p, par = p & 1;
        const double* Tp = smem_dyn + C::OFF_T + (par ^ 1) * 8 * C::LDT;
        const double* Mp = smem_dyn + C::OFF_M + (par ^ 1) * 8 * C::LDT;
        if (p > 0) {
          if (!use_red) {
            // (3a) reduces of the tiles q > p with panel p-1 first: their inputs (partials,
            // T, M') are ready since B_{p-1}, so they overlap the chain warp's update of tile p
            for (int q = p + 1 + ((d - (p + 1)) % C::DW + C::DW) % C::DW; q < C::NLT; q += C::DW) {
              const int l0 = 8 * q;
              const int r0i = rix<C>(j0 - 8 + 2 * t, l0 + g), r1i = rix<C>(j0 - 8 + 2 * t + 1, l0 + g);
              double st[2];
              sum_partials(Zp + q * 64, C::NLT * 64, st);
              double zt[2] = {R[r0i], R[r1i]};
              dmma(zt, st[0], Mp[(2 * t) * C::LDT + g]);
              dmma(zt, st[1], Mp[(2 * t + 1) * C::LDT + g]);
              double wv[2] = {0.0, 0.0};
              dmma(wv, zt[0], Tp[(2 * t) * C::LDT + g]);
              dmma(wv, zt[1], Tp[(2 * t + 1) * C::LDT + g]);
              R[r0i] -= wv[0];
              R[r1i] -= wv[1];
              double vt[2] = {0.0, 0.0};
              dmma(vt, wv[0], Mp[g * C::LDT + 2 * t]);
              dmma(vt, wv[1], Mp[g * C::LDT + 2 * t + 1]);
              *reinterpret_cast<double2*>(Ws + q * 64 + 2 * lane) = make_double2(-vt[0], -vt[1]);
            }
            if (d == 0) TR(1, 2);
            named_bar(BAR_DATA, C::DW * 32);
            if (d == 0) TR(1, 3);
          }
          // B operands of the panel p-1 update (X^T or Y^T rows of this warp), loaded once
          // for every tile: keeps the data warps' shared-memory traffic low
          double yb[C::KWT][2];
#pragma unroll
          for (int it = 0; it < C::KWT; ++it) {
            yb[it][0] = Ytw[(2 * t) * C::LDYT + 8 * it + g];
            yb[it][1] = Ytw[(2 * t + 1) * C::LDYT + 8 * it + g];
          }
          if (use_red) {
            // (1) tile p with panel p-1 (V from the chain), then (3b) the tiles q > p (V from
            // the reducer warps)
            mbar_wait(bar_v, ph_v);
            ph_v ^= 1;
            if (d == 0) TR(1, 1);
#pragma unroll
            for (int q = 0; q < C::NLT; ++q) {
              if (q == p) {
                const double2 nw = *reinterpret_cast<const double2*>(Ws + q * 64 + 2 * lane);
#pragma unroll
                for (int it = 0; it < C::KWT; ++it) {
                  dmma(c[q][it], nw.x, yb[it][0]);
                  dmma(c[q][it], nw.y, yb[it][1]);
                }
              }
            }
            mbar_wait(bar_v2, ph_v2);
            ph_v2 ^= 1;
#pragma unroll
            for (int q = 0; q < C::NLT; ++q) {
              if (q > p) {
                const double2 nw = *reinterpret_cast<const double2*>(Ws + q * 64 + 2 * lane);
#pragma unroll
                for (int it = 0; it < C::KWT; ++it) {
                  dmma(c[q][it], nw.x, yb[it][0]);
                  dmma(c[q][it], nw.y, yb[it][1]);
                }
              }
            }
          } else {
            // (3b) applies of the tiles q > p (independent of the chain's V of tile p)
#pragma unroll
            for (int q = 0; q < C::NLT; ++q) {
              if (q > p) {
                const double2 nw = *reinterpret_cast<const double2*>(Ws + q * 64 + 2 * lane);
#pragma unroll
                for (int it = 0; it < C::KWT; ++it) {
                  dmma(c[q][it], nw.x, yb[it][0]);
                  dmma(c[q][it], nw.y, yb[it][1]);
                }
              }
            }
            // (1) tile p with panel p-1, V from the chain
            mbar_wait(bar_v, ph_v);
            ph_v ^= 1;
            if (d == 0) TR(1, 1);
#pragma unroll
            for (int q = 0; q < C::NLT; ++q) {
              if (q == p) {
                const double2 nw = *reinterpret_cast<const double2*>(Ws + q * 64 + 2 * lane);
#pragma unroll
                for (int it = 0; it < C::KWT; ++it) {
                  dmma(c[q][it], nw.x, yb[it][0]);
                  dmma(c[q][it], nw.y, yb[it][1]);
                }
              }
            }
          }
          if (flag[par ^ 1] == 0) {  // panel p-1 was explicit: the chain needs the direct Gram
            gram_partial(p, Gd);
            named_bar(BAR_GD, NALL);  // D_p
          }
        }
        double cp[C::KWT][2];
#pragma unroll
        for (int q = 0; q < C::NLT; ++q)
          if (q == p)
#pragma unroll
            for (int it = 0; it < C::KWT; ++it) { cp[it][0] = c[q][it][0]; cp[it][1] = c[q][it][1]; }
        __syncwarp();
        if (d == 0) TR(1, 4);
        // (4) X^T of panel p, partial (X^T C_q)^T of the tiles q > p, C^T C of tile p+1
#pragma unroll
        for (int it = 0; it < C::KWT; ++it)
          *reinterpret_cast<double2*>(Ytw + g * C::LDYT + 8 * it + 2 * t) = make_double2(cp[it][0], cp[it][1]);
#pragma unroll
        for (int q = 0; q < C::NLT; ++q) {
          if (q > p) {
            double z[2] = {0.0, 0.0};
#pragma unroll
            for (int it = 0; it < C::KWT; ++it) {
              dmma(z, c[q][it][0], cp[it][0]);
              dmma(z, c[q][it][1], cp[it][1]);
            }
            *reinterpret_cast<double2*>(Zp + (d * C::NLT + q) * 64 + 2 * lane) = make_double2(z[0], z[1]);
          }
        }
        if (p + 1 < C::NLT) gram_partial(p + 1, Gp);
        if (d == 0) TR(1, 5);
        named_bar(BAR_ALL, NB);  // B_p
        if (d == 0) TR(1, 6);
        if (flag[par] == 0) {
          double* Tc = smem_dyn + C::OFF_T + par * 8 * C::LDT;
          double* Mc = smem_dyn + C::OFF_M + par * 8 * C::LDT;
          factor_panel_all<C, C::DW, BAR_DATA>(cp, R, j0, Ytw, Tc, U, taus, scs, P, d, lane);
          if (d == 0) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const int e = 2 * lane + k, r = e >> 3, cc = e & 7;
              Mc[r * C::LDT + cc] = r == cc ? 1.0 : 0.0;
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
              *reinterpret_cast<double2*>(Zp + (d * C::NLT + q) * 64 + 2 * lane) = make_double2(z[0], z[1]);
            }
          }
          named_bar(BAR_DATA, C::DW * 32);
          named_bar(BAR_ALL, NB);  // F_p
        }
      });
    }
    if (C::DIRECT && d == 0) src.finish(S, lane, 32);  // S final since the last load's barriers
    named_bar(BAR_ALL, NB);  // R final
  }

  double* out = r_out + cta * C::NP * C::NP;
  for (int idx = (warp == chain_w ? 0 : (d + 1) * 32) + lane; idx < C::NP * C::NP; idx += (C::DW + 1) * 32) {
    const int r = idx / C::NP, c2 = idx - r * C::NP;
    out[idx] = c2 >= r ? R[rix<C>(r, c2)] : 0.0;
  }
}
