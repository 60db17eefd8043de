// jq_headtail.cu — the Figaro head/tail operators on the GPU (SPEC.md:107-165,
// PAPER.md:49-51) and the Claim-1 assembly of the reduced matrix.
//
// head(M) = (1/sqrt(m)) sum_i M_i;  tail row r (i = r+1) = (sqrt(i) M_i - S_i/sqrt(i)) / sqrt(i+1)
// with S_i the in-group prefix sum.  The prefix is computed by a deterministic
// reduce-then-scan with FIXED tile boundaries (TILE_ROWS rows), so results do not
// depend on the grid size or on timing (SPEC.md:302 asks for run-to-run
// determinism; decoupled look-back would not give it):
//   1. segscan_tile_kernel  one warp per tile: in-tile segmented column sums,
//                           partial group totals (HBM-bound: reads x once);
//   2. segscan_carry_kernel per column, sequential over tiles: exclusive carry;
//   3. group_fixup_kernel   adds the carry to groups that span tiles.
// The figaro_r path consumes the carries inside the fused TSQR loader
// (jq_tsqr.cu) and never writes the reduced matrix; reduce_* / head_tail (the
// API that returns the matrix itself) use the emit kernels below.
#include <algorithm>
#include <cmath>

#include "jq_internal.cuh"
#include "jq_segscan.cuh"

namespace jq {

constexpr int MAXC = 16;  // columns per lane (cols <= 512)

// One warp per TILE_ROWS tile (segscan_tile, jq_segscan.cuh); MC columns per lane.
template <int MC>
__global__ void __launch_bounds__(256) segscan_tile_kernel(
    const double* __restrict__ x, int64_t rows, int cols, const int32_t* __restrict__ gid,
    int64_t ntiles, double* __restrict__ agg, int* __restrict__ flag, double* __restrict__ totals) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= ntiles) return;
  segscan_tile<8, MC>(x, rows, cols, gid, t, agg, flag, totals, lane);
}

// <= 64 columns: the narrow tile pass (fewer registers -> more warps, 16 rows in flight)
template <int SL>
__global__ void __launch_bounds__(256, 4) segscan_tile_narrow_kernel(
    const double* __restrict__ x, int64_t rows, int cols, const int32_t* __restrict__ gid,
    int64_t ntiles, double* __restrict__ agg, int* __restrict__ flag, double* __restrict__ totals) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= ntiles) return;
  segscan_tile_narrow<SL == 1 ? 16 : 8, SL>(x, rows, cols, gid, t, agg, flag, totals, lane);  // 4 KB per warp in flight
}

// keyed, <= 16 columns: several rows per warp load (32 rows in flight per warp)
template <int CP>
__global__ void __launch_bounds__(256, 2) segscan_tile_tiny_kernel(
    const double* __restrict__ x, int64_t rows, int cols, const int32_t* __restrict__ gid,
    int64_t ntiles, double* __restrict__ agg, int* __restrict__ flag, double* __restrict__ totals) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= ntiles) return;
  segscan_tile_tiny<CP>(x, rows, cols, gid, t, agg, flag, totals, lane);
}

static bool narrow_tiles() {
  static const bool on = [] {
    const char* e = getenv("JQ_SEGSCAN_GENERIC");
    return !(e && e[0] == '1');
  }();
  return on;
}

// Segmented carry over tiles, two-level with FIXED association (deterministic):
//   carry[0] = 0; carry[t+1] = flag[t] ? agg[t] : carry[t] + agg[t]
// Level 1: thread (column, block of CB tiles) folds its block into (flag, sum);
// level 2: one thread per column scans the block aggregates; level 3: each
// (column, block) thread replays its block from the block's carry-in.
constexpr int CB = 64;

__global__ void carry_block_kernel(const double* __restrict__ agg, const int* __restrict__ flag, int64_t ntiles,
                                   int cols, int64_t nblk, double* __restrict__ bagg, int* __restrict__ bflag) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < nblk * cols;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = idx / cols;
    const int c = (int)(idx - b * cols);
    double cur = 0.0;
    int f = 0;
    const int64_t t1 = min(ntiles, (b + 1) * CB);
    for (int64_t t = b * CB; t < t1; ++t) {
      const double a = agg[t * cols + c];
      if (flag[t]) { cur = a; f = 1; } else cur += a;
    }
    bagg[b * cols + c] = cur;
    if (c == 0) bflag[b] = f;
  }
}

__global__ void carry_top_kernel(double* __restrict__ bagg, const int* __restrict__ bflag, int64_t nblk, int cols) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  double cur = 0.0;  // exclusive carry into block b, written in place
  // loads of 16 blocks issued together (the in-place stores would otherwise serialise
  // every load behind the previous iteration); same additions in the same order
  constexpr int U = 16;
  int64_t b = 0;
  for (; b + U <= nblk; b += U) {
    double a[U];
    int f[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a[u] = bagg[(b + u) * cols + c];
      f[u] = bflag[b + u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      bagg[(b + u) * cols + c] = cur;
      cur = f[u] ? a[u] : cur + a[u];
    }
  }
  for (; b < nblk; ++b) {
    const double a = bagg[b * cols + c];
    bagg[b * cols + c] = cur;
    cur = bflag[b] ? a : cur + a;
  }
}

__global__ void carry_apply_kernel(const double* __restrict__ agg, const int* __restrict__ flag, int64_t ntiles,
                                   int cols, int64_t nblk, const double* __restrict__ bin, double* __restrict__ carry) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < nblk * cols;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = idx / cols;
    const int c = (int)(idx - b * cols);
    double cur = bin[b * cols + c];
    const int64_t t1 = min(ntiles, (b + 1) * CB);
    for (int64_t t = b * CB; t < t1; ++t) {
      carry[t * cols + c] = cur;
      const double a = agg[t * cols + c];
      cur = flag[t] ? a : cur + a;
    }
  }
}

// totals[g] += carry[last tile of g] for groups that began before that tile.
__global__ void group_fixup_kernel(const int64_t* __restrict__ gstart, const int64_t* __restrict__ gcount,
                                   const int64_t* __restrict__ d_ngroups, int64_t single_rows,
                                   int cols, const double* __restrict__ carry, double* __restrict__ totals) {
  const int64_t ng = d_ngroups ? d_ngroups[0] : 1;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < ng * cols;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = idx / cols;
    const int c = (int)(idx - g * cols);
    const int64_t st = gstart ? gstart[g] : 0;
    const int64_t cnt = gcount ? gcount[g] : single_rows;
    if (cnt <= 0) continue;
    const int64_t tl = (st + cnt - 1) / TILE_ROWS;
    if (st < tl * TILE_ROWS) totals[g * cols + c] += carry[tl * cols + c];
  }
}

size_t segscan_ws_bytes(int64_t rows, int64_t cols, int64_t groups_cap) {
  int64_t nt = std::max<int64_t>(1, cdiv(rows, TILE_ROWS));
  int64_t nb = cdiv(nt, CB);
  return 2 * ws_bytes(size_t(nt) * cols, 8) + ws_bytes(nt, 4) + ws_bytes(size_t(nb) * cols, 8) + ws_bytes(nb, 4) +
         ws_bytes(size_t(std::max<int64_t>(groups_cap, 1)) * cols, 8);
}

// The scan in three steps, so the tile pass (the only HBM-heavy one) can run inside
// another kernel (SideScan): begin = workspace + zeroed totals, tiles = the tile pass,
// end = the carry scan over tiles and the fix-up of groups that span tiles.
int segscan_begin(jq_ctx* ctx, const double* x, int64_t rows, int64_t cols, const int32_t* gid,
                  int64_t groups_cap, SegScan* s, SideScan* side) {
  if (cols > 32 * MAXC) return fail(JQ_E_INVALID, "more than 512 columns per table");
  s->ntiles = std::max<int64_t>(1, cdiv(rows, TILE_ROWS));
  s->rows = rows;
  s->cols = cols;
  s->carry = ws_alloc<double>(ctx, size_t(s->ntiles) * cols);
  s->tile_agg = ws_alloc<double>(ctx, size_t(s->ntiles) * cols);
  s->tile_flag = ws_alloc<int>(ctx, s->ntiles);
  s->totals = ws_alloc<double>(ctx, size_t(std::max<int64_t>(groups_cap, 1)) * cols);
  if (!s->carry || !s->tile_agg || !s->tile_flag || !s->totals)
    return fail(JQ_E_OOM, "workspace exhausted (head/tail scan)");
  JQ_CUDA(cudaMemsetAsync(s->totals, 0, size_t(std::max<int64_t>(groups_cap, 1)) * cols * 8, ctx->stream));
  *side = SideScan{};
  if (rows == 0) {
    JQ_CUDA(cudaMemsetAsync(s->carry, 0, size_t(s->ntiles) * cols * 8, ctx->stream));
    return JQ_OK;
  }
  side->x = x;
  side->rows = rows;
  side->cols = (int)cols;
  side->gid = gid;
  side->ntiles = s->ntiles;
  side->agg = s->tile_agg;
  side->flag = s->tile_flag;
  side->totals = s->totals;
  return JQ_OK;
}

int segscan_tiles(jq_ctx* ctx, const SideScan& side) {
  if (!side.x || side.ntiles == 0) return JQ_OK;
  const int wpb = 8;
  const int k = ctx->tile_launches < 4 && ctx->tev[0] ? ctx->tile_launches : -1;
  if (k >= 0) cudaEventRecord(ctx->tev[2 * k], ctx->stream);
  const unsigned grid = (unsigned)cdiv(side.ntiles, wpb);
  static const bool tiny = [] {  // JQ_SEGSCAN_TINY=0: keyed <= 16 columns on the narrow pass (A/B)
    const char* e = getenv("JQ_SEGSCAN_TINY");
    return !(e && e[0] == '0');
  }();
  if (narrow_tiles() && tiny && side.gid && side.cols <= 8)
    segscan_tile_tiny_kernel<8><<<grid, 32 * wpb, 0, ctx->stream>>>(
        side.x, side.rows, side.cols, side.gid, side.ntiles, side.agg, side.flag, side.totals);
  else if (narrow_tiles() && tiny && side.gid && side.cols <= 16)
    segscan_tile_tiny_kernel<16><<<grid, 32 * wpb, 0, ctx->stream>>>(
        side.x, side.rows, side.cols, side.gid, side.ntiles, side.agg, side.flag, side.totals);
  else if (narrow_tiles() && side.cols <= 32)
    segscan_tile_narrow_kernel<1><<<grid, 32 * wpb, 0, ctx->stream>>>(
        side.x, side.rows, side.cols, side.gid, side.ntiles, side.agg, side.flag, side.totals);
  else if (narrow_tiles() && side.cols <= 64)
    segscan_tile_narrow_kernel<2><<<grid, 32 * wpb, 0, ctx->stream>>>(
        side.x, side.rows, side.cols, side.gid, side.ntiles, side.agg, side.flag, side.totals);
  else if (side.cols <= 256)
    segscan_tile_kernel<8><<<grid, 32 * wpb, 0, ctx->stream>>>(
        side.x, side.rows, side.cols, side.gid, side.ntiles, side.agg, side.flag, side.totals);
  else
    segscan_tile_kernel<16><<<grid, 32 * wpb, 0, ctx->stream>>>(
        side.x, side.rows, side.cols, side.gid, side.ntiles, side.agg, side.flag, side.totals);
  JQ_CHECK_LAUNCH(ctx);
  if (k >= 0) {  // algorithmic bytes: the rows read once (+ their segment ids)
    cudaEventRecord(ctx->tev[2 * k + 1], ctx->stream);
    ctx->tile_bytes += 8.0 * side.rows * side.cols + (side.gid ? 4.0 * side.rows : 0.0);
    ctx->tile_launches = k + 1;
  }
  return JQ_OK;
}

int segscan_end(jq_ctx* ctx, const int64_t* gstart, const int64_t* gcount, const int64_t* d_ngroups,
                int64_t groups_cap, SegScan* s) {
  if (s->rows == 0) return JQ_OK;
  const int64_t cols = s->cols;
  {
    const int64_t nblk = cdiv(s->ntiles, CB);
    double* bagg = ws_alloc<double>(ctx, size_t(nblk) * cols);
    int* bflag = ws_alloc<int>(ctx, nblk);
    if (!bagg || !bflag) return fail(JQ_E_OOM, "workspace exhausted (carry scan)");
    const unsigned gb = (unsigned)std::min<int64_t>(cdiv(nblk * cols, 128), 148 * 16);
    carry_block_kernel<<<gb, 128, 0, ctx->stream>>>(s->tile_agg, s->tile_flag, s->ntiles, (int)cols, nblk, bagg, bflag);
    JQ_CHECK_LAUNCH(ctx);
    carry_top_kernel<<<(unsigned)cdiv(cols, 64), 64, 0, ctx->stream>>>(bagg, bflag, nblk, (int)cols);
    JQ_CHECK_LAUNCH(ctx);
    carry_apply_kernel<<<gb, 128, 0, ctx->stream>>>(s->tile_agg, s->tile_flag, s->ntiles, (int)cols, nblk, bagg,
                                                   s->carry);
    JQ_CHECK_LAUNCH(ctx);
  }
  group_fixup_kernel<<<(unsigned)std::min<int64_t>(cdiv(std::max<int64_t>(groups_cap, 1) * cols, 256), 4096),
                       256, 0, ctx->stream>>>(gstart, gcount, d_ngroups, s->rows, (int)cols, s->carry,
                                              s->totals);
  JQ_CHECK_LAUNCH(ctx);
  return JQ_OK;
}

int segscan_dev(jq_ctx* ctx, const double* x, int64_t rows, int64_t cols, const int32_t* gid,
                const int64_t* gstart, const int64_t* gcount, const int64_t* d_ngroups,
                int64_t groups_cap, SegScan* s) {
  SideScan side;
  JQ_TRY(segscan_begin(ctx, x, rows, cols, gid, groups_cap, s, &side));
  JQ_TRY(segscan_tiles(ctx, side));
  return segscan_end(ctx, gstart, gcount, d_ngroups, groups_cap, s);
}

// ------------------------------------------------------------------ emit kernels
// Tail rows of every segment: row r of x with in-group index rr >= 1 goes to output
// row base(g) + rr - 1, columns [col0, col0 + cols), scaled by sqrt(count(g)); columns
// [0, col0) of that output row are zeroed (the exact-zero block).
//   tail_rr = (sqrt(rr) x - S / sqrt(rr)) / sqrt(rr + 1) sqrt(c) = a1 x - a2 S,
//   a2 = sqrt(c) / sqrt(rr (rr + 1)),  a1 = rr a2   (MUFU rsqrt + one cubic step).
// One warp per TILE_ROWS tile; lane j derives the scalars of row j of each batch of
// 32 rows (shuffled to the warp when the row is processed) and four rows' loads are
// issued before their sequential prefix updates.
template <int MC>  // columns per lane: cols <= 32 MC (few registers -> many warps in flight)
__global__ void __launch_bounds__(256) tail_emit_kernel(
    const double* __restrict__ x, int64_t rows, int cols, const int32_t* __restrict__ gid,
    const int64_t* __restrict__ gstart, const int64_t* __restrict__ scale_count, double scale_all,
    const int64_t* __restrict__ out_base, int64_t out_base_all, int out_ld, int col0,
    const double* __restrict__ carry, int64_t ntiles, double* __restrict__ out) {
  const unsigned FULLM = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= ntiles) return;
  const int64_t r0 = t * TILE_ROWS, r1 = min(rows, r0 + TILE_ROWS);
  double s[MC];
#pragma unroll
  for (int k = 0; k < MC; ++k) s[k] = (k * 32 + lane < cols) ? carry[t * cols + k * 32 + lane] : 0.0;
  for (int64_t rb = r0; rb < r1; rb += 32) {
    int kind = 0;  // 0 no output (key absent), 1 group start (head row), 2 tail row
    double a1 = 0.0, a2 = 0.0;
    int64_t orow = 0;
    {
      const int64_t r = rb + lane;
      if (r < r1) {
        const int g = gid ? gid[r] : 0;
        if (g >= 0) {
          const int64_t rr = r - (gid ? gstart[g] : 0);
          if (rr == 0) {
            kind = 1;
          } else {
            kind = 2;
            const double rd = (double)rr;
            const double c = scale_count ? (double)scale_count[g] : scale_all;
            a2 = (c * rsqrt_nr(c)) * rsqrt_nr(rd * (rd + 1.0));
            a1 = rd * a2;
            orow = (gid ? out_base[g] : out_base_all) + rr - 1;
          }
        }
      }
    }
    const int nb = r1 - rb < 32 ? (int)(r1 - rb) : 32;
    for (int j0 = 0; j0 < nb; j0 += 4) {
      double v[4][MC];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double* row = x + (rb + j0 + u) * cols;
        const bool in = j0 + u < nb;
#pragma unroll
        for (int k = 0; k < MC; ++k) {
          const int c = k * 32 + lane;
          v[u][k] = (in && c < cols) ? __ldg(row + c) : 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = j0 + u;
        const int kj = __shfl_sync(FULLM, kind, j & 31);
        const double b1 = __shfl_sync(FULLM, a1, j & 31), b2 = __shfl_sync(FULLM, a2, j & 31);
        const int64_t oj = __shfl_sync(FULLM, orow, j & 31);
        if (j >= nb || kj == 0) continue;
        if (kj == 1) {
#pragma unroll
          for (int k = 0; k < MC; ++k) s[k] = v[u][k];
          continue;
        }
        double* orw = out + oj * out_ld;
        for (int c = lane; c < col0; c += 32) orw[c] = 0.0;
#pragma unroll
        for (int k = 0; k < MC; ++k) {
          const int c = k * 32 + lane;
          if (c < cols) orw[col0 + c] = fma(b1, v[u][k], -b2 * s[k]);
          s[k] += v[u][k];
        }
      }
    }
  }
}

// Top block rows: A row i of group g -> output row red_off[g] + (i - a_start[g]):
// [sqrt(m2g) A_i | totals_b[g] / sqrt(m2g)].  One warp per row, lanes
// over the columns; the row scale from MUFU rsqrt + one cubic step.
__global__ void top_emit_kernel(const double* __restrict__ a, int64_t m1, int n1,
                                const int32_t* __restrict__ gid_a, const int64_t* __restrict__ a_start,
                                const int64_t* __restrict__ b_count, int64_t m2_all,
                                const int64_t* __restrict__ red_off, const double* __restrict__ b_totals,
                                int n2, double* __restrict__ out) {
  const int n = n1 + n2;
  const int lane = threadIdx.x & 31;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < m1;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int g = gid_a ? gid_a[i] : 0;
    if (g < 0) continue;
    const double m2g = gid_a ? (double)b_count[g] : (double)m2_all;
    const double rs = rsqrt_nr(m2g), sq = m2g * rs;
    const int64_t orow = gid_a ? red_off[g] + (i - a_start[g]) : i;
    const double* arow = a + i * n1;
    const double* brow = b_totals + (int64_t)g * n2;
    double* o = out + orow * n;
    for (int c = lane; c < n; c += 32) o[c] = c < n1 ? __ldg(arow + c) * sq : brow[c - n1] * rs;
  }
}

static void launch_tail_emit(jq_ctx* ctx, int cols, unsigned grid, const double* x, int64_t rows,
                             const int32_t* gid, const int64_t* gstart, const int64_t* scale_count,
                             double scale_all, const int64_t* out_base, int64_t out_base_all, int out_ld,
                             int col0, const double* carry, int64_t ntiles, double* out) {
  if (cols <= 64)
    tail_emit_kernel<2><<<grid, 256, 0, ctx->stream>>>(x, rows, cols, gid, gstart, scale_count, scale_all,
                                                       out_base, out_base_all, out_ld, col0, carry, ntiles, out);
  else if (cols <= 128)
    tail_emit_kernel<4><<<grid, 256, 0, ctx->stream>>>(x, rows, cols, gid, gstart, scale_count, scale_all,
                                                       out_base, out_base_all, out_ld, col0, carry, ntiles, out);
  else if (cols <= 256)
    tail_emit_kernel<8><<<grid, 256, 0, ctx->stream>>>(x, rows, cols, gid, gstart, scale_count, scale_all,
                                                       out_base, out_base_all, out_ld, col0, carry, ntiles, out);
  else
    tail_emit_kernel<16><<<grid, 256, 0, ctx->stream>>>(x, rows, cols, gid, gstart, scale_count, scale_all,
                                                        out_base, out_base_all, out_ld, col0, carry, ntiles, out);
}

__global__ void tail_base_kernel(const int64_t* __restrict__ red_off, const int64_t* __restrict__ a_count,
                                 const int64_t* __restrict__ d_ng, int64_t* __restrict__ base) {
  const int64_t ng = d_ng[0];
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ng; g += (int64_t)gridDim.x * blockDim.x)
    base[g] = red_off[g] + a_count[g];
}

__global__ void head_row_kernel(const double* __restrict__ totals, int cols, double m, double* __restrict__ out) {
  for (int c = threadIdx.x; c < cols; c += blockDim.x) out[c] = totals[c] / sqrt(m);
}

__global__ void group_bounds_kernel(const int64_t* __restrict__ red_off, const int64_t* __restrict__ d_ng,
                                    int64_t* __restrict__ bounds) {
  const int64_t ng = d_ng[0];
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ng; g += (int64_t)gridDim.x * blockDim.x) {
    bounds[2 * g] = red_off[g];
    bounds[2 * g + 1] = red_off[g + 1];
  }
}

static unsigned grid_for(int64_t work, int threads = 256, int64_t cap = 148 * 16) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(work, threads), cap));
}

// The reduced matrix in SPEC row order into dout (total_rows x
// (n1 + n2), device): scan of B, top rows [sqrt(m2g) A_g | head(B_g)], tail rows
// [0 | sqrt(m1g) tail(B_g)].  gr = grouping (keyed) or nullptr (Cartesian).  Shared by
// jq_reduce and figaro_r's wide path (n1 + n2 > 256: reduce, then jq_wide.cu's TSQR).
int reduce_emit_dev(jq_ctx* ctx, const double* da, int64_t m1, int64_t n1, const double* db, int64_t m2,
                    int64_t n2, const Groups* gr, int64_t cap, int64_t total_rows, double* dout) {
  const bool keyed = gr != nullptr;
  const int64_t n = n1 + n2;
  if (n2 == 0)  // bottom rows are exact-zero rows of width n1
    JQ_CUDA(cudaMemsetAsync(dout, 0, total_rows * n * 8, ctx->stream));
  SegScan ss;
  const int64_t cols_b = std::max<int64_t>(n2, 1);
  if (n2 > 0) {
    JQ_TRY(segscan_dev(ctx, db, m2, n2, keyed ? gr->gid_b : nullptr, keyed ? gr->b_start : nullptr,
                       keyed ? gr->b_count : nullptr, keyed ? gr->d_n : nullptr, cap, &ss));
  } else {
    JQ_TRY(segscan_dev(ctx, db, 0, cols_b, nullptr, nullptr, nullptr, nullptr, cap, &ss));
  }
  top_emit_kernel<<<grid_for(m1 * 32), 256, 0, ctx->stream>>>(
      da, m1, (int)n1, keyed ? gr->gid_a : nullptr, keyed ? gr->a_start : nullptr,
      keyed ? gr->b_count : nullptr, m2, keyed ? gr->red_off : nullptr, ss.totals, (int)n2, dout);
  JQ_CHECK_LAUNCH(ctx);
  if (n2 > 0) {
    int64_t* base = nullptr;
    if (keyed) {
      base = ws_alloc<int64_t>(ctx, cap);
      if (!base) return fail(JQ_E_OOM, "workspace exhausted (reduce)");
      tail_base_kernel<<<grid_for(cap), 256, 0, ctx->stream>>>(gr->red_off, gr->a_count, gr->d_n, base);
      JQ_CHECK_LAUNCH(ctx);
    }
    launch_tail_emit(ctx, (int)n2, (unsigned)cdiv(ss.ntiles, 8), db, m2, keyed ? gr->gid_b : nullptr,
                     keyed ? gr->b_start : nullptr, keyed ? gr->a_count : nullptr, (double)m1, base, m1, (int)n,
                     (int)n1, ss.carry, ss.ntiles, dout);
    JQ_CHECK_LAUNCH(ctx);
  }
  return JQ_OK;
}

size_t reduce_emit_ws_bytes(int64_t m2, int64_t n2, int64_t cap) {
  return segscan_ws_bytes(m2, std::max<int64_t>(n2, 1), cap) + ws_bytes(cap, 8) + 4096;
}

// ------------------------------------------------------------------ public API
}  // namespace jq

using namespace jq;

extern "C" int jq_head_tail(jq_ctx* ctx, const double* m, int64_t rows, int64_t cols, double* out) {
  if (!ctx) return fail(JQ_E_INVALID, "null context");
  JQ_NVTX("jq_head_tail");
  if (rows <= 0) return fail(JQ_E_INVALID, "head/tail undefined for a matrix with 0 rows");
  if (cols <= 0) return JQ_OK;
  if (cols > 512) return fail(JQ_E_INVALID, "more than 512 columns");
  JQ_TRY(begin_call(ctx));
  size_t need = stage_bytes(m, rows * cols) + stage_bytes((const double*)out, rows * cols) +
                segscan_ws_bytes(rows, cols, 1);
  JQ_TRY(ws_reserve(ctx, need));
  const double* dm;
  double* dout;
  JQ_TRY(stage_in(ctx, m, rows * cols, &dm));
  JQ_TRY(stage_out(ctx, out, rows * cols, &dout));
  SegScan ss;
  JQ_TRY(segscan_dev(ctx, dm, rows, cols, nullptr, nullptr, nullptr, nullptr, 1, &ss));
  head_row_kernel<<<1, 256, 0, ctx->stream>>>(ss.totals, (int)cols, (double)rows, dout);
  JQ_CHECK_LAUNCH(ctx);
  launch_tail_emit(ctx, (int)cols, (unsigned)cdiv(ss.ntiles, 8), dm, rows, nullptr, nullptr, nullptr, 1.0, nullptr,
                   1, (int)cols, 0, ss.carry, ss.ntiles, dout);
  JQ_CHECK_LAUNCH(ctx);
  JQ_TRY(copy_out(ctx, out, (const double*)dout, rows * cols));
  return sync_and_check_flags(ctx);
}

extern "C" int jq_colsums(jq_ctx* ctx, const double* x, int64_t rows, int64_t cols, double* sums) {
  if (!ctx) return fail(JQ_E_INVALID, "null context");
  JQ_NVTX("jq_colsums");
  if (cols <= 0) return JQ_OK;
  if (cols > 512) return fail(JQ_E_INVALID, "more than 512 columns");
  JQ_TRY(begin_call(ctx));
  JQ_TRY(ws_reserve(ctx, stage_bytes(x, rows * cols) + stage_bytes((const double*)sums, cols) +
                             segscan_ws_bytes(rows, cols, 1)));
  const double* dx;
  double* ds;
  JQ_TRY(stage_in(ctx, x, rows * cols, &dx));
  JQ_TRY(stage_out(ctx, sums, cols, &ds));
  SegScan ss;
  JQ_TRY(segscan_dev(ctx, dx, rows, cols, nullptr, nullptr, nullptr, nullptr, 1, &ss));
  JQ_CUDA(cudaMemcpyAsync(ds, ss.totals, cols * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  JQ_TRY(copy_out(ctx, sums, (const double*)ds, cols));
  return sync_and_check_flags(ctx);
}

extern "C" int jq_reduce(jq_ctx* ctx, const double* a, int64_t m1, int64_t n1, const int64_t* ka,
                         const double* b, int64_t m2, int64_t n2, const int64_t* kb, double* out,
                         int64_t out_capacity, int64_t* out_rows, int64_t* group_bounds) {
  if (!ctx) return fail(JQ_E_INVALID, "null context");
  JQ_NVTX("jq_reduce");
  if ((ka == nullptr) != (kb == nullptr)) return fail(JQ_E_KEYS, "both tables must carry keys, or neither");
  if (n1 < 0 || n2 < 0 || n1 > 512 || n2 > 512) return fail(JQ_E_INVALID, "column counts must lie in 0..512");
  const bool keyed = ka != nullptr;
  if (!keyed && (m1 <= 0 || m2 <= 0)) return fail(JQ_E_INVALID, "reduce_cartesian needs non-empty inputs");
  JQ_TRY(begin_call(ctx));
  const int64_t n = n1 + n2;
  const int64_t cap = keyed ? std::max<int64_t>(1, std::min(m1, m2)) : 1;
  size_t need = stage_bytes(a, m1 * n1) + stage_bytes(b, m2 * n2) + stage_bytes(ka, m1) +
                stage_bytes(kb, m2) + (keyed ? group_ws_bytes(m1, m2) : 0) +
                segscan_ws_bytes(m2, std::max<int64_t>(n2, 1), cap) + ws_bytes(cap, 8) + 4096;
  if (out) need += stage_bytes((const double*)out, out_capacity * n);
  if (group_bounds) need += ws_bytes(2 * cap, 8);
  JQ_TRY(ws_reserve(ctx, need));
  const int64_t *dka = nullptr, *dkb = nullptr;
  JQ_TRY(stage_in(ctx, ka, m1, &dka));
  JQ_TRY(stage_in(ctx, kb, m2, &dkb));
  Groups gr;
  int64_t ng = 1, total_rows = m1 + m2 - 1;
  if (keyed) {
    JQ_TRY(group_keys_dev(ctx, dka, m1, dkb, m2, &gr));
    int64_t hn[2];
    JQ_CUDA(cudaMemcpyAsync(hn, gr.d_n, 16, cudaMemcpyDeviceToHost, ctx->stream));
    JQ_TRY(sync_and_check_flags(ctx));
    ng = hn[0];
    total_rows = hn[1];
  }
  if (out_rows) *out_rows = total_rows;
  if (group_bounds && ng > 0) {
    if (keyed) {
      int64_t* db = ws_alloc<int64_t>(ctx, 2 * ng);
      group_bounds_kernel<<<grid_for(ng), 256, 0, ctx->stream>>>(gr.red_off, gr.d_n, db);
      JQ_CHECK_LAUNCH(ctx);
      JQ_CUDA(cudaMemcpyAsync(group_bounds, db, 2 * ng * 8, cudaMemcpyDefault, ctx->stream));
    } else {
      group_bounds[0] = 0;
      group_bounds[1] = total_rows;
    }
  }
  if (!out || total_rows == 0) return sync_and_check_flags(ctx);
  if (out_capacity < total_rows) return fail(JQ_E_INVALID, "output buffer too small for the reduced matrix");
  const double *da, *db;
  double* dout;
  JQ_TRY(stage_in(ctx, a, m1 * n1, &da));
  JQ_TRY(stage_in(ctx, b, m2 * n2, &db));
  JQ_TRY(stage_out(ctx, out, total_rows * n, &dout));
  JQ_TRY(reduce_emit_dev(ctx, da, m1, n1, db, m2, n2, keyed ? &gr : nullptr, keyed ? std::max<int64_t>(ng, 1) : 1,
                         total_rows, dout));
  JQ_TRY(copy_out(ctx, out, (const double*)dout, total_rows * n));
  return sync_and_check_flags(ctx);
}
