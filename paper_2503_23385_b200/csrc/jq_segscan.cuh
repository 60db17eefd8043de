// jq_segscan.cuh — the per-tile pass of the head/tail segmented scan, one warp per
// TILE_ROWS tile.  Shared by segscan_tile_kernel (jq_headtail.cu) and by the spare
// warps of the warp-specialised TSQR leaf (jq_tsqr_ws.cuh), which run the tile pass
// of the other side's tails while the leaf factors this side: the same function, so
// the same bits either way.
#pragma once
#include "jq_internal.cuh"

namespace jq {

constexpr int SEG_MAXC = 8;  // columns per lane (cols <= 256); the standalone kernel also has 16 (<= 512)

// Tile t.  Segment id of row r: gid[r] (or 0 when gid is null = one segment).  Writes
// agg[t] (sum of the segment open at the tile end, restricted to the tile), flag[t]
// (tile contains a segment start) and, for each segment that ends inside the tile, its
// in-tile partial sum into totals[seg].  Rows are loaded BATCH at a time (a lone warp
// must keep enough bytes in flight); the additions happen row by row in the same order
// as with any other batching.
template <int BATCH = 8, int MAXCL = SEG_MAXC>
__device__ __forceinline__ void segscan_tile(const double* __restrict__ x, int64_t rows, int cols,
                                             const int32_t* __restrict__ gid, int64_t t, double* __restrict__ agg,
                                             int* __restrict__ flag, double* __restrict__ totals, int lane) {
  const int64_t r0 = t * TILE_ROWS, r1 = min(rows, r0 + TILE_ROWS);
  if (!gid && cols <= 64) {
    // one segment (Cartesian): plain column sums into 4 accumulators per column (row r
    // into accumulator r % 4) and a fixed-order combine (deterministic); the segment
    // starts at global row 0
    double a[2][4];
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int u = 0; u < 4; ++u) a[k][u] = 0.0;
    const bool h0 = lane < cols, h1 = lane + 32 < cols;
    int64_t r = r0;
    for (; r + BATCH <= r1; r += BATCH) {
      double v[2][BATCH];
#pragma unroll
      for (int u = 0; u < BATCH; ++u) {
        const double* row = x + (r + u) * cols;
        v[0][u] = h0 ? __ldg(row + lane) : 0.0;
        v[1][u] = h1 ? __ldg(row + lane + 32) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < BATCH; ++u) { a[0][u & 3] += v[0][u]; a[1][u & 3] += v[1][u]; }
    }
    for (; r + 4 <= r1; r += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double* row = x + (r + u) * cols;
        a[0][u] += h0 ? __ldg(row + lane) : 0.0;
        a[1][u] += h1 ? __ldg(row + lane + 32) : 0.0;
      }
    }
    for (; r < r1; ++r) {
      const double* row = x + r * cols;
      if (h0) a[0][0] += __ldg(row + lane);
      if (h1) a[1][0] += __ldg(row + lane + 32);
    }
    const double s0 = (a[0][0] + a[0][1]) + (a[0][2] + a[0][3]);
    const double s1 = (a[1][0] + a[1][1]) + (a[1][2] + a[1][3]);
    if (r1 == rows) {
      if (h0) totals[lane] = s0;
      if (h1) totals[lane + 32] = s1;
    }
    if (h0) agg[t * cols + lane] = s0;
    if (h1) agg[t * cols + lane + 32] = s1;
    if (lane == 0) flag[t] = r0 == 0;
    return;
  }
  int seg = gid ? gid[r0] : 0;
  int any_start = (r0 == 0) || (gid && gid[r0 - 1] != seg);
  if (gid && cols <= 64) {
    // keyed, <= 64 columns: the loads of BATCH rows are issued before their sequential
    // segment logic (same additions in the same order as the generic loop below)
    const bool h0 = lane < cols, h1 = lane + 32 < cols;
    double s0 = 0.0, s1 = 0.0;
    int64_t r = r0;
    auto row_step = [&](int64_t rr, int sr, double v0, double v1) {
      const bool start = (rr == 0) || (rr > r0 && sr != seg);
      if (start && rr > r0) {
        if (seg >= 0) {
          if (h0) totals[(int64_t)seg * cols + lane] = s0;
          if (h1) totals[(int64_t)seg * cols + lane + 32] = s1;
        }
        any_start = 1;
      }
      seg = sr;
      s0 = start ? v0 : s0 + v0;
      s1 = start ? v1 : s1 + v1;
    };
    for (; r + BATCH <= r1; r += BATCH) {
      int g8[BATCH];
      double v[2][BATCH];
#pragma unroll
      for (int u = 0; u < BATCH; ++u) {
        g8[u] = gid[r + u];
        const double* row = x + (r + u) * cols;
        v[0][u] = h0 ? __ldg(row + lane) : 0.0;
        v[1][u] = h1 ? __ldg(row + lane + 32) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < BATCH; ++u) row_step(r + u, g8[u], v[0][u], v[1][u]);
    }
    for (; r < r1; ++r) {
      const double* row = x + r * cols;
      row_step(r, gid[r], h0 ? __ldg(row + lane) : 0.0, h1 ? __ldg(row + lane + 32) : 0.0);
    }
    const bool ends_here = (r1 == rows) || (gid[r1] != seg);
    if (ends_here && seg >= 0) {
      if (h0) totals[(int64_t)seg * cols + lane] = s0;
      if (h1) totals[(int64_t)seg * cols + lane + 32] = s1;
    }
    if (h0) agg[t * cols + lane] = s0;
    if (h1) agg[t * cols + lane + 32] = s1;
    if (lane == 0) flag[t] = any_start;
    return;
  }
  double s[MAXCL];
#pragma unroll
  for (int k = 0; k < MAXCL; ++k) s[k] = 0.0;
  for (int64_t r = r0; r < r1; ++r) {
    const int sr = gid ? gid[r] : 0;
    const bool start = (r == 0) || (r > r0 && sr != seg);
    if (start && r > r0) {
      // previous segment ended at r-1 inside this tile
      if (seg >= 0)
#pragma unroll
        for (int k = 0; k < MAXCL; ++k)
          if (k * 32 + lane < cols) totals[(int64_t)seg * cols + k * 32 + lane] = s[k];
      any_start = 1;
    }
    seg = sr;
    const double* row = x + r * cols;
#pragma unroll
    for (int k = 0; k < MAXCL; ++k) {
      const int c = k * 32 + lane;
      if (c < cols) {
        const double v = __ldg(row + c);
        s[k] = start ? v : s[k] + v;
      }
    }
  }
  // open segment at the tile end
  const bool ends_here = (r1 == rows) || (gid && gid[r1] != seg);
  if (ends_here && seg >= 0)
#pragma unroll
    for (int k = 0; k < MAXCL; ++k)
      if (k * 32 + lane < cols) totals[(int64_t)seg * cols + k * 32 + lane] = s[k];
#pragma unroll
  for (int k = 0; k < MAXCL; ++k)
    if (k * 32 + lane < cols) agg[t * cols + k * 32 + lane] = s[k];
  if (lane == 0) flag[t] = any_start;
}

// The same tile pass for <= 32 * SL columns with fewer registers and more rows in flight
// (the standalone segscan_tile_kernel; the generic path above stays for wider tables and
// for the TSQR leaf's spare warps).  Identical additions in identical order: keyed rows
// run the same sequential segment logic; Cartesian row r goes to accumulator r % 4 and
// the last r1 % 4 rows of the tile to accumulator 0, as in segscan_tile.
template <int BATCH, int SL>
__device__ __forceinline__ void segscan_tile_narrow(const double* __restrict__ x, int64_t rows, int cols,
                                                    const int32_t* __restrict__ gid, int64_t t,
                                                    double* __restrict__ agg, int* __restrict__ flag,
                                                    double* __restrict__ totals, int lane) {
  static_assert(BATCH % 4 == 0 && (SL == 1 || SL == 2), "narrow tile pass shape");
  const int64_t r0 = t * TILE_ROWS, r1 = min(rows, r0 + TILE_ROWS);
  bool h[SL];
#pragma unroll
  for (int k = 0; k < SL; ++k) h[k] = lane + 32 * k < cols;
  if (!gid) {
    double a[SL][4];
#pragma unroll
    for (int k = 0; k < SL; ++k)
#pragma unroll
      for (int u = 0; u < 4; ++u) a[k][u] = 0.0;
    int64_t r = r0;
    for (; r + BATCH <= r1; r += BATCH) {
      double v[SL][BATCH];
#pragma unroll
      for (int u = 0; u < BATCH; ++u)
#pragma unroll
        for (int k = 0; k < SL; ++k) v[k][u] = h[k] ? __ldg(x + (r + u) * cols + lane + 32 * k) : 0.0;
#pragma unroll
      for (int u = 0; u < BATCH; ++u)
#pragma unroll
        for (int k = 0; k < SL; ++k) a[k][u & 3] += v[k][u];
    }
    for (; r + 4 <= r1; r += 4)
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int k = 0; k < SL; ++k) a[k][u] += h[k] ? __ldg(x + (r + u) * cols + lane + 32 * k) : 0.0;
    for (; r < r1; ++r)
#pragma unroll
      for (int k = 0; k < SL; ++k)
        if (h[k]) a[k][0] += __ldg(x + r * cols + lane + 32 * k);
#pragma unroll
    for (int k = 0; k < SL; ++k) {
      const double sk = (a[k][0] + a[k][1]) + (a[k][2] + a[k][3]);
      if (h[k]) {
        if (r1 == rows) totals[lane + 32 * k] = sk;
        agg[t * cols + lane + 32 * k] = sk;
      }
    }
    if (lane == 0) flag[t] = r0 == 0;
    return;
  }
  int seg = gid[r0];
  int any_start = (r0 == 0) || (gid[r0 - 1] != seg);
  double s[SL];
#pragma unroll
  for (int k = 0; k < SL; ++k) s[k] = 0.0;
  auto row_step = [&](int64_t rr, int sr, const double* v) {
    const bool start = (rr == 0) || (rr > r0 && sr != seg);
    if (start && rr > r0) {
      if (seg >= 0)
#pragma unroll
        for (int k = 0; k < SL; ++k)
          if (h[k]) totals[(int64_t)seg * cols + lane + 32 * k] = s[k];
      any_start = 1;
    }
    seg = sr;
#pragma unroll
    for (int k = 0; k < SL; ++k) s[k] = start ? v[k] : s[k] + v[k];
  };
  int64_t r = r0;
  for (; r + BATCH <= r1; r += BATCH) {
    int g[BATCH];
    double v[BATCH][SL];
#pragma unroll
    for (int u = 0; u < BATCH; ++u) {
      g[u] = gid[r + u];
#pragma unroll
      for (int k = 0; k < SL; ++k) v[u][k] = h[k] ? __ldg(x + (r + u) * cols + lane + 32 * k) : 0.0;
    }
    bool uniform = r != 0;  // every row continues the open segment: plain sequential sums
#pragma unroll
    for (int u = 0; u < BATCH; ++u) uniform = uniform && g[u] == seg;
    if (uniform) {
#pragma unroll
      for (int u = 0; u < BATCH; ++u)
#pragma unroll
        for (int k = 0; k < SL; ++k) s[k] = s[k] + v[u][k];
    } else {
#pragma unroll
      for (int u = 0; u < BATCH; ++u) row_step(r + u, g[u], v[u]);
    }
  }
  for (; r < r1; ++r) {
    double v[SL];
#pragma unroll
    for (int k = 0; k < SL; ++k) v[k] = h[k] ? __ldg(x + r * cols + lane + 32 * k) : 0.0;
    row_step(r, gid[r], v);
  }
  const bool ends_here = (r1 == rows) || (gid[r1] != seg);
#pragma unroll
  for (int k = 0; k < SL; ++k)
    if (h[k]) {
      if (ends_here && seg >= 0) totals[(int64_t)seg * cols + lane + 32 * k] = s[k];
      agg[t * cols + lane + 32 * k] = s[k];
    }
  if (lane == 0) flag[t] = any_start;
}

// Keyed tile pass for <= CP columns (CP = 8 or 16): a warp load covers R = 32 / CP rows
// (lane = (row slot, column)), 32 rows per iteration in flight -- twice the bytes of the
// narrow pass, whose lanes 16-31 sit idle on a 16-column row -- and lanes 0 .. cols-1 run
// the same row-by-row segment logic on the values shuffled to them: the same additions in
// the same order as segscan_tile_narrow, so the same bits.
template <int CP>
__device__ __forceinline__ void segscan_tile_tiny(const double* __restrict__ x, int64_t rows, int cols,
                                                  const int32_t* __restrict__ gid, int64_t t,
                                                  double* __restrict__ agg, int* __restrict__ flag,
                                                  double* __restrict__ totals, int lane) {
  constexpr int R = 32 / CP, RB = 32, NI = RB / R;
  const int64_t r0 = t * TILE_ROWS, r1 = min(rows, r0 + TILE_ROWS);
  const int slot = lane / CP, col = lane % CP;
  const bool h = lane < cols;  // a processing lane: slot 0 and a real column
  int seg = gid[r0];
  int any_start = (r0 == 0) || (gid[r0 - 1] != seg);
  double s = 0.0;
  auto row_step = [&](int64_t rr, int sr, double v) {
    const bool start = (rr == 0) || (rr > r0 && sr != seg);
    if (start && rr > r0) {
      if (seg >= 0 && h) totals[(int64_t)seg * cols + lane] = s;
      any_start = 1;
    }
    seg = sr;
    s = start ? v : s + v;
  };
  int64_t r = r0;
  for (; r + RB <= r1; r += RB) {
    int g[RB];
    double v[NI];  // load u: row r + u R + slot, column col
#pragma unroll
    for (int u = 0; u < RB; ++u) g[u] = gid[r + u];
#pragma unroll
    for (int u = 0; u < NI; ++u) v[u] = col < cols ? __ldg(x + (r + (int64_t)u * R + slot) * cols + col) : 0.0;
    bool uniform = r != 0;
#pragma unroll
    for (int u = 0; u < RB; ++u) uniform = uniform && g[u] == seg;
    if (uniform) {
#pragma unroll
      for (int u = 0; u < NI; ++u)
#pragma unroll
        for (int j = 0; j < R; ++j) s = s + __shfl_sync(0xffffffffu, v[u], j * CP + col);
    } else {
#pragma unroll
      for (int u = 0; u < NI; ++u)
#pragma unroll
        for (int j = 0; j < R; ++j)
          row_step(r + u * R + j, g[u * R + j], __shfl_sync(0xffffffffu, v[u], j * CP + col));
    }
  }
  for (; r < r1; ++r) row_step(r, gid[r], h ? __ldg(x + r * cols + lane) : 0.0);
  const bool ends_here = (r1 == rows) || (gid[r1] != seg);
  if (h) {
    if (ends_here && seg >= 0) totals[(int64_t)seg * cols + lane] = s;
    agg[t * cols + lane] = s;
  }
  if (lane == 0) flag[t] = any_start;
}

}  // namespace jq
