// jq_group.cu — join-key grouping on the GPU, bit-exact with the reference's
// grouping (keys sorted non-decreasing, groups = key values
// present on BOTH sides, ascending key order :223, reduced-row count
// sum_g (m1g + m2g - 1) :184).  The numpy restatement in oracle/joins.py
// (`group_keys`: unique -> intersect1d -> cumsum) is the parity target.
//
// Pipeline (all integer, hence deterministic):
//   per 2048-key tile (both sides in one launch): run heads + sortedness check ->
//   tile offsets (one CTA) -> run tables (start, key) + run id per row (one launch) ->
//   binary-search match of A runs in B runs ->
//   scan of match flags = group ids in ascending key order -> group tables,
//   red_off = exclusive scan of (a_count + b_count - 1) -> per-row group ids.
// Tables that arrive unsorted are sorted first, opt-in, by the GPU stable LSD radix
// sort of jq_sort.cu (bit-exact with np.argsort(kind="stable")); the default keeps the
// SPEC's ValueError for unsorted keys.
#include <algorithm>

#include "jq_internal.cuh"

namespace jq {

// ------------------------------------------------------------------ scan (int64)
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;  // (load_keys8 and the run-id stores assume 8)
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t* warp_sums, int64_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < SCAN_THREADS / 32 ? warp_sums[lane] : 0;
    int64_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < SCAN_THREADS / 32) warp_sums[lane] = wi - w;
    if (lane == SCAN_THREADS / 32 - 1) *total = wi;
  }
  __syncthreads();
  int64_t r = warp_sums[warp] + incl - v;
  __syncthreads();
  return r;
}

__global__ void scan_reduce_kernel(const int64_t* __restrict__ in, int64_t n, const int64_t* n_dev,
                                   int64_t* __restrict__ partial) {
  if (n_dev) n = min(n, n_dev[0]);
  __shared__ int64_t ws[SCAN_THREADS / 32];
  __shared__ int64_t tot;
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
  int64_t s = 0;
#pragma unroll
  for (int u = 0; u < SCAN_ITEMS; ++u)
    if (base + u < n) s += in[base + u];
  block_exclusive_scan(s, ws, &tot);
  if (threadIdx.x == 0) partial[blockIdx.x] = tot;
}

// In-place exclusive scan of c[0 .. nt) by ONE block of SCAN_THREADS threads; returns the
// total.  Rounds of SCAN_TILE values, SCAN_ITEMS consecutive values per thread loaded
// together (one global round trip per 2048 values instead of per 256).  Integer: the
// result does not depend on the association.
__device__ __forceinline__ int64_t block_scan_inplace(int64_t* c, int64_t nt, int64_t* ws, int64_t* tot) {
  int64_t carry = 0;
  for (int64_t b0 = 0; b0 < nt; b0 += SCAN_TILE) {
    const int64_t i0 = b0 + (int64_t)threadIdx.x * SCAN_ITEMS;
    int64_t v[SCAN_ITEMS], sum = 0;
#pragma unroll
    for (int u = 0; u < SCAN_ITEMS; ++u) {
      v[u] = i0 + u < nt ? c[i0 + u] : 0;
      sum += v[u];
    }
    int64_t run = carry + block_exclusive_scan(sum, ws, tot);
#pragma unroll
    for (int u = 0; u < SCAN_ITEMS; ++u)
      if (i0 + u < nt) {
        c[i0 + u] = run;
        run += v[u];
      }
    carry += *tot;
    __syncthreads();
  }
  return carry;
}

__global__ void scan_partials_kernel(int64_t* partial, int64_t nb) {
  __shared__ int64_t ws[SCAN_THREADS / 32];
  __shared__ int64_t tot;
  const int64_t carry = block_scan_inplace(partial, nb, ws, &tot);
  if (threadIdx.x == 0) partial[nb] = carry;
}

__global__ void scan_apply_kernel(const int64_t* __restrict__ in, int64_t n, const int64_t* n_dev,
                                  const int64_t* __restrict__ partial, int64_t nb, int64_t* __restrict__ out) {
  if (n_dev) n = min(n, n_dev[0]);
  __shared__ int64_t ws[SCAN_THREADS / 32];
  __shared__ int64_t tot;
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE + threadIdx.x * SCAN_ITEMS;
  int64_t v[SCAN_ITEMS], s = 0;
#pragma unroll
  for (int u = 0; u < SCAN_ITEMS; ++u) {
    v[u] = base + u < n ? in[base + u] : 0;
    s += v[u];
  }
  int64_t ex = block_exclusive_scan(s, ws, &tot) + partial[blockIdx.x];
#pragma unroll
  for (int u = 0; u < SCAN_ITEMS; ++u) {
    if (base + u < n) out[base + u] = ex;
    ex += v[u];
  }
  if (base <= n && n < base + SCAN_ITEMS) out[n] = partial[nb];  // total at [len]
  if (n == 0 && blockIdx.x == 0 && threadIdx.x == 0) out[0] = 0;
}

size_t scan_ws_bytes(int64_t n) { return ws_bytes(size_t(cdiv(std::max<int64_t>(n, 1), SCAN_TILE)) + 1, 8); }

int scan_i64_dev(jq_ctx* ctx, const int64_t* in, int64_t n, const int64_t* n_dev, int64_t* out) {
  int64_t nb = std::max<int64_t>(1, cdiv(n + 1, SCAN_TILE));
  int64_t* partial = ws_alloc<int64_t>(ctx, nb + 1);
  if (!partial) return fail(JQ_E_OOM, "workspace exhausted (scan)");
  scan_reduce_kernel<<<(unsigned)nb, SCAN_THREADS, 0, ctx->stream>>>(in, n, n_dev, partial);
  JQ_CHECK_LAUNCH(ctx);
  scan_partials_kernel<<<1, SCAN_THREADS, 0, ctx->stream>>>(partial, nb);
  JQ_CHECK_LAUNCH(ctx);
  scan_apply_kernel<<<(unsigned)nb, SCAN_THREADS, 0, ctx->stream>>>(in, n, n_dev, partial, nb, out);
  JQ_CHECK_LAUNCH(ctx);
  return JQ_OK;
}

// ------------------------------------------------------------------ grouping kernels
static unsigned gridn(int64_t n, int threads = 256) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, threads), 148 * 32));
}
#define GRID_STRIDE(i, n)                                                        \
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n);      \
       i += (int64_t)gridDim.x * blockDim.x)

__global__ void check_sorted_kernel(const int64_t* __restrict__ k, int64_t n, int bit, int* flags) {
  int bad = 0;
  GRID_STRIDE(i, n - 1) bad |= k[i] > k[i + 1];
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flags, bit);
}

// match A runs against B runs (both ascending): match[u] = index of equal key in B or -1
__global__ void match_kernel(const int64_t* __restrict__ ka_run, const int64_t* __restrict__ nra_p,
                             const int64_t* __restrict__ kb_run, const int64_t* __restrict__ nrb_p,
                             int64_t* __restrict__ match, int64_t* __restrict__ mflag) {
  const int64_t nra = nra_p[0], nrb = nrb_p[0];
  GRID_STRIDE(u, nra) {
    const int64_t key = ka_run[u];
    int64_t lo = 0, hi = nrb;  // first index with kb_run >= key
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (kb_run[mid] < key) lo = mid + 1; else hi = mid;
    }
    const bool hit = lo < nrb && kb_run[lo] == key;
    match[u] = hit ? lo : -1;
    mflag[u] = hit ? 1 : 0;
  }
}

__global__ void group_tables_kernel(const int64_t* __restrict__ match, const int64_t* __restrict__ gidx,
                                    const int64_t* __restrict__ nra_p, int64_t m1,
                                    const int64_t* __restrict__ ra_start, const int64_t* __restrict__ ra_key,
                                    const int64_t* __restrict__ nrb_p, int64_t m2,
                                    const int64_t* __restrict__ rb_start, int64_t* __restrict__ keys,
                                    int64_t* __restrict__ a_start, int64_t* __restrict__ a_count,
                                    int64_t* __restrict__ b_start, int64_t* __restrict__ b_count,
                                    int64_t* __restrict__ rowcnt, int32_t* __restrict__ ra_to_g,
                                    int32_t* __restrict__ rb_to_g) {
  const int64_t nra = nra_p[0], nrb = nrb_p[0];
  GRID_STRIDE(u, nra) {
    const int64_t v = match[u];
    if (v < 0) { ra_to_g[u] = -1; continue; }
    const int64_t gi = gidx[u];
    const int64_t as = ra_start[u], ae = (u + 1 < nra) ? ra_start[u + 1] : m1;
    const int64_t bs = rb_start[v], be = (v + 1 < nrb) ? rb_start[v + 1] : m2;
    keys[gi] = ra_key[u];
    a_start[gi] = as; a_count[gi] = ae - as;
    b_start[gi] = bs; b_count[gi] = be - bs;
    rowcnt[gi] = (ae - as) + (be - bs) - 1;
    ra_to_g[u] = (int32_t)gi;
    rb_to_g[v] = (int32_t)gi;
  }
}

__global__ void fill_i32_kernel(int32_t* p, int64_t n, int32_t v) { GRID_STRIDE(i, n) p[i] = v; }

__global__ void finish_counts_kernel(const int64_t* __restrict__ gscan, const int64_t* __restrict__ nra,
                                     const int64_t* __restrict__ red_off, int64_t* d_n) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const int64_t g = gscan[nra[0]];  // total matched = scan at [len]
    d_n[0] = g;
    d_n[1] = red_off[g];
  }
}

// ---- fused run detection, both sides in one launch each (round 2: 14 -> 3 launches)
// Tile t of the concatenated key streams (A tiles, then B tiles; SCAN_TILE keys each).
struct RunSides {
  const int64_t* k[2];
  int64_t m[2];
  int64_t tiles0;      // tiles of side A
  int64_t* cnt;        // [tilesA + tilesB] run heads per tile -> exclusive offsets (in place)
  int64_t* rs[2];      // run start row
  int64_t* rk[2];      // run key
  int32_t* runid[2];   // run index of every row
  int32_t* r_to_g_b;   // side B runs -> group (initialised to -1 here)
  int* flags;
};
__device__ __forceinline__ void run_tile(const RunSides& rs, int64_t& t, int& side, int64_t& i0, int64_t& i1) {
  side = t < rs.tiles0 ? 0 : 1;
  if (side) t -= rs.tiles0;
  i0 = t * SCAN_TILE;
  i1 = min(rs.m[side], i0 + SCAN_TILE);
}
// the thread's SCAN_ITEMS consecutive keys k[b .. b+7] (0 past i1) and the key before
// them: 16-byte loads when the key array is 16-byte aligned and the 8 keys are whole
// (4 LDG.128 + 1 LDG.64 instead of 16 LDG.64)
__device__ __forceinline__ void load_keys8(const int64_t* __restrict__ k, int64_t b, int64_t i1, int64_t (&key)[SCAN_ITEMS],
                                           int64_t& prev) {
  prev = b > 0 && b - 1 < i1 ? __ldg(k + b - 1) : 0;
  if (((reinterpret_cast<uintptr_t>(k) & 15) == 0) && b + SCAN_ITEMS <= i1) {
    const longlong2* k2 = reinterpret_cast<const longlong2*>(k + b);
#pragma unroll
    for (int u = 0; u < SCAN_ITEMS / 2; ++u) {
      const longlong2 v = __ldg(k2 + u);
      key[2 * u] = v.x;
      key[2 * u + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int u = 0; u < SCAN_ITEMS; ++u) key[u] = b + u < i1 ? __ldg(k + b + u) : 0;
  }
}

// heads per tile + the sortedness check (unsorted keys raise)
__global__ void __launch_bounds__(SCAN_THREADS) run_count_kernel(RunSides rs) {
  __shared__ int64_t ws[SCAN_THREADS / 32];
  __shared__ int64_t tot;
  int64_t t = blockIdx.x, i0, i1;
  int side;
  run_tile(rs, t, side, i0, i1);
  const int64_t* k = rs.k[side];
  int64_t h = 0;
  int bad = 0;
  const int64_t b = i0 + threadIdx.x * SCAN_ITEMS;
  int64_t key[SCAN_ITEMS], prev;
  load_keys8(k, b, i1, key, prev);
#pragma unroll
  for (int u = 0; u < SCAN_ITEMS; ++u) {
    const int64_t i = b + u;
    if (i < i1) {
      const int64_t ki = key[u];
      if (i == 0) h += 1;
      else {
        const int64_t kp = u == 0 ? prev : key[u - 1];
        h += ki != kp;
        bad |= kp > ki;
      }
    }
  }
  block_exclusive_scan(h, ws, &tot);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(rs.flags, side ? FLAG_UNSORTED_B : FLAG_UNSORTED_A);
  if (threadIdx.x == 0) rs.cnt[blockIdx.x] = tot;
}
// exclusive offsets of the per-tile counts, per side (one CTA); runs of A / B -> nr[0..1]
__global__ void __launch_bounds__(SCAN_THREADS) run_offsets_kernel(int64_t* cnt, int64_t tiles0, int64_t tiles1,
                                                                   int64_t* nr) {
  __shared__ int64_t ws[SCAN_THREADS / 32];
  __shared__ int64_t tot;
  for (int side = 0; side < 2; ++side) {
    int64_t* c = cnt + (side ? tiles0 : 0);
    const int64_t nt = side ? tiles1 : tiles0;
    const int64_t carry = block_scan_inplace(c, nt, ws, &tot);
    if (threadIdx.x == 0) nr[side] = carry;
  }
}
// run tables (start row, key) at the heads, run id of every row; B's run -> group map = -1
__global__ void __launch_bounds__(SCAN_THREADS) run_tables_fused_kernel(RunSides rs) {
  __shared__ int64_t ws[SCAN_THREADS / 32];
  __shared__ int64_t tot;
  int64_t t = blockIdx.x, i0, i1;
  int side;
  run_tile(rs, t, side, i0, i1);
  const int64_t* k = rs.k[side];
  const int64_t b = i0 + threadIdx.x * SCAN_ITEMS;
  int64_t key[SCAN_ITEMS], prev;
  int hd[SCAN_ITEMS];
  int64_t h = 0;
  load_keys8(k, b, i1, key, prev);
#pragma unroll
  for (int u = 0; u < SCAN_ITEMS; ++u) {
    const int64_t i = b + u;
    hd[u] = 0;
    if (i < i1) {
      hd[u] = (i == 0 || (u == 0 ? prev : key[u - 1]) != key[u]) ? 1 : 0;
      h += hd[u];
    }
  }
  int64_t run = rs.cnt[blockIdx.x] + block_exclusive_scan(h, ws, &tot);  // heads before this thread
  int32_t rid[SCAN_ITEMS];
#pragma unroll
  for (int u = 0; u < SCAN_ITEMS; ++u) {
    const int64_t i = b + u;
    rid[u] = 0;
    if (i < i1) {
      if (hd[u]) {
        rs.rs[side][run] = i;
        rs.rk[side][run] = key[u];
        if (side) rs.r_to_g_b[run] = -1;
        ++run;
      }
      rid[u] = (int32_t)(run - 1);
    }
  }
  int32_t* out = rs.runid[side] + b;
  if (((reinterpret_cast<uintptr_t>(out) & 15) == 0) && b + SCAN_ITEMS <= i1) {  // two 16-byte stores
    reinterpret_cast<int4*>(out)[0] = make_int4(rid[0], rid[1], rid[2], rid[3]);
    reinterpret_cast<int4*>(out)[1] = make_int4(rid[4], rid[5], rid[6], rid[7]);
  } else {
#pragma unroll
    for (int u = 0; u < SCAN_ITEMS; ++u)
      if (b + u < i1) out[u] = rid[u];
  }
}

// gid[i] = run_to_group[runid[i]] for both sides, four rows per thread (16-byte loads and
// stores; the run ids and gid arrays are workspace allocations, 256-byte aligned)
__device__ __forceinline__ void row_gid_side(const int32_t* __restrict__ runid, int64_t m,
                                             const int32_t* __restrict__ r_to_g, int32_t* __restrict__ gid,
                                             int64_t q) {
  const int64_t i = 4 * q;
  if (i + 4 <= m) {
    const int4 r = __ldg(reinterpret_cast<const int4*>(runid + i));
    reinterpret_cast<int4*>(gid + i)[0] = make_int4(__ldg(r_to_g + r.x), __ldg(r_to_g + r.y), __ldg(r_to_g + r.z),
                                                    __ldg(r_to_g + r.w));
  } else {
    for (int64_t j = i; j < m; ++j) gid[j] = r_to_g[runid[j]];
  }
}
__global__ void row_gid2_kernel(const int32_t* __restrict__ runid_a, int64_t m1, const int32_t* __restrict__ ra_to_g,
                                int32_t* __restrict__ gid_a, const int32_t* __restrict__ runid_b, int64_t m2,
                                const int32_t* __restrict__ rb_to_g, int32_t* __restrict__ gid_b) {
  const int64_t qa = (m1 + 3) / 4, qb = (m2 + 3) / 4;
  GRID_STRIDE(q, qa + qb) {
    if (q < qa) row_gid_side(runid_a, m1, ra_to_g, gid_a, q);
    else row_gid_side(runid_b, m2, rb_to_g, gid_b, q - qa);
  }
}

size_t group_ws_bytes(int64_t m1, int64_t m2) {
  const int64_t m = std::max<int64_t>(1, m1), mb = std::max<int64_t>(1, m2);
  const int64_t cap = std::max<int64_t>(1, std::min(m1, m2));
  size_t b = 0;
  // heads, scans (n+1), run_start, run_key per side
  b += 2 * ws_bytes(m + 1, 8) + 2 * ws_bytes(m, 8) + scan_ws_bytes(m);
  b += 2 * ws_bytes(mb + 1, 8) + 2 * ws_bytes(mb, 8) + scan_ws_bytes(mb);
  // match, mflag, gidx (runs of A), ra_to_g, rb_to_g
  b += 2 * ws_bytes(m, 8) + ws_bytes(m + 1, 8) + ws_bytes(m, 4) + ws_bytes(mb, 4) + scan_ws_bytes(m);
  // group tables + red_off + rowcnt
  b += 6 * ws_bytes(cap + 1, 8) + scan_ws_bytes(cap);
  // gid per row, counters
  b += ws_bytes(m, 4) + ws_bytes(mb, 4) + ws_bytes(8, 8);
  return b;
}

int group_keys_dev(jq_ctx* ctx, const int64_t* ka, int64_t m1, const int64_t* kb, int64_t m2, Groups* g) {
  const int64_t cap = std::max<int64_t>(1, std::min(m1, m2));
  const int64_t M1 = std::max<int64_t>(1, m1), M2 = std::max<int64_t>(1, m2);
  int32_t* runid_a = ws_alloc<int32_t>(ctx, M1);
  int64_t* rs_a = ws_alloc<int64_t>(ctx, M1);
  int64_t* rk_a = ws_alloc<int64_t>(ctx, M1);
  int32_t* runid_b = ws_alloc<int32_t>(ctx, M2);
  int64_t* tile_cnt = ws_alloc<int64_t>(ctx, cdiv(M1, SCAN_TILE) + cdiv(M2, SCAN_TILE) + 2);
  int64_t* rs_b = ws_alloc<int64_t>(ctx, M2);
  int64_t* rk_b = ws_alloc<int64_t>(ctx, M2);
  int64_t* match = ws_alloc<int64_t>(ctx, M1);
  int64_t* mflag = ws_alloc<int64_t>(ctx, M1);
  int64_t* gidx = ws_alloc<int64_t>(ctx, M1 + 1);
  int32_t* ra_to_g = ws_alloc<int32_t>(ctx, M1);
  int32_t* rb_to_g = ws_alloc<int32_t>(ctx, M2);
  int64_t* counters = ws_alloc<int64_t>(ctx, 8);
  g->cap = cap;
  g->keys = ws_alloc<int64_t>(ctx, cap + 1);
  g->a_start = ws_alloc<int64_t>(ctx, cap + 1);
  g->a_count = ws_alloc<int64_t>(ctx, cap + 1);
  g->b_start = ws_alloc<int64_t>(ctx, cap + 1);
  g->b_count = ws_alloc<int64_t>(ctx, cap + 1);
  int64_t* rowcnt = ws_alloc<int64_t>(ctx, cap + 1);
  g->red_off = ws_alloc<int64_t>(ctx, cap + 1);
  g->gid_a = ws_alloc<int32_t>(ctx, M1);
  g->gid_b = ws_alloc<int32_t>(ctx, M2);
  if (!g->gid_b || !counters || !rowcnt) return fail(JQ_E_OOM, "workspace exhausted (grouping)");
  g->d_n = counters;  // [0] groups, [1] reduced rows ; [2] runs A, [3] runs B
  int64_t* nra = counters + 2;
  int64_t* nrb = counters + 3;
  JQ_CUDA(cudaMemsetAsync(counters, 0, 8 * sizeof(int64_t), ctx->stream));

  if (m1 == 0 || m2 == 0) {
    if (m1 > 1) {
      check_sorted_kernel<<<gridn(m1), 256, 0, ctx->stream>>>(ka, m1, FLAG_UNSORTED_A, ctx->d_flags);
      JQ_CHECK_LAUNCH(ctx);
    }
    if (m2 > 1) {
      check_sorted_kernel<<<gridn(m2), 256, 0, ctx->stream>>>(kb, m2, FLAG_UNSORTED_B, ctx->d_flags);
      JQ_CHECK_LAUNCH(ctx);
    }
    JQ_CUDA(cudaMemsetAsync(g->red_off, 0, 8, ctx->stream));
    if (m1) { fill_i32_kernel<<<gridn(m1), 256, 0, ctx->stream>>>(g->gid_a, m1, -1); JQ_CHECK_LAUNCH(ctx); }
    if (m2) { fill_i32_kernel<<<gridn(m2), 256, 0, ctx->stream>>>(g->gid_b, m2, -1); JQ_CHECK_LAUNCH(ctx); }
    return JQ_OK;
  }
  if (m1 >= (int64_t(1) << 31) || m2 >= (int64_t(1) << 31))
    return fail(JQ_E_INVALID, "grouping supports fewer than 2^31 rows per table");
  // runs of both sides: heads per tile (+ sortedness), tile offsets, run tables + run ids
  RunSides rsd;
  rsd.k[0] = ka; rsd.k[1] = kb;
  rsd.m[0] = m1; rsd.m[1] = m2;
  const int64_t ta = cdiv(m1, SCAN_TILE), tb = cdiv(m2, SCAN_TILE);
  rsd.tiles0 = ta;
  rsd.cnt = tile_cnt;
  rsd.rs[0] = rs_a; rsd.rs[1] = rs_b;
  rsd.rk[0] = rk_a; rsd.rk[1] = rk_b;
  rsd.runid[0] = runid_a; rsd.runid[1] = runid_b;
  rsd.r_to_g_b = rb_to_g;
  rsd.flags = ctx->d_flags;
  run_count_kernel<<<(unsigned)(ta + tb), SCAN_THREADS, 0, ctx->stream>>>(rsd);
  JQ_CHECK_LAUNCH(ctx);
  run_offsets_kernel<<<1, SCAN_THREADS, 0, ctx->stream>>>(tile_cnt, ta, tb, nra);  // nra, nrb = nra + 1
  JQ_CHECK_LAUNCH(ctx);
  run_tables_fused_kernel<<<(unsigned)(ta + tb), SCAN_THREADS, 0, ctx->stream>>>(rsd);
  JQ_CHECK_LAUNCH(ctx);
  // intersect
  match_kernel<<<gridn(m1), 256, 0, ctx->stream>>>(rk_a, nra, rk_b, nrb, match, mflag);
  JQ_CHECK_LAUNCH(ctx);
  JQ_TRY(scan_i64_dev(ctx, mflag, m1, nra, gidx));
  group_tables_kernel<<<gridn(m1), 256, 0, ctx->stream>>>(match, gidx, nra, m1, rs_a, rk_a, nrb, m2, rs_b,
                                                          g->keys, g->a_start, g->a_count, g->b_start,
                                                          g->b_count, rowcnt, ra_to_g, rb_to_g);
  JQ_CHECK_LAUNCH(ctx);
  // number of groups is gidx[nra]; red_off = exclusive scan of rowcnt over it
  int64_t* ng_dev = counters + 4;
  finish_counts_kernel<<<1, 32, 0, ctx->stream>>>(gidx, nra, gidx, ng_dev);  // ng_dev[0] = groups
  JQ_CHECK_LAUNCH(ctx);
  JQ_TRY(scan_i64_dev(ctx, rowcnt, cap, ng_dev, g->red_off));
  finish_counts_kernel<<<1, 32, 0, ctx->stream>>>(gidx, nra, g->red_off, g->d_n);
  JQ_CHECK_LAUNCH(ctx);
  row_gid2_kernel<<<gridn((m1 + 3) / 4 + (m2 + 3) / 4), 256, 0, ctx->stream>>>(runid_a, m1, ra_to_g, g->gid_a,
                                                                               runid_b, m2, rb_to_g, g->gid_b);
  JQ_CHECK_LAUNCH(ctx);
  return JQ_OK;
}

}  // namespace jq

using namespace jq;

extern "C" int jq_group_keys(jq_ctx* ctx, const int64_t* ka, int64_t m1, const int64_t* kb, int64_t m2,
                             int64_t capacity, int64_t* n_groups, int64_t* keys, int64_t* a_start,
                             int64_t* a_count, int64_t* b_start, int64_t* b_count, int64_t* red_off) {
  if (!ctx) return fail(JQ_E_INVALID, "null context");
  JQ_NVTX("jq_group_keys");
  if (!ka && m1 > 0) return fail(JQ_E_KEYS, "left table has no keys");
  if (!kb && m2 > 0) return fail(JQ_E_KEYS, "right table has no keys");
  JQ_TRY(begin_call(ctx));
  JQ_TRY(ws_reserve(ctx, stage_bytes(ka, m1) + stage_bytes(kb, m2) + group_ws_bytes(m1, m2)));
  const int64_t *dka, *dkb;
  JQ_TRY(stage_in(ctx, ka, m1, &dka));
  JQ_TRY(stage_in(ctx, kb, m2, &dkb));
  Groups gr;
  JQ_TRY(group_keys_dev(ctx, dka, m1, dkb, m2, &gr));
  int64_t hn[2] = {0, 0};
  JQ_CUDA(cudaMemcpyAsync(hn, gr.d_n, 16, cudaMemcpyDeviceToHost, ctx->stream));
  JQ_TRY(sync_and_check_flags(ctx));
  const int64_t ng = hn[0];
  if (n_groups) *n_groups = ng;
  if (ng > capacity) return fail(JQ_E_INVALID, "group output capacity too small");
  if (ng > 0) {
    JQ_TRY(copy_out(ctx, keys, (const int64_t*)gr.keys, ng));
    JQ_TRY(copy_out(ctx, a_start, (const int64_t*)gr.a_start, ng));
    JQ_TRY(copy_out(ctx, a_count, (const int64_t*)gr.a_count, ng));
    JQ_TRY(copy_out(ctx, b_start, (const int64_t*)gr.b_start, ng));
    JQ_TRY(copy_out(ctx, b_count, (const int64_t*)gr.b_count, ng));
  }
  JQ_TRY(copy_out(ctx, red_off, (const int64_t*)gr.red_off, ng + 1));
  return sync_and_check_flags(ctx);
}
