// jq_group.cu — join-key grouping on the GPU, bit-exact with the reference's
// grouping (keys sorted non-decreasing, groups = key values
// present on BOTH sides, ascending key order :223, reduced-row count
// sum_g (m1g + m2g - 1) :184).  The numpy restatement in oracle/joins.py
// (`group_keys`: unique -> intersect1d -> cumsum) is the parity target.
//
// Pipeline (all integer, hence deterministic):
//   sortedness check -> run heads -> exclusive scan = run id per row ->
//   run tables (start, key) -> binary-search match of A runs in B runs ->
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
constexpr int SCAN_ITEMS = 8;
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

__global__ void scan_partials_kernel(int64_t* partial, int64_t nb) {
  __shared__ int64_t ws[SCAN_THREADS / 32];
  __shared__ int64_t tot;
  int64_t carry = 0;
  for (int64_t b0 = 0; b0 < nb; b0 += SCAN_THREADS) {
    int64_t i = b0 + threadIdx.x;
    int64_t v = i < nb ? partial[i] : 0;
    int64_t ex = block_exclusive_scan(v, ws, &tot);
    if (i < nb) partial[i] = carry + ex;
    carry += tot;
    __syncthreads();
  }
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

__global__ void run_head_kernel(const int64_t* __restrict__ k, int64_t n, int64_t* __restrict__ head) {
  GRID_STRIDE(i, n) head[i] = (i == 0 || k[i] != k[i - 1]) ? 1 : 0;
}

// runid[i] = (exclusive scan of heads)[i] + head[i] - 1  -> written in place of the scan
__global__ void run_tables_kernel(const int64_t* __restrict__ k, int64_t n, const int64_t* __restrict__ head,
                                  int64_t* __restrict__ scan, int64_t* __restrict__ run_start,
                                  int64_t* __restrict__ run_key) {
  GRID_STRIDE(i, n) {
    if (head[i]) {
      const int64_t u = scan[i];
      run_start[u] = i;
      run_key[u] = k[i];
    }
  }
}

__global__ void runid_kernel(const int64_t* __restrict__ head, int64_t n, int64_t* __restrict__ scan) {
  GRID_STRIDE(i, n) scan[i] = scan[i] + head[i] - 1;  // run index of row i
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

__global__ void row_gid_kernel(const int64_t* __restrict__ runid, int64_t n, const int32_t* __restrict__ r_to_g,
                               int32_t* __restrict__ gid) {
  GRID_STRIDE(i, n) gid[i] = r_to_g[runid[i]];
}

__global__ void counts_kernel(const int64_t* __restrict__ head_scan_a, int64_t m1,
                              const int64_t* __restrict__ head_a, const int64_t* __restrict__ head_scan_b,
                              int64_t m2, const int64_t* __restrict__ head_b, int64_t* nra, int64_t* nrb) {
  // number of runs = runid[last] + 1 (runid written in place of the scan)
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    nra[0] = m1 ? head_scan_a[m1 - 1] + 1 : 0;
    nrb[0] = m2 ? head_scan_b[m2 - 1] + 1 : 0;
  }
}

__global__ void finish_counts_kernel(const int64_t* __restrict__ gscan, const int64_t* __restrict__ nra,
                                     const int64_t* __restrict__ red_off, int64_t* d_n) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const int64_t g = gscan[nra[0]];  // total matched = scan at [len]
    d_n[0] = g;
    d_n[1] = red_off[g];
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
  int64_t* head_a = ws_alloc<int64_t>(ctx, M1 + 1);
  int64_t* scan_a = ws_alloc<int64_t>(ctx, M1 + 1);
  int64_t* rs_a = ws_alloc<int64_t>(ctx, M1);
  int64_t* rk_a = ws_alloc<int64_t>(ctx, M1);
  int64_t* head_b = ws_alloc<int64_t>(ctx, M2 + 1);
  int64_t* scan_b = ws_alloc<int64_t>(ctx, M2 + 1);
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

  if (m1 > 1) {
    check_sorted_kernel<<<gridn(m1), 256, 0, ctx->stream>>>(ka, m1, FLAG_UNSORTED_A, ctx->d_flags);
    JQ_CHECK_LAUNCH(ctx);
  }
  if (m2 > 1) {
    check_sorted_kernel<<<gridn(m2), 256, 0, ctx->stream>>>(kb, m2, FLAG_UNSORTED_B, ctx->d_flags);
    JQ_CHECK_LAUNCH(ctx);
  }
  if (m1 == 0 || m2 == 0) {
    JQ_CUDA(cudaMemsetAsync(g->red_off, 0, 8, ctx->stream));
    if (m1) { fill_i32_kernel<<<gridn(m1), 256, 0, ctx->stream>>>(g->gid_a, m1, -1); JQ_CHECK_LAUNCH(ctx); }
    if (m2) { fill_i32_kernel<<<gridn(m2), 256, 0, ctx->stream>>>(g->gid_b, m2, -1); JQ_CHECK_LAUNCH(ctx); }
    return JQ_OK;
  }
  // runs of each side
  run_head_kernel<<<gridn(m1), 256, 0, ctx->stream>>>(ka, m1, head_a);
  JQ_CHECK_LAUNCH(ctx);
  JQ_TRY(scan_i64_dev(ctx, head_a, m1, nullptr, scan_a));
  run_tables_kernel<<<gridn(m1), 256, 0, ctx->stream>>>(ka, m1, head_a, scan_a, rs_a, rk_a);
  JQ_CHECK_LAUNCH(ctx);
  runid_kernel<<<gridn(m1), 256, 0, ctx->stream>>>(head_a, m1, scan_a);
  JQ_CHECK_LAUNCH(ctx);
  run_head_kernel<<<gridn(m2), 256, 0, ctx->stream>>>(kb, m2, head_b);
  JQ_CHECK_LAUNCH(ctx);
  JQ_TRY(scan_i64_dev(ctx, head_b, m2, nullptr, scan_b));
  run_tables_kernel<<<gridn(m2), 256, 0, ctx->stream>>>(kb, m2, head_b, scan_b, rs_b, rk_b);
  JQ_CHECK_LAUNCH(ctx);
  runid_kernel<<<gridn(m2), 256, 0, ctx->stream>>>(head_b, m2, scan_b);
  JQ_CHECK_LAUNCH(ctx);
  counts_kernel<<<1, 32, 0, ctx->stream>>>(scan_a, m1, head_a, scan_b, m2, head_b, nra, nrb);
  JQ_CHECK_LAUNCH(ctx);
  // intersect
  match_kernel<<<gridn(m1), 256, 0, ctx->stream>>>(rk_a, nra, rk_b, nrb, match, mflag);
  JQ_CHECK_LAUNCH(ctx);
  JQ_TRY(scan_i64_dev(ctx, mflag, m1, nra, gidx));
  fill_i32_kernel<<<gridn(m2), 256, 0, ctx->stream>>>(rb_to_g, m2, -1);
  JQ_CHECK_LAUNCH(ctx);
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
  row_gid_kernel<<<gridn(m1), 256, 0, ctx->stream>>>(scan_a, m1, ra_to_g, g->gid_a);
  JQ_CHECK_LAUNCH(ctx);
  row_gid_kernel<<<gridn(m2), 256, 0, ctx->stream>>>(scan_b, m2, rb_to_g, g->gid_b);
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
