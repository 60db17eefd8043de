// jq_sort.cu — stable LSD radix sort of int64 join keys on the GPU, and the row
// gather that applies the permutation to a table.
//
// The reference requires keys sorted non-decreasing and raises otherwise
// (SPEC.md:204-206); tables that arrive unsorted (or the C3 generator, SURVEY.md §8d:
// keys drawn per row, then a stable sort of (key, row) permutes the data rows) are
// sorted here first, opt-in (joins.sort_by_key / figaro_r(..., sort=True)).  The
// permutation equals numpy's np.argsort(keys, kind="stable") bit for bit: stable LSD
// radix sort on the keys with the sign bit flipped (unsigned order == signed order),
// ties kept in row order.
//
// Per 8-bit digit pass (passes whose digit is the same for every key are skipped: one
// histogram pass over the keys decides, e.g. 3 of 8 passes for keys < 2^24):
//   tile_hist_kernel    per 4096-key tile histogram, stored digit-major [256][tiles]
//   scan_i64_dev        exclusive scan of that matrix = each (digit, tile)'s output base
//   scatter_kernel      stable in-tile ranks (warp match_any + per-warp digit counts,
//                       rounds in element order) -> scatter (key, row) to base + rank
// Integer only, hence deterministic and bit-exact.
#include <algorithm>
#include <cstring>

#include "jq_internal.cuh"

namespace jq {

constexpr int RS_THREADS = 256;
constexpr int RS_ITEMS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;   // keys per tile
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr uint64_t SIGN = 0x8000000000000000ull;

__device__ __forceinline__ uint32_t digit_of(int64_t k, int shift) {
  return (uint32_t)(((uint64_t)k ^ SIGN) >> shift) & 0xFFu;
}

// one pass over the keys: the 8 digit histograms (8 x 256 counters)
__global__ void __launch_bounds__(RS_THREADS) digit_hist_kernel(const int64_t* __restrict__ keys, int64_t m,
                                                                unsigned long long* __restrict__ hist) {
  __shared__ unsigned int h[8][256];
  for (int i = threadIdx.x; i < 8 * 256; i += RS_THREADS) (&h[0][0])[i] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)RS_THREADS + threadIdx.x; i < m; i += (int64_t)gridDim.x * RS_THREADS) {
    const uint64_t u = (uint64_t)__ldg(keys + i) ^ SIGN;
#pragma unroll
    for (int p = 0; p < 8; ++p) atomicAdd(&h[p][(u >> (8 * p)) & 0xFF], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 8 * 256; i += RS_THREADS) {
    const unsigned int v = (&h[0][0])[i];
    if (v) atomicAdd(hist + i, (unsigned long long)v);
  }
}

// per-tile digit counts, digit-major: cnt[d * ntiles + tile]
__global__ void __launch_bounds__(RS_THREADS) tile_hist_kernel(const int64_t* __restrict__ keys, int64_t m,
                                                               int shift, int64_t ntiles,
                                                               int64_t* __restrict__ cnt) {
  __shared__ unsigned int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * RS_TILE;
#pragma unroll 4
  for (int r = 0; r < RS_ITEMS; ++r) {
    const int64_t i = base + r * RS_THREADS + threadIdx.x;
    if (i < m) atomicAdd(&h[digit_of(__ldg(keys + i), shift)], 1u);
  }
  __syncthreads();
  cnt[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// Stable scatter of one tile.  Round r handles keys base + r*256 + tid, so the element
// order is (round, warp, lane); within a round a key's rank among equal digits is
// (earlier warps' counts) + (earlier lanes of its warp, __match_any_sync); across rounds
// a running per-digit count.  rows_in == nullptr: row index = position (first pass).
__global__ void __launch_bounds__(RS_THREADS) scatter_kernel(const int64_t* __restrict__ keys_in,
                                                             const int64_t* __restrict__ rows_in, int64_t m,
                                                             int shift, int64_t ntiles,
                                                             const int64_t* __restrict__ offs,
                                                             int64_t* __restrict__ keys_out,
                                                             int64_t* __restrict__ rows_out) {
  __shared__ int64_t base[256];       // running output position per digit
  __shared__ unsigned int wc[RS_WARPS][256];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  base[tid] = offs[(int64_t)tid * ntiles + blockIdx.x];
#pragma unroll
  for (int w = 0; w < RS_WARPS; ++w) wc[w][tid] = 0;
  __syncthreads();
  const int64_t t0 = (int64_t)blockIdx.x * RS_TILE;
  const unsigned lt = (1u << lane) - 1u;
  for (int r = 0; r < RS_ITEMS; ++r) {
    const int64_t i = t0 + r * RS_THREADS + tid;
    const bool live = i < m;
    int64_t k = 0, row = 0;
    uint32_t d = 256 + lane;  // dead lanes: a digit of their own (never matches a live one)
    if (live) {
      k = __ldg(keys_in + i);
      row = rows_in ? __ldg(rows_in + i) : i;
      d = digit_of(k, shift);
    }
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const unsigned wrank = __popc(peers & lt);
    if (live && wrank == 0) wc[warp][d] = __popc(peers);
    __syncthreads();
    {
      // digit tid: exclusive prefix over the warps, then advance the running base
      unsigned int run = 0;
#pragma unroll
      for (int w = 0; w < RS_WARPS; ++w) {
        const unsigned int c = wc[w][tid];
        wc[w][tid] = run;
        run += c;
      }
      // the base read below happens before this thread's update: sync first
      __syncthreads();
      if (live) {
        const int64_t pos = base[d] + wc[warp][d] + wrank;
        keys_out[pos] = k;
        rows_out[pos] = row;
      }
      __syncthreads();
      base[tid] += run;
#pragma unroll
      for (int w = 0; w < RS_WARPS; ++w) wc[w][tid] = 0;
      __syncthreads();
    }
  }
}

// out[i, :] = x[perm[i], :] (row-major).  L lanes per row (L = the row's 16-byte (or
// 8-byte) items rounded up to a power of two, <= 32), 32 / L rows per warp: every row
// is one contiguous read, no per-element integer division.
template <class V>
__global__ void gather_rows_kernel(const V* __restrict__ x, int64_t rows, int64_t items, int lshift,
                                   const int64_t* __restrict__ perm, V* __restrict__ out, int* flags) {
  const int L = 1 << lshift;
  const int lane = threadIdx.x & 31, sub = lane >> lshift, c0 = lane & (L - 1);
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int rpw = 32 >> lshift;
  for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w * rpw < rows; w += warps) {
    const int64_t i = w * rpw + sub;
    if (i >= rows) continue;
    const int64_t pi = __ldg(perm + i);
    if (pi < 0 || pi >= rows) {  // a caller's bad permutation: flag it, never read out of bounds
      if (c0 == 0) atomicOr(flags, FLAG_BADINDEX);
      continue;
    }
    const V* src = x + pi * items;
    V* dst = out + i * items;
    for (int64_t c = c0; c < items; c += L) dst[c] = __ldg(src + c);
  }
}

__global__ void iota_kernel(int64_t* __restrict__ out, int64_t m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = i;
}

size_t sort_ws_bytes(int64_t m) {
  const int64_t ntiles = std::max<int64_t>(1, cdiv(m, RS_TILE));
  return 4 * ws_bytes(std::max<int64_t>(m, 1), 8) + 2 * ws_bytes(size_t(256) * ntiles + 1, 8) +
         scan_ws_bytes(256 * ntiles) + ws_bytes(8 * 256, 8);
}

// Stable sort of keys[m] (device): sorted keys and the permutation (sorted position ->
// original row) into keys_out / perm_out (device, m each).
int sort_keys_dev(jq_ctx* ctx, const int64_t* keys, int64_t m, int64_t* keys_out, int64_t* perm_out) {
  if (m == 0) return JQ_OK;
  const int64_t ntiles = cdiv(m, RS_TILE);
  int64_t* kb[2] = {ws_alloc<int64_t>(ctx, m), ws_alloc<int64_t>(ctx, m)};
  int64_t* rb[2] = {ws_alloc<int64_t>(ctx, m), ws_alloc<int64_t>(ctx, m)};
  int64_t* cnt = ws_alloc<int64_t>(ctx, size_t(256) * ntiles + 1);
  int64_t* offs = ws_alloc<int64_t>(ctx, size_t(256) * ntiles + 1);
  unsigned long long* hist = ws_alloc<unsigned long long>(ctx, 8 * 256);
  if (!kb[1] || !rb[1] || !cnt || !offs || !hist) return fail(JQ_E_OOM, "workspace exhausted (radix sort)");
  // which digit passes move anything (one read of the keys, one host sync)
  JQ_CUDA(cudaMemsetAsync(hist, 0, 8 * 256 * 8, ctx->stream));
  digit_hist_kernel<<<(unsigned)std::min<int64_t>(cdiv(m, RS_THREADS), int64_t(ctx->sms) * 8), RS_THREADS, 0,
                      ctx->stream>>>(keys, m, hist);
  JQ_CHECK_LAUNCH(ctx);
  unsigned long long hh[8 * 256];
  JQ_CUDA(cudaMemcpyAsync(hh, hist, sizeof(hh), cudaMemcpyDeviceToHost, ctx->stream));
  JQ_CUDA(cudaStreamSynchronize(ctx->stream));
  const int64_t* kin = keys;
  const int64_t* rin = nullptr;  // implicit row index on the first executed pass
  int cur = 0;
  for (int p = 0; p < 8; ++p) {
    bool trivial = false;
    for (int d = 0; d < 256; ++d) trivial |= (int64_t)hh[p * 256 + d] == m;
    if (trivial) continue;
    tile_hist_kernel<<<(unsigned)ntiles, RS_THREADS, 0, ctx->stream>>>(kin, m, 8 * p, ntiles, cnt);
    JQ_CHECK_LAUNCH(ctx);
    JQ_TRY(scan_i64_dev(ctx, cnt, 256 * ntiles, nullptr, offs));
    scatter_kernel<<<(unsigned)ntiles, RS_THREADS, 0, ctx->stream>>>(kin, rin, m, 8 * p, ntiles, offs, kb[cur],
                                                                   rb[cur]);
    JQ_CHECK_LAUNCH(ctx);
    kin = kb[cur];
    rin = rb[cur];
    cur ^= 1;
  }
  if (rin == nullptr) {  // every pass trivial: all keys equal, identity permutation
    JQ_CUDA(cudaMemcpyAsync(keys_out, keys, m * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    iota_kernel<<<(unsigned)std::min<int64_t>(cdiv(m, 256), int64_t(ctx->sms) * 16), 256, 0, ctx->stream>>>(perm_out,
                                                                                                         m);
    JQ_CHECK_LAUNCH(ctx);
    return JQ_OK;
  }
  JQ_CUDA(cudaMemcpyAsync(keys_out, kin, m * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  JQ_CUDA(cudaMemcpyAsync(perm_out, rin, m * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  return JQ_OK;
}

int gather_rows_dev(jq_ctx* ctx, const double* x, int64_t rows, int64_t cols, const int64_t* perm, double* out) {
  if (rows == 0 || cols == 0) return JQ_OK;
  const bool vec = (cols % 2 == 0) && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  const int64_t items = vec ? cols / 2 : cols;
  int lshift = 0;
  while ((1 << lshift) < items && lshift < 5) ++lshift;
  const int64_t warps = cdiv(rows, 32 >> lshift);
  const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(warps, 8), int64_t(ctx->sms) * 16);
  if (vec)
    gather_rows_kernel<double2><<<blocks, 256, 0, ctx->stream>>>(reinterpret_cast<const double2*>(x), rows, items,
                                                                 lshift, perm, reinterpret_cast<double2*>(out),
                                                                 ctx->d_flags);
  else
    gather_rows_kernel<double><<<blocks, 256, 0, ctx->stream>>>(x, rows, items, lshift, perm, out, ctx->d_flags);
  JQ_CHECK_LAUNCH(ctx);
  return JQ_OK;
}

}  // namespace jq

using namespace jq;

extern "C" int jq_sort_keys(jq_ctx* ctx, const int64_t* keys, int64_t m, int64_t* keys_out, int64_t* perm_out) {
  if (!ctx) return fail(JQ_E_INVALID, "null context");
  JQ_NVTX("jq_sort_keys");
  if (m < 0) return fail(JQ_E_INVALID, "negative size");
  if (m > 0 && (!keys || !perm_out)) return fail(JQ_E_INVALID, "null keys or permutation output");
  if (m == 0) return JQ_OK;
  JQ_TRY(begin_call(ctx));
  JQ_TRY(ws_reserve(ctx, stage_bytes(keys, m) + stage_bytes((const int64_t*)keys_out, m) +
                             stage_bytes((const int64_t*)perm_out, m) + sort_ws_bytes(m)));
  const int64_t* dk;
  int64_t *dko = nullptr, *dp;
  JQ_TRY(stage_in(ctx, keys, m, &dk));
  JQ_TRY(stage_out(ctx, perm_out, m, &dp));
  if (keys_out) JQ_TRY(stage_out(ctx, keys_out, m, &dko));
  int64_t* tmpk = dko ? dko : ws_alloc<int64_t>(ctx, m);
  if (!tmpk) return fail(JQ_E_OOM, "workspace exhausted (radix sort)");
  JQ_TRY(sort_keys_dev(ctx, dk, m, tmpk, dp));
  if (keys_out) JQ_TRY(copy_out(ctx, keys_out, (const int64_t*)dko, m));
  JQ_TRY(copy_out(ctx, perm_out, (const int64_t*)dp, m));
  return sync_and_check_flags(ctx);
}

extern "C" int jq_gather_rows(jq_ctx* ctx, const double* x, int64_t rows, int64_t cols, const int64_t* perm,
                              double* out) {
  if (!ctx) return fail(JQ_E_INVALID, "null context");
  JQ_NVTX("jq_gather_rows");
  if (rows < 0 || cols < 0) return fail(JQ_E_INVALID, "negative size");
  if (rows == 0 || cols == 0) return JQ_OK;
  if (!x || !perm || !out) return fail(JQ_E_INVALID, "null argument");
  JQ_TRY(begin_call(ctx));
  JQ_TRY(ws_reserve(ctx, stage_bytes(x, rows * cols) + stage_bytes(perm, rows) +
                             stage_bytes((const double*)out, rows * cols)));
  const double* dx;
  const int64_t* dp;
  double* dout;
  JQ_TRY(stage_in(ctx, x, rows * cols, &dx));
  JQ_TRY(stage_in(ctx, perm, rows, &dp));
  JQ_TRY(stage_out(ctx, out, rows * cols, &dout));
  JQ_TRY(gather_rows_dev(ctx, dx, rows, cols, dp, dout));
  JQ_TRY(copy_out(ctx, out, (const double*)dout, rows * cols));
  return sync_and_check_flags(ctx);
}
