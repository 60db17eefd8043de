// jq_gen.cu — synthetic inputs on the device (PAPER.md:72:
// "The data in each column follows a uniform distribution in the range (0, 1)").
//
// Counter-based SplitMix64 (element k = row * cols + col of table `seed`):
//   u_k = ((mix64(seed + (k+1) * 0x9E3779B97F4A7C15) >> 11) + 0.5) * 2^-53
// bit-identical to oracle/datagen.py, so any shard / GPU can regenerate any
// element.  Zipf keys: the sorted multiset of searchsorted(cdf, u_row, 'right')
// built as a histogram + scan + run-length fill (integer, hence bit-exact with
// numpy's stable sort of the same keys).
#include <algorithm>

#include "jq_internal.cuh"

namespace jq {

__global__ void gen_uniform_kernel(uint64_t seed, int64_t count, int64_t k0, double* __restrict__ out) {
  // two elements per thread per step, 16-byte stores when aligned
  for (int64_t i = 2 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x); i < count;
       i += 2 * (int64_t)gridDim.x * blockDim.x) {
    const double u0 = splitmix_uniform(seed, (uint64_t)(k0 + i));
    if (i + 1 < count) {
      const double u1 = splitmix_uniform(seed, (uint64_t)(k0 + i + 1));
      if ((reinterpret_cast<uintptr_t>(out + i) & 15) == 0) {
        *reinterpret_cast<double2*>(out + i) = make_double2(u0, u1);
      } else {
        out[i] = u0;
        out[i + 1] = u1;
      }
    } else {
      out[i] = u0;
    }
  }
}

__global__ void zipf_hist_kernel(uint64_t seed, int64_t rows, const double* __restrict__ cdf, int64_t universe,
                                 unsigned long long* __restrict__ hist) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x) {
    const double u = splitmix_uniform(seed, (uint64_t)i);
    int64_t lo = 0, hi = universe;  // first index with cdf > u  (searchsorted 'right')
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (cdf[mid] <= u) lo = mid + 1; else hi = mid;
    }
    atomicAdd(hist + lo, 1ull);
  }
}

// unsorted Zipf keys, one per row: key_i = searchsorted(cdf, u_i, 'right') (oracle zipf_keys)
__global__ void zipf_keys_kernel(uint64_t seed, int64_t rows, const double* __restrict__ cdf, int64_t universe,
                                 int64_t* __restrict__ keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += (int64_t)gridDim.x * blockDim.x) {
    const double u = splitmix_uniform(seed, (uint64_t)i);
    int64_t lo = 0, hi = universe;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(cdf + mid) <= u) lo = mid + 1; else hi = mid;
    }
    keys[i] = lo;
  }
}

__global__ void zipf_fill_kernel(const int64_t* __restrict__ off, int64_t universe, int64_t rows,
                                 int64_t* __restrict__ keys) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < rows; p += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = universe;  // last key with off[key] <= p
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (off[mid] <= p) lo = mid; else hi = mid;
    }
    keys[p] = lo;
  }
}

}  // namespace jq

using namespace jq;

extern "C" int jq_gen_uniform(jq_ctx* ctx, uint64_t seed, int64_t rows, int64_t cols, int64_t row0, double* out) {
  if (!ctx) return fail(JQ_E_INVALID, "null context");
  if (rows < 0 || cols < 0 || row0 < 0) return fail(JQ_E_INVALID, "negative size");
  const int64_t count = rows * cols;
  if (count == 0) return JQ_OK;
  JQ_TRY(begin_call(ctx));
  JQ_TRY(ws_reserve(ctx, stage_bytes((const double*)out, count)));
  double* d;
  JQ_TRY(stage_out(ctx, out, count, &d));
  const int64_t blocks = std::min<int64_t>(cdiv(count, 512), int64_t(ctx->sms) * 16);
  gen_uniform_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(seed, count, row0 * cols, d);
  JQ_CHECK_LAUNCH(ctx);
  JQ_TRY(copy_out(ctx, out, (const double*)d, count));
  return sync_and_check_flags(ctx);
}

extern "C" int jq_gen_zipf_sorted_keys(jq_ctx* ctx, uint64_t seed, int64_t rows, const double* cdf,
                                       int64_t universe, int64_t* keys_out) {
  if (!ctx) return fail(JQ_E_INVALID, "null context");
  if (rows < 0 || universe <= 0) return fail(JQ_E_INVALID, "bad Zipf geometry");
  if (rows == 0) return JQ_OK;
  JQ_TRY(begin_call(ctx));
  JQ_TRY(ws_reserve(ctx, stage_bytes(cdf, universe) + stage_bytes((const int64_t*)keys_out, rows) +
                             2 * ws_bytes(universe + 1, 8) + scan_ws_bytes(universe)));
  const double* dcdf;
  int64_t* dkeys;
  JQ_TRY(stage_in(ctx, cdf, universe, &dcdf));
  JQ_TRY(stage_out(ctx, keys_out, rows, &dkeys));
  int64_t* hist = ws_alloc<int64_t>(ctx, universe + 1);
  int64_t* off = ws_alloc<int64_t>(ctx, universe + 1);
  JQ_CUDA(cudaMemsetAsync(hist, 0, (universe + 1) * 8, ctx->stream));
  const int64_t blocks = std::min<int64_t>(cdiv(rows, 256), int64_t(ctx->sms) * 16);
  zipf_hist_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(seed, rows, dcdf, universe,
                                                              reinterpret_cast<unsigned long long*>(hist));
  JQ_CHECK_LAUNCH(ctx);
  JQ_TRY(scan_i64_dev(ctx, hist, universe, nullptr, off));
  zipf_fill_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(off, universe, rows, dkeys);
  JQ_CHECK_LAUNCH(ctx);
  JQ_TRY(copy_out(ctx, keys_out, (const int64_t*)dkeys, rows));
  return sync_and_check_flags(ctx);
}

extern "C" int jq_gen_zipf_keys(jq_ctx* ctx, uint64_t seed, int64_t rows, const double* cdf, int64_t universe,
                                int64_t* keys_out) {
  if (!ctx) return fail(JQ_E_INVALID, "null context");
  if (rows < 0 || universe <= 0) return fail(JQ_E_INVALID, "bad Zipf geometry");
  if (rows == 0) return JQ_OK;
  JQ_TRY(begin_call(ctx));
  JQ_TRY(ws_reserve(ctx, stage_bytes(cdf, universe) + stage_bytes((const int64_t*)keys_out, rows)));
  const double* dcdf;
  int64_t* dkeys;
  JQ_TRY(stage_in(ctx, cdf, universe, &dcdf));
  JQ_TRY(stage_out(ctx, keys_out, rows, &dkeys));
  const int64_t blocks = std::min<int64_t>(cdiv(rows, 256), int64_t(ctx->sms) * 16);
  zipf_keys_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(seed, rows, dcdf, universe, dkeys);
  JQ_CHECK_LAUNCH(ctx);
  JQ_TRY(copy_out(ctx, keys_out, (const int64_t*)dkeys, rows));
  return sync_and_check_flags(ctx);
}
