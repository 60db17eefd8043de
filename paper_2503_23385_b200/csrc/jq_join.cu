// jq_join.cu — the brute-force side of the oracle module on the GPU:
// the join matrix itself (materialize_cartesian / materialize_natural_join) and the R
// of the join matrix computed WITHOUT the Figaro reduction -- the performance foil of
// the paper's figures (the role cuSOLVER plays there).  The streamed
// variant generates the join rows inside the TSQR data warps (JoinSrc, jq_tsqr.cu), so
// joins far larger than HBM can be factored; the materialised one writes them.
#include <algorithm>
#include <vector>

#include "jq_internal.cuh"

namespace jq {

// One warp per join row: [A_i | B_j] with (i, j) = join_row(v).
__global__ void materialize_kernel(JoinArgs ja, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
  const int n1 = (int)ja.n1, n2 = (int)ja.n2, n = n1 + n2;
  for (int64_t v = w0; v < ja.rows; v += nw) {
    int64_t ia, ib;
    join_row(ja, v, ia, ib);
    double* o = out + v * n;
    for (int c = lane; c < n; c += 32) o[c] = c < n1 ? __ldg(ja.a + ia * n1 + c) : __ldg(ja.b + ib * n2 + (c - n1));
  }
}

// Join geometry: Cartesian (jo = nullptr, rows = m1 m2) or, for keyed tables, the
// matched groups of group_keys_dev and their join-row offsets (prefix of m1g m2g, on
// the host: brute force is for joins whose row count fits int64 comfortably).
static int join_geometry(jq_ctx* ctx, const int64_t* dka, int64_t m1, const int64_t* dkb, int64_t m2,
                         JoinArgs* ja) {
  ja->jo = nullptr;
  ja->ng = 1;
  if (!dka) {
    ja->rows = m1 * m2;
    return JQ_OK;
  }
  Groups gr;
  JQ_TRY(group_keys_dev(ctx, dka, m1, dkb, m2, &gr));
  int64_t hn[2];
  JQ_CUDA(cudaMemcpyAsync(hn, gr.d_n, 16, cudaMemcpyDeviceToHost, ctx->stream));
  JQ_TRY(sync_and_check_flags(ctx));
  const int64_t ng = hn[0];
  ja->ng = ng;
  ja->rows = 0;
  if (ng == 0) return JQ_OK;
  std::vector<int64_t> ac(ng), bc(ng), jo(ng + 1);
  JQ_CUDA(cudaMemcpyAsync(ac.data(), gr.a_count, ng * 8, cudaMemcpyDeviceToHost, ctx->stream));
  JQ_CUDA(cudaMemcpyAsync(bc.data(), gr.b_count, ng * 8, cudaMemcpyDeviceToHost, ctx->stream));
  JQ_CUDA(cudaStreamSynchronize(ctx->stream));
  jo[0] = 0;
  for (int64_t g = 0; g < ng; ++g) jo[g + 1] = jo[g] + ac[g] * bc[g];
  int64_t* djo = ws_alloc<int64_t>(ctx, ng + 1);
  if (!djo) return fail(JQ_E_OOM, "workspace exhausted (join offsets)");
  JQ_CUDA(cudaMemcpyAsync(djo, jo.data(), (ng + 1) * 8, cudaMemcpyHostToDevice, ctx->stream));
  JQ_CUDA(cudaStreamSynchronize(ctx->stream));  // jo (host) goes out of scope
  ja->jo = djo;
  ja->a_start = gr.a_start;
  ja->b_start = gr.b_start;
  ja->b_count = gr.b_count;
  ja->rows = jo[ng];
  return JQ_OK;
}

static int check_join_args(int64_t m1, int64_t n1, const int64_t* ka, int64_t m2, int64_t n2, const int64_t* kb) {
  if ((ka == nullptr) != (kb == nullptr)) return fail(JQ_E_KEYS, "both tables must carry keys, or neither");
  if (m1 < 0 || m2 < 0 || n1 < 0 || n2 < 0) return fail(JQ_E_INVALID, "negative size");
  if (n1 + n2 == 0) return fail(JQ_E_INVALID, "the join has no columns");
  if (n1 + n2 > 256) return fail(JQ_E_INVALID, "n1 + n2 above 256 is not supported");
  if (!ka && (m1 == 0 || m2 == 0)) return fail(JQ_E_INVALID, "materialize_cartesian needs non-empty inputs");
  return JQ_OK;
}

}  // namespace jq

using namespace jq;

extern "C" int jq_materialize(jq_ctx* ctx, const double* a, int64_t m1, int64_t n1, const int64_t* ka,
                              const double* b, int64_t m2, int64_t n2, const int64_t* kb, double* out,
                              int64_t out_capacity, int64_t* out_rows) {
  if (!ctx) return fail(JQ_E_INVALID, "null context");
  JQ_TRY(check_join_args(m1, n1, ka, m2, n2, kb));
  JQ_TRY(begin_call(ctx));
  const int64_t n = n1 + n2;
  size_t need = stage_bytes(a, m1 * n1) + stage_bytes(b, m2 * n2) + stage_bytes(ka, m1) + stage_bytes(kb, m2) +
                (ka ? group_ws_bytes(m1, m2) + ws_bytes(std::min(m1, m2) + 2, 8) : 0) + 4096;
  if (out) need += stage_bytes((const double*)out, out_capacity * n);
  JQ_TRY(ws_reserve(ctx, need));
  const int64_t *dka = nullptr, *dkb = nullptr;
  JQ_TRY(stage_in(ctx, ka, m1, &dka));
  JQ_TRY(stage_in(ctx, kb, m2, &dkb));
  JoinArgs ja{};
  ja.m1 = m1; ja.n1 = n1; ja.m2 = m2; ja.n2 = n2;
  JQ_TRY(join_geometry(ctx, dka, m1, dkb, m2, &ja));
  if (out_rows) *out_rows = ja.rows;
  if (!out || ja.rows == 0) return sync_and_check_flags(ctx);
  if (out_capacity < ja.rows) return fail(JQ_E_INVALID, "output buffer too small for the join matrix");
  double* dout;
  JQ_TRY(stage_in(ctx, a, m1 * n1, &ja.a));
  JQ_TRY(stage_in(ctx, b, m2 * n2, &ja.b));
  JQ_TRY(stage_out(ctx, out, ja.rows * n, &dout));
  const unsigned grid = (unsigned)std::min<int64_t>(cdiv(ja.rows * 32, 256), int64_t(ctx->sms) * 16);
  materialize_kernel<<<grid, 256, 0, ctx->stream>>>(ja, dout);
  JQ_CHECK_LAUNCH(ctx);
  JQ_TRY(copy_out(ctx, out, (const double*)dout, ja.rows * n));
  return sync_and_check_flags(ctx);
}

extern "C" int jq_join_r_bruteforce(jq_ctx* ctx, const double* a, int64_t m1, int64_t n1, const int64_t* ka,
                                    const double* b, int64_t m2, int64_t n2, const int64_t* kb, double* r) {
  if (!ctx) return fail(JQ_E_INVALID, "null context");
  JQ_TRY(check_join_args(m1, n1, ka, m2, n2, kb));
  JQ_TRY(begin_call(ctx));
  const int64_t n = n1 + n2;
  JQ_TRY(ws_reserve(ctx, stage_bytes(a, m1 * n1) + stage_bytes(b, m2 * n2) + stage_bytes(ka, m1) +
                             stage_bytes(kb, m2) + stage_bytes((const double*)r, n * n) +
                             (ka ? group_ws_bytes(m1, m2) + ws_bytes(std::min(m1, m2) + 2, 8) : 0) +
                             tsqr_ws_bytes(std::max<int64_t>(m1, 1) * std::max<int64_t>(m2, 1), n, ctx->sms)));
  const int64_t *dka = nullptr, *dkb = nullptr;
  JQ_TRY(stage_in(ctx, ka, m1, &dka));
  JQ_TRY(stage_in(ctx, kb, m2, &dkb));
  JoinArgs ja{};
  ja.m1 = m1; ja.n1 = n1; ja.m2 = m2; ja.n2 = n2;
  JQ_TRY(join_geometry(ctx, dka, m1, dkb, m2, &ja));
  double* dr;
  JQ_TRY(stage_in(ctx, a, m1 * n1, &ja.a));
  JQ_TRY(stage_in(ctx, b, m2 * n2, &ja.b));
  JQ_TRY(stage_out(ctx, r, n * n, &dr));
  JQ_TRY(join_tsqr_dev(ctx, ja, dr, true));
  JQ_TRY(copy_out(ctx, r, (const double*)dr, n * n));
  return sync_and_check_flags(ctx);
}
