// jq_api.cu — context, error plumbing, workspace and the figaro_r / figaro_svd
// orchestration of libjoinqr.so (include/joinqr.h).
//
// figaro_r on the device, no host round trip between stages:
//   [keys]  group_keys_dev        bit-exact grouping (jq_group.cu)
//           segscan_dev(B)        head/tail prefix carries + group heads (jq_headtail.cu)
//           figaro_tsqr_dev       fused Claim-1 assembly + TSQR leaves + tree (jq_tsqr.cu)
//           -> canonical R, exact zeros below the diagonal.
// Validation flags (unsorted keys, Jacobi non-convergence) are raised on the
// device and read once at the end of the call.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <utility>
#include <string>
#include <vector>

#include "jq_internal.cuh"

namespace jq {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

int ws_reserve(jq_ctx* ctx, size_t bytes) {
  bytes += 4096;
  if (bytes <= ctx->ws.cap) return JQ_OK;
  if (ctx->ws.base) {
    JQ_CUDA(cudaStreamSynchronize(ctx->stream));
    JQ_CUDA(cudaFree(ctx->ws.base));
    ctx->ws.base = nullptr;
    ctx->ws.cap = 0;
  }
  size_t cap = bytes + bytes / 8;
  cudaError_t e = cudaMalloc(&ctx->ws.base, cap);
  if (e != cudaSuccess) {
    cudaGetLastError();
    ctx->ws.base = nullptr;
    return fail(JQ_E_OOM, "cannot allocate " + std::to_string(cap >> 20) + " MiB of device workspace");
  }
  ctx->ws.cap = cap;
  return JQ_OK;
}

int begin_call(jq_ctx* ctx) {
  JQ_CUDA(cudaSetDevice(ctx->device));
  ws_reset(ctx);
  ctx->tile_launches = 0;
  ctx->tile_bytes = 0.0;
  JQ_CUDA(cudaMemsetAsync(ctx->d_flags, 0, sizeof(int), ctx->stream));
  return JQ_OK;
}

int sync_and_check_flags(jq_ctx* ctx) {
  JQ_CUDA(cudaMemcpyAsync(ctx->h_flags, ctx->d_flags, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  JQ_CUDA(cudaStreamSynchronize(ctx->stream));
  const int f = *ctx->h_flags;
  if (f & FLAG_UNSORTED_A) return fail(JQ_E_UNSORTED, "left table keys are not sorted non-decreasing");
  if (f & FLAG_UNSORTED_B) return fail(JQ_E_UNSORTED, "right table keys are not sorted non-decreasing");
  if (f & FLAG_NOCONV) return fail(JQ_E_NOCONV, "Jacobi SVD did not converge in 64 sweeps");
  if (f & FLAG_BADINDEX) return fail(JQ_E_INVALID, "row permutation entry out of range");
  return JQ_OK;
}

void stage_event(jq_ctx* ctx, int k) {
  static const char* names[8] = {"jq: grouping", "jq: head/tail scan", "jq: scan done", "jq: TSQR leaves",
                                 "jq: TSQR tree", "jq: R done / SVD", "jq: SVD done", "jq: stage 7"};
  cudaEventRecord(ctx->ev[k], ctx->stream);
  nvtxMarkA(names[k & 7]);
}

static float ev_ms(jq_ctx* ctx, int a, int b) {
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, ctx->ev[a], ctx->ev[b]) != cudaSuccess) {
    cudaGetLastError();
    return 0.f;
  }
  return ms;
}

// Workspace needed by figaro_r_dev for these sizes (inputs already on device).
static size_t figaro_ws(int64_t m1, int64_t n1, int64_t m2, int64_t n2, bool keyed, int sms) {
  const int64_t cap = keyed ? std::max<int64_t>(1, std::min(m1, m2)) : 1;
  const int64_t n = n1 + n2;
  if (n > 256)  // wide path: the reduced matrix (<= m1 + m2 - 1 rows) + the wide TSQR
    return (keyed ? group_ws_bytes(m1, m2) : 0) + reduce_emit_ws_bytes(m2, n2, cap) +
           ws_bytes(size_t(m1 + m2) * n, 8) + wide_tsqr_ws_bytes(m1 + m2, n, sms) + ws_bytes(size_t(n) * n, 8);
  size_t dense = (keyed ? group_ws_bytes(m1, m2) : 0) + segscan_ws_bytes(m2, std::max<int64_t>(n2, 1), cap) +
                 figaro_tsqr_ws_bytes(m1, m2, n, sms) + ws_bytes(size_t(n) * n, 8);
  size_t foot = (keyed ? group_ws_bytes(m1, m2) : 0) + segscan_ws_bytes(m1, std::max<int64_t>(n1, 1), cap) +
                segscan_ws_bytes(m2, std::max<int64_t>(n2, 1), cap) + tsqr_ws_bytes(m1 + TILE_ROWS, n1, sms) +
                tsqr_ws_bytes(m2 + TILE_ROWS, n2, sms) + tsqr_ws_bytes(cap, n, sms) +
                tsqr_ws_bytes(3 * n, n, sms) + ws_bytes(size_t(cap) * n, 8) + 8 * ws_bytes(size_t(n) * n, 8) +
                tsqr_pair_ws_bytes(std::max(n1, n2), sms) +
                // carry-free leaves: block sums (the extra stack elements: tsqr_ws_bytes' slack)
                2 * ws_bytes(size_t(sms) * 32 * n, 8);
  return std::max(dense, foot);
}

// ---- footnote variant (PAPER.md:59 footnote) -------------
// Head/tail BOTH sides per key group.  With hA_g = colsum(A_g)/sqrt(m1g) and
// hB_g = colsum(B_g)/sqrt(m2g), J^T J = sum_g hr_g^T hr_g + diag(sum_g m2g TA_g^T TA_g,
// sum_g m1g TB_g^T TB_g) with the head row hr_g = [sqrt(m2g) hA_g | sqrt(m1g) hB_g]
// (same Gram as the Claim-1 matrix, hence the same canonical R).  TSQR work drops
// from 2 (m1+m2) N^2 to 2 (m1 n1^2 + m2 n2^2) + 2 G N^2.
__global__ void head_rows_kernel(const double* __restrict__ totA, int n1, const double* __restrict__ totB, int n2,
                                 const int64_t* __restrict__ a_count, const int64_t* __restrict__ b_count,
                                 int64_t ng, int64_t m1_all, int64_t m2_all, double* __restrict__ out) {
  // one warp per head row (grid-stride), lanes over the columns: the row's two scales once
  // per row, coalesced stores
  const int n = n1 + n2, lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; g < ng; g += nw) {
    const double m1g = a_count ? (double)a_count[g] : (double)m1_all;
    const double m2g = b_count ? (double)b_count[g] : (double)m2_all;
    const double sa = sqrt(m2g) / sqrt(m1g), sb = sqrt(m1g) / sqrt(m2g);
    double* row = out + g * n;
    for (int c = lane; c < n; c += 32) row[c] = c < n1 ? totA[g * n1 + c] * sa : totB[g * n2 + (c - n1)] * sb;
  }
}

// Between-block rows of carry-free leaves (Cartesian footnote).  Each leaf of side X
// took its row block k (m_k rows, column sums s_k) as a group of its own: local tails
// (prefix from 0), no local head.  The between-block part of the centred Gram of X is
//   sum_{k >= 1} v_k v_k^T,  v_k = sqrt(W_k m_k / (W_k + m_k)) (s_k / m_k - S_k / W_k)
// (W_k, S_k: rows and column sums of blocks 0..k-1; the pairwise scatter update), so
// with the footnote scale these P - 1 rows stand in for the carries.  They are written
// as dense NP-row elements behind the side's leaves at odd stack positions (the first
// tree level absorbs element 2c + 1 as rows into R = element 2c; the even elements in
// between are zero R's, block_stack_layout), so the side's own tree takes them in.
// One thread per column (both sides), blocks in a fixed order: deterministic.  Also
// the global head row [sqrt(m2) hA | sqrt(m1) hB] from the block sums.
struct BlockSide {
  const double* sums;
  int64_t p, blk, m;
  int nc;
  double scale;       // sqrt(rows of the other side)
  double* stack;      // the side's leaf stack (p leaves, then the extra elements)
  int64_t first_d;    // stack index of the first dense element
  int np;             // the side's leaf width (stack elements are np x np)
};
__global__ void block_rows_kernel(BlockSide sa, BlockSide sb, double* __restrict__ head) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= sa.nc + sb.nc) return;
  const BlockSide& sd = c < sa.nc ? sa : sb;
  const int cc = c < sa.nc ? c : c - sa.nc;
  const int np = sd.np;
  const size_t nn = size_t(np) * np;
  double W = 0.0, Sk = 0.0;
  for (int64_t k = 0; k < sd.p; ++k) {
    const double mk = (double)min(sd.blk, sd.m - k * sd.blk);
    const double sk = sd.sums[k * sd.nc + cc];
    if (k > 0) {
      const int64_t r = k - 1, j = r / np;
      sd.stack[(sd.first_d + 2 * j) * nn + (r - j * np) * np + cc] =
          sd.scale * sqrt(W * mk / (W + mk)) * (sk / mk - Sk / W);
    }
    W += mk;
    Sk += sk;
  }
  head[c] = sd.scale * (Sk / sqrt((double)sd.m));  // sqrt(m_other) * total / sqrt(m)
}

// extra stack elements behind p leaves: a zero R when p is even, then D0, Z, D1, ..., so
// every dense element D_j sits at an odd index; returns the new count
static int64_t block_stack_layout(int64_t p, int np, int64_t* first_d) {
  const int64_t e = p > 1 ? cdiv(p - 1, np) : 0;
  if (e == 0) { *first_d = p; return p; }
  const int64_t pad = (p % 2 == 0) ? 1 : 0;
  *first_d = p + pad;
  return p + pad + 2 * e - 1;
}

// [blockdiag(R_A, R_B); R_H]: two n x n factors (the first already upper triangular)
__global__ void footnote_stack_kernel(const double* __restrict__ rh, const double* __restrict__ ra, int n1,
                                      const double* __restrict__ rb, int n2, double* __restrict__ out) {
  const int n = n1 + n2;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < 2 * n * n; idx += gridDim.x * blockDim.x) {
    const int k = idx / (n * n), rem = idx - k * n * n, r = rem / n, c = rem - r * n;
    double v;
    if (k == 1) v = rh ? rh[rem] : 0.0;
    else v = (r < n1 && c < n1) ? ra[r * n1 + c] : (r >= n1 && c >= n1) ? rb[(r - n1) * n2 + (c - n1)] : 0.0;
    out[idx] = v;
  }
}

// blockdiag(R_A, R_B) (n x n): the two tail factors already form an upper-triangular R
__global__ void blockdiag_kernel(const double* __restrict__ ra, int n1, const double* __restrict__ rb, int n2,
                                 double* __restrict__ out) {
  const int n = n1 + n2;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n * n; idx += gridDim.x * blockDim.x) {
    const int r = idx / n, c = idx - r * n;
    out[idx] = (r < n1 && c < n1) ? ra[r * n1 + c] : (r >= n1 && c >= n1) ? rb[(r - n1) * n2 + (c - n1)] : 0.0;
  }
}

// Absorb `count` rows (row-major count x n) into the upper-triangular R (n x n, row-major,
// in place) by Givens rotations, row after row, column j of the row zeroed against R[j][j]
// (one CTA, thread = column; row j + 1 of R is fetched while step j runs).  For the few
// head rows of the footnote variant (one for a Cartesian product) this replaces the
// head-row TSQR and the 3-factor stack (two NP x NP combines).
constexpr int GIVENS_THREADS = 256;
__global__ void __launch_bounds__(GIVENS_THREADS) givens_absorb_kernel(double* __restrict__ R,
                                                                       const double* __restrict__ rows, int count,
                                                                       int n) {
  __shared__ double w[GIVENS_THREADS];
  __shared__ double rot[2];
  const int k = threadIdx.x;
  for (int row = 0; row < count; ++row) {
    if (k < n) w[k] = rows[(size_t)row * n + k];
    double rj = k < n ? R[k] : 0.0;  // R[0][k]
    __syncthreads();
    for (int j = 0; j < n; ++j) {
      const double rnext = (j + 1 < n && k < n) ? R[(size_t)(j + 1) * n + k] : 0.0;
      if (k == j) {
        const double a = rj, b = w[j];
        double c = 1.0, s = 0.0;
        if (b != 0.0) {
          const double r = hypot(a, b);
          c = a / r;
          s = b / r;
        }
        rot[0] = c;
        rot[1] = s;
      }
      __syncthreads();
      if (k >= j && k < n) {
        const double c = rot[0], s = rot[1], wk = w[k];
        R[(size_t)j * n + k] = fma(c, rj, s * wk);
        w[k] = k == j ? 0.0 : fma(-s, rj, c * wk);
      }
      rj = rnext;
      __syncthreads();
    }
  }
}

// R from blockdiag(R_A, R_B) and `ng` head rows (few): blockdiag, then Givens.
static int footnote_small_head(jq_ctx* ctx, const double* ra, int64_t n1, const double* rb, int64_t n2,
                               const double* heads, int64_t ng, bool canonical, double* tmp, double* r_out) {
  const int64_t n = n1 + n2;
  double* R = canonical ? tmp : r_out;
  blockdiag_kernel<<<(unsigned)cdiv(n * n, 256), 256, 0, ctx->stream>>>(n1 > 0 ? ra : nullptr, (int)n1,
                                                                        n2 > 0 ? rb : nullptr, (int)n2, R);
  JQ_CHECK_LAUNCH(ctx);
  if (ng > 0) {
    givens_absorb_kernel<<<1, GIVENS_THREADS, 0, ctx->stream>>>(R, heads, (int)ng, (int)n);
    JQ_CHECK_LAUNCH(ctx);
  }
  if (canonical) JQ_TRY(canonicalize_dev(ctx, R, n, r_out));
  return JQ_OK;
}
constexpr int64_t FOOTNOTE_GIVENS_MAX_HEADS = 8;

// Cartesian footnote variant with carry-free leaves (default; JQ_FOOTNOTE_CARRY=scan
// restores the scan-carried leaves for A/B tests): no prefix-scan pass at all -- each
// leaf transforms its own row block (FigaroArgs::blk_sums), block_rows_kernel turns the
// block sums into each side's between-block rows (taken in by the side's own tree) and
// the head row (absorbed by Givens rotations).
static bool carry_free_leaves() {
  static const bool on = [] {
    const char* e = getenv("JQ_FOOTNOTE_CARRY");
    return !(e && !strcmp(e, "scan"));
  }();
  return on;
}
constexpr int64_t BLOCK_LEAVES_MAX_PER_SM = 32;  // bound on leaves per side (workspace)

static int figaro_r_footnote_blocks(jq_ctx* ctx, const double* a, int64_t m1, int64_t n1, const double* b,
                                    int64_t m2, int64_t n2, double* r_out) {
  const int64_t n = n1 + n2;
  const int64_t pmax = int64_t(ctx->sms) * BLOCK_LEAVES_MAX_PER_SM;
  stage_event(ctx, 2);  // no scan stage
  double* ra = ws_alloc<double>(ctx, n1 * n1);
  double* rb = ws_alloc<double>(ctx, n2 * n2);
  double* rh = ws_alloc<double>(ctx, n * n);
  double* sums_a = ws_alloc<double>(ctx, pmax * n1);
  double* sums_b = ws_alloc<double>(ctx, pmax * n2);
  double* head = ws_alloc<double>(ctx, n);
  if (!ra || !rb || !rh || !sums_a || !sums_b || !head)
    return fail(JQ_E_OOM, "workspace exhausted (footnote variant, carry-free leaves)");
  ctx->record_tsqr_events = false;
  ctx->timing.tsqr_ctas = 0;
  ctx->timing.reduced_rows = 0;
  stage_event(ctx, 3);
  FigaroArgs fa{};
  fa.b = a; fa.m2 = m1; fa.n2 = n1;
  fa.m1_global = m2; fa.m2_global = m1;
  fa.blk_sums = sums_a;
  FigaroArgs fb{};
  fb.b = b; fb.m2 = m2; fb.n2 = n2;
  fb.m1_global = m1; fb.m2_global = m2;
  fb.blk_sums = sums_b;
  LeafSet la{}, lb{};
  int rc = figaro_tsqr_leaves(ctx, fa, &la);
  if (!rc) rc = figaro_tsqr_leaves(ctx, fb, &lb);
  if (!rc && (la.count > pmax || lb.count > pmax)) rc = fail(JQ_E_INVALID, "too many TSQR leaves for the block sums");
  if (rc) { ctx->record_tsqr_events = true; return rc; }
  // between-block rows into each side's stack (zeroed extra elements first)
  BlockSide sd[2];
  LeafSet* ls[2] = {&la, &lb};
  const double* sums[2] = {sums_a, sums_b};
  const int64_t ms[2] = {m1, m2}, mo[2] = {m2, m1}, ns[2] = {n1, n2};
  for (int k = 0; k < 2; ++k) {
    LeafSet& L = *ls[k];
    const size_t nn = size_t(L.np) * L.np;
    int64_t first_d = 0;
    const int64_t cnt = block_stack_layout(L.count, L.np, &first_d);
    if (cnt > L.count) JQ_CUDA(cudaMemsetAsync(L.leaves + L.count * nn, 0, (cnt - L.count) * nn * 8, ctx->stream));
    sd[k] = BlockSide{sums[k], L.count, L.rows_per_leaf, ms[k], (int)ns[k], sqrt((double)mo[k]), L.leaves, first_d,
                     L.np};
    L.count = cnt;
  }
  block_rows_kernel<<<(unsigned)cdiv(n, 128), 128, 0, ctx->stream>>>(sd[0], sd[1], head);
  JQ_CHECK_LAUNCH(ctx);
  rc = tsqr_finish_pair(ctx, la, lb, ra, rb);
  if (rc) { ctx->record_tsqr_events = true; return rc; }
  stage_event(ctx, 4);
  rc = footnote_small_head(ctx, ra, n1, rb, n2, head, 1, true, rh, r_out);
  ctx->record_tsqr_events = true;
  stage_event(ctx, 5);
  return rc;
}

// JQ_FOOTNOTE_SERIAL_TREES=1: the keyed footnote's side trees on the main stream, after
// the leaves and before the head rows (A/B)
static bool serial_trees() {
  static const bool on = [] {
    const char* e = getenv("JQ_FOOTNOTE_SERIAL_TREES");
    return e && e[0] == '1';
  }();
  return on;
}
static int ensure_aux(jq_ctx* ctx) {
  if (!ctx->aux_stream) {
    JQ_CUDA(cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking));
    for (auto& e : ctx->aev) JQ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  return JQ_OK;
}

static int figaro_r_footnote_dev(jq_ctx* ctx, const double* a, int64_t m1, int64_t n1, const int64_t* ka,
                                 const double* b, int64_t m2, int64_t n2, const int64_t* kb, double* r_out) {
  const bool keyed = ka != nullptr;
  const int64_t n = n1 + n2;
  stage_event(ctx, 0);
  Groups gr;
  int64_t ng = 1;
  if (keyed) {
    JQ_TRY(group_keys_dev(ctx, ka, m1, kb, m2, &gr));
    int64_t hn[2];
    JQ_CUDA(cudaMemcpyAsync(hn, gr.d_n, 16, cudaMemcpyDeviceToHost, ctx->stream));
    JQ_CUDA(cudaStreamSynchronize(ctx->stream));
    ng = hn[0];
  }
  stage_event(ctx, 1);
  // per-group arrays (scan totals: memset and written per group) sized by the ACTUAL
  // group count, known on the host here -- not by the min(m1, m2) capacity of the
  // grouping tables (at C3 that was 2 x 2.56 GB of memset per call)
  const int64_t cap = keyed ? std::max<int64_t>(ng, 1) : 1;
  if (!keyed && n1 > 0 && n2 > 0 && carry_free_leaves()) return figaro_r_footnote_blocks(ctx, a, m1, n1, b, m2, n2, r_out);
  // A's scan in full; the tile pass of B's scan (the HBM-heavy part) runs on the spare
  // warps of A's TSQR leaf (FigaroArgs::side), B's carries right after it
  SegScan sa{}, sb{};
  SideScan side_b;
  if (n1 > 0)
    JQ_TRY(segscan_dev(ctx, a, m1, n1, keyed ? gr.gid_a : nullptr, keyed ? gr.a_start : nullptr,
                       keyed ? gr.a_count : nullptr, keyed ? gr.d_n : nullptr, cap, &sa));
  if (n2 > 0) JQ_TRY(segscan_begin(ctx, b, m2, n2, keyed ? gr.gid_b : nullptr, cap, &sb, &side_b));
  stage_event(ctx, 2);
  double* ra = ws_alloc<double>(ctx, std::max<int64_t>(n1 * n1, 1));
  double* rb = ws_alloc<double>(ctx, std::max<int64_t>(n2 * n2, 1));
  double* rh = ws_alloc<double>(ctx, n * n);
  double* stack = ws_alloc<double>(ctx, 2 * n * n);
  double* heads = ws_alloc<double>(ctx, std::max<int64_t>(ng, 1) * n);
  if (!ra || !rb || !rh || !stack || !heads) return fail(JQ_E_OOM, "workspace exhausted (footnote variant)");
  ctx->record_tsqr_events = false;
  ctx->timing.tsqr_ctas = 0;
  ctx->timing.reduced_rows = 0;
  stage_event(ctx, 3);
  // tails of A scaled by sqrt(m2g): the "B-part" of a source with an empty A-part
  FigaroArgs fa{};
  LeafSet leaves_a{};
  bool trees_on_aux = false;  // the side trees run on the aux stream (joined before the stack)
  auto join_trees = [&]() {
    if (trees_on_aux) cudaStreamWaitEvent(ctx->stream, ctx->aev[1], 0);
    trees_on_aux = false;
  };
  if (n1 > 0) {
    fa.b = a; fa.m2 = m1; fa.n2 = n1;
    fa.gid_b = keyed ? gr.gid_a : nullptr;
    fa.b_start = keyed ? gr.a_start : nullptr;
    fa.a_count = keyed ? gr.b_count : nullptr;
    fa.b_carry = sa.carry;
    fa.m1_global = m2; fa.m2_global = m1; fa.b_row0 = 0;
    fa.side = side_b;
    // both sides present: leaves now, the two trees later in shared launches
    int rc = n2 > 0 ? figaro_tsqr_leaves(ctx, fa, &leaves_a) : figaro_tsqr_dev(ctx, fa, ra, false);
    if (rc) { ctx->record_tsqr_events = true; return rc; }
  } else {
    JQ_TRY(segscan_tiles(ctx, side_b));
  }
  if (n2 > 0) {
    int rc = segscan_end(ctx, keyed ? gr.b_start : nullptr, keyed ? gr.b_count : nullptr, keyed ? gr.d_n : nullptr,
                         cap, &sb);
    if (rc) { ctx->record_tsqr_events = true; return rc; }
    FigaroArgs fb{};
    fb.b = b; fb.m2 = m2; fb.n2 = n2;
    fb.gid_b = keyed ? gr.gid_b : nullptr;
    fb.b_start = keyed ? gr.b_start : nullptr;
    fb.a_count = keyed ? gr.a_count : nullptr;
    fb.b_carry = sb.carry;
    fb.m1_global = m1; fb.m2_global = m2; fb.b_row0 = 0;
    if (n1 > 0) {
      LeafSet leaves_b{};
      rc = figaro_tsqr_leaves(ctx, fb, &leaves_b);
      if (!rc && ng > FOOTNOTE_GIVENS_MAX_HEADS && !serial_trees()) {
        // the two sides' trees (latency-bound, a few CTAs per level) on the aux stream,
        // beside the head rows' TSQR on this one; joined before the stack below
        rc = ensure_aux(ctx);
        if (!rc) {
          cudaEventRecord(ctx->aev[0], ctx->stream);
          cudaStreamWaitEvent(ctx->aux_stream, ctx->aev[0], 0);
          cudaStream_t main_stream = ctx->stream;
          ctx->stream = ctx->aux_stream;
          rc = tsqr_finish_pair(ctx, leaves_a, leaves_b, ra, rb);
          ctx->stream = main_stream;
          cudaEventRecord(ctx->aev[1], ctx->aux_stream);
          trees_on_aux = true;
        }
      } else if (!rc) {
        rc = tsqr_finish_pair(ctx, leaves_a, leaves_b, ra, rb);
      }
    } else {
      rc = figaro_tsqr_dev(ctx, fb, rb, false);
    }
    if (rc) { ctx->record_tsqr_events = true; return rc; }
  }
  stage_event(ctx, 4);
  if (ng <= FOOTNOTE_GIVENS_MAX_HEADS) {
    if (ng > 0) {
      head_rows_kernel<<<(unsigned)std::min<int64_t>(cdiv(ng, 8), 4096), 256, 0, ctx->stream>>>(
          sa.totals, (int)n1, sb.totals, (int)n2, keyed ? gr.a_count : nullptr, keyed ? gr.b_count : nullptr,
          ng, m1, m2, heads);
      JQ_CHECK_LAUNCH(ctx);
    }
    const int rc = footnote_small_head(ctx, ra, n1, rb, n2, heads, ng, true, rh, r_out);
    ctx->record_tsqr_events = true;
    stage_event(ctx, 5);
    return rc;
  }
  // head rows (G x n) -> R_H, then [blockdiag(R_A, R_B); R_H] -> canonical R
  if (ng > 0) {
    head_rows_kernel<<<(unsigned)std::min<int64_t>(cdiv(ng, 8), 4096), 256, 0, ctx->stream>>>(
        sa.totals, (int)n1, sb.totals, (int)n2, keyed ? gr.a_count : nullptr, keyed ? gr.b_count : nullptr,
        ng, m1, m2, heads);
    JQ_CHECK_LAUNCH(ctx);
    int rc = tsqr_dense_dev(ctx, heads, ng, n, rh, false);
    join_trees();
    if (rc) { ctx->record_tsqr_events = true; return rc; }
  } else {
    JQ_CUDA(cudaMemsetAsync(rh, 0, n * n * 8, ctx->stream));
  }
  join_trees();
  if (getenv("JQ_DEBUG_FOOTNOTE")) {
    cudaStreamSynchronize(ctx->stream);
    auto nan_count = [&](const double* d, int64_t cnt) {
      std::vector<double> h(cnt);
      cudaMemcpy(h.data(), d, cnt * 8, cudaMemcpyDeviceToHost);
      int64_t k = 0; double mx = 0;
      for (double v : h) { k += (v != v); mx = std::max(mx, std::fabs(v)); }
      return std::make_pair(k, mx);
    };
    auto a1 = nan_count(ra, n1 * n1), b1 = nan_count(rb, n2 * n2), h1 = nan_count(rh, n * n),
         hh = nan_count(heads, ng * n);
    fprintf(stderr, "footnote debug: R_A nan=%ld max=%g  R_B nan=%ld max=%g  R_H nan=%ld max=%g  heads nan=%ld max=%g\n",
            (long)a1.first, a1.second, (long)b1.first, b1.second, (long)h1.first, h1.second, (long)hh.first, hh.second);
  }
  footnote_stack_kernel<<<(unsigned)cdiv(2 * n * n, 256), 256, 0, ctx->stream>>>(
      rh, n1 > 0 ? ra : nullptr, (int)n1, n2 > 0 ? rb : nullptr, (int)n2, stack);
  JQ_CHECK_LAUNCH(ctx);
  int rc = tsqr_stack_dev(ctx, stack, 2, n, r_out, true);
  ctx->record_tsqr_events = true;
  stage_event(ctx, 5);
  return rc;
}

// The shard's own between-shard row per side (carry-free leaves on a row shard): the
// shard is block number k of the global group with W = row0 rows and column sums
// `prefix` before it, and local sums s = sum of its leaves' block sums (fixed order), so
//   v = scale sqrt(W m / (W + m)) (s / m - prefix / W)      (W > 0; none for shard 0).
// rows[0] = [v_A | 0], rows[1] = [0 | v_B]; a side with W = 0 gets a zero row.
__global__ void shard_rows_kernel(BlockSide sa, const double* __restrict__ pre_a, int64_t row0_a, BlockSide sb,
                                  const double* __restrict__ pre_b, int64_t row0_b, double* __restrict__ rows) {
  const int n = sa.nc + sb.nc;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const bool side_a = c < sa.nc;
  const BlockSide& sd = side_a ? sa : sb;
  const int cc = side_a ? c : c - sa.nc;
  double sl = 0.0;
  for (int64_t k = 0; k < sd.p; ++k) sl += sd.sums[k * sd.nc + cc];
  const double W = (double)(side_a ? row0_a : row0_b), ml = (double)sd.m;
  const double* pre = side_a ? pre_a : pre_b;
  const double v = (W > 0.0 && ml > 0.0) ? sd.scale * sqrt(W * ml / (W + ml)) * (sl / ml - pre[cc] / W) : 0.0;
  rows[(side_a ? 0 : n) + c] = v;
  rows[(side_a ? n : 0) + c] = 0.0;
}

// Rows that complete the Gram of key groups split by rows across shards (multi-GPU
// co-partition; the Cartesian product is one group split over every
// rank).  Each shard factored its part of group g as a carry-free block: local tails
// scaled by sqrt(m2g) / sqrt(m1g) (jq_figaro_r_shard_local).  What the parts' R's miss
// is, per group, the head row [sqrt(m2g) SA / sqrt(m1g) | sqrt(m1g) SB / sqrt(m2g)] and
// per side one between-part row per part k >= 1 (pairwise scatter update, as
// block_rows_kernel):  v_k = scale sqrt(W m_k / (W + m_k)) (s_k / m_k - S / W).
// One CTA per group, one thread per column, parts in order: deterministic.  Rows of a
// group: head, A rows, B rows from row0[g]; the caller zero-fills `out`.
__global__ void split_group_rows_kernel(const double* __restrict__ sums, const int64_t* __restrict__ prows,
                                        const int64_t* __restrict__ first_part, const int64_t* __restrict__ row0,
                                        const int64_t* __restrict__ na_rows, int n1, int n2,
                                        double* __restrict__ out) {
  const int64_t g = blockIdx.x;
  const int n = n1 + n2;
  const int64_t k0 = first_part[g], k1 = first_part[g + 1];
  double m1g = 0.0, m2g = 0.0;
  for (int64_t k = k0; k < k1; ++k) {
    m1g += (double)prows[2 * k];
    m2g += (double)prows[2 * k + 1];
  }
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    const bool side_a = c < n1;
    const double scale = sqrt(side_a ? m2g : m1g);
    int64_t r = row0[g] + 1 + (side_a ? 0 : na_rows[g]);
    double W = 0.0, S = 0.0;
    for (int64_t k = k0; k < k1; ++k) {
      const double mk = (double)prows[2 * k + (side_a ? 0 : 1)];
      if (mk <= 0.0) continue;
      const double sk = sums[k * n + c];
      if (W > 0.0) out[r++ * n + c] = scale * sqrt(W * mk / (W + mk)) * (sk / mk - S / W);
      W += mk;
      S += sk;
    }
    const double mx = side_a ? m1g : m2g;
    out[row0[g] * n + c] = (mx > 0.0) ? scale * (S / sqrt(mx)) : 0.0;
  }
}

// Column sums of the shard (A then B) from its leaves' block sums, in block order.
__global__ void block_total_kernel(BlockSide sa, BlockSide sb, double* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= sa.nc + sb.nc) return;
  const BlockSide& sd = c < sa.nc ? sa : sb;
  const int cc = c < sa.nc ? c : c - sa.nc;
  double t = 0.0;
  for (int64_t k = 0; k < sd.p; ++k) t += sd.sums[k * sd.nc + cc];
  out[c] = t;
}

// Carry-free leaves on one Cartesian row shard: the shard's leaves take their blocks as
// groups (block_rows_kernel: within-shard between-block rows into the shard's trees),
// shard_rows_kernel adds the shard's own between-shard row per side (from a_prefix /
// a_row0, b_prefix / b_row0), and shard 0 adds the global head row: at most three rows
// for the Givens absorb.  The stacked shard R's then have the Gram of the whole join.
static int footnote_shard_blocks(jq_ctx* ctx, const double* a, int64_t a_rows, int64_t n1, int64_t m1,
                                 int64_t a_row0, const double* a_prefix, const double* a_total, const double* b,
                                 int64_t b_rows, int64_t n2, int64_t m2, int64_t b_row0, const double* b_prefix,
                                 const double* b_total, bool include_head, double* r_out,
                                 double* sums_out = nullptr) {
  const int64_t n = n1 + n2;
  const int64_t pmax = int64_t(ctx->sms) * BLOCK_LEAVES_MAX_PER_SM;
  stage_event(ctx, 2);  // no scan stage
  double* ra = ws_alloc<double>(ctx, n1 * n1);
  double* rb = ws_alloc<double>(ctx, n2 * n2);
  double* rh = ws_alloc<double>(ctx, n * n);
  double* sums_a = ws_alloc<double>(ctx, pmax * n1);
  double* sums_b = ws_alloc<double>(ctx, pmax * n2);
  double* rows = ws_alloc<double>(ctx, 3 * n);
  if (!ra || !rb || !rh || !sums_a || !sums_b || !rows)
    return fail(JQ_E_OOM, "workspace exhausted (footnote shard, carry-free leaves)");
  ctx->record_tsqr_events = false;
  stage_event(ctx, 3);
  FigaroArgs fa{};
  fa.b = a; fa.m2 = a_rows; fa.n2 = n1;
  fa.m1_global = m2; fa.m2_global = m1;
  fa.blk_sums = sums_a;
  FigaroArgs fb{};
  fb.b = b; fb.m2 = b_rows; fb.n2 = n2;
  fb.m1_global = m1; fb.m2_global = m2;
  fb.blk_sums = sums_b;
  LeafSet la{}, lb{};
  int rc = figaro_tsqr_leaves(ctx, fa, &la);
  if (!rc) rc = figaro_tsqr_leaves(ctx, fb, &lb);
  if (!rc && (la.count > pmax || lb.count > pmax)) rc = fail(JQ_E_INVALID, "too many TSQR leaves for the block sums");
  if (rc) { ctx->record_tsqr_events = true; return rc; }
  BlockSide sd[2];
  LeafSet* ls[2] = {&la, &lb};
  const double* sums[2] = {sums_a, sums_b};
  const int64_t ms[2] = {a_rows, b_rows}, mo[2] = {m2, m1}, ns[2] = {n1, n2};
  for (int k = 0; k < 2; ++k) {
    LeafSet& L = *ls[k];
    const size_t nn = size_t(L.np) * L.np;
    int64_t first_d = 0;
    const int64_t cnt = block_stack_layout(L.count, L.np, &first_d);
    if (cnt > L.count) JQ_CUDA(cudaMemsetAsync(L.leaves + L.count * nn, 0, (cnt - L.count) * nn * 8, ctx->stream));
    sd[k] = BlockSide{sums[k], L.count, L.rows_per_leaf, ms[k], (int)ns[k], sqrt((double)mo[k]), L.leaves, first_d,
                     L.np};
  }
  // the shard's rows (uses the leaf counts before the layout change), then the blocks'
  shard_rows_kernel<<<(unsigned)cdiv(n, 128), 128, 0, ctx->stream>>>(sd[0], a_prefix, a_row0, sd[1], b_prefix,
                                                                    b_row0, rows + (include_head ? n : 0));
  JQ_CHECK_LAUNCH(ctx);
  block_rows_kernel<<<(unsigned)cdiv(n, 128), 128, 0, ctx->stream>>>(sd[0], sd[1], rh);  // rh: scratch head
  JQ_CHECK_LAUNCH(ctx);
  if (sums_out) {
    block_total_kernel<<<(unsigned)cdiv(n, 128), 128, 0, ctx->stream>>>(sd[0], sd[1], sums_out);
    JQ_CHECK_LAUNCH(ctx);
  }
  for (int k = 0; k < 2; ++k) ls[k]->count = block_stack_layout(ls[k]->count, ls[k]->np, &sd[k].first_d);
  rc = tsqr_finish_pair(ctx, la, lb, ra, rb);
  if (rc) { ctx->record_tsqr_events = true; return rc; }
  stage_event(ctx, 4);
  if (include_head) {
    head_rows_kernel<<<(unsigned)cdiv(n, 256), 256, 0, ctx->stream>>>(a_total, (int)n1, b_total, (int)n2, nullptr,
                                                                        nullptr, 1, m1, m2, rows);
    JQ_CHECK_LAUNCH(ctx);
  }
  rc = footnote_small_head(ctx, ra, n1, rb, n2, rows, include_head ? 3 : 2, false, rh, r_out);
  ctx->record_tsqr_events = true;
  stage_event(ctx, 5);
  return rc;
}

// Footnote variant on one Cartesian row shard: tails of the local A rows (global
// row index a_row0 + i, prefix a_prefix, scale sqrt(m2)) and of the local B rows,
// plus the global head row when include_head.  Output: local R (n x n, not canonical).
static int footnote_shard_dev(jq_ctx* ctx, const double* a, int64_t a_rows, int64_t n1, int64_t m1, int64_t a_row0,
                              const double* a_prefix, const double* a_total, const double* b, int64_t b_rows,
                              int64_t n2, int64_t m2, int64_t b_row0, const double* b_prefix,
                              const double* b_total, bool include_head, double* r_out) {
  const int64_t n = n1 + n2;
  if (n1 > 0 && n2 > 0 && carry_free_leaves())
    return footnote_shard_blocks(ctx, a, a_rows, n1, m1, a_row0, a_prefix, a_total, b, b_rows, n2, m2, b_row0,
                                 b_prefix, b_total, include_head, r_out);
  SegScan sa{}, sb{};
  SideScan side_b;  // B's tile pass on the spare warps of A's leaf (as in figaro_r_footnote_dev)
  if (n1 > 0) JQ_TRY(segscan_dev(ctx, a, a_rows, n1, nullptr, nullptr, nullptr, nullptr, 1, &sa));
  if (n2 > 0) JQ_TRY(segscan_begin(ctx, b, b_rows, n2, nullptr, 1, &sb, &side_b));
  stage_event(ctx, 2);
  double* ra = ws_alloc<double>(ctx, std::max<int64_t>(n1 * n1, 1));
  double* rb = ws_alloc<double>(ctx, std::max<int64_t>(n2 * n2, 1));
  double* rh = ws_alloc<double>(ctx, n * n);
  double* heads = ws_alloc<double>(ctx, n);
  if (!ra || !rb || !rh || !heads) return fail(JQ_E_OOM, "workspace exhausted (footnote shard)");
  ctx->record_tsqr_events = false;
  stage_event(ctx, 3);
  int rc = JQ_OK;
  if (n1 > 0) {
    FigaroArgs fa{};
    fa.b = a; fa.m2 = a_rows; fa.n2 = n1;
    fa.b_carry = sa.carry; fa.b_prefix0 = a_prefix;
    fa.m1_global = m2; fa.m2_global = m1; fa.b_row0 = a_row0;
    fa.side = side_b;
    rc = figaro_tsqr_dev(ctx, fa, ra, false);
  } else {
    rc = segscan_tiles(ctx, side_b);
  }
  if (!rc && n2 > 0) rc = segscan_end(ctx, nullptr, nullptr, nullptr, 1, &sb);
  if (!rc && n2 > 0) {
    FigaroArgs fb{};
    fb.b = b; fb.m2 = b_rows; fb.n2 = n2;
    fb.b_carry = sb.carry; fb.b_prefix0 = b_prefix;
    fb.m1_global = m1; fb.m2_global = m2; fb.b_row0 = b_row0;
    rc = figaro_tsqr_dev(ctx, fb, rb, false);
  }
  ctx->record_tsqr_events = true;
  if (rc) return rc;
  stage_event(ctx, 4);
  // one head row at most: blockdiag(R_A, R_B) plus a Givens absorb of the head row
  if (include_head) {
    head_rows_kernel<<<(unsigned)cdiv(n, 256), 256, 0, ctx->stream>>>(a_total, (int)n1, b_total, (int)n2, nullptr,
                                                                        nullptr, 1, m1, m2, heads);
    JQ_CHECK_LAUNCH(ctx);
  }
  rc = footnote_small_head(ctx, ra, n1, rb, n2, heads, include_head ? 1 : 0, false, rh, r_out);
  stage_event(ctx, 5);
  return rc;
}

// Variant 2 (auto, the default): the footnote variant from 1e8 reduced elements up
// (measured crossover: C2 2e6 x 32 is faster dense, C3 2e7 x 64 and C5 2e6 x 256 footnote).
static bool use_footnote(const jq_ctx* ctx, int64_t rows, int64_t n) {
  if (ctx->variant == 2) return double(rows) * double(n) > 1e8;
  return ctx->variant == 1;
}

// Device-resident figaro_r: R (n x n, canonical) into r_out (device).
// Wide joins (n1 + n2 > 256): the reduced matrix is emitted into the workspace
// (reduce_emit_dev, SPEC row order) and factored by the wide TSQR (jq_wide.cu).
static int figaro_r_wide(jq_ctx* ctx, const double* a, int64_t m1, int64_t n1, const int64_t* ka,
                         const double* b, int64_t m2, int64_t n2, const int64_t* kb, double* r_out) {
  const bool keyed = ka != nullptr;
  const int64_t n = n1 + n2;
  ctx->timing.tsqr_ctas = 0;
  stage_event(ctx, 0);
  Groups gr;
  int64_t total = m1 + m2 - 1, ng = 1;
  if (keyed) {
    JQ_TRY(group_keys_dev(ctx, ka, m1, kb, m2, &gr));
    int64_t hn[2];
    JQ_CUDA(cudaMemcpyAsync(hn, gr.d_n, 16, cudaMemcpyDeviceToHost, ctx->stream));
    JQ_CUDA(cudaStreamSynchronize(ctx->stream));
    ng = hn[0];
    total = hn[1];
  }
  const int64_t cap = keyed ? std::max<int64_t>(ng, 1) : 1;
  stage_event(ctx, 1);
  ctx->timing.reduced_rows = total;
  if (total <= 0) {  // empty join: R = 0
    JQ_CUDA(cudaMemsetAsync(r_out, 0, size_t(n) * n * 8, ctx->stream));
    for (int k = 2; k <= 5; ++k) stage_event(ctx, k);
    return JQ_OK;
  }
  double* red = ws_alloc<double>(ctx, size_t(total) * n);
  if (!red) return fail(JQ_E_OOM, "workspace exhausted (wide reduced matrix)");
  JQ_TRY(reduce_emit_dev(ctx, a, m1, n1, b, m2, n2, keyed ? &gr : nullptr, cap, total, red));
  stage_event(ctx, 2);
  JQ_TRY(wide_tsqr_dev(ctx, red, total, n, r_out, true));
  stage_event(ctx, 5);
  return JQ_OK;
}

static int figaro_r_dev(jq_ctx* ctx, const double* a, int64_t m1, int64_t n1, const int64_t* ka,
                        const double* b, int64_t m2, int64_t n2, const int64_t* kb, double* r_out) {
  if (n1 + n2 > 256) return figaro_r_wide(ctx, a, m1, n1, ka, b, m2, n2, kb, r_out);
  if (use_footnote(ctx, m1 + m2, n1 + n2)) return figaro_r_footnote_dev(ctx, a, m1, n1, ka, b, m2, n2, kb, r_out);
  const bool keyed = ka != nullptr;
  ctx->timing.tsqr_ctas = 0;
  ctx->timing.reduced_rows = 0;
  stage_event(ctx, 0);
  Groups gr;
  int64_t ng = 1;
  if (keyed) {
    JQ_TRY(group_keys_dev(ctx, ka, m1, kb, m2, &gr));
    int64_t hn[2];  // the group count sizes the per-group scan totals (see the footnote path)
    JQ_CUDA(cudaMemcpyAsync(hn, gr.d_n, 16, cudaMemcpyDeviceToHost, ctx->stream));
    JQ_CUDA(cudaStreamSynchronize(ctx->stream));
    ng = hn[0];
  }
  stage_event(ctx, 1);
  SegScan ss;
  const int64_t cap = keyed ? std::max<int64_t>(ng, 1) : 1;
  if (n2 > 0)
    JQ_TRY(segscan_dev(ctx, b, m2, n2, keyed ? gr.gid_b : nullptr, keyed ? gr.b_start : nullptr,
                       keyed ? gr.b_count : nullptr, keyed ? gr.d_n : nullptr, cap, &ss));
  stage_event(ctx, 2);
  FigaroArgs fa{};
  fa.a = a; fa.m1 = m1; fa.n1 = n1;
  fa.b = b; fa.m2 = m2; fa.n2 = n2;
  fa.gid_a = keyed ? gr.gid_a : nullptr;
  fa.gid_b = keyed ? gr.gid_b : nullptr;
  fa.a_count = keyed ? gr.a_count : nullptr;
  fa.b_count = keyed ? gr.b_count : nullptr;
  fa.b_start = keyed ? gr.b_start : nullptr;
  fa.b_totals = n2 > 0 ? ss.totals : nullptr;
  fa.b_carry = n2 > 0 ? ss.carry : nullptr;
  fa.b_prefix0 = nullptr;
  fa.m1_global = m1; fa.m2_global = m2; fa.b_row0 = 0;
  JQ_TRY(figaro_tsqr_dev(ctx, fa, r_out, true));
  return JQ_OK;
}

// ---- host-resident Cartesian inputs: streamed pipeline ------------------------
// Each table is copied in row pieces (~512 MB, TILE_ROWS multiples) on a copy
// stream into two alternating device buffers while the previous piece's
// head/tail scan and TSQR run on the compute stream, so the PCIe transfer (the
// bound of an end-to-end call from host memory) overlaps the compute.  Per piece:
// segscan (carries relative to the piece) + prefix carried across pieces, the
// piece's rows as a row shard of the virtual reduced matrix (FigaroArgs.b_row0 /
// b_prefix0, exactly the multi-GPU shard machinery), one local R folded into a
// running R by a 2-factor TSQR.  Deterministic for a fixed piece size.
__global__ void vec_add_kernel(double* __restrict__ acc, const double* __restrict__ x, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc[i] += x[i];
}
__global__ void pack2_kernel(const double* __restrict__ r0, const double* __restrict__ r1, int n,
                             double* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * n * n; i += gridDim.x * blockDim.x)
    out[i] = i < n * n ? r0[i] : r1[i - n * n];
}

// Environment overrides (read per call, for the piece-count parity sweep):
// JQ_STREAM_MIN_BYTES (default 1 GiB of host input) and JQ_PIECE_BYTES (default 512 MiB).
static int64_t env_bytes(const char* name, int64_t dflt) {
  const char* e = getenv(name);
  if (!e || !*e) return dflt;
  const long long v = atoll(e);
  return v > 0 ? (int64_t)v : dflt;
}

static bool use_streamed(const double* a, int64_t m1, int64_t n1, const double* b, int64_t m2, int64_t n2,
                         const int64_t* ka) {
  if (ka || n1 + n2 > 256) return false;
  if (is_device_ptr(a) || is_device_ptr(b)) return false;
  return (m1 * n1 + m2 * n2) * 8 >= env_bytes("JQ_STREAM_MIN_BYTES", int64_t(1) << 30);
}

// H2D of PAGEABLE host memory through a pinned staging ring: the driver would stage
// such copies itself at ~11 GB/s, synchronously; instead host threads memcpy each chunk
// (<= 512 MB) into a pinned slot (waiting only for that slot's previous DMA) and the DMA
// runs from the slot on `stream` while the next chunk is being copied.  The ring (3 slots)
// is allocated on first use and kept by the context.
int pinned_ring_copy(jq_ctx* ctx, cudaStream_t stream, void* dst, const void* src, size_t bytes) {
  constexpr int S = 3;
  const size_t slot_max = size_t(512) << 20;
  const size_t want = std::min(slot_max, bytes);
  if (!ctx->stage_pin || ctx->stage_slot < want) {
    if (ctx->stage_pin) {
      for (auto& e : ctx->sev) if (e) cudaEventSynchronize(e);
      cudaFreeHost(ctx->stage_pin);
      ctx->stage_pin = nullptr;
    }
    JQ_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ctx->stage_pin), want * S, cudaHostAllocDefault));
    ctx->stage_slot = want;
    ctx->stage_slots = S;
    for (int i = 0; i < S; ++i)
      if (!ctx->sev[i]) JQ_CUDA(cudaEventCreateWithFlags(&ctx->sev[i], cudaEventDisableTiming));
  }
  const unsigned hw = std::thread::hardware_concurrency();
  const int nt = (int)std::max(1u, std::min(hw ? hw : 1u, 16u));
  for (size_t off = 0; off < bytes; off += ctx->stage_slot) {
    const size_t len = std::min(ctx->stage_slot, bytes - off);
    const int slot = ctx->stage_next++ % S;
    JQ_CUDA(cudaEventSynchronize(ctx->sev[slot]));  // the slot's previous DMA has drained
    char* pin = ctx->stage_pin + size_t(slot) * ctx->stage_slot;
    const char* from = static_cast<const char*>(src) + off;
    const size_t part = (len + nt - 1) / nt;
    std::vector<std::thread> th;
    for (int i = 1; i < nt; ++i) {
      const size_t o = size_t(i) * part;
      if (o < len) th.emplace_back([=] { memcpy(pin + o, from + o, std::min(part, len - o)); });
    }
    memcpy(pin, from, std::min(part, len));
    for (auto& x : th) x.join();
    JQ_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, pin, len, cudaMemcpyHostToDevice, stream));
    JQ_CUDA(cudaEventRecord(ctx->sev[slot], stream));
  }
  return JQ_OK;
}

bool is_pageable(const void* p) {
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return attr.type == cudaMemoryTypeUnregistered;
}

// Host -> device copy of a staged input: large pageable sources through the pinned ring.
int h2d_copy(jq_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (bytes >= (size_t(64) << 20) && is_pageable(src)) return pinned_ring_copy(ctx, ctx->stream, dst, src, bytes);
  JQ_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return JQ_OK;
}

// Piece H2D for the streamed path (copy stream; pageable pieces through the ring).
static int h2d_piece(jq_ctx* ctx, void* dst, const void* src, size_t bytes, bool pageable, int64_t k) {
  (void)k;
  if (!pageable) {
    JQ_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->copy_stream));
    return JQ_OK;
  }
  return pinned_ring_copy(ctx, ctx->copy_stream, dst, src, bytes);
}

static int figaro_r_streamed(jq_ctx* ctx, const double* a, int64_t m1, int64_t n1, const double* b, int64_t m2,
                             int64_t n2, double* dr /* device, n x n canonical */) {
  const int64_t n = n1 + n2;
  const bool foot = use_footnote(ctx, m1 + m2, n);
  const int64_t piece_bytes = env_bytes("JQ_PIECE_BYTES", int64_t(512) << 20);
  auto prows = [&](int64_t cols) {
    int64_t pr = piece_bytes / (8 * std::max<int64_t>(cols, 1));
    return std::max<int64_t>(TILE_ROWS, pr / TILE_ROWS * TILE_ROWS);
  };
  const int64_t pa = prows(n1), pb = prows(n2);
  const int64_t buf_elems = std::max(std::min(pa, m1) * n1, std::min(pb, m2) * n2);
  if (!ctx->copy_stream) {
    JQ_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
    for (auto& e : ctx->pev) JQ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  const int64_t maxp = std::max(pa, pb);
  JQ_TRY(ws_reserve(ctx, 2 * ws_bytes(buf_elems, 8) + 12 * ws_bytes(n * n, 8) + 8 * ws_bytes(n, 8) +
                             segscan_ws_bytes(maxp, std::max<int64_t>(std::max(n1, n2), 1), 1) +
                             figaro_tsqr_ws_bytes(maxp, TILE_ROWS, n, ctx->sms) +
                             tsqr_ws_bytes(3 * n, n, ctx->sms) + tsqr_ws_bytes(TILE_ROWS, n, ctx->sms)));
  double* buf[2] = {ws_alloc<double>(ctx, buf_elems), ws_alloc<double>(ctx, buf_elems)};
  double* racc[2] = {ws_alloc<double>(ctx, n * n), ws_alloc<double>(ctx, n * n)};  // per side (dense: [0] only)
  double* rpiece = ws_alloc<double>(ctx, n * n);
  double* pair = ws_alloc<double>(ctx, 2 * n * n);
  double* pre[2] = {ws_alloc<double>(ctx, std::max<int64_t>(n1, 1)), ws_alloc<double>(ctx, std::max<int64_t>(n2, 1))};
  double* heads = ws_alloc<double>(ctx, n);
  double* rh = ws_alloc<double>(ctx, n * n);
  if (!buf[1] || !rh) return fail(JQ_E_OOM, "workspace exhausted (streamed figaro)");
  JQ_CUDA(cudaMemsetAsync(pre[0], 0, std::max<int64_t>(n1, 1) * 8, ctx->stream));
  JQ_CUDA(cudaMemsetAsync(pre[1], 0, std::max<int64_t>(n2, 1) * 8, ctx->stream));
  const size_t mark = ctx->ws.used;
  ctx->timing.tsqr_ctas = 0;
  ctx->timing.reduced_rows = 0;
  ctx->record_tsqr_events = false;
  stage_event(ctx, 0);
  int64_t k = 0;  // global piece counter (buffer parity)
  bool first[2] = {true, true};
  // side 0 = A, side 1 = B.  Dense: B first (top rows need head(B)), footnote: any order.
  const int order[2] = {foot ? 0 : 1, foot ? 1 : 0};
  const bool pageable[2] = {n1 > 0 && is_pageable(a), n2 > 0 && is_pageable(b)};
  for (int oi = 0; oi < 2; ++oi) {
    const int side = order[oi];
    const double* host = side == 0 ? a : b;
    const int64_t m = side == 0 ? m1 : m2, cols = side == 0 ? n1 : n2;
    if (cols == 0) continue;
    const int64_t pr = side == 0 ? pa : pb;
    for (int64_t r0 = 0; r0 < m; r0 += pr, ++k) {
      const int64_t rows = std::min(pr, m - r0);
      const int bi = int(k & 1);
      ctx->ws.used = mark;
      // copy piece k into buf[bi] once piece k-2 (same buffer) has been consumed
      if (k >= 2) JQ_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->pev[2 + bi], 0));
      JQ_TRY(h2d_piece(ctx, buf[bi], host + r0 * cols, size_t(rows * cols * 8), pageable[side], k));
      JQ_CUDA(cudaEventRecord(ctx->pev[bi], ctx->copy_stream));
      JQ_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->pev[bi], 0));
      SegScan ss{};
      JQ_TRY(segscan_dev(ctx, buf[bi], rows, cols, nullptr, nullptr, nullptr, nullptr, 1, &ss));
      FigaroArgs fa{};
      const int rs = foot ? side : 0;  // running-R slot
      double* pfx = pre[side];
      const int64_t nn = foot ? cols : n;
      if (!foot && side == 0) {
        // dense top rows [sqrt(m2) A_i | head(B)]: head from the complete B total
        fa.a = buf[bi]; fa.m1 = rows; fa.n1 = n1; fa.n2 = n2;
        fa.b_totals = pre[1]; fa.m1_global = m1; fa.m2_global = m2;
      } else {
        // tails: the "B-part" of a source with an empty A-part (dense: n1 zero columns first)
        fa.n1 = foot ? 0 : n1;
        fa.b = buf[bi]; fa.m2 = rows; fa.n2 = cols;
        fa.b_carry = ss.carry; fa.b_prefix0 = pfx; fa.b_row0 = r0;
        fa.m1_global = side == 0 ? m2 : m1;   // tails of A scale by sqrt(m2), of B by sqrt(m1)
        fa.m2_global = m;
      }
      JQ_TRY(figaro_tsqr_dev(ctx, fa, rpiece, false));
      if (!(!foot && side == 0)) {
        vec_add_kernel<<<1, 256, 0, ctx->stream>>>(pfx, ss.totals, (int)cols);  // prefix += piece sum
        JQ_CHECK_LAUNCH(ctx);
      }
      JQ_CUDA(cudaEventRecord(ctx->pev[2 + bi], ctx->stream));
      if (first[rs]) {
        JQ_CUDA(cudaMemcpyAsync(racc[rs], rpiece, nn * nn * 8, cudaMemcpyDeviceToDevice, ctx->stream));
        first[rs] = false;
      } else {
        pack2_kernel<<<(unsigned)cdiv(2 * nn * nn, 256), 256, 0, ctx->stream>>>(racc[rs], rpiece, (int)nn, pair);
        JQ_CHECK_LAUNCH(ctx);
        JQ_TRY(tsqr_stack_dev(ctx, pair, 2, nn, racc[rs], false));
      }
    }
  }
  ctx->ws.used = mark;
  stage_event(ctx, 4);
  int rc = JQ_OK;
  if (!foot) {
    canonicalize_dev(ctx, racc[0], n, dr);
  } else {
    head_rows_kernel<<<(unsigned)cdiv(n, 256), 256, 0, ctx->stream>>>(pre[0], (int)n1, pre[1], (int)n2, nullptr,
                                                                        nullptr, 1, m1, m2, heads);
    JQ_CHECK_LAUNCH(ctx);
    rc = footnote_small_head(ctx, racc[0], n1, racc[1], n2, heads, 1, true, rh, dr);
  }
  ctx->record_tsqr_events = true;
  stage_event(ctx, 5);
  stage_event(ctx, 1);
  stage_event(ctx, 2);
  stage_event(ctx, 3);
  return rc;
}

static void record_timing(jq_ctx* ctx, bool svd) {
  jq_timing& t = ctx->timing;
  t.group_ms = ev_ms(ctx, 0, 1);
  t.scan_ms = ev_ms(ctx, 1, 2);
  t.tsqr_ms = ev_ms(ctx, 3, 4);
  t.tree_ms = ev_ms(ctx, 4, 5);
  t.svd_ms = svd ? ev_ms(ctx, 5, 6) : 0.0;
  t.total_ms = ev_ms(ctx, 0, svd ? 6 : 5);
  t.scan_tile_ms = 0.0;
  for (int k = 0; k < ctx->tile_launches; ++k) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, ctx->tev[2 * k], ctx->tev[2 * k + 1]) != cudaSuccess) {
      cudaGetLastError();
      ms = 0.f;
    }
    t.scan_tile_ms += ms;
  }
  t.scan_tile_bytes = ctx->tile_launches ? ctx->tile_bytes : 0.0;
}

static int check_tables(int64_t m1, int64_t n1, const int64_t* ka, int64_t m2, int64_t n2, const int64_t* kb) {
  if ((ka == nullptr) != (kb == nullptr)) return fail(JQ_E_KEYS, "both tables must carry keys, or neither");
  if (m1 < 0 || m2 < 0 || n1 < 0 || n2 < 0) return fail(JQ_E_INVALID, "negative size");
  if (n1 + n2 == 0) return fail(JQ_E_INVALID, "the join has no columns");
  if (n1 + n2 > 512) return fail(JQ_E_INVALID, "n1 + n2 above 512 is not supported");
  if (!ka && (m1 == 0 || m2 == 0)) return fail(JQ_E_INVALID, "reduce_cartesian needs non-empty inputs");
  return JQ_OK;
}

}  // namespace jq

using namespace jq;

extern "C" {

int jq_version(void) { return 100; }
const char* jq_last_error(void) { return g_err.c_str(); }

int jq_ctx_create(int device, jq_ctx** out) {
  if (!out) return fail(JQ_E_INVALID, "null output pointer");
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(JQ_E_NODEV, "no CUDA device is visible (libjoinqr needs a B200 / sm_100a GPU)");
  }
  if (device < 0 || device >= count) return fail(JQ_E_NODEV, "device index out of range");
  JQ_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  JQ_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) return fail(JQ_E_NODEV, std::string("libjoinqr is built for sm_100a; device is ") + prop.name);
  jq_ctx* ctx = new jq_ctx();
  ctx->device = device;
  ctx->sms = prop.multiProcessorCount;
  JQ_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
  ctx->stream = ctx->own_stream;
  JQ_CUDA(cudaMalloc(&ctx->d_flags, sizeof(int)));
  JQ_CUDA(cudaMallocHost(&ctx->h_flags, sizeof(int)));
  for (auto& e : ctx->ev) JQ_CUDA(cudaEventCreate(&e));
  for (auto& e : ctx->tev) JQ_CUDA(cudaEventCreate(&e));
  *out = ctx;
  return JQ_OK;
}

int jq_ctx_destroy(jq_ctx* ctx) {
  if (!ctx) return JQ_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  if (ctx->ws.base) cudaFree(ctx->ws.base);
  if (ctx->d_flags) cudaFree(ctx->d_flags);
  if (ctx->h_flags) cudaFreeHost(ctx->h_flags);
  for (auto& e : ctx->ev) if (e) cudaEventDestroy(e);
  for (auto& e : ctx->tev) if (e) cudaEventDestroy(e);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->stage_pin) cudaFreeHost(ctx->stage_pin);
  for (auto& e : ctx->sev) if (e) cudaEventDestroy(e);
  if (ctx->aux_stream) cudaStreamDestroy(ctx->aux_stream);
  for (auto& e : ctx->aev) if (e) cudaEventDestroy(e);
  for (auto& e : ctx->pev) if (e) cudaEventDestroy(e);
  delete ctx;
  return JQ_OK;
}

int jq_ctx_set_stream(jq_ctx* ctx, void* s) {
  if (!ctx) return fail(JQ_E_INVALID, "null context");
  ctx->stream = s ? reinterpret_cast<cudaStream_t>(s) : ctx->own_stream;
  return JQ_OK;
}

int jq_ctx_sync(jq_ctx* ctx) {
  if (!ctx) return fail(JQ_E_INVALID, "null context");
  JQ_CUDA(cudaStreamSynchronize(ctx->stream));
  return JQ_OK;
}

int jq_ctx_set_variant(jq_ctx* ctx, int variant) {
  if (!ctx) return fail(JQ_E_INVALID, "null context");
  if (variant < 0 || variant > 2) return fail(JQ_E_INVALID, "variant must be 0 (dense), 1 (footnote) or 2 (auto)");
  ctx->variant = variant;
  return JQ_OK;
}

int jq_last_timing(jq_ctx* ctx, jq_timing* out) {
  if (!ctx || !out) return fail(JQ_E_INVALID, "null argument");
  *out = ctx->timing;
  return JQ_OK;
}

int64_t jq_kernel_launches(jq_ctx* ctx) { return ctx ? ctx->launches : 0; }

int jq_canonicalize(jq_ctx* ctx, const double* r, int64_t n, double* out) {
  if (!ctx) return fail(JQ_E_INVALID, "null context");
  JQ_NVTX("jq_canonicalize");
  if (n <= 0) return JQ_OK;
  JQ_TRY(begin_call(ctx));
  JQ_TRY(ws_reserve(ctx, stage_bytes(r, n * n) + stage_bytes((const double*)out, n * n)));
  const double* dr;
  double* dout;
  JQ_TRY(stage_in(ctx, r, n * n, &dr));
  JQ_TRY(stage_out(ctx, out, n * n, &dout));
  JQ_TRY(canonicalize_dev(ctx, dr, n, dout));
  JQ_TRY(copy_out(ctx, out, (const double*)dout, n * n));
  return sync_and_check_flags(ctx);
}

int jq_householder_r(jq_ctx* ctx, const double* m, int64_t rows, int64_t cols, double* r) {
  if (!ctx) return fail(JQ_E_INVALID, "null context");
  JQ_NVTX("jq_householder_r");
  if (cols <= 0) return fail(JQ_E_INVALID, "householder_r needs at least one column");
  if (cols > 512) return fail(JQ_E_INVALID, "more than 512 columns");
  if (rows < 0) return fail(JQ_E_INVALID, "negative row count");
  JQ_TRY(begin_call(ctx));
  JQ_TRY(ws_reserve(ctx, stage_bytes(m, rows * cols) + stage_bytes((const double*)r, cols * cols) +
                             tsqr_ws_bytes(rows, cols, ctx->sms)));
  const double* dm;
  double* dr;
  JQ_TRY(stage_in(ctx, m, rows * cols, &dm));
  JQ_TRY(stage_out(ctx, r, cols * cols, &dr));
  JQ_TRY(tsqr_dense_dev(ctx, dm, rows, cols, dr, false));
  JQ_TRY(copy_out(ctx, r, (const double*)dr, cols * cols));
  return sync_and_check_flags(ctx);
}

int jq_figaro_r(jq_ctx* ctx, const double* a, int64_t m1, int64_t n1, const int64_t* ka,
                const double* b, int64_t m2, int64_t n2, const int64_t* kb, double* r) {
  if (!ctx) return fail(JQ_E_INVALID, "null context");
  JQ_NVTX("jq_figaro_r");
  JQ_TRY(check_tables(m1, n1, ka, m2, n2, kb));
  JQ_TRY(begin_call(ctx));
  const int64_t n = n1 + n2;
  if (use_streamed(a, m1, n1, b, m2, n2, ka)) {
    double* dr = nullptr;
    if (is_device_ptr(r)) {
      dr = r;
    } else {
      JQ_CUDA(cudaMallocAsync(&dr, n * n * 8, ctx->stream));
    }
    int rc = figaro_r_streamed(ctx, a, m1, n1, b, m2, n2, dr);
    if (rc == JQ_OK && dr != r) rc = copy_out(ctx, r, (const double*)dr, n * n);
    int rc2 = sync_and_check_flags(ctx);
    if (dr != r) cudaFreeAsync(dr, ctx->stream);
    record_timing(ctx, false);
    return rc ? rc : rc2;
  }
  JQ_TRY(ws_reserve(ctx, stage_bytes(a, m1 * n1) + stage_bytes(b, m2 * n2) + stage_bytes(ka, m1) +
                             stage_bytes(kb, m2) + stage_bytes((const double*)r, n * n) +
                             figaro_ws(m1, n1, m2, n2, ka != nullptr, ctx->sms)));
  const double *da, *db;
  const int64_t *dka, *dkb;
  double* dr;
  JQ_TRY(stage_in(ctx, a, m1 * n1, &da));
  JQ_TRY(stage_in(ctx, b, m2 * n2, &db));
  JQ_TRY(stage_in(ctx, ka, m1, &dka));
  JQ_TRY(stage_in(ctx, kb, m2, &dkb));
  JQ_TRY(stage_out(ctx, r, n * n, &dr));
  JQ_TRY(figaro_r_dev(ctx, da, m1, n1, dka, db, m2, n2, dkb, dr));
  JQ_TRY(copy_out(ctx, r, (const double*)dr, n * n));
  int rc = sync_and_check_flags(ctx);
  record_timing(ctx, false);
  return rc;
}

int jq_figaro_svd(jq_ctx* ctx, const double* a, int64_t m1, int64_t n1, const int64_t* ka,
                  const double* b, int64_t m2, int64_t n2, const int64_t* kb, int want_v,
                  double* values, double* v, double* r) {
  if (!ctx) return fail(JQ_E_INVALID, "null context");
  JQ_NVTX("jq_figaro_svd");
  JQ_TRY(check_tables(m1, n1, ka, m2, n2, kb));
  JQ_TRY(begin_call(ctx));
  const int64_t n = n1 + n2;
  JQ_TRY(ws_reserve(ctx, stage_bytes(a, m1 * n1) + stage_bytes(b, m2 * n2) + stage_bytes(ka, m1) +
                             stage_bytes(kb, m2) + stage_bytes((const double*)values, n) +
                             stage_bytes((const double*)v, n * n) + ws_bytes(n * n, 8) +
                             figaro_ws(m1, n1, m2, n2, ka != nullptr, ctx->sms) + svd_ws_bytes(n)));
  const double *da, *db;
  const int64_t *dka, *dkb;
  double *dval, *dv = nullptr;
  JQ_TRY(stage_in(ctx, a, m1 * n1, &da));
  JQ_TRY(stage_in(ctx, b, m2 * n2, &db));
  JQ_TRY(stage_in(ctx, ka, m1, &dka));
  JQ_TRY(stage_in(ctx, kb, m2, &dkb));
  JQ_TRY(stage_out(ctx, values, n, &dval));
  if (want_v) JQ_TRY(stage_out(ctx, v, n * n, &dv));
  double* dr = ws_alloc<double>(ctx, n * n);
  JQ_TRY(figaro_r_dev(ctx, da, m1, n1, dka, db, m2, n2, dkb, dr));
  JQ_TRY(svd_dev(ctx, dr, n, want_v, dval, dv));
  stage_event(ctx, 6);
  JQ_TRY(copy_out(ctx, values, (const double*)dval, n));
  if (want_v) JQ_TRY(copy_out(ctx, v, (const double*)dv, n * n));
  if (r) JQ_TRY(copy_out(ctx, r, (const double*)dr, n * n));
  int rc = sync_and_check_flags(ctx);
  record_timing(ctx, true);
  return rc;
}

int jq_figaro_r_shard(jq_ctx* ctx, const double* a, int64_t a_rows, int64_t n1, int64_t m1, int64_t a_row0,
                      const double* a_prefix, const double* a_total, const double* b, int64_t b_rows, int64_t n2,
                      int64_t m2, int64_t b_row0, const double* b_prefix, const double* b_total, int include_head,
                      double* r_local) {
  if (!ctx) return fail(JQ_E_INVALID, "null context");
  JQ_NVTX("jq_figaro_r_shard");
  if (a_rows < 0 || b_rows < 0 || n1 < 0 || n2 < 0 || n1 + n2 == 0 || n1 + n2 > 256)
    return fail(JQ_E_INVALID, "bad shard geometry");
  if (m1 <= 0 || m2 <= 0 || b_row0 < 0 || b_row0 + b_rows > m2 || a_row0 < 0 || a_row0 + a_rows > m1)
    return fail(JQ_E_INVALID, "bad global sizes for the shard");
  const bool foot = use_footnote(ctx, m1 + m2, n1 + n2);
  if (foot && (!a_prefix || !a_total)) return fail(JQ_E_INVALID, "footnote shards need a_prefix and a_total");
  JQ_TRY(begin_call(ctx));
  const int64_t n = n1 + n2;
  JQ_TRY(ws_reserve(ctx, stage_bytes(a, a_rows * n1) + stage_bytes(b, b_rows * n2) + stage_bytes(a_prefix, n1) +
                             stage_bytes(a_total, n1) + stage_bytes(b_prefix, n2) + stage_bytes(b_total, n2) +
                             stage_bytes((const double*)r_local, n * n) +
                             figaro_ws(a_rows, n1, b_rows, n2, false, ctx->sms)));
  const double *da, *db, *dapre = nullptr, *datot = nullptr, *dpre, *dtot;
  double* dr;
  JQ_TRY(stage_in(ctx, a, a_rows * n1, &da));
  JQ_TRY(stage_in(ctx, b, b_rows * n2, &db));
  JQ_TRY(stage_in(ctx, a_prefix, n1, &dapre));
  JQ_TRY(stage_in(ctx, a_total, n1, &datot));
  JQ_TRY(stage_in(ctx, b_prefix, n2, &dpre));
  JQ_TRY(stage_in(ctx, b_total, n2, &dtot));
  JQ_TRY(stage_out(ctx, r_local, n * n, &dr));
  ctx->timing.tsqr_ctas = 0;
  ctx->timing.reduced_rows = 0;
  stage_event(ctx, 0);
  stage_event(ctx, 1);
  int rc = JQ_OK;
  if (!foot) {
    SegScan ss{};
    if (n2 > 0) JQ_TRY(segscan_dev(ctx, db, b_rows, n2, nullptr, nullptr, nullptr, nullptr, 1, &ss));
    stage_event(ctx, 2);
    FigaroArgs fa{};
    fa.a = da; fa.m1 = a_rows; fa.n1 = n1;
    fa.b = db; fa.m2 = b_rows; fa.n2 = n2;
    fa.b_totals = dtot;
    fa.b_carry = n2 > 0 ? ss.carry : nullptr;
    fa.b_prefix0 = dpre;
    fa.m1_global = m1; fa.m2_global = m2; fa.b_row0 = b_row0;
    JQ_TRY(figaro_tsqr_dev(ctx, fa, dr, false));
  } else {
    JQ_TRY(footnote_shard_dev(ctx, da, a_rows, n1, m1, a_row0, dapre, datot, db, b_rows, n2, m2, b_row0, dpre,
                              dtot, include_head != 0, dr));
  }
  JQ_TRY(copy_out(ctx, r_local, (const double*)dr, n * n));
  rc = sync_and_check_flags(ctx);
  record_timing(ctx, false);
  return rc;
}

int jq_figaro_r_shard_local(jq_ctx* ctx, const double* a, int64_t a_rows, int64_t n1, int64_t m1, const double* b,
                            int64_t b_rows, int64_t n2, int64_t m2, double* r_local, double* sums) {
  if (!ctx) return fail(JQ_E_INVALID, "null context");
  JQ_NVTX("jq_figaro_r_shard_local");
  if (a_rows <= 0 || b_rows <= 0 || n1 <= 0 || n2 <= 0 || n1 + n2 > 256)
    return fail(JQ_E_INVALID, "bad shard geometry (both sides need rows and columns)");
  if (m1 < a_rows || m2 < b_rows) return fail(JQ_E_INVALID, "bad global sizes for the shard");
  if (!r_local || !sums) return fail(JQ_E_INVALID, "null output");
  JQ_TRY(begin_call(ctx));
  const int64_t n = n1 + n2;
  JQ_TRY(ws_reserve(ctx, stage_bytes(a, a_rows * n1) + stage_bytes(b, b_rows * n2) +
                             stage_bytes((const double*)r_local, n * n) + stage_bytes((const double*)sums, n) +
                             figaro_ws(a_rows, n1, b_rows, n2, false, ctx->sms)));
  const double *da, *db;
  double *dr, *ds;
  JQ_TRY(stage_in(ctx, a, a_rows * n1, &da));
  JQ_TRY(stage_in(ctx, b, b_rows * n2, &db));
  JQ_TRY(stage_out(ctx, r_local, n * n, &dr));
  JQ_TRY(stage_out(ctx, sums, n, &ds));
  ctx->timing.tsqr_ctas = 0;
  ctx->timing.reduced_rows = 0;
  stage_event(ctx, 0);
  stage_event(ctx, 1);
  JQ_TRY(footnote_shard_blocks(ctx, da, a_rows, n1, m1, 0, nullptr, nullptr, db, b_rows, n2, m2, 0, nullptr, nullptr,
                               false, dr, ds));
  JQ_TRY(copy_out(ctx, r_local, (const double*)dr, n * n));
  JQ_TRY(copy_out(ctx, sums, (const double*)ds, n));
  const int rc = sync_and_check_flags(ctx);
  record_timing(ctx, false);
  return rc;
}

int jq_split_group_rows(jq_ctx* ctx, const double* part_sums, const int64_t* part_rows,
                        const int64_t* part_group, int64_t nparts, int64_t n1, int64_t n2, double* rows,
                        int64_t rows_capacity, int64_t* n_rows) {
  if (!ctx) return fail(JQ_E_INVALID, "null context");
  JQ_NVTX("jq_split_group_rows");
  if (nparts < 0 || n1 < 0 || n2 < 0 || n1 + n2 == 0 || n1 + n2 > 1024) return fail(JQ_E_INVALID, "bad geometry");
  if (nparts > 0 && (!part_sums || !part_rows || !part_group)) return fail(JQ_E_INVALID, "null argument");
  const int64_t n = n1 + n2;
  // group layout on the host (part_rows / part_group are small host arrays)
  std::vector<int64_t> first{0}, row0, na;
  int64_t total = 0;
  for (int64_t k = 0; k < nparts; ++k) {
    if (part_rows[2 * k] < 0 || part_rows[2 * k + 1] < 0) return fail(JQ_E_INVALID, "negative part size");
    if (k > 0 && part_group[k] < part_group[k - 1]) return fail(JQ_E_INVALID, "parts must be ordered by group");
    if (k + 1 == nparts || part_group[k + 1] != part_group[k]) first.push_back(k + 1);
  }
  const int64_t ng = (int64_t)first.size() - 1;
  for (int64_t g = 0; g < ng; ++g) {
    int64_t ca = 0, cb = 0;
    for (int64_t k = first[g]; k < first[g + 1]; ++k) {
      ca += part_rows[2 * k] > 0;
      cb += part_rows[2 * k + 1] > 0;
    }
    row0.push_back(total);
    na.push_back(std::max<int64_t>(ca - 1, 0));
    total += 1 + std::max<int64_t>(ca - 1, 0) + std::max<int64_t>(cb - 1, 0);
  }
  if (n_rows) *n_rows = total;
  if (!rows) return JQ_OK;
  if (total > rows_capacity) return fail(JQ_E_INVALID, "row output capacity too small");
  if (total == 0) return JQ_OK;
  JQ_TRY(begin_call(ctx));
  JQ_TRY(ws_reserve(ctx, stage_bytes(part_sums, nparts * n) + stage_bytes((const double*)rows, total * n) +
                             4 * ws_bytes(nparts * 2 + ng + 2, 8)));
  const double* dsums;
  double* dout;
  JQ_TRY(stage_in(ctx, part_sums, nparts * n, &dsums));
  JQ_TRY(stage_out(ctx, rows, total * n, &dout));
  int64_t* meta = ws_alloc<int64_t>(ctx, 2 * nparts + (ng + 1) + 2 * ng);
  if (!meta) return fail(JQ_E_OOM, "workspace exhausted (split group rows)");
  std::vector<int64_t> hm(part_rows, part_rows + 2 * nparts);
  hm.insert(hm.end(), first.begin(), first.end());
  hm.insert(hm.end(), row0.begin(), row0.end());
  hm.insert(hm.end(), na.begin(), na.end());
  JQ_CUDA(cudaMemcpyAsync(meta, hm.data(), hm.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
  JQ_CUDA(cudaMemsetAsync(dout, 0, total * n * 8, ctx->stream));
  split_group_rows_kernel<<<(unsigned)ng, 256, 0, ctx->stream>>>(dsums, meta, meta + 2 * nparts,
                                                                  meta + 2 * nparts + ng + 1,
                                                                  meta + 2 * nparts + ng + 1 + ng, (int)n1, (int)n2,
                                                                  dout);
  JQ_CHECK_LAUNCH(ctx);
  JQ_TRY(copy_out(ctx, rows, (const double*)dout, total * n));
  return sync_and_check_flags(ctx);
}

int jq_tsqr_stack(jq_ctx* ctx, const double* rs, int64_t count, int64_t n, double* r) {
  if (!ctx) return fail(JQ_E_INVALID, "null context");
  JQ_NVTX("jq_tsqr_stack");
  if (count <= 0 || n <= 0 || n > 512) return fail(JQ_E_INVALID, "bad R stack geometry");
  JQ_TRY(begin_call(ctx));
  JQ_TRY(ws_reserve(ctx, stage_bytes(rs, count * n * n) + stage_bytes((const double*)r, n * n) +
                             (n > 256 ? wide_tsqr_ws_bytes(count * n, n, ctx->sms)
                                      : 2 * ws_bytes(size_t(count + 1) * 256 * 256, 8))));
  const double* drs;
  double* dr;
  JQ_TRY(stage_in(ctx, rs, count * n * n, &drs));
  JQ_TRY(stage_out(ctx, r, n * n, &dr));
  JQ_TRY(tsqr_stack_dev(ctx, drs, count, n, dr, true));
  JQ_TRY(copy_out(ctx, r, (const double*)dr, n * n));
  return sync_and_check_flags(ctx);
}

}  // extern "C"
