// jq_internal.cuh — context, error plumbing, workspace and device helpers shared
// by the libjoinqr.so translation units.  Target: sm_100a (B200) only.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "joinqr.h"

namespace jq {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

#define JQ_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return ::jq::fail(e_ == cudaErrorMemoryAllocation ? JQ_E_OOM : JQ_E_CUDA,    \
                        std::string(#call) + ": " + cudaGetErrorString(e_));       \
  } while (0)

#define JQ_TRY(expr)          \
  do {                        \
    int rc_ = (expr);         \
    if (rc_ != JQ_OK) return rc_; \
  } while (0)

// NVTX (SURVEY.md §5 tracing): a range per public call (JQ_NVTX) and a mark per
// pipeline stage boundary (stage_event), visible in Nsight Systems / Compute timelines.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define JQ_NVTX(name) ::jq::NvtxRange jq_nvtx_range_(name)

// Count launches of our own kernels (evidence for bench.py "gpu_launches").
#define JQ_LAUNCHED(ctx) ((ctx)->launches++)
#define JQ_CHECK_LAUNCH(ctx)                                                       \
  do {                                                                             \
    JQ_LAUNCHED(ctx);                                                              \
    cudaError_t e_ = cudaGetLastError();                                           \
    if (e_ != cudaSuccess)                                                         \
      return ::jq::fail(JQ_E_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
  } while (0)

// ---------------------------------------------------------------- context
struct Workspace {
  char* base = nullptr;
  size_t cap = 0;
  size_t used = 0;
};

// Device-side error flags raised by validation kernels (read once per call).
enum DevFlag : int { FLAG_UNSORTED_A = 1, FLAG_UNSORTED_B = 2, FLAG_NOCONV = 4, FLAG_BADINDEX = 8 };

}  // namespace jq

struct jq_ctx {
  int device = 0;
  int sms = 148;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  jq::Workspace ws;
  int* d_flags = nullptr;    // device error flags
  int* h_flags = nullptr;    // pinned mirror
  int variant = 2;              // 0 dense Claim-1, 1 footnote (head/tail of both sides), 2 auto
  bool record_tsqr_events = true;
  int64_t launches = 0;
  jq_timing timing{};
  cudaEvent_t ev[8]{};
  cudaStream_t copy_stream = nullptr;   // host -> device piece copies (streamed figaro)
  cudaEvent_t pev[4]{};                 // piece copied / consumed events
  // pinned staging ring for PAGEABLE host inputs of the streamed path (host threads
  // memcpy a piece into a slot while the previous slot's DMA runs)
  char* stage_pin = nullptr;
  size_t stage_slot = 0;
  int stage_slots = 0;
  int64_t stage_next = 0;
  cudaEvent_t sev[4]{};
  cudaStream_t aux_stream = nullptr;    // V replay beside the Jacobi sweeps (jq_svd.cu)
  cudaEvent_t aev[2]{};
  // the head/tail tile pass timed on its own (up to 4 launches per call; bench roofline)
  cudaEvent_t tev[8]{};
  int tile_launches = 0;
  double tile_bytes = 0.0;
};

namespace jq {

// 1/x and 1/sqrt(x) from the MUFU approximations (~1e-6 relative) plus ONE cubically
// convergent correction each: r (1 + e + e^2) and y (1 + e/2 + 3e^2/8), measured at
// <= 2.2e-16 relative (tools/microbench/approx_acc.cu) -- the accuracy of two Newton
// steps with a shorter dependent chain (3 and 4 fp64 ops) on the panel's critical path.
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x * y, y, 1.0);
  return fma(y * e, fma(0.375, e, 0.5), y);
}


// Grow-only bump allocator on the context workspace.  reset() at the start of
// every public call; alloc() 256-byte aligned.  Growing synchronises the device
// (cudaFree) and invalidates earlier allocations, so callers size everything up
// front with reserve().
int ws_reserve(jq_ctx* ctx, size_t bytes);
inline void ws_reset(jq_ctx* ctx) { ctx->ws.used = 0; }
template <class T>
T* ws_alloc(jq_ctx* ctx, size_t count) {
  size_t bytes = (count * sizeof(T) + 255) & ~size_t(255);
  if (ctx->ws.used + bytes > ctx->ws.cap) return nullptr;
  T* p = reinterpret_cast<T*>(ctx->ws.base + ctx->ws.used);
  ctx->ws.used += bytes;
  return p;
}
inline size_t ws_bytes(size_t count, size_t elem) { return (count * elem + 255) & ~size_t(255); }

bool is_device_ptr(const void* p);
bool is_pageable(const void* p);
// H2D of a staged input on ctx->stream (large pageable sources via a pinned ring)
int h2d_copy(jq_ctx* ctx, void* dst, const void* src, size_t bytes);

// Input staging: returns a device pointer for `p` (device pointers pass through;
// host buffers are copied into workspace memory on the context stream).
template <class T>
int stage_in(jq_ctx* ctx, const T* p, size_t count, const T** out) {
  if (p == nullptr || count == 0 || is_device_ptr(p)) { *out = p; return JQ_OK; }
  T* d = ws_alloc<T>(ctx, count);
  if (!d) return fail(JQ_E_OOM, "workspace exhausted while staging input");
  JQ_TRY(h2d_copy(ctx, d, p, count * sizeof(T)));
  *out = d;
  return JQ_OK;
}
template <class T>
int stage_out(jq_ctx* ctx, T* p, size_t count, T** out) {
  if (p == nullptr || count == 0 || is_device_ptr(p)) { *out = p; return JQ_OK; }
  T* d = ws_alloc<T>(ctx, count);
  if (!d) return fail(JQ_E_OOM, "workspace exhausted while staging output");
  *out = d;
  return JQ_OK;
}
template <class T>
int copy_out(jq_ctx* ctx, T* host_or_dev, const T* dev, size_t count) {
  if (host_or_dev == nullptr || count == 0 || host_or_dev == dev) return JQ_OK;
  JQ_CUDA(cudaMemcpyAsync(host_or_dev, dev, count * sizeof(T), cudaMemcpyDefault, ctx->stream));
  return JQ_OK;
}
// host bytes that stage_in would need for this pointer
template <class T>
size_t stage_bytes(const T* p, size_t count) {
  return (p == nullptr || count == 0 || is_device_ptr(p)) ? 0 : ws_bytes(count, sizeof(T));
}

int sync_and_check_flags(jq_ctx* ctx);   // stream sync + read device flags
// ctx->ev[k] (stage timing, jq_timing) + an NVTX mark naming the stage that begins there
void stage_event(jq_ctx* ctx, int k);
int begin_call(jq_ctx* ctx);              // device select + ws reset + clear flags

// ---------------------------------------------------------------- device helpers
__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ __device__ inline double splitmix_uniform(uint64_t seed, uint64_t k) {
  uint64_t x = mix64(seed + (k + 1) * 0x9E3779B97F4A7C15ull);
  return ((double)(x >> 11) + 0.5) * 1.1102230246251565e-16;  // 2^-53
}

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------- cross-TU entry points
// Grouping (jq_group.cu).  Device outputs: per-group arrays sized `cap`, per-row
// group ids (int32, -1 = unmatched) for each side, n_groups on device.
struct Groups {
  int64_t cap = 0;
  int64_t* keys = nullptr;
  int64_t* a_start = nullptr;
  int64_t* a_count = nullptr;
  int64_t* b_start = nullptr;
  int64_t* b_count = nullptr;
  int64_t* red_off = nullptr;  // cap + 1
  int32_t* gid_a = nullptr;    // m1
  int32_t* gid_b = nullptr;    // m2
  int64_t* d_n = nullptr;      // [0] = n_groups, [1] = total reduced rows
};
size_t group_ws_bytes(int64_t m1, int64_t m2);
int group_keys_dev(jq_ctx* ctx, const int64_t* ka, int64_t m1, const int64_t* kb, int64_t m2,
                   Groups* g);

// Head/tail prefix pass (jq_headtail.cu).  For a row-major matrix x (rows x cols)
// split into segments (gid per row, nullptr = one segment), compute per tile of
// TILE_ROWS rows the exclusive in-segment prefix at the tile start (carry) and
// per-group column totals.
constexpr int TILE_ROWS = 1024;
struct SegScan {
  int64_t ntiles = 0;
  int64_t rows = 0, cols = 0;
  double* carry = nullptr;   // ntiles x cols
  double* tile_agg = nullptr;
  int* tile_flag = nullptr;
  double* totals = nullptr;  // ngroups_cap x cols (group sums)
};
// The tile pass of a segmented scan as a job description: run by segscan_tiles, or by
// the spare warps of a TSQR leaf (FigaroArgs::side) while it factors the other side.
struct SideScan {
  const double* x = nullptr;  // nullptr: nothing to do
  int64_t rows = 0;
  int cols = 0;
  const int32_t* gid = nullptr;
  int64_t ntiles = 0;
  double* agg = nullptr;
  int* flag = nullptr;
  double* totals = nullptr;
};
size_t segscan_ws_bytes(int64_t rows, int64_t cols, int64_t groups_cap);
int segscan_begin(jq_ctx* ctx, const double* x, int64_t rows, int64_t cols, const int32_t* gid,
                  int64_t groups_cap, SegScan* s, SideScan* side);
int segscan_tiles(jq_ctx* ctx, const SideScan& side);
int segscan_end(jq_ctx* ctx, const int64_t* gstart, const int64_t* gcount, const int64_t* d_ngroups,
                int64_t groups_cap, SegScan* s);
int segscan_dev(jq_ctx* ctx, const double* x, int64_t rows, int64_t cols, const int32_t* gid,
                const int64_t* gstart, const int64_t* gcount, const int64_t* d_ngroups,
                int64_t groups_cap, SegScan* s);
// exclusive scan of int64 values; n_dev (optional) holds the live length <= n;
// out has n + 1 entries (out[len] = total).  Deterministic (integer).
size_t scan_ws_bytes(int64_t n);
int scan_i64_dev(jq_ctx* ctx, const int64_t* in, int64_t n, const int64_t* n_dev, int64_t* out);

// TSQR (jq_tsqr.cu).
struct FigaroSrc;  // defined in jq_tsqr.cu
int tsqr_dense_dev(jq_ctx* ctx, const double* m, int64_t rows, int64_t cols, double* r_out,
                   bool canonical);
int tsqr_stack_dev(jq_ctx* ctx, const double* rs, int64_t count, int64_t n, double* r_out,
                   bool canonical);
size_t tsqr_ws_bytes(int64_t rows, int64_t n, int sms);
// Figaro fused streaming TSQR: virtual rows built on the fly from A, B, heads and
// prefix carries.  Geometry / tables in FigaroArgs.
struct FigaroArgs {
  const double* a; int64_t m1, n1;
  const double* b; int64_t m2, n2;
  const int32_t* gid_a;          // nullptr = Cartesian
  const int32_t* gid_b;
  const int64_t* a_count;        // per group
  const int64_t* b_count;
  const int64_t* b_start;
  const double* b_totals;        // per group column sums of B (ngroups x n2)
  const double* b_carry;         // per TILE_ROWS tile exclusive prefix (ntiles x n2)
  const double* b_prefix0;       // shard: sum of B rows before this shard (n2), or nullptr
  // Cartesian shard extras (jq_figaro_r_shard): global sizes and row offset of B
  int64_t m1_global, m2_global, b_row0;
  SideScan side;                 // tile pass of another scan to run alongside (or nothing)
  // carry-free leaves (Cartesian footnote): every leaf's row block is its own group --
  // prefix from 0 at the block start, block row index -- and the leaf writes its block's
  // column sums to blk_sums[leaf][n2]; the between-block rows replace the carries
  // (block_heads_kernel).  blk_rows is set by the launcher (the leaf's rows).
  double* blk_sums;
  int64_t blk_rows;
};
int figaro_tsqr_dev(jq_ctx* ctx, const FigaroArgs& fa, double* r_out, bool canonical);
// TSQR leaves of a source without their tree (footnote: both sides' trees run in shared
// launches, tsqr_finish_pair); R's are NOT canonical
struct LeafSet {
  double* leaves;  // count NP x NP factors
  double* tmp;     // ceil(count / 2) factors (the single-stack tree's ping-pong buffer)
  int64_t count;
  int np, n;
  int64_t rows_per_leaf;
};
int figaro_tsqr_leaves(jq_ctx* ctx, const FigaroArgs& fa, LeafSet* out);
int tsqr_finish_pair(jq_ctx* ctx, const LeafSet& x, const LeafSet& y, double* rx, double* ry);
size_t tsqr_pair_ws_bytes(int64_t n, int sms);

// The join matrix itself (brute force): row v = [A_i | B_j], rows by
// key, then left row, then right row.  Cartesian when jo == nullptr (i = v / m2).
struct JoinArgs {
  const double* a; int64_t m1, n1;
  const double* b; int64_t m2, n2;
  const int64_t* jo;       // keyed: join-row offset of each matched group (ng + 1)
  const int64_t* a_start;  // keyed: per matched group
  const int64_t* b_start;
  const int64_t* b_count;
  int64_t ng;
  int64_t rows;            // join rows
};
// join row v -> (A row, B row)
__device__ __forceinline__ void join_row(const JoinArgs& ja, int64_t v, int64_t& ia, int64_t& ib) {
  if (!ja.jo) {
    ia = v / ja.m2;
    ib = v - ia * ja.m2;
    return;
  }
  int64_t lo = 0, hi = ja.ng - 1;  // last group with jo[g] <= v
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (__ldg(ja.jo + mid) <= v) lo = mid; else hi = mid - 1;
  }
  const int64_t local = v - __ldg(ja.jo + lo), bc = __ldg(ja.b_count + lo);
  const int64_t q = local / bc;
  ia = __ldg(ja.a_start + lo) + q;
  ib = __ldg(ja.b_start + lo) + (local - q * bc);
}
// canonical-or-not R of the join matrix, its rows generated inside the TSQR (never written)
int join_tsqr_dev(jq_ctx* ctx, const JoinArgs& ja, double* r_out, bool canonical);
size_t figaro_tsqr_ws_bytes(int64_t m1, int64_t m2, int64_t n, int sms);

// The reduced matrix into device memory (jq_headtail.cu; gr = nullptr: Cartesian).
int reduce_emit_dev(jq_ctx* ctx, const double* da, int64_t m1, int64_t n1, const double* db, int64_t m2,
                    int64_t n2, const Groups* gr, int64_t cap, int64_t total_rows, double* dout);
size_t reduce_emit_ws_bytes(int64_t m2, int64_t n2, int64_t cap);
// Wide Householder TSQR, 256 < n <= 512 (jq_wide.cu).
int wide_tsqr_dev(jq_ctx* ctx, const double* m, int64_t rows, int64_t n, double* r_out, bool canonical);
size_t wide_tsqr_ws_bytes(int64_t rows, int64_t n, int sms);

// SVD (jq_svd.cu).
size_t svd_ws_bytes(int64_t n);
int svd_dev(jq_ctx* ctx, const double* r, int64_t n, int want_v, double* values, double* v);

// small kernels
int canonicalize_dev(jq_ctx* ctx, const double* r, int64_t n, double* out);

}  // namespace jq
