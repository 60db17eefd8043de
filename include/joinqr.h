/*
 * joinqr.h — C ABI of libjoinqr.so, the B200 (sm_100a) implementation of the
 * Figaro two-table QR / SVD hot path (arXiv 2503.23385, BASELINE.json north_star).
 *
 * The reference (/root/reference) exposes this path only as a Python API —
 * package `joinqr`, 41 lazily resolved names (pkg/src/joinqr/__init__.py:20-62) —
 * and ships no FFI.  Each entry point below replaces one reference operation and
 * cites the SPEC.md lines that define it (the reference modules themselves are
 * absent; SPEC.md is the de-facto implementation).  The Python
 * mirror paper_2503_23385_b200/ binds these through ctypes.
 *
 * Conventions
 *   - Plain pointers and sizes, no torch types.  Matrices are row-major float64
 *     with a row stride equal to the column count (numpy C-contiguous,
 *     pkg/src/joinqr/matrix.py:13-22).  Keys are int64.
 *   - Every pointer may be HOST memory (pageable or pinned) or DEVICE memory of
 *     the context's GPU; the library detects which (cudaPointerGetAttributes).
 *     Host inputs are copied in and outputs copied out inside the call; device
 *     pointers are used in place (no host round trip).
 *   - Calls are stream-ordered on the context stream and return after the
 *     result is complete (synchronous), except the *_async entry points.
 *   - Return 0 on success, else a JQ_E_* code; jq_last_error() gives the
 *     message (thread-local).  Errors map to the reference's exception types:
 *     JQ_E_INVALID / JQ_E_UNSORTED / JQ_E_KEYS -> ValueError (matrix.py:19,21,
 *     SPEC.md:196,206,280), JQ_E_NOCONV -> RuntimeError,
 *     JQ_E_OOM -> MemoryError, JQ_E_CUDA / JQ_E_NODEV -> RuntimeError.
 *   - One context per host thread; calls on one context are serialised.
 */
#ifndef JOINQR_H
#define JOINQR_H

#include <stdint.h>

#if defined(__GNUC__)
#define JQ_API __attribute__((visibility("default")))
#else
#define JQ_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define JQ_OK 0
#define JQ_E_INVALID 1
#define JQ_E_UNSORTED 2
#define JQ_E_KEYS 3
#define JQ_E_NOCONV 4
#define JQ_E_OOM 5
#define JQ_E_CUDA 6
#define JQ_E_NODEV 7

typedef struct jq_ctx jq_ctx;

/* Per-stage device time of the last figaro call on a context (CUDA events, ms). */
typedef struct jq_timing {
  double group_ms;   /* key grouping (0 for a Cartesian product)            */
  double scan_ms;    /* head/tail prefix pass (segmented column sums)        */
  double tsqr_ms;    /* streamed assembly + TSQR leaves                      */
  double tree_ms;    /* TSQR tree combine + canonicalisation                 */
  double svd_ms;     /* Jacobi SVD (0 for figaro_r)                          */
  double total_ms;   /* first event to last event                            */
  int64_t tsqr_ctas; /* leaves of the TSQR tree                              */
  int64_t reduced_rows; /* rows streamed into the TSQR (incl. zero padding)  */
  double scan_tile_ms;    /* the head/tail tile-pass kernel(s) alone (<= 4 launches) */
  double scan_tile_bytes; /* their algorithmic bytes (rows read once + segment ids)  */
} jq_timing;

/* ---- library / context ------------------------------------------------- */
JQ_API int jq_version(void);                                 /* 100 * major + minor */
JQ_API const char* jq_last_error(void);
JQ_API int jq_ctx_create(int device, jq_ctx** out);
JQ_API int jq_ctx_destroy(jq_ctx* ctx);
/* Use a caller stream (e.g. torch.cuda.current_stream().cuda_stream); NULL
 * restores the context's own (non-blocking) stream.  The legacy default stream
 * must be passed as cudaStreamLegacy ((void*)0x1), not as NULL: the own stream
 * does not wait for work queued on the legacy stream. */
JQ_API int jq_ctx_set_stream(jq_ctx* ctx, void* cuda_stream);
JQ_API int jq_ctx_sync(jq_ctx* ctx);
/* Internal variant switch: 0 = dense Claim-1 reduced matrix (north star),
 * 1 = footnote variant (head/tail of both sides, PAPER.md:59 footnote),
 * 2 = auto (default): footnote from (m1 + m2) * (n1 + n2) > 1e8, else dense.
 * All variants return the same canonical R within the parity tolerance. */
JQ_API int jq_ctx_set_variant(jq_ctx* ctx, int variant);
JQ_API int jq_last_timing(jq_ctx* ctx, jq_timing* out);
/* Number of launches of this library's kernels since context creation. */
JQ_API int64_t jq_kernel_launches(jq_ctx* ctx);

/* ---- headtail ---------------------------------------- */
/* out (rows x cols): row 0 = head(m), rows 1.. = tail(m) (
 * head :115-123, tail :125-133).  rows = 0 -> JQ_E_INVALID. */
JQ_API int jq_head_tail(jq_ctx* ctx, const double* m, int64_t rows, int64_t cols, double* out);

/* ---- join-reduce ------------------------------------- */
/* Grouping of two sorted key columns, ascending matched key order
 * (SPEC.md:205, :223).  Output arrays hold up to `capacity` groups
 * (min(m1, m2) always suffices); red_off holds n_groups + 1 entries,
 * red_off[g+1] - red_off[g] = a_count[g] + b_count[g] - 1.
 * Unsorted keys -> JQ_E_UNSORTED. */
JQ_API int jq_group_keys(jq_ctx* ctx, const int64_t* ka, int64_t m1, const int64_t* kb, int64_t m2,
                  int64_t capacity, int64_t* n_groups, int64_t* keys, int64_t* a_start,
                  int64_t* a_count, int64_t* b_start, int64_t* b_count, int64_t* red_off);

/* Claim-1 reduced matrix in SPEC row order (reduce_cartesian SPEC.md:189-200
 * when ka == kb == NULL, reduce_natural_join SPEC.md:202-210 otherwise).
 * out == NULL only reports *out_rows.  Otherwise out holds out_capacity rows of
 * n1 + n2 doubles; group_bounds (optional, 2 * n_groups int64) receives the
 * per-group [start, stop) row ranges. */
JQ_API int jq_reduce(jq_ctx* ctx, const double* a, int64_t m1, int64_t n1, const int64_t* ka,
              const double* b, int64_t m2, int64_t n2, const int64_t* kb,
              double* out, int64_t out_capacity, int64_t* out_rows, int64_t* group_bounds);

/* ---- qr ---------------------------------------------- */
/* n x n upper-triangular R of m (cols = n), R^T R = m^T m, NOT sign-canonical
 * (householder_r SPEC.md:250-258; zero-row padding when rows < cols :296). */
JQ_API int jq_householder_r(jq_ctx* ctx, const double* m, int64_t rows, int64_t cols, double* r);
/* Negate rows with a negative diagonal entry. */
JQ_API int jq_canonicalize(jq_ctx* ctx, const double* r, int64_t n, double* out);
/* Canonical R of the join matrix (figaro_r); n = n1 + n2. */
JQ_API int jq_figaro_r(jq_ctx* ctx, const double* a, int64_t m1, int64_t n1, const int64_t* ka,
                const double* b, int64_t m2, int64_t n2, const int64_t* kb, double* r);

/* ---- svd --------------------------------------------- */
/* Descending singular values (and V when want_v != 0) of an n x n R by
 * one-sided Jacobi.  Non-convergence -> JQ_E_NOCONV. */
JQ_API int jq_svd_of_r(jq_ctx* ctx, const double* r, int64_t n, int want_v, double* values, double* v);
/* figaro_r followed by svd_of_r; r (optional) receives R. */
JQ_API int jq_figaro_svd(jq_ctx* ctx, const double* a, int64_t m1, int64_t n1, const int64_t* ka,
                  const double* b, int64_t m2, int64_t n2, const int64_t* kb, int want_v,
                  double* values, double* v, double* r);

/* ---- data-io generator --------------------------------- */
/* rows x cols uniform(0,1) block starting at table row row0 of the SplitMix64
 * table `seed` (oracle/datagen.py documents the bit recipe). */
JQ_API int jq_gen_uniform(jq_ctx* ctx, uint64_t seed, int64_t rows, int64_t cols, int64_t row0, double* out);
/* Sorted Zipf(s) keys over [0, universe) for a table of `rows` rows: the sorted
 * multiset of searchsorted(cdf, u_row, 'right') (cdf given, universe entries). */
JQ_API int jq_gen_zipf_sorted_keys(jq_ctx* ctx, uint64_t seed, int64_t rows, const double* cdf,
                            int64_t universe, int64_t* keys_out);
/* Unsorted Zipf keys, one per row in generation order: keys_out[i] =
 * searchsorted(cdf, u_i, 'right') (SURVEY.md §8d C3 recipe, before the stable sort). */
JQ_API int jq_gen_zipf_keys(jq_ctx* ctx, uint64_t seed, int64_t rows, const double* cdf, int64_t universe,
                            int64_t* keys_out);

/* ---- data-io: CSV ingest -------------------------------- */
/* Row and cell counts of a CSV table (comma separated, optional single header
 * line, blank lines skipped); host only, multithreaded over the mmapped file. */
JQ_API int jq_csv_scan(const char* path, int has_header, int64_t* rows, int64_t* cols);
/* Parse the table into data (rows x (cols - [key_col >= 0]) f64, row-major) and
 * keys (rows int64, key_col >= 0) -- host or device buffers.  Device outputs are
 * streamed through pinned staging slots with the H2D copies on the context stream
 * overlapping the parse.  Errors (JQ_E_INVALID) name the file line: ragged row,
 * unparsable cell, non-finite value, unsorted keys.  Replaces read_table's parser
 * (SPEC.md:458). */
JQ_API int jq_csv_parse(jq_ctx* ctx, const char* path, int has_header, int key_col, int64_t rows, int64_t cols,
                        double* data, int64_t* keys);

/* ---- key sort for unsorted tables (opt-in; SPEC.md:204-206 raises by default) ---- */
/* Stable LSD radix sort of m int64 keys: perm_out[i] = the original row of sorted
 * position i, equal to np.argsort(keys, kind="stable") bit for bit; keys_out
 * (optional) = keys[perm_out].  Replaces the caller-side sort the reference
 * requires before reduce_natural_join / figaro_r. */
JQ_API int jq_sort_keys(jq_ctx* ctx, const int64_t* keys, int64_t m, int64_t* keys_out, int64_t* perm_out);
/* out[i, :] = x[perm[i], :] for a row-major rows x cols table (perm entries must lie
 * in [0, rows)): applies jq_sort_keys' permutation to the data rows. */
JQ_API int jq_gather_rows(jq_ctx* ctx, const double* x, int64_t rows, int64_t cols, const int64_t* perm,
                          double* out);

/* ---- row-sharded multi-GPU building blocks -------------- */
/* Column sums of a row block (fixed-order, deterministic): sums[cols]. */
JQ_API int jq_colsums(jq_ctx* ctx, const double* x, int64_t rows, int64_t cols, double* sums);
/* Local R of one shard of a Cartesian product.  The shard holds A rows
 * [a_row0, a_row0 + a_rows) of an m1-row table and B rows [b_row0, b_row0 + b_rows)
 * of an m2-row table; x_prefix = sum of the rows of X before the shard and
 * x_total = sum of all rows of X (n1 / n2 doubles each, from an all-gather of
 * jq_colsums).  Dense variant: the Claim-1 rows of the shard (a_prefix/a_total
 * unused).  Footnote variant: tails of both sides plus, when include_head != 0,
 * the single head row (exactly one rank passes 1).  r_local is n x n, not
 * canonical; the stack of all ranks' r_local has the join's R (jq_tsqr_stack). */
JQ_API int jq_figaro_r_shard(jq_ctx* ctx, const double* a, int64_t a_rows, int64_t n1, int64_t m1,
                             int64_t a_row0, const double* a_prefix, const double* a_total,
                             const double* b, int64_t b_rows, int64_t n2, int64_t m2, int64_t b_row0,
                             const double* b_prefix, const double* b_total, int include_head,
                             double* r_local);
/* Footnote variant with carry-free leaves on one Cartesian row shard (A rows
 * a_rows of an m1-row table, B rows b_rows of an m2-row table, n1, n2 > 0): the
 * shard's local R (its blocks' tails and between-block rows, scaled by sqrt(m2) /
 * sqrt(m1); no head row, no between-shard row) and sums[n1 + n2] = the shard's
 * column sums (A then B).  Needs no prefix: the between-shard rows and the head row
 * follow from the all-gathered sums (paper_2503_23385_b200/sharded.py), so one
 * all-gather carries R and sums.  Replaces the carry exchange of jq_figaro_r_shard
 * for the same R (SPEC.md:278-286 by Gram). */
JQ_API int jq_figaro_r_shard_local(jq_ctx* ctx, const double* a, int64_t a_rows, int64_t n1, int64_t m1,
                                   const double* b, int64_t b_rows, int64_t n2, int64_t m2, double* r_local,
                                   double* sums);
/* Rows completing the join Gram of key groups split by rows across shards
 * (SURVEY.md §8e co-partition; a Cartesian product is one group split over every
 * rank).  Part k (ordered by part_group[k], groups contiguous, parts of a group in
 * shard order) holds part_rows[2k] A rows and part_rows[2k+1] B rows of its group and
 * was factored by jq_figaro_r_shard_local with the group's m1g / m2g (the sums of the
 * group's parts) -- part_sums[k] is that call's sums (n1 + n2).  Writes per group the
 * head row [sqrt(m2g) hA | sqrt(m1g) hB] and one between-part row per side and part
 * after the first (pairwise scatter update).  rows == NULL only reports *n_rows.
 * part_rows / part_group are host arrays; part_sums and rows host or device.
 * Replaces the host-side prefix / head arithmetic of the carry exchange. */
JQ_API int jq_split_group_rows(jq_ctx* ctx, const double* part_sums, const int64_t* part_rows,
                               const int64_t* part_group, int64_t nparts, int64_t n1, int64_t n2, double* rows,
                               int64_t rows_capacity, int64_t* n_rows);
/* Canonical R of the row stack [R_0; R_1; ...; R_{count-1}] (each n x n), by
 * the fixed binary TSQR tree — identical on every rank for the same input. */
JQ_API int jq_tsqr_stack(jq_ctx* ctx, const double* rs, int64_t count, int64_t n, double* r);

/* ---- brute force (oracle module): the join matrix itself -------- */
/* materialize_cartesian (ka == kb == NULL) / materialize_natural_join
 * (SPEC.md:387): rows [A_i | B_j] ordered by key, then left row, then right row.
 * out == NULL only reports *out_rows; otherwise out holds out_capacity rows of
 * n1 + n2 doubles. */
JQ_API int jq_materialize(jq_ctx* ctx, const double* a, int64_t m1, int64_t n1, const int64_t* ka,
                   const double* b, int64_t m2, int64_t n2, const int64_t* kb, double* out,
                   int64_t out_capacity, int64_t* out_rows);
/* Canonical R of the join matrix by TSQR over its rows, generated on the fly and
 * never written: baseline_r without the materialisation -- the
 * performance foil of figaro_r. */
JQ_API int jq_join_r_bruteforce(jq_ctx* ctx, const double* a, int64_t m1, int64_t n1, const int64_t* ka,
                         const double* b, int64_t m2, int64_t n2, const int64_t* kb, double* r);

#ifdef __cplusplus
}
#endif
#endif /* JOINQR_H */
