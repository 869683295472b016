/*
 * alnnls.h — C ABI of the B200-native anti-lopsided NNLS solver.
 *
 * This is the drop-in boundary for the reference's hot path
 *   antilop::solve_nnls  (/root/reference/proj/include/antilop/nnls.hpp:129-144)
 *   antilop::solve_nqp   (/root/reference/proj/include/antilop/nqp.hpp:215-339)
 *   antilop::gram / transpose_matvec / masked_matvec / matvec
 *                        (/root/reference/proj/include/antilop/linalg.hpp:160-219)
 *   antilop::rescale / unscale (/root/reference/proj/include/antilop/nnls.hpp:41-96)
 * The reference is a header-only C++ library with no FFI; its public C++ API is
 * re-declared on top of this ABI by the headers in include/antilop/ (see INTEGRATION.md).
 *
 * Conventions
 *  - Plain pointers and sizes only. Matrices are column-major fp64, leading
 *    dimension = rows unless an explicit ld is passed (reference linalg.hpp:116).
 *  - Every entry point returns an alnnls_status. Exceptions never cross the ABI:
 *    EINVAL  <-> std::invalid_argument   (reference detail::require, linalg.hpp:22-24)
 *    ERANGE  <-> std::out_of_range       (linalg.hpp:199)
 *    ENUMERIC<-> antilop::NumericFailure (nqp.hpp:136-145); the trace up to the
 *                failing iteration stays retrievable with alnnls_get_trace.
 *    ECUDA / ENOMEM / ENCCL / ENODEV: device-side failures (no reference analogue).
 *  - A context (alnnls_ctx) owns device memory, streams and events for one GPU.
 *    It is single-threaded; independent contexts may run concurrently.
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point fails with ENODEV.
 */
#ifndef ALNNLS_H
#define ALNNLS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ALNNLS_ABI_VERSION 2

typedef enum alnnls_status {
  ALNNLS_OK = 0,
  ALNNLS_EINVAL = 1,
  ALNNLS_ENUMERIC = 2,
  ALNNLS_ECUDA = 3,
  ALNNLS_ENOMEM = 4,
  ALNNLS_ENCCL = 5,
  ALNNLS_ERANGE = 6,
  ALNNLS_ECAPACITY = 7, /* caller buffer too small */
  ALNNLS_ENODEV = 8
} alnnls_status;

/* Same order as antilop::Termination (nqp.hpp:47-54). */
typedef enum alnnls_termination {
  ALNNLS_EMPTY_PASSIVE_SET = 0,
  ALNNLS_GRADIENT_BELOW_EPSILON = 1,
  ALNNLS_MAX_ITERS = 2,
  ALNNLS_TIME_CAP = 3,
  ALNNLS_STALLED = 4,
  ALNNLS_ZERO_CURVATURE = 5
} alnnls_termination;

/* Numerics profile. EXACT replicates the reference operation sequence bit for
 * bit (rounded product then rounded sum, one ascending chain per output). */
typedef enum alnnls_profile { ALNNLS_PROFILE_EXACT = 0, ALNNLS_PROFILE_FAST = 1 } alnnls_profile;

/* antilop::SolverConfig (nqp.hpp:71-99) as POD. Unset optionals have has_* = 0.
 * Defaults are resolved against the retained dimension m exactly like
 * resolve_epsilon / resolve_max_iters (nqp.hpp:84-98). */
typedef struct alnnls_config {
  int32_t has_epsilon;
  double epsilon;
  int32_t has_max_iters;
  uint64_t max_iters;
  int32_t has_time_cap;
  double time_cap_s;
  uint64_t stall_window; /* reference default 50 */
  uint64_t trace_every;  /* reference default 1; 0 is treated as 1 (nqp.hpp:222) */
  int32_t profile;       /* alnnls_profile */
  int32_t record_multiplies; /* fill SolveStats::multiplies_per_iter */
  int32_t nesterov_restart;  /* SolverConfig::nesterov_restart (accelerated solver only) */
} alnnls_config;

/* antilop::IterRecord (nqp.hpp:103-110). has_alpha = 0 on the final record. */
typedef struct alnnls_iter_record {
  uint64_t iter;
  double f;
  double grad_bar_sq;
  uint64_t passive_count;
  double elapsed_s;
  double alpha;
  int64_t has_alpha;
} alnnls_iter_record;

/* Scalars of one solve (NnlsResult / SolveResult without the arrays). */
typedef struct alnnls_summary {
  int32_t termination;   /* alnnls_termination */
  int32_t numeric_failure; /* 1 when the solve ended in NumericFailure */
  uint64_t iterations;   /* SolveResult::iterations() = last record's iter */
  uint64_t trace_len;
  uint64_t mult_len;
  uint64_t n;            /* original dimension (NNLS) or m (NQP) */
  uint64_t m;            /* retained dimension */
  uint64_t n_dropped;
  double min_iterate;
  double residual_sq;    /* NNLS only: ||Ax-b||^2 recomputed from A, b (nnls.hpp:142) */
  double f_final;        /* last trace record's f */
  double gbs_final;      /* last trace record's grad_bar_sq */
  uint64_t multiplies_total; /* sum of multiplies_per_iter (algorithmic GEMV work) */
  /* device timings (CUDA events around each phase; seconds) */
  double t_setup_s;
  double t_loop_s;
  double t_finish_s;
  double t_total_s;
} alnnls_summary;

/* Per-column result of a batched solve (one NnlsResult without arrays). */
typedef struct alnnls_column_result {
  int32_t termination;
  int32_t numeric_failure;
  uint64_t iterations;
  double residual_sq;
  double f_final;
  double gbs_final;
  uint64_t multiplies_total;
} alnnls_column_result;

typedef struct alnnls_ctx alnnls_ctx;

/* ---- lifecycle ---------------------------------------------------------- */
int alnnls_abi_version(void);
/* Fills a config with the reference defaults (SolverConfig{}). */
void alnnls_config_default(alnnls_config* cfg);
/* Creates a context on CUDA device `device`; ENODEV without an sm_100 GPU. */
int alnnls_create(alnnls_ctx** out, int device);
void alnnls_destroy(alnnls_ctx* ctx);
/* Message of the last failure on this context (never NULL). */
const char* alnnls_last_error(const alnnls_ctx* ctx);
/* Device properties seen by the context. */
int alnnls_device_info(alnnls_ctx* ctx, int* sm_count, int* cc_major, int* cc_minor);

/* ---- hot path: host buffers (H2D/D2H inside) ---------------------------- */
/* solve_nnls(A, b, cfg) — nnls.hpp:129-144. A is d x n column-major (lda = d). */
int alnnls_solve_nnls(alnnls_ctx* ctx, uint64_t d, uint64_t n, const double* A,
                      const double* b, const alnnls_config* cfg, alnnls_summary* out);
/* solve_nqp(p, cfg, start) — nqp.hpp:215-339. Q is m x m column-major and must be
 * exactly symmetric (nqp.hpp:37-41); start may be NULL. */
int alnnls_solve_nqp(alnnls_ctx* ctx, uint64_t m, const double* Q, const double* q,
                     const double* start, const alnnls_config* cfg, alnnls_summary* out);

/* ---- hot path: device-resident inputs ---------------------------------- */
int alnnls_solve_nnls_device(alnnls_ctx* ctx, uint64_t d, uint64_t n, const double* dA,
                             uint64_t lda, const double* db, const alnnls_config* cfg,
                             alnnls_summary* out);
int alnnls_solve_nqp_device(alnnls_ctx* ctx, uint64_t m, const double* dQ, uint64_t ldq,
                            const double* dq, const double* dstart,
                            const alnnls_config* cfg, alnnls_summary* out);

/* ---- results of the last solve on ctx ----------------------------------- */
/* NNLS: x has n entries (unscaled, dropped columns 0). NQP: x has m entries. */
int alnnls_get_x(alnnls_ctx* ctx, double* x, uint64_t len);
/* Rescaled-space solution y (m) and maintained gradient final_grad (m). */
int alnnls_get_inner_x(alnnls_ctx* ctx, double* y, uint64_t len);
int alnnls_get_final_grad(alnnls_ctx* ctx, double* g, uint64_t len);
int alnnls_get_trace(alnnls_ctx* ctx, alnnls_iter_record* rec, uint64_t cap);
int alnnls_get_multiplies(alnnls_ctx* ctx, uint64_t* mults, uint64_t cap);
/* Vector-CTA phase times of the last device loop, accumulated (ns):
 * [0] stop-test chains, [1] rest of P1 + barrier, [2] den chain, [3] changed set,
 * [4] barrier + P2 + barrier, [5] df chain, [6] update + next mask, [7] barrier. */
int alnnls_get_phase_ns(alnnls_ctx* ctx, uint64_t* ns, uint64_t cap);
/* Device-side timing on the context's stream (CUDA events): start, then stop
 * returns the elapsed seconds between the two records. */
int alnnls_timer_start(alnnls_ctx* ctx);
int alnnls_timer_stop(alnnls_ctx* ctx, double* seconds);
/* Number of this library's kernels launched on the context so far. */
uint64_t alnnls_launch_count(const alnnls_ctx* ctx);
/* The device loop kernel of the last solve on the context (ALNNLS_LOOP_*): the
 * general loop as a cooperative grid or as one thread-block cluster, the small-m
 * cluster loop with its state in distributed shared memory (the environment
 * variable ALNNLS_SMALL=0 disables it), the FAST one-pass loop, or 0 (none). */
enum {
  ALNNLS_LOOP_NONE = 0,
  ALNNLS_LOOP_GRID = 1,
  ALNNLS_LOOP_CLUSTER = 2,
  ALNNLS_LOOP_SMALL = 3,
  ALNNLS_LOOP_FAST = 4
};
int alnnls_last_loop_kernel(const alnnls_ctx* ctx);
/* rescale bookkeeping of the last NNLS solve/setup (nnls.hpp:32-37). */
int alnnls_get_scale(alnnls_ctx* ctx, double* scale, uint64_t cap);
int alnnls_get_retained(alnnls_ctx* ctx, uint64_t* idx, uint64_t cap);
int alnnls_get_dropped(alnnls_ctx* ctx, uint64_t* idx, uint64_t cap);

/* ---- setup kernels (K1-K3) and dense helpers, for parity and reuse ------- */
/* rescale(gram(A), -A^T b) on device; afterwards Q (m x m), q (m), scale,
 * retained and dropped are retrievable. out->m / n_dropped are set. */
int alnnls_setup(alnnls_ctx* ctx, uint64_t d, uint64_t n, const double* A, const double* b,
                 alnnls_summary* out);
int alnnls_get_Q(alnnls_ctx* ctx, double* Q, uint64_t cap);
int alnnls_get_q(alnnls_ctx* ctx, double* q, uint64_t cap);
/* rescale(H, h) — nnls.hpp:41-83, host H (n x n) and h (n). EINVAL on an
 * asymmetric H or a negative diagonal, like the reference. */
int alnnls_rescale(alnnls_ctx* ctx, uint64_t n, const double* H, const double* h,
                   alnnls_summary* out);
/* gram(A) — linalg.hpp:160-174: H (n x n) = A^T A, exactly symmetric. */
int alnnls_gram(alnnls_ctx* ctx, uint64_t d, uint64_t n, const double* A, double* H);
/* transpose_matvec(A, v) — linalg.hpp:209-219. */
int alnnls_transpose_matvec(alnnls_ctx* ctx, uint64_t rows, uint64_t cols, const double* M,
                            const double* v, double* y);
/* matvec(M, v) — linalg.hpp:179-188. */
int alnnls_matvec(alnnls_ctx* ctx, uint64_t rows, uint64_t cols, const double* M,
                  const double* v, double* y);
/* masked_matvec(M, v, mask) — linalg.hpp:193-206. ERANGE on an index >= cols.
 * *multiply_count (if non-NULL) is incremented by rows*mask_len. */
int alnnls_masked_matvec(alnnls_ctx* ctx, uint64_t rows, uint64_t cols, const double* M,
                         const double* v, const uint64_t* mask, uint64_t mask_len, double* y,
                         uint64_t* multiply_count);

/* ---- batched multi-RHS (NMF H-update; one solve_nnls per column of B) ---- */
/* X (n x nrhs, column-major) and per-column results are written by the call.
 * Column j is bitwise equal to solve_nnls(A, B[:, j], cfg) under EXACT. */
int alnnls_solve_nnls_batched(alnnls_ctx* ctx, uint64_t d, uint64_t n, const double* A,
                              uint64_t nrhs, const double* B, const alnnls_config* cfg,
                              double* X, alnnls_column_result* cols, alnnls_summary* out);
int alnnls_solve_nnls_batched_device(alnnls_ctx* ctx, uint64_t d, uint64_t n,
                                     const double* dA, uint64_t nrhs, const double* dB,
                                     const alnnls_config* cfg, double* dX,
                                     alnnls_column_result* cols, alnnls_summary* out);

/* ---- Anti+Acc baseline: accelerated.hpp ---------------------
 * solve_accelerated (accelerated.hpp:21-117): Nesterov projected gradient with
 * the fixed step 1/||Q||_F (||Q||_F one ascending chain, linalg.hpp:222-226);
 * config.nesterov_restart enables the restart. solve_anti_accelerated
 * (:121-139): rescale, solve_accelerated, unscale, residual. Bitwise the
 * reference under EXACT; results through the same alnnls_get_* accessors. */
int alnnls_solve_accelerated(alnnls_ctx* ctx, uint64_t m, const double* Q, const double* q,
                             const alnnls_config* cfg, alnnls_summary* out);
int alnnls_solve_accelerated_device(alnnls_ctx* ctx, uint64_t m, const double* dQ, uint64_t ldq,
                                    const double* dq, const alnnls_config* cfg,
                                    alnnls_summary* out);
int alnnls_solve_anti_accelerated(alnnls_ctx* ctx, uint64_t d, uint64_t n, const double* A,
                                  const double* b, const alnnls_config* cfg, alnnls_summary* out);
int alnnls_solve_anti_accelerated_device(alnnls_ctx* ctx, uint64_t d, uint64_t n, const double* dA,
                                         uint64_t lda, const double* db, const alnnls_config* cfg,
                                         alnnls_summary* out);

/* ---- multi-GPU exact setup by row blocks -----------
 * A is split into row blocks A_0, A_1, ... (ranks). Every sum of the
 * reference setup is one ascending chain over the rows (gram linalg.hpp:168,
 * transpose_matvec :215, residual_norm_sq nnls.hpp:119-122), so a block can
 * continue the chain states left by the blocks before it: feeding the blocks
 * in row order reproduces the single-GPU results bit for bit.
 * Gram states are kept per upper-triangular 128 x 128 output tile
 * (ALNNLS_GRAM_TILE_DOUBLES doubles per tile, an opaque layout); all buffers
 * are device pointers, and the calls return after their work is complete. */
#define ALNNLS_GRAM_TILE_DOUBLES 16384
uint64_t alnnls_gram_tiles(uint64_t n);
/* Tiles [tile_lo, tile_hi) over the block (rows x n, ld lda): from dpin
 * (states after the earlier blocks, tile t at (t - tile_lo) * TILE_DOUBLES;
 * NULL = first block) to dpout (same layout), or, when dpout is NULL, the
 * finished Gram entries of those tiles into dH (n x n, column-major). */
int alnnls_gram_rowblock_device(alnnls_ctx* ctx, uint64_t rows, uint64_t n, const double* dA,
                                uint64_t lda, uint64_t tile_lo, uint64_t tile_hi,
                                const double* dpin, double* dpout, double* dH);
/* A^T b chains over the block: dout[j] = dpin[j] (or 0) + sum over the block rows
 * in order (transpose_matvec, before the negation of nnls.hpp:133-134). */
int alnnls_atb_rowblock_device(alnnls_ctx* ctx, uint64_t rows, uint64_t n, const double* dA,
                               uint64_t lda, const double* db, const double* dpin, double* dout);
/* solve_nnls from the finished Gram dH (n x n) and A^T b chains dAtb: rescale,
 * solve_nqp, unscale (nnls.hpp:133-141). The residual needs A and b and is
 * formed by the ranks with alnnls_residual_rowblock_device; out->residual_sq is 0. */
int alnnls_solve_nnls_gram_device(alnnls_ctx* ctx, uint64_t n, const double* dH,
                                  const double* dAtb, const alnnls_config* cfg,
                                  alnnls_summary* out);
/* residual_norm_sq over the block's rows, continuing the ordered chain from s_in
 * (0 for the first block): *s_out = ((s_in + r_0^2) + r_1^2) + ..., r = A_blk x - b_blk. */
int alnnls_residual_rowblock_device(alnnls_ctx* ctx, uint64_t rows, uint64_t n, const double* dA,
                                    uint64_t lda, const double* db, const double* dx, double s_in,
                                    double* s_out);

/* ---- multi-GPU setup by partial Grams + one allreduce --
 * BASELINE.json configs[4] as written: every rank forms the partial Gram of its
 * row block and the partials are summed with one allreduce (the caller's NCCL
 * over NVLink), then one rank runs alnnls_solve_nnls_gram_device. Replaces the
 * reference's gram (linalg.hpp:160-174) and transpose_matvec (linalg.hpp:209-
 * 219) for a row block; the cross-rank sum order is NCCL's, so the result is
 * within rounding of the reference's H, not bitwise (use the row-block chain
 * entries above for that).
 * dH (n x n, column-major, both triangles) = A_blk^T A_blk and, when db is not
 * NULL, datb = A_blk^T b_blk. profile ALNNLS_PROFILE_FAST forms dH on the fp64
 * tensor cores (needs lda even and 16-byte aligned dA), EXACT with the chain
 * SYRK. dH and datb may be adjacent in one buffer so that a single allreduce
 * moves both. Returns after the work is complete. */
int alnnls_gram_partial_device(alnnls_ctx* ctx, uint64_t rows, uint64_t n, const double* dA,
                               uint64_t lda, const double* db, int profile, double* dH,
                               double* datb);

/* Packed upper triangle of a symmetric n x n matrix (device pointers): entry
 * (i, j), i <= j, at j*(j+1)/2 + i. pack: dP <- upper(dH); unpack: dH <- dP,
 * mirrored to both triangles. The allreduce setup moves n(n+1)/2 doubles with
 * them instead of n^2 (rowblock.allreduce_setup). Return after completion. */
int alnnls_pack_upper_device(alnnls_ctx* ctx, uint64_t n, const double* dH, double* dP);
int alnnls_unpack_upper_device(alnnls_ctx* ctx, uint64_t n, const double* dP, double* dH);

/* ---- finish: unscale + residual (nnls.hpp:141-142) ------------------------
 * x = unscale(y, sys, n) (nnls.hpp:87-96) with the rescale bookkeeping (scale,
 * retained, dropped) of the last setup / solve / rescale on ctx, and
 * *residual_sq = residual_norm_sq(A, b, x) (nnls.hpp:115-123), recomputed from
 * A (d x n, column-major) and b. y has m = the retained count entries. EINVAL
 * when m or n do not match that bookkeeping (reference: "unscale: dimension
 * mismatch"). Host buffers. */
int alnnls_finish(alnnls_ctx* ctx, uint64_t d, uint64_t n, const double* A, const double* b,
                  const double* y, uint64_t m, double* x, double* residual_sq);

/* ---- batched multi-RHS across GPUs: one context per device ---------------
 * Column shards of B (contiguous, balanced like paper_1502_01645_b200/
 * sharding.py) run concurrently, one host thread per context, each through
 * alnnls_solve_nnls_batched on its own device; no data-path collective (every
 * column is an independent solve_nnls). Same outputs as the one-context call
 * (column j bitwise solve_nnls(A, B[:, j], cfg) under EXACT). out: times are the
 * max over contexts, iterations / multiplies / numeric_failure are combined. On
 * failure the first failing context's status is returned and its message is
 * copied to ctxs[0]. */
int alnnls_solve_nnls_batched_multi(alnnls_ctx* const* ctxs, int nctx, uint64_t d, uint64_t n,
                                    const double* A, uint64_t nrhs, const double* B,
                                    const alnnls_config* cfg, double* X,
                                    alnnls_column_result* cols, alnnls_summary* out);
/* Dense product on device pointers, column j = matvec(A, H[:, j]) bit for bit
 * (linalg.hpp:179-188: one ascending chain of rounded products and sums per
 * entry). C (rows x cols, ldc) = A (rows x inner, lda) H (inner x cols, ldh).
 * Forms c4's right-hand sides B = A H_true identically on any host (the
 * harness's exact-order generator computes the same bits), and the NMF
 * product W H. Returns after completion. */
int alnnls_matmat_device(alnnls_ctx* ctx, uint64_t rows, uint64_t inner, uint64_t cols,
                         const double* dA, uint64_t lda, const double* dH, uint64_t ldh,
                         double* dC, uint64_t ldc);
/* ---- NMF by alternating NNLS (the paper's motivating use,
 * PAPER.md:22) -----------------------------------------------------------------
 * V (d x N) ~ W (d x k) H (k x N), W, H >= 0. Each outer iteration solves
 *   H <- argmin_{H >= 0} ||W H - V||_F^2   (one solve_nnls(W, V[:, j], cfg) per column)
 *   W <- argmin_{W >= 0} ||H^T W^T - V^T||_F^2 (one solve_nnls(H^T, V^T[:, i], cfg) per row)
 * with the batched multi-RHS solver (one shared Gram per half step; the
 * transposes are exact copies), so under EXACT every column of every half step
 * is bitwise the reference's solve_nnls on the same inputs. W holds the start on
 * entry and the result on exit; H is written. objective[t] (outer_iters entries,
 * may be NULL) = ||V - W H||_F^2 after iteration t's H update, summed over the
 * columns' residual_norm_sq (nnls.hpp:115-123) in column order. k <= 1024 (the
 * batched kernel's bound). Device-pointer entry (all column-major, ld = rows)
 * and host-buffer entry. */
int alnnls_nmf_device(alnnls_ctx* ctx, uint64_t d, uint64_t N, uint64_t k, const double* dV,
                      double* dW, double* dH, uint64_t outer_iters, const alnnls_config* cfg,
                      double* objective);
int alnnls_nmf(alnnls_ctx* ctx, uint64_t d, uint64_t N, uint64_t k, const double* V, double* W,
               double* H, uint64_t outer_iters, const alnnls_config* cfg, double* objective);
/* Number of visible CUDA devices (0 without a GPU; no context needed). */
int alnnls_device_count(void);

#ifdef __cplusplus
}
#endif

#endif /* ALNNLS_H */
