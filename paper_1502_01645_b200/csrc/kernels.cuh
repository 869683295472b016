// kernels.cuh — host-visible launch interface of the sm_100a kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/alnnls.h"

namespace alnnls {

// Device-resident control block of one NQP solve (written by the loop kernel).
struct LoopCtrl {
  int stop;
  int mask_len;
  int chg_len;
  int accept;
  double alpha;
  int termination;
  int numeric_failure;
  unsigned long long iterations;
  unsigned long long trace_len;
  unsigned long long mult_len;
  unsigned long long mult_total;
  double min_iterate;
  double f_final;
  double gbs_final;
  int state;        // leader -> grid broadcast after a barrier (LoopState)
  int act;          // phase-A decision: continue / stop / roll back the pending step
  int state2;       // phase-B decision: P2 / no move / stop
  int g_parity;     // which gradient buffer holds the maintained gradient
  unsigned int p1_done;  // row CTAs that finished P1 (monotonic within a launch)
  unsigned int bc_epoch; // the vector CTA's phase-B results are published (pass number)
  unsigned long long phase_ns[8];  // accumulated leader-side phase times
};

struct LoopArgs {
  const double* Q;  // m x m, column-major, leading dimension ldq
  uint64_t ldq;
  const double* q;
  int m;
  double* x;        // iterate (m)
  double* g;        // maintained gradient, ping-pong buffer 0 (m)
  double* g_alt;    // ping-pong buffer 1 (m)
  double* u;        // Q g_bar (m)
  double* gd;       // Q delta (m)
  uint32_t* mask;   // passive set, ascending (m)
  double* gP;       // g on the mask (m + 2)
  uint32_t* chg;    // changed set, ascending (m)
  double* dC;       // delta on the changed set (m + 2)
  double* candC;    // candidate x on the changed set (m)
  double* gC;       // g on the changed set (m)
  double* xP;       // x on the mask (m)
  double* qP;       // q on the mask (m)
  double* x_alt;    // x ping-pong buffer 1 (row CTAs own x and g)
  uint32_t* mask2;  // second passive-list set (ping-pong for the speculative step)
  double* gP2;
  double* xP2;
  double* qP2;
  double* uP;       // (Q g_bar) compacted to the passive list: uP[t] = u[mask[t]]
  double* gdC;      // (Q delta) compacted to the changed list: gdC[t] = gd[chg[t]]
  int* cnt;         // per row-CTA passive counts
  double* minx;     // per row-CTA min(x)
  int* badv;        // per row-CTA non-finite gradient flags
  // resolved SolverConfig (nqp.hpp:219-222)
  double eps;
  uint64_t max_iters;
  int has_time_cap;
  double time_cap_s;
  uint64_t stall_window;
  uint64_t trace_every;
  alnnls_iter_record* trace;
  uint64_t trace_cap;
  uint64_t* mults;  // may be null
  uint64_t mults_cap;
  LoopCtrl* ctrl;
  unsigned int* bar;  // grid barrier words {count, generation}, zeroed before launch
  int rows_per_cta;
  int resident;     // row CTAs keep their Q panel in shared memory (small m, gemv_resident)
  float l2_frac;    // ring copies of Q: this fraction of its lines L2 evict_last (0: no hint)
  int zero_start;   // x = 0, g = q not yet written: the loop launch initialises them
                    // (the small-m kernel in its prologue; launch_nqp_loop otherwise)
  // accelerated (Nesterov) solver only (accelerated.hpp:21-117)
  double* y;        // extrapolated point (m)
  double* xn;       // projected step from y (m)
  double* w;        // Q y (m)
  double* vy;       // y on the union list (mask holds the list, gP the x values)
  int* pcnt;        // per row-CTA passive counts of (x, grad)
  double alpha;     // 1 / ||Q||_F
  int restart;      // SolverConfig::nesterov_restart
};

// Exact device-resident solve_nqp loop (nqp.hpp:249-334). One cooperative
// launch for the whole solve; returns the launch status.
// which (optional) <- the loop kernel launched (ALNNLS_LOOP_* in alnnls.h).
cudaError_t launch_nqp_loop(const LoopArgs& a, int num_ctas, cudaStream_t stream,
                            int* which = nullptr);
// Small-m variant (small.cu): one cluster, loop state in distributed shared memory.
// cudaErrorNotSupported when the shape does not fit it (launch_nqp_loop then takes
// the general kernel).
bool nqp_small_fits(int m, int R, int num_ctas);
cudaError_t launch_nqp_small(const LoopArgs& a, int num_ctas, cudaStream_t stream);
// Accelerated (Nesterov) baseline loop (accelerated.hpp:21-117), same CTA layout.
cudaError_t launch_acc_loop(const LoopArgs& a, int num_ctas, cudaStream_t stream,
                            int* which = nullptr);
// frobenius_norm of the blocked m x m Q (linalg.hpp:222-226): one ascending chain
// over the column-major entries, then sqrt, into *out (one CTA).
cudaError_t launch_frobenius(const double* Qb, int m, int R, double* out, cudaStream_t stream);
int nqp_rows_per_cta(int m, int sm_count);
size_t nqp_loop_smem_bytes();
// true when a row CTA's Q panel (R x m) and the staged list fit its shared memory
bool nqp_resident_fits(int m, int R);

// FAST-profile single-RHS loop (fastloop.cu): one streaming pass over the passive
// columns of Q per iteration (one-pass update), fixed-tree reductions.
struct FastPart {  // one CTA's partial sums of a state (and of the try that produced it)
  double gbs, xg, qx, minx, df, el;
  int cnt, bad, nchg, pad;
};
struct FastArgs {
  const double* Q;  // blocked m x m (gemv.cuh blk_index, block rows R)
  int m;
  int R;
  const double* q;
  double* x[2];     // ping-pong states; [0] holds the start point
  double* g[2];
  double* gbar[2];  // g on the passive set, 0 elsewhere (m)
  FastPart* part[2];  // [nblk] per state slot
  double* den;      // [nblk]
  uint32_t* kl;     // [nblk * R] clamped columns per CTA
  double* kv;       // [nblk * R] their coefficients alpha g - x
  int* kc;          // [nblk]
  int local_k;      // set by launch_fast_loop: x staged in shared memory too
  float l2_frac;    // set by launch_fast_loop: fraction of Q's lines loaded L2 evict_last
  double eps;
  uint64_t max_iters;
  int has_time_cap;
  double time_cap_s;
  uint64_t stall_window;
  uint64_t trace_every;
  alnnls_iter_record* trace;
  uint64_t trace_cap;
  uint64_t* mults;
  uint64_t mults_cap;
  LoopCtrl* ctrl;
};
bool fast_loop_supported(int m, int R);
cudaError_t launch_fast_loop(const FastArgs& a, cudaStream_t stream);

// Exact masked GEMV over a row range: y[i] = sum_t M[i, list[t]] * vals[t].
// dlen (optional): the length is read on the device from *dlen (no host round trip).
cudaError_t launch_masked_gemv(const double* M, uint64_t ld, int rows, const uint32_t* list,
                               const double* vals, int len, double* y, int sm_count,
                               cudaStream_t stream, const int* dlen = nullptr);
// y = x or x_alt (m entries), whichever the finished loop's ctrl->g_parity names:
// the iterate is taken on the device, before the host has read the control block.
cudaError_t launch_copy_parity(double* y, const double* x, const double* x_alt,
                               const LoopCtrl* ctrl, int m, cudaStream_t stream);

// Setup (K1-K3): D_i^2 = H_ii chains, retained compaction, fused SYRK+rescale.
struct SetupArgs {
  const double* A;  // d x n, lda
  uint64_t lda;
  const double* b;  // d
  int d;
  int n;
  double* diag;     // n: H_ii
  int* pos;         // n: retained position or -1
  double* scale;    // m: D_a = sqrt(H_ii)
  uint32_t* retained; // m
  int* m_out;       // device scalar
  double* Q;        // m x m in the blocked layout (gemv.cuh blk_index, block rows qR)
  int m;            // retained count (known on the host before the SYRK launch)
  int qR;
  double* q;        // m
  double* H;        // optional: raw gram output (n x n, ld n), nullptr when fusing rescale
  double* hvec;     // optional: raw -A^T b (n)
  double* hvec_scratch;  // n doubles for A^T b when b is given
  // mode 2 (batched right-hand sides): QB[:, j] = q of column j of B
  const double* B;  // d x nrhs, ldb
  uint64_t ldb;
  int nrhs;
  double* QB;       // m x nrhs (ld m)
  // exact SYRK stream-K scheduling (setup.cu): partial chain states [ctas][32][512]
  // and per-CTA ready flags; sk_ctas = 0 runs one CTA per tile
  double* sk_part;
  int* sk_flag;
  int sk_ctas;
  // mode 0 row-block continuation through the stream-K kernel: every tile's chain
  // starts from tpin[t] and ends in tpout[t] ([tiles][32][512]) instead of 0 / H
  const double* tpin;
  double* tpout;
  // FAST DMMA Gram v2 (dmma.cu syrk_tma_kernel): stream-K partials and flags
  double* dm_ws;
  int* dm_flags;
  int dm_ctas;
};
// CTAs for the stream-K exact SYRK of this shape (0: use one CTA per tile).
int syrk_streamk_ctas(const SetupArgs& s, int mode, int sm_count);
cudaError_t launch_gram_diag(const SetupArgs& s, cudaStream_t stream);
// A^T b chains over `rows` rows of A, continuing from atb0 (nullptr: +0); also
// transpose_matvec, y_j = sum_i M[i,j] v_i (linalg.hpp:209-219).
cudaError_t launch_atb_chain(const double* A, uint64_t lda, int rows, int n, const double* b,
                             const double* atb0, double* atb, cudaStream_t stream);
cudaError_t launch_retained(const SetupArgs& s, cudaStream_t stream);
// mode 0: write H (and -A^T b into hvec when b != nullptr); mode 1: fused rescale into Q, q.
cudaError_t launch_syrk(const SetupArgs& s, int mode, cudaStream_t stream);
// FAST profile: the same three modes on the fp64 tensor cores (dmma.cu). Needs
// even leading dimensions and 16-byte aligned operands (syrk_dmma_supported).
// v2 (when s.dm_ws / dm_flags / dm_ctas are set): TMA-staged, stream-K persistent
// kernel; mode 0 flags: accumulate bit 0 adds into H instead of overwriting it,
// bit 1 writes the upper triangle only.
// [tile_lo, tile_hi) restricts the launch to a range of the tile order (upper
// triangle by columns: tile (ti, tj) is tj (tj + 1) / 2 + ti), v2 only; -1 = all.
cudaError_t launch_syrk_dmma(const SetupArgs& s, int mode, cudaStream_t stream, int accumulate = 0,
                             int tile_lo = -1, int tile_hi = -1);
size_t syrk_dmma_ws_doubles(int sm_count);
bool syrk_dmma_supported(const SetupArgs& s, int mode);
// q (mode 1) or hvec = -(A^T b) (mode 0) from the column chains' A^T b.
cudaError_t launch_q_from_atb(const SetupArgs& s, int mode, cudaStream_t stream);
// Rescale from a given H (n x n) and h (n) on device (nnls.hpp:41-83).
cudaError_t launch_rescale_from_h(const double* H, const double* h, int n, const int* pos,
                                  const double* scale, double* Q, int m, int qR, double* q,
                                  cudaStream_t stream);
// Exact masked GEMV on a blocked m x m matrix (block rows R).
cudaError_t launch_masked_gemv_blocked(const double* Qb, int m, int R, const uint32_t* list,
                                       const double* vals, int len, double* y,
                                       cudaStream_t stream);
// Column-major (ld) -> blocked layout, and back.
cudaError_t launch_to_blocked(const double* src, uint64_t ld, int m, int R, double* dst,
                              cudaStream_t stream);
cudaError_t launch_from_blocked(const double* src, int m, int R, double* dst, uint64_t ld,
                                cudaStream_t stream);

// K7: x = y / D scattered to the original columns (nnls.hpp:87-96).
cudaError_t launch_unscale(const double* y, const double* scale, const uint32_t* retained, int m,
                           double* x, int n, cudaStream_t stream);
// residual_norm_sq (nnls.hpp:115-123): r_i = (A x)_i - b_i, s = sum r_i^2 in order.
cudaError_t launch_residual(const double* ax, const double* b, int d, double* prod, double* out,
                            cudaStream_t stream, double s0 = 0.0);
// Compaction of the support of x (x_j != 0, ascending) for matvec(A, x).
cudaError_t launch_support(const double* x, int n, uint32_t* list, double* vals, int* len,
                           cudaStream_t stream);
// Multi-GPU exact Gram by row blocks (setup.cu syrk_rowblock_kernel): tile count,
// and continuation of tiles [tile_lo, tile_lo + ntiles) over the rows of s.A
// from chain states pin to pout ([ntiles][ALNNLS_GRAM_TILE_DOUBLES]; pout == nullptr writes s.H).
uint64_t gram_tiles(uint64_t n);
cudaError_t launch_syrk_rowblock(const SetupArgs& s, int tile_lo, int ntiles, const double* pin,
                                 double* pout, cudaStream_t stream);
cudaError_t launch_diag(const double* H, int n, double* diag, cudaStream_t stream);
cudaError_t launch_negate(const double* x, int n, double* y, cudaStream_t stream);
// g = y + q (warm start, nqp.hpp:232-233)
cudaError_t launch_add(const double* y, const double* q, double* g, int m, cudaStream_t stream);
// any non-finite entry among `count` doubles (strided columns) -> *flag = 1
cudaError_t launch_check_finite(const double* p, uint64_t rows, uint64_t cols, uint64_t ld,
                                int* flag, cudaStream_t stream);
// kind 0: any asymmetric pair of the square rows x rows matrix, kind 1: any entry
// that is not >= 0 (negative or NaN) -> *flag = 1
cudaError_t launch_check_matrix(const double* p, uint64_t rows, uint64_t cols, uint64_t ld,
                                int kind, int* flag, cudaStream_t stream);
// dir 0: packed upper triangle P (j(j+1)/2 + i) of the symmetric H; dir 1: H from P (mirrored)
cudaError_t launch_pack_upper(double* H, uint64_t n, double* P, int dir, cudaStream_t stream);
// C (rows x cols) = A (rows x inner) H (inner x cols), each column the reference's
// matvec order (bitwise matvec(A, H[:, j]))
cudaError_t launch_matmat(const double* A, uint64_t lda, int rows, int inner, const double* H,
                          uint64_t ldh, int cols, double* C, uint64_t ldc, cudaStream_t stream);
// dst (cols x rows) = src^T (rows x cols), column-major both
cudaError_t launch_transpose(const double* src, uint64_t ld_src, int rows, int cols, double* dst,
                             uint64_t ld_dst, cudaStream_t stream);
// pads: copy a rows x cols col-major block into a buffer with leading dimension ld_dst.
cudaError_t launch_copy_pad(const double* src, uint64_t ld_src, double* dst, uint64_t ld_dst,
                            uint64_t rows, uint64_t cols, cudaStream_t stream);

// Batched multi-RHS exact solve (K8).
struct BatchArgs {
  const double* Q;     // m x m, column-major (ld m)
  int m;
  const double* QB;    // m x ncols: per-column linear term q (ld m)
  int ncols;
  double* Y;           // m x ncols solution (rescaled space)
  alnnls_column_result* res;  // per column
  double eps;
  uint64_t max_iters;
  uint64_t stall_window;
  int* next_col;       // work counter (zeroed before the launch)
  int fast;            // FAST profile: the Q V passes on the fp64 tensor cores (DMMA)
  double* Qf;          // FAST, m <= 256: scratch of m_pad^2 doubles for Q in DMMA fragment order
  int qf_ready;        // Qf already holds Q (launch_qfrag): launch_batched does not rewrite it
  int total_cols;      // columns of the whole batch when this launch is one chunk of it (0: ncols)
};
cudaError_t launch_batched(const BatchArgs& a, int sm_count, cudaStream_t stream);
cudaError_t launch_qfrag(const BatchArgs& a, cudaStream_t stream);  // Q -> Qf (FAST, m <= 256)
int batched_cols_per_cta(int m);  // 0 when m is too large for the batched kernel
cudaError_t launch_unscale_batched(const double* Y, int m, const double* scale,
                                   const uint32_t* retained, double* X, int n, int ncols,
                                   cudaStream_t stream);
cudaError_t launch_residual_batched(const double* A, uint64_t lda, int d, int n, const double* X,
                                    const double* B, uint64_t ldb, int ncols,
                                    alnnls_column_result* res, cudaStream_t stream);

// FAST: the same residuals on the fp64 tensor cores (dmma.cu), n <= 256
bool residual_dmma_supported(const double* A, uint64_t lda, int d, int n, int ncols);
cudaError_t launch_residual_batched_dmma(const double* A, uint64_t lda, int d, int n,
                                         const double* X, const double* B, uint64_t ldb,
                                         int ncols, alnnls_column_result* res,
                                         cudaStream_t stream);

}  // namespace alnnls
