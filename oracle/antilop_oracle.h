/*
 * antilop_oracle.h — TEST INFRASTRUCTURE ONLY. Not part of the product.
 *
 * CPU restatement of the reference hot path (plain C11, scalar, single thread)
 * used as the parity checker by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg. Nothing in paper_1502_01645_b200/ may link or call it.
 *
 * The same signatures are exported by two implementations:
 *   oracle_*  — oracle/antilop_oracle.c, our restatement of the algorithm
 *   ref_*     — oracle/ref_shim.cpp, the reference headers themselves compiled
 *               into oracle/_ref/libantilop_ref.so (namespace renamed to
 *               antilop_ref, reference Release flags, no -march).
 * tests/test_oracle_pin.py pins the restatement to the reference bit for bit.
 */
#ifndef ANTILOP_ORACLE_H
#define ANTILOP_ORACLE_H

#include <stdint.h>

#include "../include/alnnls.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Caller-owned output buffers. Any pointer may be NULL (that output is skipped).
 * Capacities are in elements. */
typedef struct oracle_out {
  double* x;            /* NNLS: n (unscaled); NQP: m */
  uint64_t x_cap;
  double* inner_x;      /* NNLS only: rescaled-space y (m) */
  double* final_grad;   /* m */
  uint64_t vec_cap;     /* capacity of inner_x / final_grad / scale */
  alnnls_iter_record* trace;
  uint64_t trace_cap;
  uint64_t* mults;      /* multiplies_per_iter */
  uint64_t mults_cap;
  double* scale;        /* NNLS: D over retained columns */
  uint64_t* retained;   /* NNLS: cap x_cap */
  uint64_t* dropped;    /* NNLS: cap x_cap */
  alnnls_summary summary;
  char error[256];
} oracle_out;

/* linalg.hpp:160-174 */
int oracle_gram(uint64_t d, uint64_t n, const double* A, double* H);
/* linalg.hpp:209-219 */
int oracle_transpose_matvec(uint64_t rows, uint64_t cols, const double* M, const double* v,
                            double* y);
/* linalg.hpp:179-188 */
int oracle_matvec(uint64_t rows, uint64_t cols, const double* M, const double* v, double* y);
/* linalg.hpp:193-206 (returns ALNNLS_ERANGE on a bad index) */
int oracle_masked_matvec(uint64_t rows, uint64_t cols, const double* M, const double* v,
                         const uint64_t* mask, uint64_t mask_len, double* y,
                         uint64_t* multiply_count);
/* nnls.hpp:41-83. Q (m x m) and q (m) into caller buffers of capacity n*n / n. */
int oracle_rescale(uint64_t n, const double* H, const double* h, double* Q, double* q,
                   oracle_out* out);
/* nqp.hpp:215-339 */
int oracle_solve_nqp(uint64_t m, const double* Q, const double* q, const double* start,
                     const alnnls_config* cfg, oracle_out* out);
/* nnls.hpp:129-144 */
int oracle_solve_nnls(uint64_t d, uint64_t n, const double* A, const double* b,
                      const alnnls_config* cfg, oracle_out* out);
/* accelerated.hpp:21-117 and :121-139 (the Anti+Acc baseline) */
int oracle_solve_accelerated(uint64_t m, const double* Q, const double* q, const double* start,
                             const alnnls_config* cfg, oracle_out* out);
int oracle_solve_anti_accelerated(uint64_t d, uint64_t n, const double* A, const double* b,
                                  const alnnls_config* cfg, oracle_out* out);
/* linalg.hpp:222-226 */
double oracle_frobenius_norm(uint64_t rows, uint64_t cols, const double* M);
/* nqp.hpp:183-186 and :190-207 */
double oracle_objective(uint64_t m, const double* Q, const double* q, const double* x);
double oracle_kkt_error(uint64_t m, const double* Q, const double* q, const double* x);

/* Reference-compiled twins (oracle/_ref/libantilop_ref.so). */
int ref_gram(uint64_t d, uint64_t n, const double* A, double* H);
int ref_transpose_matvec(uint64_t rows, uint64_t cols, const double* M, const double* v,
                         double* y);
int ref_matvec(uint64_t rows, uint64_t cols, const double* M, const double* v, double* y);
int ref_masked_matvec(uint64_t rows, uint64_t cols, const double* M, const double* v,
                      const uint64_t* mask, uint64_t mask_len, double* y,
                      uint64_t* multiply_count);
int ref_rescale(uint64_t n, const double* H, const double* h, double* Q, double* q,
                oracle_out* out);
int ref_solve_nqp(uint64_t m, const double* Q, const double* q, const double* start,
                  const alnnls_config* cfg, oracle_out* out);
int ref_solve_accelerated(uint64_t m, const double* Q, const double* q, const double* start,
                          const alnnls_config* cfg, oracle_out* out);
int ref_solve_anti_accelerated(uint64_t d, uint64_t n, const double* A, const double* b,
                               const alnnls_config* cfg, oracle_out* out);
double ref_frobenius_norm(uint64_t rows, uint64_t cols, const double* M);
int ref_solve_nnls(uint64_t d, uint64_t n, const double* A, const double* b,
                   const alnnls_config* cfg, oracle_out* out);
double ref_objective(uint64_t m, const double* Q, const double* q, const double* x);
double ref_kkt_error(uint64_t m, const double* Q, const double* q, const double* x);
/* Gram once, then the per-column pipeline transpose_matvec -> rescale ->
 * solve_nqp -> unscale -> residual (bitwise equal to solve_nnls per column,
 * nnls.hpp:131-143). X is n x ncols. Runs columns on `threads` std::threads. */
int ref_solve_nnls_columns(uint64_t d, uint64_t n, const double* A, uint64_t ncols,
                           const double* B, const alnnls_config* cfg, double* X,
                           alnnls_column_result* cols, int threads);

#ifdef __cplusplus
}
#endif

#endif
