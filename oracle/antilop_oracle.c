/*
 * antilop_oracle.c — TEST INFRASTRUCTURE ONLY (the parity checker, never the
 * product). Plain C11 restatement of the reference hot path:
 *
 *   gram              /root/reference/proj/include/antilop/linalg.hpp:160-174
 *   matvec            linalg.hpp:179-188
 *   masked_matvec     linalg.hpp:193-206
 *   transpose_matvec  linalg.hpp:209-219
 *   rescale / unscale nnls.hpp:41-96
 *   passive_mask      nqp.hpp:149-157
 *   exact_step        nqp.hpp:162-173
 *   solve_nqp         nqp.hpp:215-339
 *   solve_nnls        nnls.hpp:129-144 (+ residual_norm_sq :115-123)
 *
 * Floating-point contract (must match the reference Release build, which is
 * x86-64 SSE2 without FMA): every `s += a*b` is a rounded product followed by
 * a rounded sum, sums are single chains in ascending index order, and nothing
 * is reassociated. Build with -ffp-contract=off and without -ffast-math or
 * -march (oracle/Makefile). tests/test_oracle_pin.py checks this file bit for
 * bit against the reference compiled from its own headers (oracle/_ref).
 */
#define _POSIX_C_SOURCE 199309L
#include "antilop_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static int fail(oracle_out* out, int code, const char* msg) {
  if (out) {
    strncpy(out->error, msg, sizeof(out->error) - 1);
    out->error[sizeof(out->error) - 1] = 0;
  }
  return code;
}

/* linalg.hpp:160-174: each upper entry is one ascending-k chain, mirrored. */
int oracle_gram(uint64_t d, uint64_t n, const double* A, double* H) {
  for (uint64_t j = 0; j < n; ++j) {
    const double* cj = A + j * d;
    for (uint64_t i = 0; i <= j; ++i) {
      const double* ci = A + i * d;
      double s = 0.0;
      for (uint64_t k = 0; k < d; ++k) s += ci[k] * cj[k];
      H[j * n + i] = s;
      H[i * n + j] = s;
    }
  }
  return ALNNLS_OK;
}

/* linalg.hpp:209-219 */
int oracle_transpose_matvec(uint64_t rows, uint64_t cols, const double* M, const double* v,
                            double* y) {
  for (uint64_t j = 0; j < cols; ++j) {
    const double* col = M + j * rows;
    double s = 0.0;
    for (uint64_t i = 0; i < rows; ++i) s += col[i] * v[i];
    y[j] = s;
  }
  return ALNNLS_OK;
}

/* linalg.hpp:179-188: column sweep, y starts at +0. */
int oracle_matvec(uint64_t rows, uint64_t cols, const double* M, const double* v, double* y) {
  for (uint64_t i = 0; i < rows; ++i) y[i] = 0.0;
  for (uint64_t j = 0; j < cols; ++j) {
    const double vj = v[j];
    const double* col = M + j * rows;
    for (uint64_t i = 0; i < rows; ++i) y[i] += col[i] * vj;
  }
  return ALNNLS_OK;
}

/* linalg.hpp:193-206: only masked columns, in the order given. */
int oracle_masked_matvec(uint64_t rows, uint64_t cols, const double* M, const double* v,
                         const uint64_t* mask, uint64_t mask_len, double* y,
                         uint64_t* multiply_count) {
  for (uint64_t i = 0; i < rows; ++i) y[i] = 0.0;
  for (uint64_t t = 0; t < mask_len; ++t) {
    const uint64_t j = mask[t];
    if (j >= cols) return ALNNLS_ERANGE;
    const double vj = v[j];
    const double* col = M + j * rows;
    for (uint64_t i = 0; i < rows; ++i) y[i] += col[i] * vj;
  }
  if (multiply_count) *multiply_count += rows * mask_len;
  return ALNNLS_OK;
}

static double dot(uint64_t n, const double* a, const double* b) { /* linalg.hpp:134-139 */
  double s = 0.0;
  for (uint64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

/* nqp.hpp:183-186 */
double oracle_objective(uint64_t m, const double* Q, const double* q, const double* x) {
  double* qx = (double*)malloc(sizeof(double) * (m ? m : 1));
  oracle_matvec(m, m, Q, x, qx);
  const double r = 0.5 * dot(m, x, qx) + dot(m, q, x);
  free(qx);
  return r;
}

/* nqp.hpp:190-207 */
double oracle_kkt_error(uint64_t m, const double* Q, const double* q, const double* x) {
  double* g = (double*)malloc(sizeof(double) * (m ? m : 1));
  oracle_matvec(m, m, Q, x, g);
  for (uint64_t i = 0; i < m; ++i) g[i] += q[i];
  double err = 0.0;
  for (uint64_t i = 0; i < m; ++i) {
    if (x[i] < 0.0) {
      free(g);
      return INFINITY;
    }
    const double ng = -g[i];
    const double v = x[i] > 0.0 ? fabs(g[i]) : ((0.0 < ng) ? ng : 0.0); /* std::max(0.0, -g) */
    if (err < v) err = v; /* std::max(err, v) keeps err on ties */
  }
  free(g);
  return err;
}

/* nnls.hpp:41-83. Writes Q (m x m), q (m) and the bookkeeping. */
int oracle_rescale(uint64_t n, const double* H, const double* h, double* Q, double* q,
                   oracle_out* out) {
  for (uint64_t j = 0; j < n; ++j)
    for (uint64_t i = 0; i < j; ++i)
      if (!(H[j * n + i] == H[i * n + j])) return fail(out, ALNNLS_EINVAL, "rescale: H must be symmetric");
  uint64_t* retained = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
  double* scale = (double*)malloc(sizeof(double) * (n ? n : 1));
  uint64_t m = 0, nd = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const double dg = H[i * n + i];
    if (!(dg >= 0.0)) {
      free(retained);
      free(scale);
      return fail(out, ALNNLS_EINVAL, "rescale: negative diagonal entry");
    }
    if (dg == 0.0) {
      if (out && out->dropped) out->dropped[nd] = i;
      ++nd;
    } else {
      retained[m] = i;
      scale[m] = sqrt(dg);
      ++m;
    }
  }
  for (uint64_t b = 0; b < m; ++b) {
    const uint64_t jb = retained[b];
    Q[b * m + b] = 1.0;
    for (uint64_t a = 0; a < b; ++a) {
      const uint64_t ja = retained[a];
      const double v = H[jb * n + ja] / (scale[a] * scale[b]);
      Q[b * m + a] = v;
      Q[a * m + b] = v;
    }
    q[b] = h[jb] / scale[b];
  }
  if (out) {
    if (out->retained) memcpy(out->retained, retained, sizeof(uint64_t) * m);
    if (out->scale) memcpy(out->scale, scale, sizeof(double) * m);
    out->summary.m = m;
    out->summary.n = n;
    out->summary.n_dropped = nd;
  }
  free(retained);
  free(scale);
  return ALNNLS_OK;
}

static void push_record(oracle_out* out, uint64_t* len, uint64_t iter, double f, double gbs,
                        uint64_t pc, double elapsed, double alpha, int has_alpha) {
  if (out && out->trace && *len < out->trace_cap) {
    alnnls_iter_record* r = &out->trace[*len];
    r->iter = iter;
    r->f = f;
    r->grad_bar_sq = gbs;
    r->passive_count = pc;
    r->elapsed_s = elapsed;
    r->alpha = has_alpha ? alpha : 0.0;
    r->has_alpha = has_alpha;
  }
  ++*len;
}

/* nqp.hpp:215-339 */
int oracle_solve_nqp(uint64_t n, const double* Q, const double* q, const double* start,
                     const alnnls_config* cfg, oracle_out* out) {
  /* resolve_epsilon / resolve_max_iters, nqp.hpp:84-98 */
  double eps;
  if (cfg->has_epsilon) {
    if (!(cfg->epsilon > 0.0)) return fail(out, ALNNLS_EINVAL, "SolverConfig: epsilon must be > 0");
    eps = cfg->epsilon;
  } else {
    eps = 1e-10 * (double)n;
  }
  uint64_t max_iters;
  if (cfg->has_max_iters) {
    if (cfg->max_iters < 1) return fail(out, ALNNLS_EINVAL, "SolverConfig: max_iters must be >= 1");
    max_iters = cfg->max_iters;
  } else {
    max_iters = 5 * n;
  }
  const uint64_t trace_every = cfg->trace_every > 0 ? cfg->trace_every : 1;
  const size_t nb = sizeof(double) * (n ? n : 1);

  double* x = (double*)calloc(1, nb);
  double* grad = (double*)malloc(nb);
  memcpy(grad, q, sizeof(double) * n);
  if (start) {
    for (uint64_t i = 0; i < n; ++i) {
      if (!(start[i] >= 0.0)) {
        free(x);
        free(grad);
        return fail(out, ALNNLS_EINVAL, "solve_nqp: start must be nonnegative");
      }
    }
    memcpy(x, start, sizeof(double) * n);
    oracle_matvec(n, n, Q, x, grad);
    for (uint64_t i = 0; i < n; ++i) grad[i] += q[i];
  }
  double min_iterate = INFINITY;
  if (n) {
    min_iterate = x[0];
    for (uint64_t i = 1; i < n; ++i)
      if (x[i] < min_iterate) min_iterate = x[i];
  } else {
    min_iterate = 0.0;
  }

  double* grad_bar = (double*)calloc(1, nb);
  double* delta = (double*)calloc(1, nb);
  double* cand = (double*)calloc(1, nb);
  double* qg = (double*)malloc(nb);
  double* gd = (double*)malloc(nb);
  uint64_t* mask = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
  uint64_t* changed = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));

  double best_gbs = INFINITY;
  uint64_t since_best = 0;
  uint64_t trace_len = 0, mult_len = 0, mult_total = 0;
  int status = ALNNLS_OK;
  int termination = ALNNLS_MAX_ITERS;
  double last_f = 0.0, last_gbs = 0.0;
  const double t0 = now_s();

  for (uint64_t k = 0;; ++k) {
    uint64_t ml = 0; /* passive_mask, nqp.hpp:149-157 */
    for (uint64_t i = 0; i < n; ++i)
      if (x[i] > 0.0 || grad[i] < 0.0) mask[ml++] = i;
    double gbs = 0.0;
    for (uint64_t t = 0; t < ml; ++t) gbs += grad[mask[t]] * grad[mask[t]];
    const double f = 0.5 * (dot(n, x, grad) + dot(n, q, x));
    const double elapsed = now_s() - t0;

    if (!isfinite(f) || !isfinite(gbs)) {
      status = fail(out, ALNNLS_ENUMERIC, "solve_nqp: non-finite objective or gradient");
      if (out) out->summary.numeric_failure = 1;
      break;
    }

    int stop = -1; /* nqp.hpp:261-275, else-if chain */
    if (ml == 0) {
      stop = ALNNLS_EMPTY_PASSIVE_SET;
    } else if (gbs < eps) {
      stop = ALNNLS_GRADIENT_BELOW_EPSILON;
    } else if (k >= max_iters) {
      stop = ALNNLS_MAX_ITERS;
    } else if (cfg->has_time_cap && elapsed >= cfg->time_cap_s) {
      stop = ALNNLS_TIME_CAP;
    } else if (gbs < best_gbs) {
      best_gbs = gbs;
      since_best = 0;
    } else if (++since_best >= cfg->stall_window) {
      stop = ALNNLS_STALLED;
    }

    if (stop < 0) {
      for (uint64_t t = 0; t < ml; ++t) grad_bar[mask[t]] = grad[mask[t]];
      uint64_t mults = 0;
      /* exact_step, nqp.hpp:162-173 */
      int have_step = 0;
      double step = 0.0;
      {
        double num = 0.0;
        for (uint64_t t = 0; t < ml; ++t) num += grad_bar[mask[t]] * grad_bar[mask[t]];
        if (num != 0.0) {
          oracle_masked_matvec(n, n, Q, grad_bar, mask, ml, qg, &mults);
          double den = 0.0;
          for (uint64_t t = 0; t < ml; ++t) den += grad_bar[mask[t]] * qg[mask[t]];
          if (den > 0.0) {
            have_step = 1;
            step = num / den;
          }
        }
      }
      for (uint64_t t = 0; t < ml; ++t) grad_bar[mask[t]] = 0.0;
      if (!have_step) stop = ALNNLS_ZERO_CURVATURE;

      if (stop < 0) {
        double alpha = step; /* halving safeguard, nqp.hpp:284-318 */
        for (int tries = 0;; ++tries) {
          uint64_t cl = 0;
          for (uint64_t t = 0; t < ml; ++t) {
            const uint64_t i = mask[t];
            double xi = x[i] - alpha * grad[i];
            if (xi < 0.0) xi = 0.0;
            if (xi != x[i]) {
              cand[i] = xi;
              delta[i] = xi - x[i];
              changed[cl++] = i;
            }
          }
          if (cl == 0) break;
          oracle_masked_matvec(n, n, Q, delta, changed, cl, gd, &mults);
          double df = 0.0;
          for (uint64_t t = 0; t < cl; ++t) {
            const uint64_t i = changed[t];
            df += (grad[i] + 0.5 * gd[i]) * delta[i];
          }
          if (df <= 0.0 || tries >= 60) {
            for (uint64_t t = 0; t < cl; ++t) {
              x[changed[t]] = cand[changed[t]];
              delta[changed[t]] = 0.0;
            }
            for (uint64_t i = 0; i < n; ++i) grad[i] += gd[i];
            break;
          }
          for (uint64_t t = 0; t < cl; ++t) delta[changed[t]] = 0.0;
          alpha *= 0.5;
        }
        if (k % trace_every == 0) push_record(out, &trace_len, k, f, gbs, ml, elapsed, alpha, 1);
        if (out && out->mults && mult_len < out->mults_cap) out->mults[mult_len] = mults;
        ++mult_len;
        mult_total += mults;
        if (n) {
          double mn = x[0];
          for (uint64_t i = 1; i < n; ++i)
            if (x[i] < mn) mn = x[i];
          if (mn < min_iterate) min_iterate = mn;
        }
        continue;
      }
    }
    push_record(out, &trace_len, k, f, gbs, ml, elapsed, 0.0, 0);
    termination = stop;
    last_f = f;
    last_gbs = gbs;
    if (out) out->summary.iterations = k;
    break;
  }

  if (out) {
    out->summary.termination = termination;
    out->summary.trace_len = trace_len;
    out->summary.mult_len = mult_len;
    out->summary.multiplies_total = mult_total;
    out->summary.min_iterate = min_iterate;
    out->summary.f_final = last_f;
    out->summary.gbs_final = last_gbs;
    out->summary.m = n;
    out->summary.t_loop_s = now_s() - t0;
    if (status == ALNNLS_OK) {
      if (out->x) memcpy(out->x, x, sizeof(double) * n);
      if (out->final_grad) memcpy(out->final_grad, grad, sizeof(double) * n);
    }
  }
  free(x);
  free(grad);
  free(grad_bar);
  free(delta);
  free(cand);
  free(qg);
  free(gd);
  free(mask);
  free(changed);
  return status;
}

/* nnls.hpp:115-123 */
static double residual_norm_sq(uint64_t d, uint64_t n, const double* A, const double* b,
                               const double* x) {
  double* ax = (double*)malloc(sizeof(double) * (d ? d : 1));
  oracle_matvec(d, n, A, x, ax);
  double s = 0.0;
  for (uint64_t i = 0; i < d; ++i) {
    const double r = ax[i] - b[i];
    s += r * r;
  }
  free(ax);
  return s;
}

typedef int (*inner_solver)(uint64_t m, const double* Q, const double* q, const double* start,
                            const alnnls_config* cfg, oracle_out* out);

/* linalg.hpp:222-226: one ascending chain over the column-major data */
double oracle_frobenius_norm(uint64_t rows, uint64_t cols, const double* M) {
  double s = 0.0;
  for (uint64_t e = 0; e < rows * cols; ++e) s += M[e] * M[e];
  return sqrt(s);
}

/* accelerated.hpp:21-113 (solve_accelerated): Nesterov momentum projected
 * gradient with the fixed step 1/||Q||_F; start must be NULL (the reference
 * has no warm start here). */
int oracle_solve_accelerated(uint64_t n, const double* Q, const double* q, const double* start,
                             const alnnls_config* cfg, oracle_out* out) {
  (void)start;
  double eps;
  if (cfg->has_epsilon) {
    if (!(cfg->epsilon > 0.0)) return fail(out, ALNNLS_EINVAL, "SolverConfig: epsilon must be > 0");
    eps = cfg->epsilon;
  } else {
    eps = 1e-10 * (double)n;
  }
  uint64_t max_iters;
  if (cfg->has_max_iters) {
    if (cfg->max_iters < 1) return fail(out, ALNNLS_EINVAL, "SolverConfig: max_iters must be >= 1");
    max_iters = cfg->max_iters;
  } else {
    max_iters = 5 * n;
  }
  const uint64_t trace_every = cfg->trace_every > 0 ? cfg->trace_every : 1;
  const double m_norm = oracle_frobenius_norm(n, n, Q);
  const size_t nb = sizeof(double) * (n ? n : 1);
  double* x = (double*)calloc(1, nb);
  double* y = (double*)calloc(1, nb);
  double* xn = (double*)calloc(1, nb);
  double* grad = (double*)malloc(nb);
  double* gy = (double*)malloc(nb);
  double t = 1.0, f_prev = INFINITY, min_iterate = 0.0;
  double best_gbs = INFINITY;
  uint64_t since_best = 0, trace_len = 0;
  int status = ALNNLS_OK, termination = ALNNLS_MAX_ITERS;
  double last_f = 0.0, last_gbs = 0.0;
  const double t0 = now_s();
  for (uint64_t k = 0;; ++k) {
    oracle_matvec(n, n, Q, x, grad); /* :45-46 */
    for (uint64_t i = 0; i < n; ++i) grad[i] += q[i];
    uint64_t ml = 0;
    double gbs = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
      if (x[i] > 0.0 || grad[i] < 0.0) {
        ++ml;
        gbs += grad[i] * grad[i];
      }
    }
    const double f = 0.5 * (dot(n, x, grad) + dot(n, q, x));
    const double elapsed = now_s() - t0;
    if (!isfinite(f) || !isfinite(gbs)) {
      status = fail(out, ALNNLS_ENUMERIC, "solve_accelerated: non-finite objective or gradient");
      if (out) out->summary.numeric_failure = 1;
      break;
    }
    int stop = -1; /* :60-75 */
    if (ml == 0) {
      stop = ALNNLS_EMPTY_PASSIVE_SET;
    } else if (gbs < eps) {
      stop = ALNNLS_GRADIENT_BELOW_EPSILON;
    } else if (k >= max_iters) {
      stop = ALNNLS_MAX_ITERS;
    } else if (cfg->has_time_cap && elapsed >= cfg->time_cap_s) {
      stop = ALNNLS_TIME_CAP;
    } else if (m_norm == 0.0) {
      stop = ALNNLS_ZERO_CURVATURE;
    } else if (gbs < best_gbs) {
      best_gbs = gbs;
      since_best = 0;
    } else if (++since_best >= cfg->stall_window) {
      stop = ALNNLS_STALLED;
    }
    if (stop >= 0) {
      push_record(out, &trace_len, k, f, gbs, ml, elapsed, 0.0, 0);
      termination = stop;
      last_f = f;
      last_gbs = gbs;
      if (out) out->summary.iterations = k;
      break;
    }
    const double alpha = 1.0 / m_norm; /* :83-86 */
    if (k % trace_every == 0) push_record(out, &trace_len, k, f, gbs, ml, elapsed, alpha, 1);
    oracle_matvec(n, n, Q, y, gy); /* :89-94 */
    for (uint64_t i = 0; i < n; ++i) gy[i] += q[i];
    for (uint64_t i = 0; i < n; ++i) {
      const double v = y[i] - alpha * gy[i];
      xn[i] = 0.0 < v ? v : 0.0; /* std::max(0.0, v) */
    }
    const double t_next = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t)); /* :96-100 */
    const double momentum = (t - 1.0) / t_next;
    for (uint64_t i = 0; i < n; ++i) y[i] = xn[i] + momentum * (xn[i] - x[i]);
    if (cfg->nesterov_restart && f > f_prev) { /* :102-107 */
      t = 1.0;
      memcpy(y, xn, sizeof(double) * n);
    } else {
      t = t_next;
    }
    f_prev = f;
    memcpy(x, xn, sizeof(double) * n);
    double mn = 0.0; /* :110-112 */
    for (uint64_t i = 0; i < n; ++i) mn = x[i] < mn ? x[i] : mn;
    min_iterate = mn < min_iterate ? mn : min_iterate;
  }
  if (out) {
    out->summary.termination = termination;
    out->summary.trace_len = trace_len;
    out->summary.min_iterate = min_iterate;
    out->summary.f_final = last_f;
    out->summary.gbs_final = last_gbs;
    out->summary.m = n;
    out->summary.t_loop_s = now_s() - t0;
    if (status == ALNNLS_OK) {
      if (out->x) memcpy(out->x, x, sizeof(double) * n);
      if (out->final_grad) memcpy(out->final_grad, grad, sizeof(double) * n); /* :115-117 */
    }
  }
  free(x);
  free(y);
  free(xn);
  free(grad);
  free(gy);
  return status;
}

static int nnls_pipeline(uint64_t d, uint64_t n, const double* A, const double* b,
                         const alnnls_config* cfg, oracle_out* out, inner_solver solve);

/* nnls.hpp:129-144 */
int oracle_solve_nnls(uint64_t d, uint64_t n, const double* A, const double* b,
                      const alnnls_config* cfg, oracle_out* out) {
  return nnls_pipeline(d, n, A, b, cfg, out, oracle_solve_nqp);
}

/* accelerated.hpp:121-139 (solve_anti_accelerated): the same rescale / unscale /
 * residual pipeline around solve_accelerated. */
int oracle_solve_anti_accelerated(uint64_t d, uint64_t n, const double* A, const double* b,
                                  const alnnls_config* cfg, oracle_out* out) {
  return nnls_pipeline(d, n, A, b, cfg, out, oracle_solve_accelerated);
}

static int nnls_pipeline(uint64_t d, uint64_t n, const double* A, const double* b,
                         const alnnls_config* cfg, oracle_out* out, inner_solver solve) {
  const double t0 = now_s();
  double* H = (double*)malloc(sizeof(double) * (n > 0 ? n * n : 1));
  double* h = (double*)malloc(sizeof(double) * (n ? n : 1));
  oracle_gram(d, n, A, H);
  oracle_transpose_matvec(d, n, A, b, h);
  for (uint64_t i = 0; i < n; ++i) h[i] = -h[i];

  double* Q = (double*)malloc(sizeof(double) * (n > 0 ? n * n : 1));
  double* q = (double*)malloc(sizeof(double) * (n ? n : 1));
  uint64_t* retained = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
  double* scale = (double*)malloc(sizeof(double) * (n ? n : 1));
  uint64_t* dropped_user = out ? out->dropped : NULL;
  oracle_out tmp;
  memset(&tmp, 0, sizeof(tmp));
  tmp.retained = retained;
  tmp.scale = scale;
  tmp.dropped = dropped_user;
  int st = oracle_rescale(n, H, h, Q, q, &tmp);
  free(H);
  free(h);
  const uint64_t m = tmp.summary.m;
  const double t_setup = now_s() - t0;
  if (st != ALNNLS_OK) {
    if (out) memcpy(out->error, tmp.error, sizeof(out->error));
    free(Q); free(q); free(retained); free(scale);
    return st;
  }

  double* y = (double*)calloc(1, sizeof(double) * (m ? m : 1));
  if (m > 0) {
    oracle_out inner = out ? *out : tmp;
    inner.x = y;
    inner.x_cap = m;
    inner.final_grad = out ? out->final_grad : NULL;
    memset(&inner.summary, 0, sizeof(inner.summary));
    st = solve(m, Q, q, NULL, cfg, &inner);
    if (out) {
      out->summary = inner.summary;
      memcpy(out->error, inner.error, sizeof(out->error));
    }
    if (st != ALNNLS_OK) {
      free(Q); free(q); free(retained); free(scale); free(y);
      return st;
    }
  } else if (out) {
    /* detail::empty_solve_result, nnls.hpp:107-113 */
    memset(&out->summary, 0, sizeof(out->summary));
    out->summary.termination = ALNNLS_EMPTY_PASSIVE_SET;
    out->summary.trace_len = 1;
    out->summary.min_iterate = 0.0;
    if (out->trace && out->trace_cap) memset(out->trace, 0, sizeof(alnnls_iter_record));
  }

  /* unscale, nnls.hpp:87-96 */
  double* x = (double*)calloc(1, sizeof(double) * (n ? n : 1));
  for (uint64_t a = 0; a < m; ++a) x[retained[a]] = y[a] / scale[a];
  const double res = residual_norm_sq(d, n, A, b, x);
  if (out) {
    out->summary.n = n;
    out->summary.m = m;
    out->summary.n_dropped = n - m;
    out->summary.residual_sq = res;
    out->summary.t_setup_s = t_setup;
    out->summary.t_total_s = now_s() - t0;
    if (out->x) memcpy(out->x, x, sizeof(double) * n);
    if (out->inner_x) memcpy(out->inner_x, y, sizeof(double) * m);
    if (out->scale) memcpy(out->scale, scale, sizeof(double) * m);
    if (out->retained) memcpy(out->retained, retained, sizeof(uint64_t) * m);
  }
  free(Q); free(q); free(retained); free(scale); free(y); free(x);
  return ALNNLS_OK;
}
