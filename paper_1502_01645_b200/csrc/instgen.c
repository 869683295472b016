/*
 * instgen.c — seeded synthetic inputs for the five BASELINE.json configs.
 *
 * Harness code (input generation), not the solver. It reuses the reference's
 * generation SCHEME — a SplitMix64 master seed with one counter-based
 * substream per column (/root/reference/proj/include/antilop/testgen.hpp:42-76),
 * exact-count sparsity by partial Fisher-Yates (testgen.hpp:159-170) — with the
 * value laws of BASELINE.json's configs:
 *   U[0,1)  = 53-bit uniform01
 *   N(0,1)  = sqrt(-2 ln(1-u1)) cos(2 pi u2)     (two draws per normal)
 *   Exp(1)  = -ln(1-u)
 * Column j of A draws from substream(seed, j); x_true from substream(seed, n);
 * the noise of b from substream(seed, n+1); column selections from
 * substream(seed, n+2). Columns are independent, so generation is threaded
 * and insensitive to evaluation order.
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { uint64_t s; } sm64;

static inline uint64_t sm64_next(sm64* r) {
  uint64_t z = (r->s += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static inline sm64 sm64_sub(uint64_t seed, uint64_t stream) {
  uint64_t z = seed + 0x9E3779B97F4A7C15ULL * (stream + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  sm64 r = {z ^ (z >> 31)};
  return r;
}

static inline double u01(sm64* r) { return (double)(sm64_next(r) >> 11) * 0x1.0p-53; }

static inline double normal(sm64* r) {
  const double u1 = u01(r), u2 = u01(r);
  return sqrt(-2.0 * log(1.0 - u1)) * cos(6.283185307179586 * u2);
}

static inline double expo(sm64* r) { return -log(1.0 - u01(r)); }

/* Marks `count` distinct positions of [0, len) in `sel` (partial Fisher-Yates). */
static void choose(sm64* r, uint64_t len, uint64_t count, unsigned char* sel) {
  uint64_t* idx = (uint64_t*)malloc(sizeof(uint64_t) * (len ? len : 1));
  for (uint64_t i = 0; i < len; ++i) idx[i] = i;
  memset(sel, 0, len);
  for (uint64_t t = 0; t < count && t < len; ++t) {
    const uint64_t j = t + sm64_next(r) % (len - t);
    const uint64_t tmp = idx[t];
    idx[t] = idx[j];
    idx[j] = tmp;
    sel[idx[t]] = 1;
  }
  free(idx);
}

enum { LAW_U01 = 0, LAW_NORMAL = 1, LAW_ABSNORMAL = 2 };

typedef struct {
  double* A;
  uint64_t d, n, seed, j0, j1;
  int law;
  const unsigned char* scale_sel; /* columns multiplied by col_scale */
  double col_scale;
} col_job;

static void* fill_cols(void* arg) {
  col_job* jb = (col_job*)arg;
  for (uint64_t j = jb->j0; j < jb->j1; ++j) {
    sm64 r = sm64_sub(jb->seed, j);
    double* c = jb->A + j * jb->d;
    const double s = (jb->scale_sel && jb->scale_sel[j]) ? jb->col_scale : 1.0;
    for (uint64_t i = 0; i < jb->d; ++i) {
      double v;
      if (jb->law == LAW_U01) v = u01(&r);
      else if (jb->law == LAW_NORMAL) v = normal(&r);
      else v = fabs(normal(&r));
      c[i] = v * s;
    }
  }
  return NULL;
}

static void fill_matrix(double* A, uint64_t d, uint64_t n, uint64_t seed, int law,
                        const unsigned char* scale_sel, double col_scale, int threads) {
  if (threads < 1) threads = 1;
  if ((uint64_t)threads > n) threads = (int)(n ? n : 1);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  col_job* jobs = (col_job*)malloc(sizeof(col_job) * threads);
  for (int t = 0; t < threads; ++t) {
    col_job jb = {A, d, n, seed, n * t / threads, n * (t + 1) / threads, law, scale_sel, col_scale};
    jobs[t] = jb;
    pthread_create(&th[t], NULL, fill_cols, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
}

/* b = A x (column sweep, ascending — same order as the reference matvec). */
static void matvec(const double* A, uint64_t d, uint64_t n, const double* x, double* b) {
  for (uint64_t i = 0; i < d; ++i) b[i] = 0.0;
  for (uint64_t j = 0; j < n; ++j) {
    const double xj = x[j];
    if (xj == 0.0) continue;
    const double* c = A + j * d;
    for (uint64_t i = 0; i < d; ++i) b[i] += c[i] * xj;
  }
}

/* A "fraction nonzero" vector: values by law, exactly round(frac_nonzero*n) kept. */
static void sparse_vector(sm64* r, uint64_t n, double frac_nonzero, int law_exp, double* x) {
  for (uint64_t i = 0; i < n; ++i) x[i] = law_exp ? expo(r) : u01(r);
  const uint64_t nz = (uint64_t)llround(frac_nonzero * (double)n);
  unsigned char* sel = (unsigned char*)malloc(n ? n : 1);
  choose(r, n, n - nz, sel); /* positions set to zero */
  for (uint64_t i = 0; i < n; ++i)
    if (sel[i]) x[i] = 0.0;
  free(sel);
}

/* Fills a d x n matrix whose columns draw from substreams of `seed`.
 * law: 0 U[0,1), 1 N(0,1), 2 |N(0,1)|. */
int alnnls_gen_matrix(double* A, uint64_t d, uint64_t n, uint64_t seed, int law, int threads) {
  fill_matrix(A, d, n, seed, law, NULL, 1.0, threads);
  return 0;
}

/* ---- c3: A = U diag(s) V^T with U, V Haar-random orthogonal -----------------------
 * Deterministic on any host and thread count (no BLAS/LAPACK): Stewart's
 * construction Q = H_0 H_1 ... H_{n-2} S, each H_k a Householder reflection built
 * from an independent seeded Gaussian vector of length n - k (column k of a
 * seeded N(0,1) matrix, rows k..n-1), S the sign fix that makes the implied
 * triangular factor positive. Every sum runs in a fixed order and every row is
 * owned by one thread. */
typedef struct {
  double* Qr;          /* n x n row-major */
  const double* u;     /* reflector, length L (rows k..n-1 of the row space) */
  uint64_t n, k, r0, r1;
  double beta;
} refl_job;

static void* refl_rows(void* arg) {
  refl_job* jb = (refl_job*)arg;
  const uint64_t L = jb->n - jb->k;
  for (uint64_t i = jb->r0; i < jb->r1; ++i) {
    double* row = jb->Qr + i * jb->n + jb->k;
    double w = 0.0;
    for (uint64_t j = 0; j < L; ++j) w += row[j] * jb->u[j];
    const double c = jb->beta * w;
    for (uint64_t j = 0; j < L; ++j) row[j] -= c * jb->u[j];
  }
  return NULL;
}

static void haar(double* Q /* n x n column-major out */, uint64_t n, uint64_t seed, int threads) {
  double* G = (double*)malloc(sizeof(double) * n * n);
  double* Qr = (double*)calloc(n * n, sizeof(double));
  double* u = (double*)malloc(sizeof(double) * (n ? n : 1));
  double* sgn = (double*)malloc(sizeof(double) * (n ? n : 1));
  fill_matrix(G, n, n, seed, LAW_NORMAL, NULL, 1.0, threads);
  for (uint64_t i = 0; i < n; ++i) Qr[i * n + i] = 1.0;
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  refl_job* jobs = (refl_job*)malloc(sizeof(refl_job) * threads);
  for (uint64_t k = 0; k + 1 < n; ++k) {
    const uint64_t L = n - k;
    const double* v = G + k * n + k;
    double nrm2 = 0.0;
    for (uint64_t j = 0; j < L; ++j) nrm2 += v[j] * v[j];
    const double nrm = sqrt(nrm2);
    const double s0 = v[0] >= 0.0 ? 1.0 : -1.0;
    for (uint64_t j = 0; j < L; ++j) u[j] = v[j];
    u[0] += s0 * nrm; /* H v = -s0 ||v|| e_0 */
    double uu = 0.0;
    for (uint64_t j = 0; j < L; ++j) uu += u[j] * u[j];
    sgn[k] = -s0;
    if (uu == 0.0) continue;
    const double beta = 2.0 / uu;
    for (int t = 0; t < threads; ++t) {
      refl_job jb = {Qr, u, n, k, n * t / threads, n * (t + 1) / threads, beta};
      jobs[t] = jb;
      pthread_create(&th[t], NULL, refl_rows, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  }
  if (n) sgn[n - 1] = G[(n - 1) * n + (n - 1)] >= 0.0 ? 1.0 : -1.0;
  for (uint64_t i = 0; i < n; ++i) /* column-major out, columns scaled by the sign fix */
    for (uint64_t j = 0; j < n; ++j) Q[j * n + i] = Qr[i * n + j] * sgn[j];
  free(G);
  free(Qr);
  free(u);
  free(sgn);
  free(th);
  free(jobs);
}

typedef struct {
  double* A;
  const double* U;
  const double* W; /* W[j*k + t] = s_t * V[j, t] */
  uint64_t d, k, j0, j1;
} prod_job;

static void* prod_cols(void* arg) {
  prod_job* jb = (prod_job*)arg;
  for (uint64_t j = jb->j0; j < jb->j1; ++j) {
    double* a = jb->A + j * jb->d;
    for (uint64_t i = 0; i < jb->d; ++i) a[i] = 0.0;
    for (uint64_t t = 0; t < jb->k; ++t) {
      const double c = jb->W[j * jb->k + t];
      const double* ut = jb->U + t * jb->d;
      for (uint64_t i = 0; i < jb->d; ++i) a[i] += ut[i] * c;
    }
  }
  return NULL;
}

/* A (d x n, column-major) = U[:, :k] diag(s) V[:, :k]^T, s_t = 10^(-6 t / (k-1)). */
int alnnls_gen_c3_matrix(double* A, uint64_t d, uint64_t n, uint64_t seed, int threads) {
  const uint64_t k = d < n ? d : n;
  double* U = (double*)malloc(sizeof(double) * d * d);
  double* V = (double*)malloc(sizeof(double) * n * n);
  double* W = (double*)malloc(sizeof(double) * n * (k ? k : 1));
  haar(U, d, seed * 1000 + 11, threads);
  haar(V, n, seed * 1000 + 13, threads);
  for (uint64_t j = 0; j < n; ++j)
    for (uint64_t t = 0; t < k; ++t) {
      const double st = pow(10.0, -6.0 * (double)t / (double)(k > 1 ? k - 1 : 1));
      W[j * k + t] = st * V[t * n + j];
    }
  if (threads < 1) threads = 1;
  if ((uint64_t)threads > n) threads = (int)(n ? n : 1);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  prod_job* jobs = (prod_job*)malloc(sizeof(prod_job) * threads);
  for (int t = 0; t < threads; ++t) {
    prod_job jb = {A, U, W, d, k, n * t / threads, n * (t + 1) / threads};
    jobs[t] = jb;
    pthread_create(&th[t], NULL, prod_cols, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(U);
  free(V);
  free(W);
  free(th);
  free(jobs);
  return 0;
}

/*
 * BASELINE.json configs (kind 1..5). A is d x n column-major, b has d entries,
 * x_true n. kind 3 (Haar product) is assembled by the Python harness from
 * alnnls_gen_matrix draws; here it only draws x_true and b = A x_true given A.
 *   1: A U[0,1); x 50% zero, U[0,1); b = A x + 0.01 N
 *   2: A N(0,1); x 30% nonzero Exp(1); b = A x + 1e-3 N
 *   3: (A given); x 50% nonzero U[0,1); b = A x
 *   5: A |N(0,1)|, 10% of columns x 1e3; x 20% nonzero U[0,1); b = A x + 1e-3 N
 */
int alnnls_gen_config(int kind, uint64_t d, uint64_t n, uint64_t seed, double* A, double* b,
                      double* x_true, int threads) {
  unsigned char* scale_sel = NULL;
  double noise = 0.0;
  switch (kind) {
    case 1: fill_matrix(A, d, n, seed, LAW_U01, NULL, 1.0, threads); noise = 0.01; break;
    case 2: fill_matrix(A, d, n, seed, LAW_NORMAL, NULL, 1.0, threads); noise = 1e-3; break;
    case 3: break;
    case 5: {
      sm64 rs = sm64_sub(seed, n + 2);
      scale_sel = (unsigned char*)malloc(n ? n : 1);
      choose(&rs, n, (uint64_t)llround(0.1 * (double)n), scale_sel);
      fill_matrix(A, d, n, seed, LAW_ABSNORMAL, scale_sel, 1e3, threads);
      noise = 1e-3;
      break;
    }
    default: return 1;
  }
  sm64 rx = sm64_sub(seed, n);
  switch (kind) {
    case 1: sparse_vector(&rx, n, 0.5, 0, x_true); break;
    case 2: sparse_vector(&rx, n, 0.3, 1, x_true); break;
    case 3: sparse_vector(&rx, n, 0.5, 0, x_true); break;
    case 5: sparse_vector(&rx, n, 0.2, 0, x_true); break;
  }
  matvec(A, d, n, x_true, b);
  if (noise != 0.0) {
    sm64 rn = sm64_sub(seed, n + 1);
    for (uint64_t i = 0; i < d; ++i) b[i] += noise * normal(&rn);
  }
  free(scale_sel);
  return 0;
}

/* c4: H_true (k x ncols) U[0,1) with exactly round(0.4 k) zeros per column;
 * column j draws from substream(seed, 1000003 + j) so it never overlaps A's. */
int alnnls_gen_htrue(double* H, uint64_t k, uint64_t ncols, uint64_t seed, uint64_t col0) {
  unsigned char* sel = (unsigned char*)malloc(k ? k : 1);
  const uint64_t nz0 = (uint64_t)llround(0.4 * (double)k);
  for (uint64_t j = 0; j < ncols; ++j) {
    sm64 r = sm64_sub(seed, 1000003ULL + col0 + j);
    double* c = H + j * k;
    for (uint64_t i = 0; i < k; ++i) c[i] = u01(&r);
    choose(&r, k, nz0, sel);
    for (uint64_t i = 0; i < k; ++i)
      if (sel[i]) c[i] = 0.0;
  }
  free(sel);
  return 0;
}
