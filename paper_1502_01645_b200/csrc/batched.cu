// batched.cu — K8: many independent right-hand sides sharing one Gram (the NMF
// H-update, BASELINE.json config c4). Column j's result is bitwise
// solve_nnls(A, B[:, j], cfg) (reference nnls.hpp:129-144), because the
// reference recomputes the same Gram for every call and everything after the
// Gram is per column.
//
//  - q for every column: exact A^T B tile GEMM (setup.cu mode 2)
//  - batched_nqp_kernel: persistent CTAs, each advancing NB columns. Every
//    GEMV of the reference loop (Q g_bar, Q delta) becomes one pass of an exact
//    chain GEMM U = Q V over dense masked vectors: v_b[j] = 0 off the mask, and
//    adding a +-0 product to a chain that starts at +0 is exact, so each
//    U[i, b] is bitwise masked_matvec (linalg.hpp:193-206). Q (m x m, L2
//    resident) is read once per pass for all NB columns. Columns have their own
//    state machine (mask/stop tests, den, candidate, df, halving) and finished
//    columns are replaced from a global queue.
//  - unscale + residual: x = y / D; ||A x - b||^2 with one ordered chain per
//    column over the rows (nnls.hpp:87-96, :115-123).
#include <cstdio>

#include "common.cuh"
#include "kernels.cuh"

namespace alnnls {

namespace {

#ifndef ALNNLS_GEMM_JB
#define ALNNLS_GEMM_JB 8  // Q columns per register block of the batched GEMM (prefetch distance)
#endif
constexpr int kBT = 512;          // threads per batched CTA (one warp per column at NB = 16)
constexpr int kMaxCols = 16;      // NB upper bound (columns per CTA)

enum ColPhase { kIdle = 0, kNeedP1 = 1, kNeedP2 = 2 };

struct ColState {
  int phase[kMaxCols];
  int col[kMaxCols];
  unsigned long long k[kMaxCols];
  int tries[kMaxCols];
  int ml[kMaxCols];
  double alpha[kMaxCols];
  double f[kMaxCols], gbs[kMaxCols];
  double best[kMaxCols];
  unsigned long long since[kMaxCols];
  unsigned long long mults[kMaxCols];
};

// Shared-memory layout of one CTA (mp = m rounded up to 8):
//  - V, the GEMM input, row-major mp x ld (ld = NB + 2): the GEMM reads a row of
//    V with 16-byte broadcasts; the padding keeps the per-column writes (lane =
//    row) at 4-way bank sharing; rows >= m stay zero so the GEMM needs no tail.
//  - U (GEMM output), C (candidate), X (iterate), G (gradient), q (linear term):
//    column panels of mp doubles, so the GEMM's stores and every per-column walk
//    are conflict-free, and a lane can load 8 consecutive entries as 4 x 16 B.
struct BatchSmem {
  double* V;
  int ld;
  int m, mp;
  double* U;
  double* C;
  double* X;
  double* G;
  double* q;
  __device__ double& v(int i, int b) const { return V[i * ld + b]; }
  __device__ double* u(int b) const { return U + b * mp; }
  __device__ double* c(int b) const { return C + b * mp; }
  __device__ double* x(int b) const { return X + b * mp; }
  __device__ double* g(int b) const { return G + b * mp; }
  __device__ double* qc(int b) const { return q + b * mp; }
};

__host__ __device__ constexpr int batch_ld(int nb) { return nb + 2; }
__host__ __device__ constexpr int round8(int m) { return (m + 15) & ~15; }  // (16: GEMM blocks of up to 16 rows)
size_t batch_smem_bytes(int m, int nb) {
  const size_t mp = (size_t)round8(m);
  return (mp * batch_ld(nb) + 5 * mp * nb) * sizeof(double);
}

// 8 consecutive doubles (16-byte aligned) from shared memory.
__device__ __forceinline__ void load8(const double* p, double (&v)[8]) {
  const double2* w = reinterpret_cast<const double2*>(p);
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const double2 t = w[h];
    v[2 * h] = t.x;
    v[2 * h + 1] = t.y;
  }
}

// Cross-lane ordered chains. Within a 256-index round, lane L holds the terms of
// indices base + 8L .. base + 8L + 7 (computed in parallel); the running sums
// are handed from lane to lane with a shuffle, so each s[k] is the single
// ascending chain ((0 + t_0) + t_1) + ... of the reference, skipping the terms
// whose use flag is false (exact zeros). A skipped term is added as -0, which
// leaves every sum bit-identical (s + -0 = s, +0 included: a chain that starts
// at +0 never becomes -0), so the chain is pure dependent DADDs with no select.
// All lanes end with the current sums.
template <int K>
__device__ __forceinline__ void lane_chain(double (&s)[K], const double (&t)[K][8],
                                           const bool (&use)[K][8], int nsteps) {
  const int lane = threadIdx.x & 31;
  double tt[K][8];
#pragma unroll
  for (int e = 0; e < 8; ++e)
#pragma unroll
    for (int k = 0; k < K; ++k) tt[k][e] = use[k][e] ? t[k][e] : -0.0;
  // Branch-free hand-off: every lane adds its own 8 terms to the current sums
  // and the sums of lane `src` (the only ones in index order) are broadcast.
  (void)lane;
  for (int src = 0; src < nsteps; ++src) {
    double r[K];
#pragma unroll
    for (int k = 0; k < K; ++k) r[k] = s[k];
#pragma unroll
    for (int e = 0; e < 8; ++e)
#pragma unroll
      for (int k = 0; k < K; ++k) r[k] = xadd(r[k], tt[k][e]);
#pragma unroll
    for (int k = 0; k < K; ++k) s[k] = __shfl_sync(0xffffffffu, r[k], src);
  }
}
// FAST profile: the same sums as fixed trees instead of the reference's ordered
// chains (lane-local partials in index order, then an xor-shuffle tree; lane 0's
// result broadcast so every lane holds identical bits). Deterministic run to run;
// ~6x shorter than the 32-step cross-lane hand-off of lane_chain.
template <int K>
__device__ __forceinline__ void lane_accum(double (&acc)[K], const double (&t)[K][8],
                                           const bool (&use)[K][8]) {
#pragma unroll
  for (int e = 0; e < 8; ++e)
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (use[k][e]) acc[k] += t[k][e];
}
template <int K>
__device__ __forceinline__ void lane_finish(double (&s)[K], const double (&acc)[K]) {
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double v = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    s[k] = __shfl_sync(0xffffffffu, v, 0);
  }
}
__device__ __forceinline__ int chain_steps(int m, int r0) {
  const int left = (m - r0 + 7) >> 3;
  return left < 32 ? left : 32;
}

__device__ void finish_col(const BatchArgs& a, ColState& S, const BatchSmem& sm, int b, int term,
                           int numeric) {
  const int lane = threadIdx.x & 31;
  const int c = S.col[b];
  const double* xb = sm.x(b);
  for (int i = lane; i < a.m; i += 32) a.Y[(size_t)c * a.m + i] = xb[i];
  if (lane == 0) {
    alnnls_column_result r;
    r.termination = term;
    r.numeric_failure = numeric;
    r.iterations = S.k[b];
    r.residual_sq = 0.0;
    r.f_final = S.f[b];
    r.gbs_final = S.gbs[b];
    r.multiplies_total = S.mults[b];
    a.res[c] = r;
    S.phase[b] = kIdle;
  }
  __syncwarp();
}

// Top of an iteration for column b (nqp.hpp:250-275): g_bar into V, the gbs /
// x.g / q.x chains, the ordered stop tests. One warp; returns true if stopped.
__device__ bool mask_phase(const BatchArgs& a, ColState& S, const BatchSmem& sm, int b) {
  const int lane = threadIdx.x & 31;
  const double* xb = sm.x(b);
  const double* gb = sm.g(b);
  const double* qb = sm.qc(b);
  for (int i = lane; i < a.m; i += 32) {
    const double xi = xb[i], gi = gb[i];
    sm.v(i, b) = (xi > 0.0 || gi < 0.0) ? gi : 0.0;  // g_bar
  }
  // the three chains in ascending index order; terms off the mask are exact
  // zeros (g_bar = 0, x = 0) and are skipped. q.x uses x*q (same product bits).
  int cnt = 0, bad = 0;
  double s[3] = {0.0, 0.0, 0.0};
  double fa[3] = {0.0, 0.0, 0.0};
  for (int r0 = 0; r0 < a.m; r0 += 256) {
    const int base = r0 + 8 * lane;
    double t[3][8];
    bool use[3][8];
    if (base < a.m) {
      double xv[8], gv[8], qv[8];
      load8(xb + base, xv);
      load8(gb + base, gv);
      load8(qb + base, qv);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const bool p = xv[e] > 0.0 || gv[e] < 0.0;  // zero beyond m: never passive
        cnt += p;
        if (!isfinite(gv[e])) bad = 1;
        const double gbar = p ? gv[e] : 0.0;
        use[0][e] = gbar != 0.0;
        t[0][e] = xmul(gbar, gbar);
        use[1][e] = xv[e] != 0.0;
        t[1][e] = xmul(xv[e], gv[e]);
        use[2][e] = use[1][e];
        t[2][e] = xmul(xv[e], qv[e]);
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          use[k][e] = false;
          t[k][e] = 0.0;
        }
    }
    if (a.fast) lane_accum<3>(fa, t, use);
    else lane_chain<3>(s, t, use, chain_steps(a.m, r0));
  }
  if (a.fast) lane_finish<3>(s, fa);
  for (int o = 16; o > 0; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  const double gbs = s[0], xg = s[1], qx = s[2];
  int stop = -1;
  if (lane == 0) {
    const double f = xmul(0.5, xadd(xg, qx));
    const unsigned long long k = S.k[b];
    S.f[b] = f;
    S.gbs[b] = gbs;
    S.ml[b] = cnt;
    if (bad || !isfinite(f) || !isfinite(gbs)) stop = 100;
    else if (cnt == 0) stop = ALNNLS_EMPTY_PASSIVE_SET;
    else if (gbs < a.eps) stop = ALNNLS_GRADIENT_BELOW_EPSILON;
    else if (k >= a.max_iters) stop = ALNNLS_MAX_ITERS;
    else if (gbs < S.best[b]) {
      S.best[b] = gbs;
      S.since[b] = 0;
    } else if (++S.since[b] >= a.stall_window) stop = ALNNLS_STALLED;
    if (stop < 0 && !(gbs != 0.0)) stop = ALNNLS_ZERO_CURVATURE;
    if (stop < 0) S.phase[b] = kNeedP1;
  }
  stop = __shfl_sync(0xffffffffu, stop, 0);
  if (stop >= 0) finish_col(a, S, sm, b, stop == 100 ? 0 : stop, stop == 100);
  return stop >= 0;
}

// den = g_bar . (Q g_bar) over the mask (exact_step, nqp.hpp:166-172).
__device__ double den_chain(const BatchSmem& sm, int b, bool fast) {
  const int lane = threadIdx.x & 31;
  double fa[1] = {0.0};
  const double* xb = sm.x(b);
  const double* gb = sm.g(b);
  const double* ub = sm.u(b);
  double s[1] = {0.0};
  for (int r0 = 0; r0 < sm.m; r0 += 256) {
    const int base = r0 + 8 * lane;
    double t[1][8];
    bool use[1][8];
    if (base < sm.m) {
      double xv[8], gv[8], uv[8];
      load8(xb + base, xv);
      load8(gb + base, gv);
      load8(ub + base, uv);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const double gbar = (xv[e] > 0.0 || gv[e] < 0.0) ? gv[e] : 0.0;
        use[0][e] = gbar != 0.0;
        t[0][e] = xmul(gbar, uv[e]);
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        use[0][e] = false;
        t[0][e] = 0.0;
      }
    }
    if (fast) lane_accum<1>(fa, t, use);
    else lane_chain<1>(s, t, use, chain_steps(sm.m, r0));
  }
  if (fast) lane_finish<1>(s, fa);
  return s[0];
}

// df = sum over the changed set of (g + 0.5 gd) * delta (nqp.hpp:307). The
// changed set is where the candidate differs from x, and delta = cand - x is
// recomputed with the same operation cand_phase used.
__device__ double df_chain(const BatchSmem& sm, int b, bool fast) {
  const int lane = threadIdx.x & 31;
  double fa[1] = {0.0};
  const double* xb = sm.x(b);
  const double* gb = sm.g(b);
  const double* cb = sm.c(b);
  const double* ub = sm.u(b);
  double s[1] = {0.0};
  for (int r0 = 0; r0 < sm.m; r0 += 256) {
    const int base = r0 + 8 * lane;
    double t[1][8];
    bool use[1][8];
    if (base < sm.m) {
      double xv[8], gv[8], cv[8], uv[8];
      load8(xb + base, xv);
      load8(gb + base, gv);
      load8(cb + base, cv);
      load8(ub + base, uv);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const double dd = cv[e] != xv[e] ? xsub(cv[e], xv[e]) : 0.0;
        use[0][e] = dd != 0.0;
        t[0][e] = xmul(xadd(gv[e], xmul(0.5, uv[e])), dd);
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        use[0][e] = false;
        t[0][e] = 0.0;
      }
    }
    if (fast) lane_accum<1>(fa, t, use);
    else lane_chain<1>(s, t, use, chain_steps(sm.m, r0));
  }
  if (fast) lane_finish<1>(s, fa);
  return s[0];
}

// Candidate step and changed set with the column's alpha (nqp.hpp:294-303):
// C = candidate x, V = delta (0 off the changed set). Returns |changed|.
__device__ int cand_phase(const BatchArgs& a, ColState& S, const BatchSmem& sm, int b) {
  const int lane = threadIdx.x & 31;
  const double alpha = S.alpha[b];
  const double* xb = sm.x(b);
  const double* gb = sm.g(b);
  double* cb = sm.c(b);
  int cnt = 0;
  for (int i = lane; i < a.m; i += 32) {
    const double xi = xb[i], gi = gb[i];
    double d = 0.0, c = xi;
    if (xi > 0.0 || gi < 0.0) {
      double t = xsub(xi, xmul(alpha, gi));
      if (t < 0.0) t = 0.0;
      if (t != xi) {
        c = t;
        d = xsub(t, xi);
        ++cnt;
      }
    }
    cb[i] = c;
    sm.v(i, b) = d;
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  __syncwarp();
  return cnt;
}

// Loads the next RHS from the queue into slot b and runs its first stop test
// (repeats while columns stop immediately). One warp.
__device__ void refill(const BatchArgs& a, ColState& S, const BatchSmem& sm, int b) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    int c = 0;
    if (lane == 0) c = atomicAdd(a.next_col, 1);
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= a.ncols) {
      for (int i = lane; i < a.m; i += 32) sm.v(i, b) = 0.0;  // idle slots feed zeros
      if (lane == 0) S.phase[b] = kIdle;
      __syncwarp();
      return;
    }
    const double* q = a.QB + (size_t)c * a.m;
    double* xb = sm.x(b);
    double* gb = sm.g(b);
    double* qb = sm.qc(b);
    for (int i = lane; i < a.m; i += 32) {
      const double qi = __ldg(q + i);
      xb[i] = 0.0;
      gb[i] = qi;  // x = 0, grad = q (nqp.hpp:224-225)
      qb[i] = qi;
    }
    if (lane == 0) {
      S.col[b] = c;
      S.k[b] = 0;
      S.tries[b] = 0;
      S.best[b] = __longlong_as_double(0x7ff0000000000000LL);
      S.since[b] = 0;
      S.mults[b] = 0;
    }
    __syncwarp();
    if (!mask_phase(a, S, sm, b)) return;
  }
}

// One exact chain GEMM pass for a group of CG columns starting at column
// grp * CG: U[:, col] = Q V[:, col], rows i = trow + r * ROWT (ascending j per
// output). Off-mask entries of V are 0 and their +-0 products are exact no-ops
// (idle slots, pad rows j >= m with their zero Q operands too).
template <int RPT, int CG, int ROWT, int LD, int JB = 8>
__device__ __forceinline__ void gemm_pass(const BatchArgs& a, const BatchSmem& sm, int grp, int trow) {
  const int m = sm.m, mp = sm.mp;
  double acc[RPT * CG];
#pragma unroll
  for (int t = 0; t < RPT * CG; ++t) acc[t] = 0.0;
  // JB: Q columns per block; two blocks in registers (ping-pong)
  auto load_q = [&](int j0, double (&qv)[RPT][JB]) {
#pragma unroll
    for (int u = 0; u < JB; ++u) {
      const double* qc = a.Q + (size_t)(j0 + u) * m;
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const int i = trow + r * ROWT;
        qv[r][u] = (j0 + u < m && i < m) ? __ldg(qc + i) : 0.0;
      }
    }
  };
  auto block = [&](int j0, const double (&qv)[RPT][JB]) {
#pragma unroll
    for (int u = 0; u < JB; ++u) {
      const double* vrow = sm.V + (size_t)(j0 + u) * LD + grp * CG;
      double vb[CG];
#pragma unroll
      for (int b = 0; b < CG; b += 2) {
        const double2 t = *reinterpret_cast<const double2*>(vrow + b);
        vb[b] = t.x;
        vb[b + 1] = t.y;
      }
#pragma unroll
      for (int r = 0; r < RPT; ++r)
#pragma unroll
        for (int b = 0; b < CG; ++b) acc[r * CG + b] = xmac(acc[r * CG + b], qv[r][u], vb[b]);
    }
  };
  double qa[RPT][JB], qb[RPT][JB];
  load_q(0, qa);
  for (int j0 = 0; j0 < mp; j0 += 2 * JB) {  // mp is a multiple of JB; V rows >= m are zero
    const bool two = j0 + JB < mp;
    if (two) load_q(j0 + JB, qb);
    block(j0, qa);
    if (j0 + 2 * JB < mp) load_q(j0 + 2 * JB, qa);
    if (two) block(j0 + JB, qb);
  }
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int i = trow + r * ROWT;
    if (i < m) {
#pragma unroll
      for (int b = 0; b < CG; ++b) sm.U[(size_t)(grp * CG + b) * mp + i] = acc[r * CG + b];
    }
  }
}

// Column b's state machine after its GEMM pass (nqp.hpp:276-318): P1 result ->
// den, alpha, candidate step; P2 result -> df, accept (next mask / stop tests)
// or halve and retry. One warp; V of the column is ready for its next pass.
__device__ void column_step(const BatchArgs& a, ColState& S, const BatchSmem& sm, int b) {
  const int lane = threadIdx.x & 31;
  const int m = sm.m;
  const int ph = S.phase[b];
  if (ph == kIdle) return;
  if (ph == kNeedP1) {
    const double den = den_chain(sm, b, a.fast != 0);  // exact_step, nqp.hpp:166-172
    if (!(den > 0.0)) {
      finish_col(a, S, sm, b, ALNNLS_ZERO_CURVATURE, 0);
      refill(a, S, sm, b);
      return;
    }
    if (lane == 0) {
      S.alpha[b] = xdiv(S.gbs[b], den);
      S.tries[b] = 0;
      S.mults[b] += (unsigned long long)m * (unsigned long long)S.ml[b];
    }
    __syncwarp();
  } else {  // kNeedP2: gd = Q delta in U
    const double df = df_chain(sm, b, a.fast != 0);
    const bool accept = df <= 0.0 || S.tries[b] >= 60;
    if (accept) {  // x[C] = cand, grad += gd (nqp.hpp:309-313)
      double* xb = sm.x(b);
      double* gw = sm.g(b);
      const double* cb = sm.c(b);
      const double* ub = sm.u(b);
      for (int i = lane; i < m; i += 32) {
        xb[i] = cb[i];
        gw[i] = xadd(gw[i], ub[i]);
      }
      if (lane == 0) ++S.k[b];
      __syncwarp();
      if (mask_phase(a, S, sm, b)) refill(a, S, sm, b);
      return;
    }
    if (lane == 0) {
      S.alpha[b] = xmul(S.alpha[b], 0.5);  // nqp.hpp:317
      ++S.tries[b];
    }
    __syncwarp();
  }
  // candidate step with the current alpha
  const int cl = cand_phase(a, S, sm, b);
  if (cl == 0) {  // nothing moved (nqp.hpp:304): next iteration on the same state
    if (lane == 0) ++S.k[b];
    __syncwarp();
    if (mask_phase(a, S, sm, b)) refill(a, S, sm, b);
    return;
  }
  if (lane == 0) {
    S.mults[b] += (unsigned long long)m * (unsigned long long)cl;
    S.phase[b] = kNeedP2;
  }
  __syncwarp();
}

// FAST profile: the pass U = Q V on the fp64 tensor cores (mma.sync m16n8k8
// DMMA, the dmma.cu fragment layout), NB = 16 columns, m <= 256: warp w owns
// rows [16w, 16w + 16) for both 8-column halves. DMMA sums each k8 group with
// its own ordering, so this is not the reference's chain (FAST is opt-in).
__device__ __forceinline__ void dmma8(double (&c)[4], double a0, double a1, double a2, double a3,
                                      double b0, double b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
}

template <int LD>
__device__ __forceinline__ void dmma_gemm_pass16(const BatchArgs& a, const BatchSmem& sm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int m = sm.m, mp = sm.mp;
  const int r0 = warp * 16;
  if (r0 >= m) return;
  const int ra = r0 + g, rb = r0 + g + 8;
  const bool va = ra < m, vb = rb < m;
  double acc[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
  constexpr int U = 4;  // k-steps whose Q fragments load together
  for (int k0 = 0; k0 < mp; k0 += 8 * U) {
    double q[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k1 = k0 + 8 * u + t, k2 = k1 + 4;
      const double* c1 = a.Q + (size_t)k1 * m;
      const double* c2 = a.Q + (size_t)k2 * m;
      q[u][0] = va && k1 < m ? __ldg(c1 + ra) : 0.0;
      q[u][1] = vb && k1 < m ? __ldg(c1 + rb) : 0.0;
      q[u][2] = va && k2 < m ? __ldg(c2 + ra) : 0.0;
      q[u][3] = vb && k2 < m ? __ldg(c2 + rb) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k1 = k0 + 8 * u + t;
      if (k0 + 8 * u >= mp) break;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const double b0 = sm.V[(size_t)k1 * LD + 8 * nt + g];
        const double b1 = sm.V[(size_t)(k1 + 4) * LD + 8 * nt + g];
        dmma8(acc[nt], q[u][0], q[u][1], q[u][2], q[u][3], b0, b1);
      }
    }
  }
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int row = (c < 2 ? ra : rb);
      const int col = 8 * nt + 2 * t + (c & 1);
      if (row < m) sm.U[(size_t)col * mp + row] = acc[nt][c];
    }
}

__device__ __forceinline__ BatchSmem carve(double* bsm, int m, int nb) {
  BatchSmem sm;
  const int mp = round8(m);
  sm.ld = batch_ld(nb);
  sm.m = m;
  sm.mp = mp;
  sm.V = bsm;
  sm.U = bsm + (size_t)mp * sm.ld;
  sm.C = sm.U + (size_t)mp * nb;
  sm.X = sm.C + (size_t)mp * nb;
  sm.G = sm.X + (size_t)mp * nb;
  sm.q = sm.G + (size_t)mp * nb;
  const int total = mp * sm.ld + 5 * mp * nb;  // zero once: pads must read as +0
  for (int e = threadIdx.x; e < total; e += blockDim.x) bsm[e] = 0.0;
  return sm;
}

// Every pass, all threads run the GEMM for all NB columns, then one warp per
// column runs its state machine. (A warp-specialised variant -- 8 warps on the
// GEMM of one half of the columns while 8 run the other half's state machines --
// measured slower at c4: 1.71-1.86 s vs 1.65 s; with 2 warps per scheduler the
// GEMM cannot hide the L2 latency of Q.)
template <int NB>
__global__ void __launch_bounds__(kBT, 1) batched_nqp_kernel(BatchArgs a) {
  extern __shared__ __align__(16) double bsm[];
  __shared__ ColState S;
  constexpr int LD = batch_ld(NB);
  const BatchSmem sm = carve(bsm, a.m, NB);
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  constexpr int nwarps = kBT / 32;
  for (int b = warp; b < NB; b += nwarps) refill(a, S, sm, b);
  __syncthreads();
#ifndef ALNNLS_GEMM_CG
#define ALNNLS_GEMM_CG 8
#endif
  constexpr int CG = NB < ALNNLS_GEMM_CG ? NB : ALNNLS_GEMM_CG;  // columns per thread
  constexpr int GROUPS = NB / CG;
  constexpr int ROWT = kBT / GROUPS;
  constexpr int RPT = (4096 / NB + ROWT - 1) / ROWT;  // rows per thread at the largest m (4096/NB)
  const int grp = threadIdx.x / ROWT, trow = threadIdx.x % ROWT;
  for (;;) {
    int active = 0;
    for (int b = 0; b < NB; ++b) active |= S.phase[b] != kIdle;
    if (!active) break;
    if (NB == 16 && a.fast) {
      dmma_gemm_pass16<LD>(a, sm);
    } else {
      gemm_pass<RPT, CG, ROWT, LD, ALNNLS_GEMM_JB>(a, sm, grp, trow);
    }
    __syncthreads();
    for (int b = warp; b < NB; b += nwarps) column_step(a, S, sm, b);
    __syncthreads();
  }
}

// x[retained[a], j] = Y[a, j] / D_a; dropped columns 0 (nnls.hpp:87-96).
__global__ void unscale_batched_kernel(const double* Y, int m, const double* scale,
                                       const uint32_t* retained, double* X, int n, int ncols) {
  const size_t total = (size_t)m * ncols;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total;
       e += (size_t)gridDim.x * blockDim.x) {
    const size_t j = e / m, a = e % m;
    X[j * n + retained[a]] = xdiv(Y[e], scale[a]);
  }
}

// residual_norm_sq per column (nnls.hpp:115-123): (A x)_i is one chain over the
// columns of A in ascending order (matvec, linalg.hpp:182-186), then s += r_i^2 in
// ascending i. One CTA owns kRC right-hand sides and walks all row tiles in order,
// so each column's s is a single chain. A zero x_j adds a +-0 product, an exact
// no-op on a chain that starts at +0 (it can never become -0), so the MACs are
// branch-free. Each thread owns a 4 x 4 block of the tile; the next k-slab of A
// and X is loaded into registers while the current one is multiplied.
constexpr int kRT = 64;   // rows per tile
constexpr int kRC = 64;   // columns per CTA
constexpr int kRK = 16;   // k slab
__global__ void __launch_bounds__(256) residual_batched_kernel(const double* A, uint64_t lda, int d,
                                                               int n, const double* X,
                                                               const double* B, uint64_t ldb,
                                                               int ncols,
                                                               alnnls_column_result* res) {
  // the slab buffers and the finished tile share one static buffer (< 48 KB)
  __shared__ double sbuf[kRT * (kRC + 1)];
  double(*As)[kRK][kRT] = reinterpret_cast<double(*)[kRK][kRT]>(sbuf);
  double(*Xs)[kRK][kRC] = reinterpret_cast<double(*)[kRK][kRC]>(sbuf + 2 * kRK * kRT);
  double(*Cs)[kRC + 1] = reinterpret_cast<double(*)[kRC + 1]>(sbuf);
  static_assert(2 * kRK * (kRT + kRC) <= kRT * (kRC + 1), "slab buffers fit the tile buffer");
  const int c0 = blockIdx.x * kRC;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // rows tx + 16 r, columns ty + 16 c
  const int nslab = (n + kRK - 1) / kRK;
  double ssum = 0.0;  // thread t < kRC: the running chain of column c0 + t
  // slab loader: 4 A and 4 X elements per thread
  auto fetch = [&](int i0, int k0, double (&ra)[4], double (&rx)[4]) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = threadIdx.x + 256 * u;
      const int kk = e / kRT, r = e % kRT;
      const int i = i0 + r, kcol = k0 + kk;
      ra[u] = (i < d && kcol < n) ? __ldg(A + (size_t)kcol * lda + i) : 0.0;
      const int c = e / kRK, kx = e % kRK;
      const int col = c0 + c, kc2 = k0 + kx;
      rx[u] = (col < ncols && kc2 < n) ? __ldg(X + (size_t)col * n + kc2) : 0.0;
    }
  };
  auto stash = [&](int buf, const double (&ra)[4], const double (&rx)[4]) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = threadIdx.x + 256 * u;
      As[buf][e / kRT][e % kRT] = ra[u];
      Xs[buf][e % kRK][e / kRK] = rx[u];
    }
  };
  for (int i0 = 0; i0 < d; i0 += kRT) {
    double acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;
    double ra[4], rx[4];
    fetch(i0, 0, ra, rx);
    stash(0, ra, rx);
    __syncthreads();
    for (int sl = 0; sl < nslab; ++sl) {
      const int buf = sl & 1;
      if (sl + 1 < nslab) fetch(i0, (sl + 1) * kRK, ra, rx);
#pragma unroll
      for (int kk = 0; kk < kRK; ++kk) {
        double av[4], xv[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) av[r] = As[buf][kk][tx + 16 * r];
#pragma unroll
        for (int c = 0; c < 4; ++c) xv[c] = Xs[buf][kk][ty + 16 * c];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[r][c] = xmac(acc[r][c], av[r], xv[c]);
      }
      if (sl + 1 < nslab) stash(buf ^ 1, ra, rx);
      __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) Cs[tx + 16 * r][ty + 16 * c] = acc[r][c];
    __syncthreads();
    if (threadIdx.x < kRC && c0 + (int)threadIdx.x < ncols) {
      const double* bcol = B + (size_t)(c0 + threadIdx.x) * ldb;
      const int rows = min(kRT, d - i0);
      for (int r = 0; r < rows; ++r) {
        const double rr = xsub(Cs[r][threadIdx.x], __ldg(bcol + i0 + r));
        ssum = xadd(ssum, xmul(rr, rr));
      }
    }
    __syncthreads();
  }
  if (threadIdx.x < kRC && c0 + (int)threadIdx.x < ncols) res[c0 + threadIdx.x].residual_sq = ssum;
}

}  // namespace

int batched_cols_per_cta(int m) {
  // shared memory holds 5 m x NB panels; the GEMM covers m <= 4096 / NB rows
  return m <= 256 ? 16 : (m <= 512 ? 8 : (m <= 1024 ? 4 : 0));
}

cudaError_t launch_batched(const BatchArgs& a, int sm_count, cudaStream_t stream) {
  const int NB = batched_cols_per_cta(a.m);
  if (NB == 0) return cudaErrorInvalidValue;
  {
    const int mx = (int)batch_smem_bytes(1024, 4);  // the largest configuration
    if (cudaError_t e = smem_optin(batched_nqp_kernel<16>, mx)) return e;
    if (cudaError_t e = smem_optin(batched_nqp_kernel<8>, mx)) return e;
    if (cudaError_t e = smem_optin(batched_nqp_kernel<4>, mx)) return e;
  }
  const size_t smem = batch_smem_bytes(a.m, NB);
  int grid = sm_count;
  const int need = (a.ncols + NB - 1) / NB;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  if (NB == 16) batched_nqp_kernel<16><<<grid, kBT, smem, stream>>>(a);
  else if (NB == 8) batched_nqp_kernel<8><<<grid, kBT, smem, stream>>>(a);
  else batched_nqp_kernel<4><<<grid, kBT, smem, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_unscale_batched(const double* Y, int m, const double* scale,
                                   const uint32_t* retained, double* X, int n, int ncols,
                                   cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(X, 0, sizeof(double) * (size_t)n * ncols, stream);
  if (e != cudaSuccess || m == 0) return e;
  unscale_batched_kernel<<<148 * 8, 256, 0, stream>>>(Y, m, scale, retained, X, n, ncols);
  return cudaGetLastError();
}

cudaError_t launch_residual_batched(const double* A, uint64_t lda, int d, int n, const double* X,
                                    const double* B, uint64_t ldb, int ncols,
                                    alnnls_column_result* res, cudaStream_t stream) {
  if (ncols <= 0) return cudaSuccess;
  residual_batched_kernel<<<(ncols + kRC - 1) / kRC, 256, 0, stream>>>(A, lda, d, n, X, B, ldb,
                                                                         ncols, res);
  return cudaGetLastError();
}

}  // namespace alnnls
