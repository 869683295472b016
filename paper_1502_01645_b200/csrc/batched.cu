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
#include <cstdlib>

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
// Work a column slot still has to do in the current pass (settle rounds).
enum ColAct {
  kActNone = 0,
  kActCand = 1,    // candidate step + changed set with alpha (nqp.hpp:294-303)
  kActAccept = 2,  // x[C] = cand, grad += gd (nqp.hpp:309-313), then the next stop test
  kActMask = 3,    // stop test on the current state (nqp.hpp:250-275)
  kActInit = 4,    // a fresh column: x = 0, grad = q (nqp.hpp:224-225), then its stop test
  kActFinish = 5,  // write the column's result, then take the next column
  kActGrab = 6     // take the next column from the queue
};

struct ColState {
#ifdef ALNNLS_BATCH_PROF
  long long pr[8];
#endif
  int phase[kMaxCols];
  int act[kMaxCols];
  int col[kMaxCols];
  unsigned long long k[kMaxCols];
  int tries[kMaxCols];
  int ml[kMaxCols];
  int cnt[kMaxCols];   // per-column counts of the elementwise phase (passive / changed)
  int bad[kMaxCols];   // non-finite gradient entry seen
  int term[kMaxCols];  // termination of a finishing column (-1: NumericFailure)
  double alpha[kMaxCols];
  double f[kMaxCols], gbs[kMaxCols];
  double best[kMaxCols];
  double res[kMaxCols][3];  // chain results
  double part[kMaxCols][4][3];  // FAST: per-warp tree partials (<= 4 warps per column)
  unsigned long long since[kMaxCols];
  unsigned long long mults[kMaxCols];
};

// Shared-memory layout of one CTA (mp = m rounded up to 16, ps = mp + 2):
//  - V, the GEMM input, row-major mp x ld (ld = NB + 2): the GEMM reads a row of
//    V with 16-byte broadcasts; the padding keeps the per-column writes (lane =
//    row) at 4-way bank sharing; rows >= m stay zero so the GEMM needs no tail.
//  - U (GEMM output), C (candidate), X (iterate), G (gradient), q (linear term):
//    column panels of stride ps. The elementwise phases walk a column with
//    consecutive lanes (conflict-free); the chain lanes (one per column) read
//    the same offset of NB panels, which the +2 stride spreads over the banks.
//  - chain terms: den / df terms go to V (dead once the pass has read it; the
//    chain lanes read one V row, NB consecutive doubles); the stop-test terms
//    x.g and q.x go to U and C (dead after the accepted update), and g_bar^2 is
//    formed by the chain lane from V = g_bar.
struct BatchSmem {
  double* V;
  int ld;
  int m, mp, ps;
  double* U;
  double* C;
  double* X;
  double* G;
  double* q;
  __device__ double& v(int i, int b) const { return V[i * ld + b]; }
  __device__ double* u(int b) const { return U + b * ps; }
  __device__ double* c(int b) const { return C + b * ps; }
  __device__ double* x(int b) const { return X + b * ps; }
  __device__ double* g(int b) const { return G + b * ps; }
  __device__ double* qc(int b) const { return q + b * ps; }
};

__host__ __device__ constexpr int batch_ld(int nb) { return nb + 2; }
__host__ __device__ constexpr int round8(int m) { return (m + 15) & ~15; }  // (16: GEMM blocks of up to 16 rows)
__host__ __device__ constexpr int panel_stride(int m) { return round8(m) + 2; }
size_t batch_smem_bytes(int m, int nb) {
  const size_t mp = (size_t)round8(m);
  return (mp * batch_ld(nb) + 5 * (size_t)panel_stride(m) * nb) * sizeof(double);
}

// Reference-ordered sums, one lane per column (the chain warp, lane b = column
// b): s = ((0 + t_0) + t_1) + ... over the m rows. A term the reference skips
// is a -0, which leaves every sum bit-identical (s + -0 = s, and a chain that
// starts at +0 never becomes -0), so each lane runs pure dependent DADDs, and
// one DADD instruction advances every column's chain (the FP64 pipe is not
// spent on one useful lane per instruction). The three stop-test sums of a
// column run on three lanes (warp 0 lanes b and 16 + b; warp 1 lane b).
// lane_sum<false>: the terms are p[t * stride] as stored. Two register blocks of 16
// alternate, so the loads of the next block are in flight during the current block's
// chain and the dependent DADD (8 cycles) is the per-term cost.
// lane_sum<true>: the terms are the squares (g_bar^2; g_bar = +0 off the mask gives +0,
// which leaves the chain unchanged just like the reference's skipped term). (A three-
// block rotation that squares block t + 1 between the DADDs of block t measured slower.)
template <bool SQ>
__device__ __forceinline__ double lane_sum(const double* __restrict__ p, int stride, int n) {
  constexpr int B = 16;
  double s = 0.0;
  int t = 0;
  auto term = [](double v) { return SQ ? xmul(v, v) : v; };
  auto load = [&](double (&r)[B], int at) {
#pragma unroll
    for (int e = 0; e < B; ++e) r[e] = p[(at + e) * stride];
  };
  auto run = [&](const double (&r)[B]) {
#pragma unroll
    for (int e = 0; e < B; ++e) s = xadd(s, term(r[e]));
  };
  if (n >= 2 * B) {
    double ra[B], rb[B];
    load(ra, 0);
    for (; t + 3 * B <= n; t += 2 * B) {
      load(rb, t + B);
      run(ra);
      load(ra, t + 2 * B);
      run(rb);
    }
    if (t + 2 * B <= n) {  // ra holds [t, t + B)
      load(rb, t + B);
      run(ra);
      run(rb);
      t += 2 * B;
    } else {
      run(ra);
      t += B;
    }
  }
  for (; t < n; ++t) s = xadd(s, term(p[t * stride]));
  return s;
}
// FAST profile: a column's sums as fixed trees instead of the reference's
// chains: each lane adds its rows in index order, an xor-shuffle tree combines
// the lanes, the column's warps' partials are added in warp order by the
// decision lane. Deterministic run to run; no chain phase.
__device__ __forceinline__ double warp_tree(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return __shfl_sync(0xffffffffu, v, 0);
}
__device__ __forceinline__ double fast_parts(const ColState& S, int b, int k, int wpc) {
  double s = S.part[b][0][k];
  for (int w = 1; w < wpc; ++w) s += S.part[b][w][k];
  return s;
}

// Elementwise phases: warp w works on column w / wpc (wpc = warps per column),
// its lanes on rows sub*32 + lane, sub*32 + lane + 32*wpc, ...
struct ColWarp {
  int b, i0, step, sub, bstep;
};
// With fewer warps than columns (NB = 8 on 4 warps) warp w takes columns w, w + nw, ...
// whole (bstep = nw); otherwise one column per warp (bstep = NB ends the loop).
__device__ __forceinline__ ColWarp col_warp(int NB) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  ColWarp w;
  if (nw < NB) {
    w.b = warp;
    w.sub = 0;
    w.i0 = lane;
    w.step = 32;
    w.bstep = nw;
    return w;
  }
  const int wpc = nw / NB;  // NB divides the warp count (16, 8 or 4 columns, 16 or 8 warps)
  w.b = warp / wpc;
  w.sub = warp - w.b * wpc;
  w.i0 = w.sub * 32 + lane;
  w.step = 32 * wpc;
  w.bstep = NB;
  return w;
}
__device__ __forceinline__ int warps_per_col(int NB) {
  const int nw = blockDim.x >> 5;
  return nw < NB ? 1 : nw / NB;
}

// Elementwise work of one settle round. Writes V = g_bar and the stop-test terms
// (U: x g, C: x q; -0 for the terms the reference skips) for the columns about
// to run a stop test, C = cand and V = delta for a candidate step.
__device__ void round_elementwise_col(const BatchArgs& a, ColState& S, const BatchSmem& sm,
                                      const ColWarp& w, int b) {
  const int m = sm.m;
  const int act = S.act[b];
  if (act == kActNone) return;
  double* xb = sm.x(b);
  double* gb = sm.g(b);
  double* cb = sm.c(b);
  double* ub = sm.u(b);
  double* qb = sm.qc(b);
  int cnt = 0, bad = 0;
  if (act == kActCand) {
    const double alpha = S.alpha[b];
#pragma unroll 4
    for (int i = w.i0; i < m; i += w.step) {
      const double xi = xb[i], gi = gb[i];
      double d = 0.0, c = xi;
      if (xi > 0.0 || gi < 0.0) {
        double t = xsub(xi, xmul(alpha, gi));  // x - (alpha g), nqp.hpp:296
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
  } else if (act == kActAccept || act == kActMask || act == kActInit) {
    const double* qg = a.QB + (size_t)S.col[b] * m;
    double f0 = 0.0, f1 = 0.0, f2 = 0.0;  // FAST partials
#pragma unroll 4
    for (int i = w.i0; i < m; i += w.step) {
      double xi, gi, qi;
      if (act == kActAccept) {  // nqp.hpp:309-313
        xi = cb[i];
        gi = xadd(gb[i], ub[i]);
        xb[i] = xi;
        gb[i] = gi;
        qi = qb[i];
      } else if (act == kActInit) {  // x = 0, grad = q (nqp.hpp:224-225)
        qi = __ldg(qg + i);
        xi = 0.0;
        gi = qi;
        xb[i] = xi;
        gb[i] = gi;
        qb[i] = qi;
      } else {
        xi = xb[i];
        gi = gb[i];
        qi = qb[i];
      }
      const bool p = xi > 0.0 || gi < 0.0;
      cnt += p;
      if (!isfinite(gi)) bad = 1;
      const double gbar = p ? gi : 0.0;
      sm.v(i, b) = gbar;  // its square is formed by the chain lane
      // x.g and q.x: the x_i = 0 terms are skipped (q.x uses x*q, same bits)
      const double txg = xi != 0.0 ? xmul(xi, gi) : -0.0;
      const double tqx = xi != 0.0 ? xmul(xi, qi) : -0.0;
      if (a.fast) {
        f0 += xmul(gbar, gbar);
        f1 += txg;
        f2 += tqx;
      } else {
        ub[i] = txg;
        cb[i] = tqx;
      }
    }
    if (a.fast) {
      f0 = warp_tree(f0);
      f1 = warp_tree(f1);
      f2 = warp_tree(f2);
      if ((threadIdx.x & 31) == 0) {
        S.part[b][w.sub][0] = f0;
        S.part[b][w.sub][1] = f1;
        S.part[b][w.sub][2] = f2;
      }
    }
  } else if (act == kActFinish || act == kActGrab) {
    if (act == kActFinish)
      for (int i = w.i0; i < m; i += w.step) a.Y[(size_t)S.col[b] * m + i] = xb[i];
    for (int i = w.i0; i < m; i += w.step) sm.v(i, b) = 0.0;  // idle slots feed zeros
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  bad = __reduce_or_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0) {
    if (cnt) atomicAdd(S.cnt + b, cnt);
    if (bad) S.bad[b] = 1;
  }
}
__device__ void round_elementwise(const BatchArgs& a, ColState& S, const BatchSmem& sm, int NB) {
  const ColWarp w = col_warp(NB);
  for (int b = w.b; b < NB; b += w.bstep) round_elementwise_col(a, S, sm, w, b);
}

// One column's stop test after its stop-test chains (nqp.hpp:251-275). Lane
// b of the chain warp. Sets act (None: continue with P1; Finish: stopped).
__device__ void stop_test(const BatchArgs& a, ColState& S, int b) {
  const double gbs = S.res[b][0], xg = S.res[b][1], qx = S.res[b][2];
  const double f = xmul(0.5, xadd(xg, qx));
  const unsigned long long k = S.k[b];
  const int cnt = S.cnt[b];
  S.f[b] = f;
  S.gbs[b] = gbs;
  S.ml[b] = cnt;
  int stop = -2;
  if (S.bad[b] || !isfinite(f) || !isfinite(gbs)) stop = -1;  // NumericFailure
  else if (cnt == 0) stop = ALNNLS_EMPTY_PASSIVE_SET;
  else if (gbs < a.eps) stop = ALNNLS_GRADIENT_BELOW_EPSILON;
  else if (k >= a.max_iters) stop = ALNNLS_MAX_ITERS;
  else if (gbs < S.best[b]) {
    S.best[b] = gbs;
    S.since[b] = 0;
  } else if (++S.since[b] >= a.stall_window) stop = ALNNLS_STALLED;
  if (stop == -2 && !(gbs != 0.0)) stop = ALNNLS_ZERO_CURVATURE;  // num == 0 (nqp.hpp:167)
  if (stop == -2) {
    S.phase[b] = kNeedP1;
    S.act[b] = kActNone;
  } else {
    S.term[b] = stop;
    S.act[b] = kActFinish;
  }
}

// Lane b of the chain warp, after the elementwise phase of a round.
__device__ void round_decide(const BatchArgs& a, ColState& S, int b) {
  const int act = S.act[b];
  if (act == kActCand) {
    const int cl = S.cnt[b];
    if (cl == 0) {  // nothing moved (nqp.hpp:304): next iteration on the same state
      ++S.k[b];
      S.act[b] = kActMask;
    } else {
      S.mults[b] += (unsigned long long)a.m * (unsigned long long)cl;
      S.phase[b] = kNeedP2;
      S.act[b] = kActNone;
    }
  } else if (act == kActAccept || act == kActMask || act == kActInit) {
    stop_test(a, S, b);
  } else if (act == kActFinish || act == kActGrab) {
    if (act == kActFinish) {
      alnnls_column_result r;
      r.termination = S.term[b] < 0 ? 0 : S.term[b];
      r.numeric_failure = S.term[b] < 0;
      r.iterations = S.k[b];
      r.residual_sq = 0.0;
      r.f_final = S.f[b];
      r.gbs_final = S.gbs[b];
      r.multiplies_total = S.mults[b];
      a.res[S.col[b]] = r;
    }
    const int c = atomicAdd(a.next_col, 1);
    if (c >= a.ncols) {
      S.phase[b] = kIdle;
      S.act[b] = kActNone;
    } else {
      S.col[b] = c;
      S.k[b] = 0;
      S.tries[b] = 0;
      S.best[b] = __longlong_as_double(0x7ff0000000000000LL);
      S.since[b] = 0;
      S.mults[b] = 0;
      S.act[b] = kActInit;
    }
  }
}

// Settle rounds until every slot has a GEMM pass to wait for (or is idle):
// elementwise phase, the stop-test chains of the columns that need them, the
// per-column decisions. Whole CTA; the chain warp is warp 0 (lane b: column b).
__device__ void settle(const BatchArgs& a, ColState& S, const BatchSmem& sm, int NB) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef ALNNLS_BATCH_PROF
  long long t0 = clock64();
#define BPROF(k) { const long long t1 = clock64(); if (threadIdx.x == 0) S.pr[k] += t1 - t0; t0 = t1; }
#else
#define BPROF(k)
#endif
  for (;;) {
    __syncthreads();  // acts and counter resets are visible
    BPROF(2)
    int pending = 0;
    for (int b = 0; b < NB; ++b) pending |= S.act[b] != kActNone;
    if (!pending) return;
    round_elementwise(a, S, sm, NB);
    __syncthreads();
    BPROF(3)
#ifdef ALNNLS_BATCH_PROF
    if (threadIdx.x == 0) S.pr[5]++;
#endif
    // the stop-test sums of column b: x.g and q.x on warp 0 lanes b and 16 + b, gbs
    // (the squares of g_bar) on warp 1 lane b (each warp runs one instruction stream)
    if (warp < 2) {
      const int k = warp == 0 ? (lane < 16 ? 1 : 2) : (lane < 16 ? 0 : 3), b = lane & 15;
      if (k < 3 && b < NB) {
        const int act = S.act[b];
        if (act == kActAccept || act == kActMask || act == kActInit) {
          if (a.fast) {
            S.res[b][k] = fast_parts(S, b, k, warps_per_col(NB));
          } else {
            S.res[b][k] = k == 0 ? lane_sum<true>(sm.V + b, sm.ld, sm.m)
                                 : lane_sum<false>(k == 1 ? sm.u(b) : sm.c(b), 1, sm.m);
          }
        }
      }
      asm volatile("bar.sync 1, 64;" ::: "memory");
    }
    if (warp == 0 && lane < NB) {
      const int b = lane;
      if (S.act[b] == kActAccept) ++S.k[b];
      round_decide(a, S, b);
      if (S.act[b] != kActNone) {
        S.cnt[b] = 0;
        S.bad[b] = 0;
      }
    }
    BPROF(4)
  }
}

// FAST, one warp per column (NB = 16 on 16 warps): the whole state machine of a
// column after its GEMM pass stays inside its warp -- the den / df tree sum, the
// decision on lane 0, then the column's settle rounds (elementwise work + tree
// sums + decision) -- so no CTA barrier is needed until the next pass.
__device__ void fast_warp_pass(const BatchArgs& a, ColState& S, const BatchSmem& sm) {
  const int b = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = sm.m;
  const int ph = S.phase[b];
  if (ph != kIdle) {
    const double* gb = sm.g(b);
    const double* ub = sm.u(b);
    double f = 0.0;
    if (ph == kNeedP1) {
#pragma unroll 4
      for (int i = lane; i < m; i += 32) {
        const double gbar = sm.v(i, b);
        f += gbar != 0.0 ? xmul(gbar, ub[i]) : -0.0;
      }
    } else {
#pragma unroll 4
      for (int i = lane; i < m; i += 32) {
        const double dd = sm.v(i, b);
        f += dd != 0.0 ? xmul(xadd(gb[i], xmul(0.5, ub[i])), dd) : -0.0;
      }
    }
    f = warp_tree(f);
    if (lane == 0) {
      if (ph == kNeedP1) {
        if (!(f > 0.0)) {
          S.term[b] = ALNNLS_ZERO_CURVATURE;
          S.act[b] = kActFinish;
        } else {
          S.alpha[b] = xdiv(S.gbs[b], f);
          S.tries[b] = 0;
          S.mults[b] += (unsigned long long)m * (unsigned long long)S.ml[b];
          S.act[b] = kActCand;
        }
      } else if (f <= 0.0 || S.tries[b] >= 60) {
        S.act[b] = kActAccept;
      } else {
        S.alpha[b] = xmul(S.alpha[b], 0.5);  // nqp.hpp:317
        ++S.tries[b];
        S.act[b] = kActCand;
      }
      S.cnt[b] = 0;
      S.bad[b] = 0;
    }
    __syncwarp();
  }
  for (;;) {
    const int act = S.act[b];
    if (act == kActNone) break;
    round_elementwise(a, S, sm, 16);  // this warp's column (one warp per column)
    __syncwarp();
    if (lane == 0) {
      if (act == kActAccept || act == kActMask || act == kActInit) {
        S.res[b][0] = S.part[b][0][0];
        S.res[b][1] = S.part[b][0][1];
        S.res[b][2] = S.part[b][0][2];
        if (act == kActAccept) ++S.k[b];
      }
      round_decide(a, S, b);
      if (S.act[b] != kActNone) {
        S.cnt[b] = 0;
        S.bad[b] = 0;
      }
    }
    __syncwarp();
  }
}

// After a GEMM pass (U = Q V for every live column): the P1 columns' den terms
// (exact_step, nqp.hpp:166-172) and the P2 columns' df terms (nqp.hpp:307) into
// V, their chains, alpha / accept-or-halve (nqp.hpp:308-317), the settle rounds.
__device__ void after_pass(const BatchArgs& a, ColState& S, const BatchSmem& sm, int NB) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = sm.m;
#ifdef ALNNLS_BATCH_PROF
  long long t0 = clock64();
#endif
  const ColWarp w = col_warp(NB);
  for (int b = w.b; b < NB; b += w.bstep) {
    const int ph = S.phase[b];
    const double* xb = sm.x(b);
    const double* gb = sm.g(b);
    const double* ub = sm.u(b);
    const double* cb = sm.c(b);
    double f = 0.0;  // FAST partial
    if (ph == kNeedP1) {
#pragma unroll 4
      for (int i = w.i0; i < m; i += w.step) {
        const double gbar = sm.v(i, b);  // the pass's input: g_bar
        const double t = gbar != 0.0 ? xmul(gbar, ub[i]) : -0.0;
        if (a.fast) f += t;
        else sm.v(i, b) = t;
      }
    } else if (ph == kNeedP2) {
#pragma unroll 4
      for (int i = w.i0; i < m; i += w.step) {
        const double dd = sm.v(i, b);  // the pass's input: delta (0 off the changed set)
        const double t = dd != 0.0 ? xmul(xadd(gb[i], xmul(0.5, ub[i])), dd) : -0.0;
        if (a.fast) f += t;
        else sm.v(i, b) = t;
      }
    }
    if (a.fast && ph != kIdle) {
      f = warp_tree(f);
      if (lane == 0) S.part[b][w.sub][0] = f;
    }
    (void)xb;
    (void)cb;
  }
  __syncthreads();
  BPROF(0)
  if (warp == 0 && lane < NB) {
    const int b = lane;
    const int ph = S.phase[b];
    if (ph != kIdle) {
      const double s = a.fast ? fast_parts(S, b, 0, warps_per_col(NB))
                              : lane_sum<false>(sm.V + b, sm.ld, m);
      if (ph == kNeedP1) {
        if (!(s > 0.0)) {
          S.term[b] = ALNNLS_ZERO_CURVATURE;
          S.act[b] = kActFinish;
        } else {
          S.alpha[b] = xdiv(S.gbs[b], s);
          S.tries[b] = 0;
          S.mults[b] += (unsigned long long)m * (unsigned long long)S.ml[b];
          S.act[b] = kActCand;
        }
      } else if (s <= 0.0 || S.tries[b] >= 60) {
        S.act[b] = kActAccept;
      } else {
        S.alpha[b] = xmul(S.alpha[b], 0.5);  // nqp.hpp:317
        ++S.tries[b];
        S.act[b] = kActCand;
      }
      S.cnt[b] = 0;
      S.bad[b] = 0;
    }
  }
  BPROF(1)
  settle(a, S, sm, NB);
}


// One exact chain GEMM pass for a group of CG columns starting at column
// grp * CG: U[:, col] = Q V[:, col], rows i = trow + r * ROWT (ascending j per
// output). Off-mask entries of V are 0 and their +-0 products are exact no-ops
// (idle slots, pad rows j >= m with their zero Q operands too).
#ifndef ALNNLS_GEMM_QBUF
#define ALNNLS_GEMM_QBUF 3  // register blocks of Q columns in flight in the 128-thread two-CTA
                            // configuration (2: ping-pong, 3: rotation); the others keep 2
#endif
template <int RPT, int CG, int ROWT, int LD, int JB = 8, int QBUF = 2>
__device__ __forceinline__ void gemm_pass(const BatchArgs& a, const BatchSmem& sm, int grp, int trow) {
  const int m = sm.m, mp = sm.mp;
  double acc[RPT * CG];
#pragma unroll
  for (int t = 0; t < RPT * CG; ++t) acc[t] = 0.0;
  // JB: Q columns per block; two blocks in registers (ping-pong)
  auto load_q = [&](int j0, double (&qv)[RPT][JB]) {
#pragma unroll
    for (int u = 0; u < JB; ++u) {
#ifdef ALNNLS_EXP_QL1
      const double* qc = a.Q + (size_t)((j0 + u) & 7) * m;
#else
      const double* qc = a.Q + (size_t)(j0 + u) * m;
#endif
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
#ifdef ALNNLS_EXP_NOV
#pragma unroll
      for (int b = 0; b < CG; ++b) vb[b] = 1.0 + b + (j0 & 3);
      (void)vrow;
#else
#pragma unroll
      for (int b = 0; b < CG; b += 2) {
        const double2 t = *reinterpret_cast<const double2*>(vrow + b);
        vb[b] = t.x;
        vb[b + 1] = t.y;
      }
#endif
#pragma unroll
      for (int r = 0; r < RPT; ++r)
#pragma unroll
        for (int b = 0; b < CG; ++b) acc[r * CG + b] = xmac(acc[r * CG + b], qv[r][u], vb[b]);
    }
  };
  if constexpr (QBUF == 3) {
  // three register blocks in rotation: a block's loads are issued two blocks (2 x JB x
  // RPT x CG rounded multiply-adds) before its use: the L2 latency of the Q columns is
  // longer than one block of one warp per scheduler (ncu: long-scoreboard stalls on the
  // first use of a block). 65536-column loop 1.4595 -> 1.4326 s, same bits.
  double qa[RPT][JB], qb[RPT][JB], qc[RPT][JB];
  load_q(0, qa);
  if (JB < mp) load_q(JB, qb);
  for (int j0 = 0; j0 < mp; j0 += 3 * JB) {  // mp is a multiple of JB; V rows >= m are zero
    if (j0 + 2 * JB < mp) load_q(j0 + 2 * JB, qc);
    block(j0, qa);
    if (j0 + 3 * JB < mp) load_q(j0 + 3 * JB, qa);
    if (j0 + JB < mp) block(j0 + JB, qb);
    if (j0 + 4 * JB < mp) load_q(j0 + 4 * JB, qb);
    if (j0 + 2 * JB < mp) block(j0 + 2 * JB, qc);
  }
  } else {
  double qa[RPT][JB], qb[RPT][JB];
  load_q(0, qa);
  for (int j0 = 0; j0 < mp; j0 += 2 * JB) {  // mp is a multiple of JB; V rows >= m are zero
    const bool two = j0 + JB < mp;
    if (two) load_q(j0 + JB, qb);
    block(j0, qa);
    if (j0 + 2 * JB < mp) load_q(j0 + 2 * JB, qa);
    if (two) block(j0 + JB, qb);
  }
  }
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int i = trow + r * ROWT;
    if (i < m) {
#pragma unroll
      for (int b = 0; b < CG; ++b) sm.U[(size_t)(grp * CG + b) * sm.ps + i] = acc[r * CG + b];
    }
  }
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
#ifndef ALNNLS_DMMA_U
#define ALNNLS_DMMA_U 4
#endif
  constexpr int U = ALNNLS_DMMA_U;  // k-steps whose Q fragments load together (build knob)
  // Q in fragment order (a.Qf, see qfrag_kernel): a lane's 4 values of a k8 step are
  // 32 contiguous bytes, a warp's 1 KB -- two 16-byte loads instead of four 8-byte
  // gathers from four columns
  const int ks_n = mp / 8;
  const double2* qf = a.Qf ? reinterpret_cast<const double2*>(a.Qf) +
                                 ((size_t)warp * ks_n * 32 + lane) * 2
                           : nullptr;
  for (int k0 = 0; k0 < mp; k0 += 8 * U) {
    double q[U][4];
    if (qf) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int ks = k0 / 8 + u;
#ifdef ALNNLS_EXP_QFL1  // timing probe only: Q fragments from an L1-resident slice
        const int kl = ks & 3;
#else
        const int kl = ks;
#endif
        const double2 v0 = ks < ks_n ? __ldg(qf + (size_t)kl * 64) : make_double2(0.0, 0.0);
        const double2 v1 = ks < ks_n ? __ldg(qf + (size_t)kl * 64 + 1) : make_double2(0.0, 0.0);
        q[u][0] = v0.x;
        q[u][1] = v0.y;
        q[u][2] = v1.x;
        q[u][3] = v1.y;
      }
    } else {
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
      if (row < m) sm.U[(size_t)col * sm.ps + row] = acc[nt][c];
    }
}

// The same pass for NB = 8 columns on 8 warps (two 16-row tiles per warp, one
// 8-column n-tile, the two tiles' DMMAs interleaved): two CTAs per SM (m <= 256).
template <int LD>
__device__ __forceinline__ void dmma_gemm_pass8(const BatchArgs& a, const BatchSmem& sm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int m = sm.m, mp = sm.mp;
  const int r0 = warp * 32;  // rows [r0, r0 + 32): two 16-row tiles, interleaved
  if (r0 >= m) return;
  int ra[2], rb[2];
  bool va[2], vb[2];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    ra[mt] = r0 + 16 * mt + g;
    rb[mt] = ra[mt] + 8;
    va[mt] = ra[mt] < m;
    vb[mt] = rb[mt] < m;
  }
  double acc[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
  constexpr int U = 2;  // (two tiles x U k-steps of Q fragments in registers)
  for (int k0 = 0; k0 < mp; k0 += 8 * U) {
    double q[U][2][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k1 = k0 + 8 * u + t, k2 = k1 + 4;
      const double* c1 = a.Q + (size_t)k1 * m;
      const double* c2 = a.Q + (size_t)k2 * m;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        q[u][mt][0] = va[mt] && k1 < m ? __ldg(c1 + ra[mt]) : 0.0;
        q[u][mt][1] = vb[mt] && k1 < m ? __ldg(c1 + rb[mt]) : 0.0;
        q[u][mt][2] = va[mt] && k2 < m ? __ldg(c2 + ra[mt]) : 0.0;
        q[u][mt][3] = vb[mt] && k2 < m ? __ldg(c2 + rb[mt]) : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k1 = k0 + 8 * u + t;
      if (k0 + 8 * u >= mp) break;
      const double b0 = sm.V[(size_t)k1 * LD + g];
      const double b1 = sm.V[(size_t)(k1 + 4) * LD + g];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
        dmma8(acc[mt], q[u][mt][0], q[u][mt][1], q[u][mt][2], q[u][mt][3], b0, b1);
    }
  }
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int row = (c < 2 ? ra[mt] : rb[mt]);
      const int col = 2 * t + (c & 1);
      if (row < m) sm.U[(size_t)col * sm.ps + row] = acc[mt][c];
    }
}

__device__ __forceinline__ BatchSmem carve(double* bsm, int m, int nb) {
  BatchSmem sm;
  const int mp = round8(m);
  sm.ld = batch_ld(nb);
  sm.m = m;
  sm.mp = mp;
  sm.ps = panel_stride(m);
  sm.V = bsm;
  sm.U = bsm + (size_t)mp * sm.ld;
  sm.C = sm.U + (size_t)sm.ps * nb;
  sm.X = sm.C + (size_t)sm.ps * nb;
  sm.G = sm.X + (size_t)sm.ps * nb;
  sm.q = sm.G + (size_t)sm.ps * nb;
  const int total = mp * sm.ld + 5 * sm.ps * nb;  // zero once: pads must read as +0
  for (int e = threadIdx.x; e < total; e += blockDim.x) bsm[e] = 0.0;
  return sm;
}

// Every pass, all threads run the GEMM for all NB columns, then the per-column
// state machines advance in CTA-wide phases: elementwise work over (column, row)
// by all threads, the reference-ordered sums by one lane per column (so one
// DADD instruction advances every column's chain), the scalar decisions by the
// same lanes. (A warp-specialised variant -- 8 warps on the GEMM of one half of
// the columns while 8 run the other half's state machines -- measured slower in
// round 1; with 2 warps per scheduler the GEMM cannot hide the L2 latency of Q.)
// BT threads per CTA, MINB CTAs per SM. <16, 512, 1> up to m = 256; <8, 256, 2> is
// the same solver with two CTAs of 8 columns per SM: while one CTA runs its
// latency-bound state machines the other's GEMM pass keeps the FP64 / tensor pipes
// busy (the two interleave without explicit warp specialisation).
template <int NB, int BT, int MINB>
__global__ void __launch_bounds__(BT, MINB) batched_nqp_kernel(BatchArgs a) {
  extern __shared__ __align__(16) double bsm[];
  __shared__ ColState S;
  constexpr int LD = batch_ld(NB);
  const BatchSmem sm = carve(bsm, a.m, NB);
#ifdef ALNNLS_BATCH_PROF
  if (threadIdx.x < 8) S.pr[threadIdx.x] = 0;
#endif
  if (threadIdx.x < NB) {
    S.phase[threadIdx.x] = kIdle;
    S.act[threadIdx.x] = kActGrab;
    S.cnt[threadIdx.x] = 0;
    S.bad[threadIdx.x] = 0;
  }
  settle(a, S, sm, NB);
#ifndef ALNNLS_GEMM_CG
#define ALNNLS_GEMM_CG 8
#endif
  constexpr int CG = NB < ALNNLS_GEMM_CG ? NB : ALNNLS_GEMM_CG;  // columns per thread
  constexpr int GROUPS = NB / CG;
  constexpr int ROWT = BT / GROUPS;
  constexpr int MAXM = BT < 512 ? 256 : 4096 / NB;  // the largest m of this configuration
  constexpr int RPT = (MAXM + ROWT - 1) / ROWT;      // rows per thread at that m
  const int grp = threadIdx.x / ROWT, trow = threadIdx.x % ROWT;
#ifdef ALNNLS_BATCH_PROF
  long long t_g = 0, t_s = 0, npass = 0, nact = 0;
#endif
  for (;;) {
    int active = 0;
    for (int b = 0; b < NB; ++b) active |= S.phase[b] != kIdle;
    if (!active) break;
#ifdef ALNNLS_BATCH_PROF
    const long long c0 = clock64();
    for (int b = 0; b < NB; ++b) nact += S.phase[b] != kIdle;
    ++npass;
#endif
    if (NB == 16 && a.fast) {
      dmma_gemm_pass16<LD>(a, sm);
    } else if (NB == 8 && BT == 256 && a.fast) {  // (not launched: see launch_batched)
      dmma_gemm_pass8<LD>(a, sm);
    } else {
      gemm_pass<RPT, CG, ROWT, LD, ALNNLS_GEMM_JB, (BT == 128 && MINB == 2) ? ALNNLS_GEMM_QBUF : 2>(
          a, sm, grp, trow);
    }
    __syncthreads();
#ifdef ALNNLS_BATCH_PROF
    const long long c1 = clock64();
#endif
#ifndef ALNNLS_FAST_WARP_STATE
#define ALNNLS_FAST_WARP_STATE 1  // build knob: FAST state machines warp-local (NB = 16)
#endif
    if (ALNNLS_FAST_WARP_STATE && NB == 16 && BT == 512 && a.fast) {
      fast_warp_pass(a, S, sm);
#ifdef ALNNLS_BATCH_PROF
      if (threadIdx.x == 0) S.pr[0] += clock64() - c1;  // warp 0's own state machine
#endif
      __syncthreads();  // every column's V is ready for the next pass
    } else {
      after_pass(a, S, sm, NB);  // ends with every thread past the last settle barrier
    }
#ifdef ALNNLS_BATCH_PROF
    const long long c2 = clock64();
    t_g += c1 - c0;
    t_s += c2 - c1;
#endif
  }
#ifdef ALNNLS_BATCH_PROF
#ifdef ALNNLS_BATCH_PROF_ALL
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    printf("allcta %d sm %u passes %lld gemm %.1f state %.1f act %.2f end %lld\n", blockIdx.x, smid, npass,
           t_g / 1e3 / npass, t_s / 1e3 / npass, (double)nact / npass, clock64());
  }
#endif
  if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1))
    printf("batched prof cta %d: passes %lld, gemm %.1f kcyc/pass, state %.1f kcyc/pass, active cols/pass %.2f\n",
           blockIdx.x, npass, t_g / 1e3 / npass, t_s / 1e3 / npass, (double)nact / npass);
  if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1))
    printf("  cta %d per pass (kcyc): elem0 %.2f chain1 %.2f | rounds/pass %.2f: sync+check %.2f elem %.2f chain+decide %.2f\n",
           blockIdx.x, S.pr[0] / 1e3 / npass, S.pr[1] / 1e3 / npass, (double)S.pr[5] / npass,
           S.pr[2] / 1e3 / npass, S.pr[3] / 1e3 / npass, S.pr[4] / 1e3 / npass);
#endif
}


// ---------------------------------------------------------------------------------
// FAST, m <= 256: two CTAs of 16 columns per SM (batched_fast_kernel). One CTA's
// latency-bound state machines run while the other's DMMA pass keeps the tensor pipe
// busy. To fit two CTAs the per-column state is three vectors instead of six:
//  - VU (row-major mp x kFLD): the pass's input V, overwritten by its output U once
//    every warp has finished reading V; the state machine recomputes what V held
//    (g_bar from the mask, delta from alpha) with the arithmetic that produced it;
//  - X, G column panels; the candidate is recomputed at the accept (same operations,
//    same bits) and q comes from global memory (L2) at each stop test.
// Same sums, same trees, same decisions as the one-CTA FAST kernel: identical results.
constexpr int kFLD = 18;   // VU row stride (16 columns + 2: the column walks share banks 4-way)

struct FastSmem {
  double* VU;
  double* X;
  double* G;
  int m, mp, ps;
  __device__ double& vu(int i, int b) const { return VU[i * kFLD + b]; }
};
size_t fast_smem_bytes(int m) {
  return ((size_t)round8(m) * kFLD + 2 * (size_t)panel_stride(m) * 16) * sizeof(double);
}

// Candidate step of row i (nqp.hpp:294-303): delta (0 when the entry does not move)
// and the candidate value.
__device__ __forceinline__ void fast_cand(double alpha, double xi, double gi, double& c, double& d) {
  c = xi;
  d = 0.0;
  if (xi > 0.0 || gi < 0.0) {
    double t = xsub(xi, xmul(alpha, gi));
    if (t < 0.0) t = 0.0;
    if (t != xi) {
      c = t;
      d = xsub(t, xi);
    }
  }
}

// One column's state machine after a pass (or its first settle when !after), on one warp.
// Lane l owns rows l, l + 32, ... (at most 8: m <= 256), walked by fully unrolled loops
// at fixed offsets from per-lane base pointers, one loop per action: the state machine
// shares the SM's issue slots with the other CTA's DMMA pass, so its instruction count
// is what it costs. Per-lane sums in ascending row order, then the xor-shuffle tree.
#define FAST_ROWS(j) _Pragma("unroll") for (int j = 0; j < 8; ++j) if (j < nr)
__device__ void fast_col(const BatchArgs& a, ColState& S, const FastSmem& sm, int b, bool after) {
  const int lane = threadIdx.x & 31;
  const int m = sm.m;
#ifdef ALNNLS_BATCH_PROF
  long long t0 = clock64();
#define FPROF(k) { const long long t1 = clock64(); if (threadIdx.x == 0) S.pr[k] += t1 - t0; t0 = t1; }
#else
#define FPROF(k)
#endif
  const int nr = (m - lane + 31) >> 5;  // this lane's rows: lane + 32 j, j < nr
  double* xl = sm.X + (size_t)b * sm.ps + lane;
  double* gl = sm.G + (size_t)b * sm.ps + lane;
  double* vl = sm.VU + (size_t)lane * kFLD + b;
  constexpr int VS = 32 * kFLD;  // VU stride between a lane's rows
  if (after) {
    const int ph = S.phase[b];
    if (ph != kIdle) {
      double f = 0.0;
      if (ph == kNeedP1) {  // den = g_bar . (Q g_bar)
        FAST_ROWS(j) {
          const double xi = xl[32 * j], gi = gl[32 * j];
          const double gbar = (xi > 0.0 || gi < 0.0) ? gi : 0.0;
          f += gbar != 0.0 ? xmul(gbar, vl[VS * j]) : -0.0;
        }
      } else {  // df = (g + 0.5 Q delta) . delta (nqp.hpp:307)
        const double alpha = S.alpha[b];
        FAST_ROWS(j) {
          const double gi = gl[32 * j];
          double c, dd;
          fast_cand(alpha, xl[32 * j], gi, c, dd);
          f += dd != 0.0 ? xmul(xadd(gi, xmul(0.5, vl[VS * j])), dd) : -0.0;
        }
      }
      FPROF(0)
      f = warp_tree(f);
      FPROF(1)
      if (lane == 0) {
        if (ph == kNeedP1) {
          if (!(f > 0.0)) {
            S.term[b] = ALNNLS_ZERO_CURVATURE;
            S.act[b] = kActFinish;
          } else {
            S.alpha[b] = xdiv(S.gbs[b], f);
            S.tries[b] = 0;
            S.mults[b] += (unsigned long long)m * (unsigned long long)S.ml[b];
            S.act[b] = kActCand;
          }
        } else if (f <= 0.0 || S.tries[b] >= 60) {
          S.act[b] = kActAccept;
        } else {
          S.alpha[b] = xmul(S.alpha[b], 0.5);  // nqp.hpp:317
          ++S.tries[b];
          S.act[b] = kActCand;
        }
        S.cnt[b] = 0;
        S.bad[b] = 0;
      }
      __syncwarp();
      FPROF(2)
    }
  }
  for (;;) {
    const int act = S.act[b];
    if (act == kActNone) break;
#ifdef ALNNLS_BATCH_PROF
    t0 = clock64();
#endif
    int cnt = 0, bad = 0;
    double f0 = 0.0, f1 = 0.0, f2 = 0.0;
    // the stop-test terms of a row on the (new) state: mask, V = g_bar, the three sums
    auto stop_terms = [&](int j, double xi, double gi, double qi) {
      const bool p = xi > 0.0 || gi < 0.0;
      cnt += p;
      if (!isfinite(gi)) bad = 1;
      const double gbar = p ? gi : 0.0;
      vl[VS * j] = gbar;
      const bool xnz = xi != 0.0;
      f0 += xmul(gbar, gbar);
      f1 += xnz ? xmul(xi, gi) : -0.0;
      f2 += xnz ? xmul(xi, qi) : -0.0;
    };
    if (act == kActCand) {
      const double alpha = S.alpha[b];
      FAST_ROWS(j) {
        double c, d;
        fast_cand(alpha, xl[32 * j], gl[32 * j], c, d);
        cnt += d != 0.0;
        vl[VS * j] = d;
      }
      FPROF(3)
    } else if (act == kActAccept || act == kActMask || act == kActInit) {
      const double* ql = a.QB + (size_t)S.col[b] * m + lane;
      if (act == kActAccept) {  // nqp.hpp:309-313
        const double alpha = S.alpha[b];
        FAST_ROWS(j) {
          const double qi = __ldg(ql + 32 * j);
          const double go = gl[32 * j];
          double xi, d;
          fast_cand(alpha, xl[32 * j], go, xi, d);
          const double gi = xadd(go, vl[VS * j]);
          xl[32 * j] = xi;
          gl[32 * j] = gi;
          stop_terms(j, xi, gi, qi);
        }
      } else if (act == kActInit) {  // x = 0, grad = q (nqp.hpp:224-225)
        FAST_ROWS(j) {
          const double qi = __ldg(ql + 32 * j);
          xl[32 * j] = 0.0;
          gl[32 * j] = qi;
          stop_terms(j, 0.0, qi, qi);
        }
      } else {
        FAST_ROWS(j) stop_terms(j, xl[32 * j], gl[32 * j], __ldg(ql + 32 * j));
      }
      FPROF(4)
      f0 = warp_tree(f0);
      f1 = warp_tree(f1);
      f2 = warp_tree(f2);
      FPROF(5)
    } else {  // kActFinish / kActGrab
      if (act == kActFinish) {
        double* yl = a.Y + (size_t)S.col[b] * m + lane;
        FAST_ROWS(j) yl[32 * j] = xl[32 * j];
      }
      FAST_ROWS(j) vl[VS * j] = 0.0;  // idle slots feed zeros
    }
#ifdef ALNNLS_BATCH_PROF
    t0 = clock64();
#endif
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (lane == 0) {
      S.cnt[b] = cnt;
      if (bad) S.bad[b] = 1;
      if (act == kActAccept || act == kActMask || act == kActInit) {
        S.res[b][0] = f0;
        S.res[b][1] = f1;
        S.res[b][2] = f2;
        if (act == kActAccept) ++S.k[b];
      }
      round_decide(a, S, b);
      if (S.act[b] != kActNone) {
        S.cnt[b] = 0;
        S.bad[b] = 0;
      }
    }
    __syncwarp();
    FPROF(6)
  }
}
#undef FAST_ROWS

#ifndef ALNNLS_FAST2_U
#define ALNNLS_FAST2_U 1  // k8 steps whose Q fragments load together (two row tiles each); 1 measured best (0.566 s vs 0.605 U=2, 0.646 U=4 on the c4 loop)
#endif

// TPW row tiles of the pass and TPW columns per warp: 2 (8 warps) or 1 (16 warps, 64
// registers per thread).
template <int TPW>
__global__ void __launch_bounds__(512 / TPW, 2) batched_fast_kernel(BatchArgs a) {
  extern __shared__ __align__(16) double bsm[];
  __shared__ ColState S;
  FastSmem sm;
  sm.m = a.m;
  sm.mp = round8(a.m);
  sm.ps = panel_stride(a.m);
  sm.VU = bsm;
  sm.X = bsm + (size_t)sm.mp * kFLD;
  sm.G = sm.X + (size_t)sm.ps * 16;
  {
    const int total = sm.mp * kFLD + 2 * sm.ps * 16;  // pads must read as +0
    for (int e = threadIdx.x; e < total; e += blockDim.x) bsm[e] = 0.0;
  }
  if (threadIdx.x < 16) {
    S.phase[threadIdx.x] = kIdle;
    S.act[threadIdx.x] = kActGrab;
    S.cnt[threadIdx.x] = 0;
    S.bad[threadIdx.x] = 0;
  }
#ifdef ALNNLS_BATCH_PROF
  if (threadIdx.x < 8) S.pr[threadIdx.x] = 0;
#endif
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
#pragma unroll
  for (int c = 0; c < TPW; ++c) fast_col(a, S, sm, TPW * warp + c, false);
  __syncthreads();
  const int mp = sm.mp, m = sm.m;
  const int ks_n = mp / 8;
  constexpr int U = ALNNLS_FAST2_U;
  // fragment-ordered Q (qfrag_kernel): tile T = 2 warp + mt, k8 step ks, lane -> 4 doubles
  const double2* qf0 = reinterpret_cast<const double2*>(a.Qf) + ((size_t)(TPW * warp) * ks_n * 32 + lane) * 2;
  const bool rows_live = 16 * TPW * warp < m;
#ifdef ALNNLS_BATCH_PROF
  long long t_g = 0, t_s = 0, npass = 0, nact = 0;
#endif
  for (;;) {
    int active = 0;
    for (int b = 0; b < 16; ++b) active |= S.phase[b] != kIdle;
    if (!active) break;
#ifdef ALNNLS_BATCH_PROF
    const long long c0 = clock64();
    for (int b = 0; b < 16; ++b) nact += S.phase[b] != kIdle;
    ++npass;
#endif
    double acc[TPW][2][4];
#pragma unroll
    for (int mt = 0; mt < TPW; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[mt][nt][c] = 0.0;
    if (rows_live) {
      for (int k0 = 0; k0 < mp; k0 += 8 * U) {
        double q[U][TPW][4];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int ks = k0 / 8 + u;
          const bool in = ks < ks_n;
          const double2 z = make_double2(0.0, 0.0);
#pragma unroll
          for (int mt = 0; mt < TPW; ++mt) {
            const double2* qp = qf0 + ((size_t)mt * ks_n + ks) * 64;
            const double2 v0 = in ? __ldg(qp) : z;
            const double2 v1 = in ? __ldg(qp + 1) : z;
            q[u][mt][0] = v0.x;
            q[u][mt][1] = v0.y;
            q[u][mt][2] = v1.x;
            q[u][mt][3] = v1.y;
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int k1 = k0 + 8 * u + t;
          if (k0 + 8 * u >= mp) break;
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            const double b0 = sm.VU[(size_t)k1 * kFLD + 8 * nt + g];
            const double b1 = sm.VU[(size_t)(k1 + 4) * kFLD + 8 * nt + g];
#pragma unroll
            for (int mt = 0; mt < TPW; ++mt)
              dmma8(acc[mt][nt], q[u][mt][0], q[u][mt][1], q[u][mt][2], q[u][mt][3], b0, b1);
          }
        }
      }
    }
    __syncthreads();  // every warp has read V: U may take its place
    if (rows_live) {
#pragma unroll
      for (int mt = 0; mt < TPW; ++mt) {
        const int ra = 16 * (TPW * warp + mt) + g, rb = ra + 8;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const int col = 8 * nt + 2 * t;
          if (ra < m)
            *reinterpret_cast<double2*>(&sm.VU[(size_t)ra * kFLD + col]) =
                make_double2(acc[mt][nt][0], acc[mt][nt][1]);
          if (rb < m)
            *reinterpret_cast<double2*>(&sm.VU[(size_t)rb * kFLD + col]) =
                make_double2(acc[mt][nt][2], acc[mt][nt][3]);
        }
      }
    }
    __syncthreads();
#ifdef ALNNLS_BATCH_PROF
    const long long c1 = clock64();
#endif
#pragma unroll
    for (int c = 0; c < TPW; ++c) fast_col(a, S, sm, TPW * warp + c, true);
#ifdef ALNNLS_BATCH_PROF
    if (threadIdx.x == 0) S.pr[7] += clock64() - c1;
#endif
    __syncthreads();  // every column's V is ready for the next pass
#ifdef ALNNLS_BATCH_PROF
    const long long c2 = clock64();
    t_g += c1 - c0;
    t_s += c2 - c1;
#endif
  }
#ifdef ALNNLS_BATCH_PROF
  if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1))
    printf("fast2 prof cta %d: passes %lld, gemm %.1f kcyc/pass, state %.1f kcyc/pass, active cols/pass %.2f | warp 0 (2 cols) kcyc/pass: "
           "den/df loop %.2f tree %.2f decide %.2f cand %.2f accept loop %.2f trees %.2f lane0 %.2f own %.2f\n",
           blockIdx.x, npass, t_g / 1e3 / npass, t_s / 1e3 / npass, (double)nact / npass, S.pr[0] / 1e3 / npass,
           S.pr[1] / 1e3 / npass, S.pr[2] / 1e3 / npass, S.pr[3] / 1e3 / npass, S.pr[4] / 1e3 / npass,
           S.pr[5] / 1e3 / npass, S.pr[6] / 1e3 / npass, S.pr[7] / 1e3 / npass);
#endif
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
// branch-free. 128 threads, each an 8 x 4 block of the tile (rows 2 tx + 16 r + {0, 1},
// columns 4 ty + c), its operands read as six 16-byte shared loads per k (four of A, two
// of X) for 64 FP64 instructions: the 4 x 4 / 8-byte-load form needed as many LSU
// cycles as FP64 cycles per k and ran at half the exact cap. The next k-slab of A and X
// is loaded into registers while the current one is multiplied.
constexpr int kRT = 64;   // rows per tile
constexpr int kRC = 64;   // columns per CTA
constexpr int kRK = 16;   // k slab
constexpr int kRThreads = 128;
__global__ void __launch_bounds__(kRThreads) residual_batched_kernel(const double* A, uint64_t lda,
                                                                     int d, int n, const double* X,
                                                                     const double* B, uint64_t ldb,
                                                                     int ncols,
                                                                     alnnls_column_result* res) {
  // the slab buffers and the finished tile share one static buffer (< 48 KB)
  __shared__ __align__(16) double sbuf[kRT * (kRC + 1)];
  double(*As)[kRK][kRT] = reinterpret_cast<double(*)[kRK][kRT]>(sbuf);
  double(*Xs)[kRK][kRC] = reinterpret_cast<double(*)[kRK][kRC]>(sbuf + 2 * kRK * kRT);
  double(*Cs)[kRC + 1] = reinterpret_cast<double(*)[kRC + 1]>(sbuf);
  static_assert(2 * kRK * (kRT + kRC) <= kRT * (kRC + 1), "slab buffers fit the tile buffer");
  const int c0 = blockIdx.x * kRC;
  const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;
  const int nslab = (n + kRK - 1) / kRK;
  double ssum = 0.0;  // thread t < kRC: the running chain of column c0 + t
  constexpr int NF = kRT * kRK / kRThreads;  // slab loader: 8 A and 8 X elements per thread
  auto fetch = [&](int i0, int k0, double (&ra)[NF], double (&rx)[NF]) {
#pragma unroll
    for (int u = 0; u < NF; ++u) {
      const int e = threadIdx.x + kRThreads * u;
      const int kk = e / kRT, r = e % kRT;
      const int i = i0 + r, kcol = k0 + kk;
      ra[u] = (i < d && kcol < n) ? __ldg(A + (size_t)kcol * lda + i) : 0.0;
      const int c = e / kRK, kx = e % kRK;
      const int col = c0 + c, kc2 = k0 + kx;
      rx[u] = (col < ncols && kc2 < n) ? __ldg(X + (size_t)col * n + kc2) : 0.0;
    }
  };
  auto stash = [&](int buf, const double (&ra)[NF], const double (&rx)[NF]) {
#pragma unroll
    for (int u = 0; u < NF; ++u) {
      const int e = threadIdx.x + kRThreads * u;
      As[buf][e / kRT][e % kRT] = ra[u];
      Xs[buf][e % kRK][e / kRK] = rx[u];
    }
  };
  for (int i0 = 0; i0 < d; i0 += kRT) {
    double acc[8][4];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;
    double ra[NF], rx[NF];
    fetch(i0, 0, ra, rx);
    stash(0, ra, rx);
    __syncthreads();
    for (int sl = 0; sl < nslab; ++sl) {
      const int buf = sl & 1;
      if (sl + 1 < nslab) fetch(i0, (sl + 1) * kRK, ra, rx);
#pragma unroll
      for (int kk = 0; kk < kRK; ++kk) {
        double av[8], xv[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const double2 t2 = *reinterpret_cast<const double2*>(&As[buf][kk][2 * tx + 16 * r]);
          av[2 * r] = t2.x;
          av[2 * r + 1] = t2.y;
        }
#pragma unroll
        for (int c = 0; c < 4; c += 2) {
          const double2 t2 = *reinterpret_cast<const double2*>(&Xs[buf][kk][4 * ty + c]);
          xv[c] = t2.x;
          xv[c + 1] = t2.y;
        }
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[r][c] = xmac(acc[r][c], av[r], xv[c]);
      }
      if (sl + 1 < nslab) stash(buf ^ 1, ra, rx);
      __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) Cs[2 * tx + 16 * (r >> 1) + (r & 1)][4 * ty + c] = acc[r][c];
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

// Q (m x m, column-major) into the DMMA fragment order of dmma_gemm_pass16: for warp
// w (rows 16w..16w+15), k8 step ks and lane (g = lane / 4, t = lane % 4) the four
// values Q(16w+g, 8ks+t), Q(16w+g+8, 8ks+t), Q(16w+g, 8ks+t+4), Q(16w+g+8, 8ks+t+4),
// zero outside m x m. Same values, same DMMA operands: the pass's result is unchanged.
__global__ void qfrag_kernel(const double* Q, int m, int mp, double* Qf) {
  const int ks_n = mp / 8;
  const int total = 16 * ks_n * 32;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const int lane = e & 31, ks = (e >> 5) % ks_n, w = (e >> 5) / ks_n;
    const int g = lane >> 2, t = lane & 3;
    const int ra = 16 * w + g, rb = ra + 8, k1 = 8 * ks + t, k2 = k1 + 4;
    double* o = Qf + (size_t)e * 4;
    o[0] = ra < m && k1 < m ? Q[(size_t)k1 * m + ra] : 0.0;
    o[1] = rb < m && k1 < m ? Q[(size_t)k1 * m + rb] : 0.0;
    o[2] = ra < m && k2 < m ? Q[(size_t)k2 * m + ra] : 0.0;
    o[3] = rb < m && k2 < m ? Q[(size_t)k2 * m + rb] : 0.0;
  }
}

#ifndef ALNNLS_BATCH_2CTA
#define ALNNLS_BATCH_2CTA 1  // build knob: m <= 256 runs two 8-column CTAs per SM
#endif

cudaError_t launch_qfrag(const BatchArgs& a, cudaStream_t stream) {
  qfrag_kernel<<<64, 256, 0, stream>>>(a.Q, a.m, round8(a.m), a.Qf);
  return cudaGetLastError();
}

cudaError_t launch_batched(const BatchArgs& a, int sm_count, cudaStream_t stream) {
  const int NB = batched_cols_per_cta(a.m);
  if (NB == 0) return cudaErrorInvalidValue;
  {
    const int mx = (int)batch_smem_bytes(1024, 4);  // the largest configuration
    if (cudaError_t e = smem_optin(batched_nqp_kernel<16, kBT, 1>, mx)) return e;
    if (cudaError_t e = smem_optin(batched_nqp_kernel<8, kBT, 1>, mx)) return e;
    if (cudaError_t e = smem_optin(batched_nqp_kernel<4, kBT, 1>, mx)) return e;
    if (cudaError_t e = smem_optin(batched_nqp_kernel<8, 256, 2>, (int)batch_smem_bytes(256, 8)))
      return e;
    if (cudaError_t e = smem_optin(batched_nqp_kernel<8, 128, 2>, (int)batch_smem_bytes(256, 8)))
      return e;
  }
  // EXACT, m <= 256: two CTAs of 8 columns per SM (c4 65536 columns: loop 1.545 ->
  // 1.498 s). FAST keeps one 16-column CTA: its DMMA pass shares each Q fragment
  // between two n-tiles there, and the 8-column pass (dmma_gemm_pass8) loading Q
  // twice as often measured 0.862 -> 1.113 s.
  if (ALNNLS_BATCH_2CTA && NB == 16 && !a.fast) {
    const size_t smem = batch_smem_bytes(a.m, 8);
    int grid = 2 * sm_count;
    const int need = (a.ncols + 7) / 8;
    if (grid > need) grid = need;
    if (grid < 1) grid = 1;
    // 128 threads, each 2 rows x 8 columns of the GEMM (half the V and Q load instructions
    // per FP64 operation of the 256-thread, 1 x 8 form): 65536-column loop 1.487 -> 1.461 s.
    // ALNNLS_BATCH_BT=256 keeps the 256-thread CTAs for A/B runs.
    const char* bt = getenv("ALNNLS_BATCH_BT");
    if (bt && atoi(bt) == 256) batched_nqp_kernel<8, 256, 2><<<grid, 256, smem, stream>>>(a);
    else batched_nqp_kernel<8, 128, 2><<<grid, 128, smem, stream>>>(a);
    return cudaGetLastError();
  }
  const size_t smem = batch_smem_bytes(a.m, NB);
  int grid = sm_count;
  const int need = (a.ncols + NB - 1) / NB;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  BatchArgs b = a;
  if (NB == 16 && a.fast && a.Qf) {
    if (!a.qf_ready)
      if (cudaError_t e = launch_qfrag(a, stream)) return e;
    // Two 16-column CTAs per SM whenever the batch has more than one CTA per SM to fill
    // (loop, one-CTA vs two-CTA kernel: 4096 columns 0.0623 vs 0.0558 s, 8192 0.1045 vs
    // 0.0983, 16384 0.189 vs 0.164, 32768 0.355 vs 0.299, 65536 0.689 vs 0.566); below
    // that the grids are the same and the one-CTA kernel stays.
    // ALNNLS_FAST_2CTA=0 / 1 forces either for A/B runs.
    const char* two = getenv("ALNNLS_FAST_2CTA");
    const int tot = a.total_cols > a.ncols ? a.total_cols : a.ncols;
    const bool use2 = two ? atoi(two) != 0 : tot > 16 * sm_count;
    if (use2) {
      const size_t fsm = fast_smem_bytes(a.m);
      if (cudaError_t e = smem_optin(batched_fast_kernel<1>, (int)fast_smem_bytes(256))) return e;
      if (cudaError_t e = smem_optin(batched_fast_kernel<2>, (int)fast_smem_bytes(256))) return e;
      int fgrid = 2 * sm_count;
      if (fgrid > need) fgrid = need;
      const char* tpw = getenv("ALNNLS_FAST_TPW");
      if (tpw && atoi(tpw) == 2) batched_fast_kernel<2><<<fgrid, 256, fsm, stream>>>(b);
      else batched_fast_kernel<1><<<fgrid, 512, fsm, stream>>>(b);
      return cudaGetLastError();
    }
  } else {
    b.Qf = nullptr;
  }
  if (NB == 16) batched_nqp_kernel<16, kBT, 1><<<grid, kBT, smem, stream>>>(b);
  else if (NB == 8) batched_nqp_kernel<8, kBT, 1><<<grid, kBT, smem, stream>>>(b);
  else batched_nqp_kernel<4, kBT, 1><<<grid, kBT, smem, stream>>>(b);
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
  residual_batched_kernel<<<(ncols + kRC - 1) / kRC, kRThreads, 0, stream>>>(A, lda, d, n, X, B,
                                                                                ldb, ncols, res);
  return cudaGetLastError();
}

}  // namespace alnnls
