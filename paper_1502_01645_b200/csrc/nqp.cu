// nqp.cu — exact device-resident projected-gradient loop (K4-K6).
//
// Restates reference solve_nqp (/root/reference/proj/include/antilop/nqp.hpp:
// 215-339) as ONE persistent cooperative kernel: no host round trip per
// iteration; the passive mask, step, halving decision, stop tests, stall
// counter, trace records and multiply counts all live in device memory.
//
// Grid: CTA 0 is the "vector" CTA (all O(m) phases, sequential chains);
// CTAs 1..B each own a row block of the blocked Q (gemv.cuh) for the two
// masked GEMVs. Per iteration k:
//
//   P1   row CTAs: u = Q[:, P] g_P
//        vector CTA, concurrently: gbs, x.g, q.x chains (nqp.hpp:251-254),
//        f, stop tests, stall counter (nqp.hpp:257-275)                     -> barrier
//   D/C  vector CTA: den chain, alpha (exact_step, nqp.hpp:162-173), candidate
//        max(0, x - alpha g) and the changed set C (nqp.hpp:294-303)        -> barrier
//   P2   row CTAs: gd = Q[:, C] delta_C (nqp.hpp:305)        -> (own rows only)
//   F/U  row CTAs: g_next = g + gd on own rows (ping-pong buffer, so doing it
//        before the decision is safe); vector CTA: df chain (nqp.hpp:307),
//        accept -> x[C] = cand, next passive mask from g + gd, trace record;
//        reject -> alpha/2 and a new C (nqp.hpp:316-317)                    -> barrier
//
// Every sum is one sequential chain in the reference order: the vector CTA
// forms the rounded products in parallel into shared memory and one thread
// runs the dependent DADD chain, so the trajectory is bitwise the reference's.
#include <cooperative_groups.h>
#include <cstdlib>

#include "common.cuh"
#include "gemv.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace alnnls {

namespace {

#ifndef ALNNLS_RESIDENT_Q
#define ALNNLS_RESIDENT_Q 1  // build knob: Q panels resident in shared memory when they fit
#endif

#ifndef ALNNLS_P1_PREFETCH
#define ALNNLS_P1_PREFETCH 384  // build knob: columns of the next P1 prefetched into L2 after P2
                                // (c2 79.3 -> 78.7, c3 91.0 -> 90.3 us/iteration; 1536 slower)
#endif

#ifndef ALNNLS_CHAIN_CH
#define ALNNLS_CHAIN_CH 1024  // build knob: vector-CTA chain chunk (products per buffer)
#endif

constexpr int kLoopThreads = 384;  // 168 registers/thread at one CTA per SM: no spills
constexpr int kWarps = kLoopThreads / 32;
enum LoopState { kStateP2 = 1, kStateNoMove = 2, kStateNext = 3, kStateStop = 4 };

struct LeaderState {
  double best_gbs;
  unsigned long long since_best;
  double gbs, xg, qx, f;
  double elapsed;
  double alpha;
  double res[4];
  unsigned long long mults;
  int nonfinite;
  int tries;
  int mask_len;
  int act;  // phase-A decision (LoopAct), for the whole vector CTA
  unsigned long long t_mark;
  unsigned long long ph[8];
  double red[kWarps];
  int scan[40];
  int cnt[8 * kWarps + 1];  // kU x kWarps warp counts / offsets + total
};

__device__ __forceinline__ void chunk(int len, int& lo, int& hi) {
  const int nt = blockDim.x;
  const int per = (len + nt - 1) / nt;
  lo = min(len, (int)threadIdx.x * per);
  hi = min(len, lo + per);
}

__device__ __forceinline__ void phase_mark(LeaderState& L, int idx) {
  const unsigned long long t = globaltimer_ns();
  L.ph[idx] += t - L.t_mark;
  L.t_mark = t;
}

// One thread: s = ((s + p0) + p1) + ... over n products in shared memory.
// Two register blocks alternate (no register copies): the 16-byte loads of the
// next block issue ahead of the current block's chain, so the dependent DADD
// (8 cycles on B200) is the only thing on the critical path.
__device__ __forceinline__ double smem_chain(double s, const double* __restrict__ p, int n) {
  constexpr int B = 16;
  int t = 0;
  auto load = [&](double (&r)[B], int at) {
#pragma unroll
    for (int k = 0; k < B; k += 2) {
      const double2 d = *reinterpret_cast<const double2*>(p + at + k);
      r[k] = d.x;
      r[k + 1] = d.y;
    }
  };
  if (n >= 2 * B) {
    double ra[B], rb[B];
    load(ra, 0);
    for (; t + 3 * B <= n; t += 2 * B) {
      load(rb, t + B);
#pragma unroll
      for (int k = 0; k < B; ++k) s = xadd(s, ra[k]);
      load(ra, t + 2 * B);
#pragma unroll
      for (int k = 0; k < B; ++k) s = xadd(s, rb[k]);
    }
    // ra holds [t, t + B); t + B <= n < t + 3B
    if (t + 2 * B <= n) {
      load(rb, t + B);
#pragma unroll
      for (int k = 0; k < B; ++k) s = xadd(s, ra[k]);
#pragma unroll
      for (int k = 0; k < B; ++k) s = xadd(s, rb[k]);
      t += 2 * B;
    } else {
#pragma unroll
      for (int k = 0; k < B; ++k) s = xadd(s, ra[k]);
      t += B;
    }
  }
  while (t < n) {  // < 2B left: blocks of B with predicated loads
    double r[B];
#pragma unroll
    for (int k = 0; k < B; ++k) r[k] = t + k < n ? p[t + k] : 0.0;
#pragma unroll
    for (int k = 0; k < B; ++k)
      if (t + k < n) s = xadd(s, r[k]);
    t += B;
  }
  return s;
}

// Variant with one register block copied forward (the phase-A chains run hidden
// behind P1; this form keeps the loop kernel's row-CTA code faster, measured).
__device__ __forceinline__ double smem_chain_db(double s, const double* __restrict__ p, int n) {
  constexpr int B = 16;
  int t = 0;
  if (n >= 2 * B) {
    double cur[B], nx[B];
#pragma unroll
    for (int k = 0; k < B; k += 2) {
      const double2 d = *reinterpret_cast<const double2*>(p + k);
      cur[k] = d.x;
      cur[k + 1] = d.y;
    }
    for (; t + 2 * B <= n; t += B) {
#pragma unroll
      for (int k = 0; k < B; k += 2) {
        const double2 d = *reinterpret_cast<const double2*>(p + t + B + k);
        nx[k] = d.x;
        nx[k + 1] = d.y;
      }
#pragma unroll
      for (int k = 0; k < B; ++k) s = xadd(s, cur[k]);
#pragma unroll
      for (int k = 0; k < B; ++k) cur[k] = nx[k];
    }
#pragma unroll
    for (int k = 0; k < B; ++k) s = xadd(s, cur[k]);
    t += B;
  }
  for (; t < n; ++t) s = xadd(s, p[t]);
  return s;
}

// K concurrent ordered chains over len positions, products prod(k, t) formed
// in parallel by warps K..15 into double-buffered shared-memory chunks while
// lane 0 of warps 0..K-1 runs the chains. Whole vector CTA; results in L.res.
template <int K, class F>
__device__ void leader_chains(double* sbuf, size_t sbuf_bytes, LeaderState& L, int len, F prod) {
  // small chunks so the chain starts after the first 1024 products are formed
  const int CH = min(ALNNLS_CHAIN_CH, (int)(sbuf_bytes / (2 * K * sizeof(double))) & ~1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = (len + CH - 1) / CH;
  // 4 positions per thread per round: all their operand loads are in flight
  // together before the first shared-memory store
  auto produce = [&](int c, int buf, int first_thread) {
    const int b0 = c * CH;
    const int cnt = min(CH, len - b0);
    double* dst = sbuf + (size_t)buf * K * CH;
    const int nthr = (int)blockDim.x - first_thread;
    for (int i = (int)threadIdx.x - first_thread; i < cnt; i += 4 * nthr) {
      double v[4][K];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int k = 0; k < K; ++k) v[u][k] = i + u * nthr < cnt ? prod(k, b0 + i + u * nthr) : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int k = 0; k < K; ++k)
          if (i + u * nthr < cnt) dst[(size_t)k * CH + i + u * nthr] = v[u][k];
    }
  };
  double s = 0.0;
  if (nch > 0) produce(0, 0, 0);
  __syncthreads();
  for (int c = 0; c < nch; ++c) {
    if (warp < K) {
      if (lane == 0) {
        const int cnt = min(CH, len - c * CH);
        s = smem_chain(s, sbuf + (size_t)(c & 1) * K * CH + (size_t)warp * CH, cnt);
      }
    } else if (c + 1 < nch) {
      produce(c + 1, (c + 1) & 1, K * 32);
    }
    __syncthreads();
  }
  if (warp < K && lane == 0) L.res[warp] = s;
  __syncthreads();
}

// Ordered block compaction: positions are processed in super-rounds of kU
// rounds x blockDim consecutive positions (thread t takes r*blockDim + t), so a
// warp's selected entries land at consecutive output positions (coalesced
// stores); order = ascending position. Warp counts of the kU rounds are
// scanned together by warp 0.
constexpr int kU = 8;
constexpr int kSuper = kLoopThreads * kU;

__device__ __forceinline__ int super_scan(LeaderState& L) {
  __syncthreads();
  if (threadIdx.x < 32) {
    constexpr int N = kU * kWarps;
    constexpr int PER = (N + 31) / 32;
    const int lane = threadIdx.x;
    int v[PER], s = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int idx = lane * PER + j;
      v[j] = idx < N ? L.cnt[idx] : 0;
      s += v[j];
    }
    int incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    int ex = incl - s;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int idx = lane * PER + j;
      if (idx < N) {
        L.cnt[idx] = ex;
        ex += v[j];
      }
    }
    if (lane == 31) L.cnt[N] = incl;
  }
  __syncthreads();
  return L.cnt[kU * kWarps];
}

// Candidate step on the mask and the changed set C (nqp.hpp:294-303).
struct ListSet;
__device__ void leader_build_changed(const LoopArgs& a, LeaderState& L, int ml, double alpha,
                                     const struct ListSet& ls);
__device__ void leader_build_changed_impl(const LoopArgs& a, LeaderState& L, int ml, double alpha,
                                          const uint32_t* mask, const double* gP, const double* xP) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  int base = 0;
  for (int s0 = 0; s0 < ml; s0 += kSuper) {
    double xv[kU], gv[kU], cv[kU];
    uint32_t iv[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const int t = s0 + k * kLoopThreads + threadIdx.x;
      xv[k] = 0.0;
      gv[k] = 0.0;
      iv[k] = 0;
      if (t < ml) {
        xv[k] = xP[t];
        gv[k] = gP[t];
        iv[k] = mask[t];
      }
    }
    unsigned sel = 0, wp[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const bool valid = s0 + k * kLoopThreads + (int)threadIdx.x < ml;
      double xi = xsub(xv[k], xmul(alpha, gv[k]));  // x - (alpha g), nqp.hpp:296
      if (xi < 0.0) xi = 0.0;
      cv[k] = xi;
      const bool f = valid && xi != xv[k];
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      wp[k] = __popc(bal & lt);
      if (lane == 0) L.cnt[k * kWarps + warp] = __popc(bal);
      if (f) sel |= 1u << k;
    }
    const int total = super_scan(L);
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      if (sel & (1u << k)) {
        const int pos = base + L.cnt[k * kWarps + warp] + (int)wp[k];
        a.chg[pos] = iv[k];
        a.candC[pos] = cv[k];
        a.dC[pos] = xsub(cv[k], xv[k]);
        a.gC[pos] = gv[k];
      }
    }
    base += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    a.ctrl->chg_len = base;
    if (base > 0) L.mults += (unsigned long long)a.m * (unsigned long long)base;
  }
  __syncthreads();
}

__device__ void write_record(const LoopArgs& a, unsigned long long k, double f, double gbs,
                             int pc, double elapsed, double alpha, int has_alpha) {
  LoopCtrl* c = a.ctrl;
  const unsigned long long idx = c->trace_len;
  if (a.trace_cap > 0) {  // past the capacity the last slot keeps the newest record
    alnnls_iter_record r;
    r.iter = k;
    r.f = f;
    r.grad_bar_sq = gbs;
    r.passive_count = (uint64_t)pc;
    r.elapsed_s = elapsed;
    r.alpha = has_alpha ? alpha : 0.0;
    r.has_alpha = has_alpha;
    a.trace[idx < a.trace_cap ? idx : a.trace_cap - 1] = r;
  }
  c->trace_len = idx + 1;
}

// Stepped-iteration bookkeeping (nqp.hpp:319-326). Vector CTA thread 0.
__device__ void push_step(const LoopArgs& a, unsigned long long k, double f, double gbs, int ml,
                          double el, double alpha, unsigned long long mults) {
  if (k % a.trace_every == 0) write_record(a, k, f, gbs, ml, el, alpha, 1);
  const unsigned long long idx = a.ctrl->mult_len;
  if (a.mults && idx < a.mults_cap) a.mults[idx] = mults;
  a.ctrl->mult_len = idx + 1;
  a.ctrl->mult_total += mults;
}

__device__ void stop_final(const LoopArgs& a, unsigned long long k, double f, double gbs, int ml,
                           double el, int term) {
  write_record(a, k, f, gbs, ml, el, 0.0, 0);
  a.ctrl->termination = term;
  a.ctrl->iterations = k;
  a.ctrl->f_final = f;
  a.ctrl->gbs_final = gbs;
}

// ---- row-CTA phases: own x and g, build the passive-mask lists in parallel ----------
struct ListSet {
  uint32_t* mask;
  double* gP;
  double* xP;
  double* qP;
};

__device__ void leader_build_changed(const LoopArgs& a, LeaderState& L, int ml, double alpha,
                                     const ListSet& ls) {
  leader_build_changed_impl(a, L, ml, alpha, ls.mask, ls.gP, ls.xP);
}

struct RowShared {
  int wc[kWarps + 1];
  double wm[kWarps];
  int t_lo, t_hi, base, total;
  int lpos[2][kLoopThreads];  // passive-list position of each own row (-1: not passive), per list parity
};

// Passive flags of own rows of (x, g): count -> cnt[b], min(x) -> minx[b],
// any non-finite g -> badv[b]. Whole row CTA.
__device__ void row_count(const LoopArgs& a, RowShared& S, int blk, int row0, int nrows,
                          const double* x, const double* g) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int c = 0, bad = 0;
  double mn = __longlong_as_double(0x7ff0000000000000LL);
  for (int t = threadIdx.x; t < nrows; t += blockDim.x) {
    const double xi = x[row0 + t], gi = g[row0 + t];
    c += (xi > 0.0 || gi < 0.0) ? 1 : 0;
    if (!isfinite(gi)) bad = 1;
    mn = fmin(mn, xi);
  }
  for (int o = 16; o > 0; o >>= 1) {
    c += __shfl_xor_sync(0xffffffffu, c, o);
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  }
  if (lane == 0) {
    S.wc[warp] = c;
    S.wm[warp] = mn;
  }
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    int tot = 0;
    double m2 = __longlong_as_double(0x7ff0000000000000LL);
    for (int w = 0; w < kWarps; ++w) {
      tot += S.wc[w];
      m2 = fmin(m2, S.wm[w]);
    }
    a.cnt[blk] = tot;
    a.minx[blk] = m2;
    a.badv[blk] = bad;
  }
}

// Speculative update of own rows (nqp.hpp:309-313): x_next = x with x[C] = cand,
// g_next = g + gd; then row_count on the result.
// Own range [t_lo, t_hi) of the ascending changed list, by ONE warp (an idle
// warp of the P2 GEMV runs it while the GEMV streams Q): a 32-ary sample, then a
// scan of the bucket holding each bound.
__device__ void own_changed_range(const LoopArgs& a, RowShared& S, int row0, int nrows, int cl) {
  const int lane = threadIdx.x & 31;
  const int step = (cl + 31) / 32;
  const int v = lane * step < cl ? (int)__ldcg(a.chg + lane * step) : 0x7fffffff;
  const int c_lo = __popc(__ballot_sync(0xffffffffu, v < row0));
  const int c_hi = __popc(__ballot_sync(0xffffffffu, v < row0 + nrows));
  const int b_lo = max(0, c_lo - 1) * step, b_hi = max(0, c_hi - 1) * step;
  int n_lo = 0, n_hi = 0;
  for (int j0 = 0; j0 < step; j0 += 32) {
    const int j = j0 + lane;
    const int w1 = j < step && b_lo + j < cl ? (int)__ldcg(a.chg + b_lo + j) : 0x7fffffff;
    const int w2 = j < step && b_hi + j < cl ? (int)__ldcg(a.chg + b_hi + j) : 0x7fffffff;
    n_lo += __popc(__ballot_sync(0xffffffffu, w1 < row0));
    n_hi += __popc(__ballot_sync(0xffffffffu, w2 < row0 + nrows));
  }
  if (lane == 0) {
    S.t_lo = c_lo == 0 ? 0 : b_lo + n_lo;
    S.t_hi = c_hi == 0 ? 0 : b_hi + n_hi;
  }
}

// have_range: own_changed_range already ran (during the P2 GEMV).
__device__ void row_apply(const LoopArgs& a, RowShared& S, int blk, int row0, int nrows,
                          const double* xc, const double* gc, double* xn, double* gn, int cl,
                          bool have_range = false) {
  for (int t = threadIdx.x; t < nrows; t += blockDim.x) {
    const int i = row0 + t;
    gn[i] = xadd(gc[i], a.gd[i]);
    xn[i] = xc[i];
  }
  // own range [t_lo, t_hi) of the ascending changed list: a two-round
  // blockDim-ary search (two L2 round trips instead of a 2 log2(cl)-deep chain)
  if (!have_range) {
    const int nt = blockDim.x;
    const int step = (cl + nt - 1) / nt;  // round 1 samples chg[0], chg[step], ...
    const int i = threadIdx.x * step;
    const int v = i < cl ? (int)__ldcg(a.chg + i) : 0x7fffffff;
    const int c_lo = __syncthreads_count(v < row0);          // samples below row0
    const int c_hi = __syncthreads_count(v < row0 + nrows);
    // the boundary lies in (sample c-1, sample c]: scan that bucket
    const int b_lo = max(0, c_lo - 1) * step, b_hi = max(0, c_hi - 1) * step;
    const int j = threadIdx.x;
    const int w1 = j < step && b_lo + j < cl ? (int)__ldcg(a.chg + b_lo + j) : 0x7fffffff;
    const int w2 = j < step && b_hi + j < cl ? (int)__ldcg(a.chg + b_hi + j) : 0x7fffffff;
    const int n_lo = __syncthreads_count(j < step && b_lo + j < cl && w1 < row0);
    const int n_hi = __syncthreads_count(j < step && b_hi + j < cl && w2 < row0 + nrows);
    if (threadIdx.x == 0) {
      S.t_lo = c_lo == 0 ? 0 : b_lo + n_lo;
      S.t_hi = c_hi == 0 ? 0 : b_hi + n_hi;
    }
  }
  __syncthreads();
  for (int t = S.t_lo + threadIdx.x; t < S.t_hi; t += blockDim.x) {
    const uint32_t j = __ldcg(a.chg + t);
    xn[j] = __ldcg(a.candC + t);
    a.gdC[t] = a.gd[j];  // own rows of P2's result, compacted for the next df chain
  }
  __syncthreads();
  row_count(a, S, blk, row0, nrows, xn, gn);
}

// Writes own rows' entries of the ascending passive list at the global offset
// sum(cnt[0..blk)). Returns the list length (sum of all cnt). Whole row CTA.
__device__ int row_lists(const LoopArgs& a, RowShared& S, int blk, int nblk, int row0, int nrows,
                         const double* x, const double* g, const ListSet& L, int par) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
    int before = 0, all = 0;
    int cv[6];  // nblk <= 192: all loads in flight together
#pragma unroll
    for (int r = 0; r < 6; ++r) cv[r] = lane + 32 * r < nblk ? __ldcg(a.cnt + lane + 32 * r) : 0;
#pragma unroll
    for (int r = 0; r < 6; ++r) {
      all += cv[r];
      if (lane + 32 * r < blk) before += cv[r];
    }
    for (int o = 16; o > 0; o >>= 1) {
      before += __shfl_xor_sync(0xffffffffu, before, o);
      all += __shfl_xor_sync(0xffffffffu, all, o);
    }
    if (lane == 0) {
      S.base = before;
      S.total = all;
    }
  }
  // one round: nrows <= blockDim.x (checked on the host)
  const int t = threadIdx.x;
  double xi = 0.0, gi = 0.0;
  bool f = false;
  if (t < nrows) {
    xi = x[row0 + t];
    gi = g[row0 + t];
    f = xi > 0.0 || gi < 0.0;
  }
  const unsigned bal = __ballot_sync(0xffffffffu, f);
  if (lane == 0) S.wc[warp] = __popc(bal);
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = S.base;
    for (int w = 0; w < kWarps; ++w) {
      const int c = S.wc[w];
      S.wc[w] = run;
      run += c;
    }
  }
  __syncthreads();
  if (f) {
    const int pos = S.wc[warp] + __popc(bal & ((1u << lane) - 1u));
    L.mask[pos] = (uint32_t)(row0 + t);
    L.gP[pos] = gi;
    L.xP[pos] = xi;
    L.qP[pos] = __ldg(a.q + row0 + t);
    S.lpos[par][t] = pos;
  } else if (t < nrows) {
    S.lpos[par][t] = -1;
  }
  return S.total;
}

// ---- vector-CTA chains with per-chain lengths ------------------------------------------
template <int K, class F>
__device__ void leader_chains_var(double* sbuf, size_t sbuf_bytes, LeaderState& L,
                                  const int (&len)[K], F prod) {
  const int CH = min(ALNNLS_CHAIN_CH, (int)(sbuf_bytes / (2 * K * sizeof(double))) & ~1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int mx = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) mx = max(mx, len[k]);
  const int nch = (mx + CH - 1) / CH;
  auto produce = [&](int c, int buf, int first_thread) {
    const int b0 = c * CH;
    double* dst = sbuf + (size_t)buf * K * CH;
    const int nthr = (int)blockDim.x - first_thread;
    for (int i = (int)threadIdx.x - first_thread; i < CH; i += 2 * nthr) {
      double v[2][K];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int ii = i + u * nthr;
          v[u][k] = ii < CH && b0 + ii < len[k] ? prod(k, b0 + ii) : 0.0;
        }
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int ii = i + u * nthr;
          if (ii < CH && b0 + ii < len[k]) dst[(size_t)k * CH + ii] = v[u][k];
        }
    }
  };
  double s = 0.0;
  if (nch > 0) produce(0, 0, 0);
  __syncthreads();
  for (int c = 0; c < nch; ++c) {
    if (warp < K) {
      if (lane == 0) {
        const int cnt = max(0, min(CH, len[warp] - c * CH));
        s = smem_chain_db(s, sbuf + (size_t)(c & 1) * K * CH + (size_t)warp * CH, cnt);
      }
    } else if (c + 1 < nch) {
      produce(c + 1, (c + 1) & 1, K * 32);
    }
    __syncthreads();
  }
  if (warp < K && lane == 0) L.res[warp] = s;
  __syncthreads();
}

enum LoopAct { kActCont = 1, kActStop = 2, kActRollback = 3 };
enum LoopState2 { kS2P2 = 1, kS2NoMove = 2, kS2Stop = 3 };

// Speculation state of the vector CTA: the last stepped iteration is applied
// before its df (nqp.hpp:307-308) is known; df runs during the next P1 and a
// rejection (rare: the halving safeguard) rolls the step back.
struct Pending {
  int on;
  unsigned long long k;
  double f, gbs, el, alpha;
  int ml, cl, tries;
  unsigned long long mults;
};

// Barrier over all CTAs of the loop. Small problems launch the whole grid as ONE
// thread-block cluster (<= 16 CTAs, same GPC): the hardware cluster barrier
// (release/acquire at cluster scope, L1 invalidated) replaces the cooperative
// grid barrier (1.2 us measured; a nanosleep-backoff barrier in common.cuh
// measured slower).
template <bool kCluster>
struct AllCtas {
  cg::grid_group grid;
  __device__ AllCtas() : grid(cg::this_grid()) {}
  __device__ __forceinline__ void sync() {
    if constexpr (kCluster) {
      asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
                   "barrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else {
      grid.sync();
    }
  }
};

template <bool kCluster>
__global__ void __launch_bounds__(kLoopThreads, 1) nqp_loop_kernel(LoopArgs a) {
  AllCtas<kCluster> grid;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ LeaderState L;
  __shared__ Pending PD;
  __shared__ RowShared RS;
  __shared__ double s_min_x;
  const bool leader = blockIdx.x == 0;
  const int R = a.rows_per_cta;
  const int nblk = (int)gridDim.x - 1;
  const int blk = (int)blockIdx.x - 1;
  const int row0 = leader ? 0 : blk * R;
  const int nrows = leader ? 0 : max(0, min(a.m - row0, R));
  const double* qblk = a.Q + (size_t)(leader ? 0 : blk) * R * a.m;
  RowRing ring;
  // small m: the row block of Q stays in shared memory for the whole solve
  const bool resident = a.resident != 0;
  double* Qs = reinterpret_cast<double*>(smem);
  uint32_t* s_list = reinterpret_cast<uint32_t*>(Qs + (size_t)R * a.m);
  double* s_vals = reinterpret_cast<double*>(s_list + ((a.m + 8) & ~1));
  if (!leader) {
    if (resident) {
      const double2* src = reinterpret_cast<const double2*>(qblk);
      double2* dst = reinterpret_cast<double2*>(Qs);
      for (int e = threadIdx.x; e < R * a.m / 2; e += blockDim.x) dst[e] = __ldg(src + e);
      __syncthreads();
    } else {
      ring_setup(ring, smem, kRingSmemBytes, nrows, R, kWarps);
      if (a.l2_frac > 0.f) ring.l2pol = l2_evict_last_fraction(a.l2_frac);
    }
  }
  double* sbuf = reinterpret_cast<double*>(smem);
  double* xb[2] = {a.x, a.x_alt};
  double* gb[2] = {a.g, a.g_alt};
  const ListSet ls[2] = {{a.mask, a.gP, a.xP, a.qP}, {a.mask2, a.gP2, a.xP2, a.qP2}};
  int xp = 0, lp = 0;      // state / list parity (identical in every CTA)
  int ml_l[2] = {0, 0};    // list lengths per parity (row CTAs)

  // ---- prologue: passive lists of the start point ---------------------------------------
  const uint64_t t0 = globaltimer_ns();
  if (!leader) row_count(a, RS, blk, row0, nrows, xb[0], gb[0]);
  grid.sync();
  if (!leader) ml_l[0] = row_lists(a, RS, blk, nblk, row0, nrows, xb[0], gb[0], ls[0], 0);
  if (leader && threadIdx.x == 0) {
    a.ctrl->trace_len = 0;
    a.ctrl->mult_len = 0;
    a.ctrl->mult_total = 0;
    a.ctrl->numeric_failure = 0;
    a.ctrl->g_parity = 0;
    a.ctrl->p1_done = 0;
    a.ctrl->bc_epoch = 0;
    L.best_gbs = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    L.since_best = 0;
    L.t_mark = t0;
    for (int i = 0; i < 8; ++i) L.ph[i] = 0;
    PD.on = 0;
  }
  grid.sync();
  if (leader && threadIdx.x == 0) {  // min_iterate starts at min(start) (nqp.hpp:237)
    double mn = __longlong_as_double(0x7ff0000000000000LL);
    for (int b = 0; b < nblk; ++b) mn = fmin(mn, __ldcg(a.minx + b));
    a.ctrl->min_iterate = a.m ? mn : 0.0;
  }

  unsigned long long k = 0;  // iteration whose stop test runs next (vector CTA)
  unsigned int npass = 0;    // phase-A passes (identical in every CTA)
  for (;;) {
    // ===== phase A: P1 (row CTAs) || stop-test chains + pending df (vector CTA) =====
    ++npass;
    if (!leader) {
      // u = Q g_bar over own rows, also compacted to the passive list for den
      if (resident)
        gemv_resident(Qs, R, s_list, s_vals, row0, nrows, ls[lp].mask, ls[lp].gP, ml_l[lp], a.u,
                      RS.lpos[lp], a.uP);
      else
        gemv_rows(ring, qblk, R, true, row0, nrows, ls[lp].mask, ls[lp].gP, ml_l[lp], a.u,
                  RS.lpos[lp], a.uP);
      __syncthreads();
      if (threadIdx.x == 0) {  // publish: uP of own rows is complete (release)
        __threadfence();
        atomicAdd(&a.ctrl->p1_done, 1u);
      }
    } else {
      __shared__ int s_ml, s_bad;
      __shared__ double s_mn;
      if (threadIdx.x < 32) {  // gather the row CTAs' partials of the current state
        int c = 0, bd = 0;
        double mn = __longlong_as_double(0x7ff0000000000000LL);
        int cv[6], bv[6];
        double mv[6];
#pragma unroll
        for (int r = 0; r < 6; ++r) {  // nblk <= 192: all loads in flight together
          const int b = threadIdx.x + 32 * r;
          cv[r] = b < nblk ? __ldcg(a.cnt + b) : 0;
          bv[r] = b < nblk ? __ldcg(a.badv + b) : 0;
          mv[r] = b < nblk ? __ldcg(a.minx + b) : __longlong_as_double(0x7ff0000000000000LL);
        }
#pragma unroll
        for (int r = 0; r < 6; ++r) {
          c += cv[r];
          bd |= bv[r];
          mn = fmin(mn, mv[r]);
        }
        for (int o = 16; o > 0; o >>= 1) {
          c += __shfl_xor_sync(0xffffffffu, c, o);
          bd |= __shfl_xor_sync(0xffffffffu, bd, o);
          mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        }
        if (threadIdx.x == 0) {
          s_ml = c;
          s_bad = bd;
          s_mn = mn;
        }
      }
      __syncthreads();
      const int ml = s_ml;
      const ListSet cur = ls[lp];
      const int lens[4] = {ml, ml, ml, PD.on ? PD.cl : 0};
      const double *gP = cur.gP, *xP = cur.xP, *qP = cur.qP;
      const double *gC = a.gC, *dC = a.dC, *gdC = a.gdC;
      // gbs: g_i^2; dot(x, grad): x_i g_i; dot(q, x): q_i x_i (terms off the mask are
      // exact zeros since x_i = 0 there); df of the pending step (nqp.hpp:307)
      leader_chains_var<4>(sbuf, kRingSmemBytes, L, lens, [&](int c, int t) {
        if (c == 0) return xmul(gP[t], gP[t]);
        if (c == 1) return xmul(xP[t], gP[t]);
        if (c == 2) return xmul(qP[t], xP[t]);
        return xmul(xadd(gC[t], xmul(0.5, __ldcg(gdC + t))), dC[t]);
      });
      if (threadIdx.x == 0) {
        const double gbs = L.res[0];
        const double f = xmul(0.5, xadd(L.res[1], L.res[2]));
        const double el = (double)(globaltimer_ns() - t0) * 1e-9;
        const double best0 = L.best_gbs;
        const unsigned long long since0 = L.since_best;
        int stop = -1;
        if (s_bad || !isfinite(f) || !isfinite(gbs)) {
          stop = 100;  // NumericFailure (nqp.hpp:257-259)
        } else if (ml == 0) {
          stop = ALNNLS_EMPTY_PASSIVE_SET;
        } else if (gbs < a.eps) {
          stop = ALNNLS_GRADIENT_BELOW_EPSILON;
        } else if (k >= a.max_iters) {
          stop = ALNNLS_MAX_ITERS;
        } else if (a.has_time_cap && el >= a.time_cap_s) {
          stop = ALNNLS_TIME_CAP;
        } else if (gbs < L.best_gbs) {
          L.best_gbs = gbs;
          L.since_best = 0;
        } else if (++L.since_best >= a.stall_window) {
          stop = ALNNLS_STALLED;
        }
        if (stop < 0 && !(gbs != 0.0)) stop = ALNNLS_ZERO_CURVATURE;  // num == 0 (nqp.hpp:167)
        int act = stop >= 0 ? kActStop : kActCont;
        if (PD.on) {
          const double df = L.res[3];
          if (!(df <= 0.0 || PD.tries >= 60)) {  // reject: roll back (nqp.hpp:316-317)
            L.best_gbs = best0;
            L.since_best = since0;
            PD.alpha = xmul(PD.alpha, 0.5);
            ++PD.tries;
            act = kActRollback;
          } else {  // accept the pending step: its bookkeeping is now final
            if (a.m && s_mn < a.ctrl->min_iterate) a.ctrl->min_iterate = s_mn;
            push_step(a, PD.k, PD.f, PD.gbs, PD.ml, PD.el, PD.alpha, PD.mults);
            PD.on = 0;
          }
        }
        if (act == kActStop) {
          if (stop == 100) a.ctrl->numeric_failure = 1;
          else stop_final(a, k, f, gbs, ml, el, stop);
        }
        L.f = f;
        L.gbs = gbs;
        L.elapsed = el;
        L.mask_len = ml;
        a.ctrl->act = act;
        L.act = act;
        phase_mark(L, 0);
        __threadfence();
        // the den chain needs every row CTA's P1 (no grid barrier here: the row
        // CTAs go straight on to B_C, where they learn act and the changed set)
        if (act == kActCont) {
          const unsigned int target = npass * (unsigned int)nblk;
          while (ld_acquire_u32(&a.ctrl->p1_done) < target) {
          }
        }
        phase_mark(L, 1);
      }
      __syncthreads();
    }
    // rows: act is read after B_C; the leader acts on it now
    int act = leader ? L.act : 0;
    if (leader && act == kActRollback) {  // back to the state before the rejected step
      xp ^= 1;
      lp ^= 1;
    }

    // ===== phase B (vector CTA): den chain, alpha, changed set ==========================
    if (leader && act != kActStop) {
      const ListSet cur = ls[lp];
      __shared__ int s_zc;
      if (act == kActCont) {
        const int ml = L.mask_len;
        const double* gP = cur.gP;
        const double* uP = a.uP;
        leader_chains<1>(sbuf, kRingSmemBytes, L, ml,
                         [&](int, int t) { return xmul(gP[t], __ldcg(uP + t)); });
        if (threadIdx.x == 0) {
          const double den = L.res[0];
          L.mults = (unsigned long long)a.m * (unsigned long long)ml;
          L.tries = 0;
          s_zc = !(den > 0.0);
          if (s_zc) stop_final(a, k, L.f, L.gbs, ml, L.elapsed, ALNNLS_ZERO_CURVATURE);
          else L.alpha = xdiv(L.gbs, den);
          phase_mark(L, 2);
        }
      } else if (threadIdx.x == 0) {
        s_zc = 0;
        L.alpha = PD.alpha;
        L.mask_len = PD.ml;
      }
      __syncthreads();
      __shared__ unsigned long long s_m0;
      if (!s_zc) {
        if (threadIdx.x == 0) {  // den-pass multiplies; build_changed adds m*|C| to L.mults
          s_m0 = L.mults;
          L.mults = 0;
        }
        __syncthreads();
        const unsigned long long m0 = s_m0;
        leader_build_changed(a, L, L.mask_len, L.alpha, cur);
        if (threadIdx.x == 0) {
          const int cl = a.ctrl->chg_len;
          if (act == kActCont) {
            L.mults += m0;
            if (cl == 0) {  // nothing moved (nqp.hpp:304): step recorded, state unchanged
              push_step(a, k, L.f, L.gbs, L.mask_len, L.elapsed, L.alpha, L.mults);
            } else {        // speculate: apply now, check df during the next P1
              PD.on = 1;
              PD.k = k;
              PD.f = L.f;
              PD.gbs = L.gbs;
              PD.el = L.elapsed;
              PD.ml = L.mask_len;
              PD.alpha = L.alpha;
              PD.tries = 0;
              PD.mults = L.mults;
            }
            ++k;
          } else {
            PD.mults += L.mults;
            if (cl == 0) {  // halving made the step vanish: record it unchanged
              push_step(a, PD.k, PD.f, PD.gbs, PD.ml, PD.el, PD.alpha, PD.mults);
              PD.on = 0;
            }
          }
          PD.cl = cl;
          a.ctrl->state2 = cl == 0 ? kS2NoMove : kS2P2;
        }
      } else if (threadIdx.x == 0) {
        a.ctrl->state2 = kS2Stop;
      }
      if (threadIdx.x == 0) {
        phase_mark(L, 3);
        __threadfence();
      }
    }
    // B_C: only the vector CTA's results flow here (act, the changed set), so the
    // grid variant signals them one way (a release store the row CTAs poll) instead
    // of a grid barrier; the cluster variant keeps its hardware barrier
    if constexpr (kCluster) {
      grid.sync();
    } else if (leader) {
      __threadfence();  // every vector-CTA thread's writes of the changed set
      __syncthreads();
      if (threadIdx.x == 0) st_release_u32(&a.ctrl->bc_epoch, npass);
    } else {
      if (threadIdx.x == 0)
        while (ld_acquire_u32(&a.ctrl->bc_epoch) < npass) {
        }
      __syncthreads();
    }
    if (!leader) {
      act = __ldcg(&a.ctrl->act);  // after the barrier: L2 read, no sys-scope volatile
      if (act == kActRollback) {
        xp ^= 1;
        lp ^= 1;
      }
    }
    if (act == kActStop) break;
    const int st2 = __ldcg(&a.ctrl->state2);
    if (st2 == kS2Stop) break;
    if (st2 == kS2NoMove) continue;

    // ===== P2, speculative update, next passive lists ====================================
    const int cl = __ldcg(&a.ctrl->chg_len);
    // a warp the P2 GEMV leaves idle finds this CTA's slice of the changed list
    const int idle_w = resident ? kWarps : ring.P + ring.cons_warps;
    if (!leader) {
      if (resident) {
        gemv_resident(Qs, R, s_list, s_vals, row0, nrows, a.chg, a.dC, cl, a.gd);
      } else {
        if ((int)(threadIdx.x >> 5) == idle_w) own_changed_range(a, RS, row0, nrows, cl);
        gemv_rows(ring, qblk, R, true, row0, nrows, a.chg, a.dC, cl, a.gd);
#if ALNNLS_P1_PREFETCH
        // the next P1's first stages: its passive list is not built yet, but it is
        // mostly this iteration's; prefetch this CTA's panel runs of the first
        // columns of the current list into L2 while the barriers and lists run
        if ((int)(threadIdx.x >> 5) < ring.P) {
          const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
          const int npf = min(ml_l[lp], ALNNLS_P1_PREFETCH);
          const uint32_t* lst = ls[lp].mask;
          for (int l0 = w * 32; l0 < npf; l0 += ring.P * 32) {
            const int l = l0 + lane;
            const bool valid = l < npf;
            const uint32_t j = valid ? __ldcg(lst + l) : 0u;
            const uint32_t jp = __shfl_up_sync(0xffffffffu, j, 1);
            const bool start = valid && (lane == 0 || j != jp + 1u);
            const uint32_t starts = __ballot_sync(0xffffffffu, start);
            if (start) {
              const uint32_t later = starts & ~((2u << lane) - 1u);
              int end = later ? __ffs(later) - 1 : 32;
              end = min(end, npf - l0);
              bulk_prefetch_l2(qblk + (size_t)j * R, (uint32_t)((end - lane) * R * 8));
            }
          }
        }
#endif
      }
    }
    // no grid barrier after P2: row_apply reads only its own rows of gd, and the
    // leader's df chain reads gdC only after B0
    __syncthreads();
    if (leader && threadIdx.x == 0) phase_mark(L, 4);
    if (!leader)
      row_apply(a, RS, blk, row0, nrows, xb[xp], gb[xp], xb[xp ^ 1], gb[xp ^ 1], cl,
                idle_w < kWarps);
    grid.sync();  // B_cnt
    if (leader && threadIdx.x == 0) phase_mark(L, 5);
    if (!leader)
      ml_l[lp ^ 1] = row_lists(a, RS, blk, nblk, row0, nrows, xb[xp ^ 1], gb[xp ^ 1], ls[lp ^ 1],
                               lp ^ 1);
    grid.sync();  // B0
    if (leader && threadIdx.x == 0) phase_mark(L, 6);
    xp ^= 1;
    lp ^= 1;
  }
  if (leader && threadIdx.x == 0) {
    a.ctrl->g_parity = xp;
    for (int i = 0; i < 8; ++i) a.ctrl->phase_ns[i] = L.ph[i];
  }
}

// ==== Accelerated (Nesterov) baseline: accelerated.hpp:21-117 =========================
// Per iteration k (reference order): grad = Q x + q; the stop tests on (x, grad);
// grad_y = Q y + q; x' = max(0, y - alpha grad_y) with alpha = 1/||Q||_F;
// t' = (1 + sqrt(1 + 4t^2))/2; y' = x' + ((t-1)/t') (x' - x) (or x' after a
// restart); x = x'. Both products run in ONE pass over Q: the union of the
// supports of x and y is streamed once and every row carries two chains (a zero
// x_j or y_j adds +-0, an exact no-op, so each chain equals the reference's
// matvec over all columns). Vector CTA: the gbs / x.g / q.x chains (over all m
// positions, skipped terms added as -0), stop tests and trace. Row CTAs: the
// pass, the elementwise updates and the next union list.

// Row phase after the pass: grad = u + q and grad_y = w + q (linalg.hpp:185 then
// accelerated.hpp:46, :90), x' = max(0, y - alpha grad_y); passive counts.
__device__ void acc_rows_after_pass(const LoopArgs& a, RowShared& S, int blk, int row0, int nrows) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int c = 0, bad = 0;
  for (int t = threadIdx.x; t < nrows; t += blockDim.x) {
    const int i = row0 + t;
    const double gi = xadd(a.u[i], a.q[i]);
    const double gyi = xadd(a.w[i], a.q[i]);
    a.g[i] = gi;
    const double v = xsub(a.y[i], xmul(a.alpha, gyi));
    a.xn[i] = 0.0 < v ? v : 0.0;  // std::max(0.0, v)
    c += (a.x[i] > 0.0 || gi < 0.0) ? 1 : 0;
    if (!isfinite(gi)) bad = 1;
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) S.wc[warp] = c;
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < kWarps; ++w) tot += S.wc[w];
    a.pcnt[blk] = tot;
    a.badv[blk] = bad;
  }
}

// Row phase after the stop test: y' and x = x' (accelerated.hpp:96-108); count the
// union flags (x_i != 0 or y_i != 0) for the next pass.
__device__ void acc_rows_update(const LoopArgs& a, RowShared& S, int blk, int row0, int nrows,
                                double momentum, int restart) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int c = 0;
  for (int t = threadIdx.x; t < nrows; t += blockDim.x) {
    const int i = row0 + t;
    const double xn = a.xn[i];
    const double yi = restart ? xn : xadd(xn, xmul(momentum, xsub(xn, a.x[i])));
    a.y[i] = yi;
    a.x[i] = xn;
    c += (xn != 0.0 || yi != 0.0) ? 1 : 0;
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) S.wc[warp] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < kWarps; ++w) tot += S.wc[w];
    a.cnt[blk] = tot;
  }
}

// Union list of own rows at the global offset sum(cnt[0..blk)), values x and y.
__device__ int acc_rows_list(const LoopArgs& a, RowShared& S, int blk, int nblk, int row0,
                             int nrows) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
    int before = 0, all = 0;
    int cv[6];
#pragma unroll
    for (int r = 0; r < 6; ++r) cv[r] = lane + 32 * r < nblk ? __ldcg(a.cnt + lane + 32 * r) : 0;
#pragma unroll
    for (int r = 0; r < 6; ++r) {
      all += cv[r];
      if (lane + 32 * r < blk) before += cv[r];
    }
    for (int o = 16; o > 0; o >>= 1) {
      before += __shfl_xor_sync(0xffffffffu, before, o);
      all += __shfl_xor_sync(0xffffffffu, all, o);
    }
    if (lane == 0) {
      S.base = before;
      S.total = all;
    }
  }
  const int t = threadIdx.x;  // one round: nrows <= blockDim.x
  double xi = 0.0, yi = 0.0;
  bool f = false;
  if (t < nrows) {
    xi = a.x[row0 + t];
    yi = a.y[row0 + t];
    f = xi != 0.0 || yi != 0.0;
  }
  const unsigned bal = __ballot_sync(0xffffffffu, f);
  if (lane == 0) S.wc[warp] = __popc(bal);
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = S.base;
    for (int w = 0; w < kWarps; ++w) {
      const int c = S.wc[w];
      S.wc[w] = run;
      run += c;
    }
  }
  __syncthreads();
  if (f) {
    const int pos = S.wc[warp] + __popc(bal & ((1u << lane) - 1u));
    a.mask[pos] = (uint32_t)(row0 + t);
    a.gP[pos] = xi;
    a.vy[pos] = yi;
  }
  return S.total;
}

template <bool kCluster>
__global__ void __launch_bounds__(kLoopThreads, 1) acc_loop_kernel(LoopArgs a) {
  AllCtas<kCluster> grid;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ LeaderState L;
  __shared__ RowShared RS;
  const bool leader = blockIdx.x == 0;
  const int R = a.rows_per_cta;
  const int nblk = (int)gridDim.x - 1;
  const int blk = (int)blockIdx.x - 1;
  const int row0 = leader ? 0 : blk * R;
  const int nrows = leader ? 0 : max(0, min(a.m - row0, R));
  const double* qblk = a.Q + (size_t)(leader ? 0 : blk) * R * a.m;
  RowRing ring;
  if (!leader) ring_setup(ring, smem, kRingSmemBytes, nrows, R, kWarps);
  double* sbuf = reinterpret_cast<double*>(smem);
  const uint64_t t0 = globaltimer_ns();
  if (leader && threadIdx.x == 0) {
    a.ctrl->trace_len = 0;
    a.ctrl->mult_len = 0;
    a.ctrl->mult_total = 0;
    a.ctrl->numeric_failure = 0;
    a.ctrl->g_parity = 0;
    a.ctrl->min_iterate = 0.0;  // result.min_iterate = 0 (:32); x' >= 0 keeps it there
    L.best_gbs = __longlong_as_double(0x7ff0000000000000LL);
    L.since_best = 0;
    L.f = __longlong_as_double(0x7ff0000000000000LL);  // f_prev = +inf
  }
  int len = 0;       // union list length (x = y = 0 at the start: empty)
  double t = 1.0;    // every thread carries the same momentum sequence
  for (unsigned long long k = 0;; ++k) {
    // ===== pass: u = Q x, w = Q y over the union list; then grad, grad_y, x' =====
    if (!leader)
      gemv_rows(ring, qblk, R, true, row0, nrows, a.mask, a.gP, len, a.u, nullptr, nullptr,
                a.vy, a.w);
    __syncthreads();  // own rows of u, w written by the consumer warps
    if (!leader) acc_rows_after_pass(a, RS, blk, row0, nrows);
    grid.sync();
    // ===== vector CTA: chains and the ordered stop tests (accelerated.hpp:45-81) =====
    if (leader) {
      const double *x = a.x, *g = a.g, *q = a.q;
      const int m = a.m;
      const int lens[3] = {m, m, m};
      leader_chains_var<3>(sbuf, kRingSmemBytes, L, lens, [&](int c, int i) {
        const double xi = __ldcg(x + i), gi = __ldcg(g + i);
        if (c == 0) return (xi > 0.0 || gi < 0.0) ? xmul(gi, gi) : -0.0;  // gbs over the mask
        if (c == 1) return xi != 0.0 ? xmul(xi, gi) : -0.0;               // dot(x, grad)
        return xi != 0.0 ? xmul(__ldcg(q + i), xi) : -0.0;                // dot(q, x)
      });
      if (threadIdx.x == 0) {
        int ml = 0, bad = 0;
        for (int b = 0; b < nblk; ++b) {
          ml += __ldcg(a.pcnt + b);
          bad |= __ldcg(a.badv + b);
        }
        const double gbs = L.res[0];
        const double f = xmul(0.5, xadd(L.res[1], L.res[2]));
        const double el = (double)(globaltimer_ns() - t0) * 1e-9;
        int stop = -1;
        if (bad || !isfinite(f) || !isfinite(gbs)) stop = 100;  // NumericFailure (:55-58)
        else if (ml == 0) stop = ALNNLS_EMPTY_PASSIVE_SET;
        else if (gbs < a.eps) stop = ALNNLS_GRADIENT_BELOW_EPSILON;
        else if (k >= a.max_iters) stop = ALNNLS_MAX_ITERS;
        else if (a.has_time_cap && el >= a.time_cap_s) stop = ALNNLS_TIME_CAP;
        else if (a.alpha == __longlong_as_double(0x7ff0000000000000LL))  // m_norm == 0
          stop = ALNNLS_ZERO_CURVATURE;
        else if (gbs < L.best_gbs) {
          L.best_gbs = gbs;
          L.since_best = 0;
        } else if (++L.since_best >= a.stall_window) {
          stop = ALNNLS_STALLED;
        }
        int act = kActCont;
        if (stop == 100) {
          a.ctrl->numeric_failure = 1;
          act = kActStop;
        } else if (stop >= 0) {
          stop_final(a, k, f, gbs, ml, el, stop);
          act = kActStop;
        } else {
          if (k % a.trace_every == 0) write_record(a, k, f, gbs, ml, el, a.alpha, 1);
          if (a.restart && f > L.f) act = kActRollback;  // restart (:102-105)
        }
        L.f = f;  // f_prev
        a.ctrl->act = act;
        __threadfence();
      }
    }
    grid.sync();
    const int act = __ldcg(&a.ctrl->act);  // after the grid barrier: L2 read, no sys-scope volatile
    if (act == kActStop) break;
    // ===== y', x = x' (accelerated.hpp:96-108), next union list =====
    const double t_next = xmul(0.5, xadd(1.0, __dsqrt_rn(xadd(1.0, xmul(xmul(4.0, t), t)))));
    const double momentum = xdiv(xsub(t, 1.0), t_next);
    const int rs = act == kActRollback;
    if (!leader) acc_rows_update(a, RS, blk, row0, nrows, momentum, rs);
    t = rs ? 1.0 : t_next;
    grid.sync();
    if (!leader) len = acc_rows_list(a, RS, blk, nblk, row0, nrows);
    grid.sync();
  }
}

__global__ void __launch_bounds__(kLoopThreads, 1) frobenius_kernel(const double* Qb, int m, int R,
                                                                    double* out) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ LeaderState L;
  double* sbuf = reinterpret_cast<double*>(smem);
  // column-major order: entry e = j*m + i (m*m < 2^31, checked on the host)
  leader_chains<1>(sbuf, kRingSmemBytes, L, m * m, [&](int, int e) {
    const int j = e / m, i = e - j * m;
    const double v = __ldg(Qb + blk_index(i, j, m, R));
    return xmul(v, v);
  });
  if (threadIdx.x == 0) *out = __dsqrt_rn(L.res[0]);
}

}  // namespace

size_t nqp_loop_smem_bytes() { return kRingSmemBytes; }
bool nqp_resident_fits(int m, int R) {
  return ALNNLS_RESIDENT_Q && R <= kLoopThreads && resident_smem_bytes(R, m) <= kRingSmemBytes;
}

// Rows per block of the blocked Q: the vector CTA takes one SM, the row
// blocks share the rest.
// Small m: the loop runs as ONE thread-block cluster, the rows split over 7 row
// CTAs (portable cluster of 8) up to m = 448, over 15 (non-portable 16) up to
// m = 640; at most 64 rows per row CTA. Larger m: the cooperative grid (whose row
// CTAs keep their Q panels resident in shared memory up to m ~ 1870). c1 (m = 300): 22.7 us/iteration on 76
// cooperative CTAs -> 19.3 (cluster of 16) -> 18.6 (cluster of 8).
#ifndef ALNNLS_CLUSTER_ROWS
#define ALNNLS_CLUSTER_ROWS 64  // 0 disables the cluster launch policy (build knob)
#endif
#ifndef ALNNLS_CLUSTER16_MAX_M
#define ALNNLS_CLUSTER16_MAX_M 640  // build knob: top of the 16-CTA cluster tier
#endif
int nqp_rows_per_cta(int m, int sm_count) {
  // measured (tools/ab_run.sh, us/iteration, cluster of 16 vs grid with resident Q
  // panels): m = 500 18.2 vs 21.3, 600 22.9 vs 23.7, 800 28.3 vs 25.0, 900 28.1 vs 25.9
  if (ALNNLS_CLUSTER_ROWS > 0 && m <= ALNNLS_CLUSTER16_MAX_M &&
      m <= 15 * ALNNLS_CLUSTER_ROWS) {
    const int ctas = m <= 7 * ALNNLS_CLUSTER_ROWS ? 7 : 15;
    int r = (m + ctas - 1) / ctas;
    r = (r + 3) & ~3;
    return r < 4 ? 4 : r;
  }
  const int nb = sm_count > 1 ? sm_count - 1 : 1;
  int r = (m + nb - 1) / nb;
  r = (r + 3) & ~3;
  if (r < 4) r = 4;
  return r;
}

// One loop launch: a single thread-block cluster when the grid fits one (<= 16
// CTAs, non-portable sizes allowed, and the occupancy query finds a GPC for it),
// else a cooperative grid.
template <class KC, class KG>
cudaError_t launch_loop(KC kcluster, KG kgrid, const LoopArgs& a, int num_ctas,
                        cudaStream_t stream, int* which = nullptr,
                        size_t smem_bytes = nqp_loop_smem_bytes(), int threads = kLoopThreads) {
  // attributes are per device (func_attr_once keys them by the current device)
  if (cudaError_t e = smem_optin(kgrid, (int)smem_bytes)) return e;
  if (cudaError_t e = smem_optin(kcluster, (int)smem_bytes)) return e;
  const bool cluster_ok =
      func_attr_once(reinterpret_cast<const void*>(kcluster),
                     cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
  (void)cudaGetLastError();
  LoopArgs args = a;
  if (cluster_ok && num_ctas <= 16) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(num_ctas);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem_bytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = num_ctas;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, kcluster, &cfg) == cudaSuccess && nclusters > 0) {
      if (which) *which = ALNNLS_LOOP_CLUSTER;
      return cudaLaunchKernelEx(&cfg, kcluster, args);
    }
    (void)cudaGetLastError();  // no cluster of this size fits: cooperative grid instead
  }
  if (which) *which = ALNNLS_LOOP_GRID;
  void* params[] = {&args};
  return cudaLaunchCooperativeKernel((void*)kgrid, dim3(num_ctas), dim3(threads), params,
                                     smem_bytes, stream);
}

cudaError_t launch_nqp_loop(const LoopArgs& a, int num_ctas, cudaStream_t stream, int* which) {
  // small m: the cluster loop with its state in distributed shared memory (small.cu);
  // ALNNLS_SMALL=0 in the environment forces the general kernel (A/B and parity tests)
  const char* knob = getenv("ALNNLS_SMALL");
  if (!(knob && knob[0] == '0')) {
    const cudaError_t e = launch_nqp_small(a, num_ctas, stream);
    if (e != cudaErrorNotSupported) {
      if (which) *which = ALNNLS_LOOP_SMALL;
      return e;
    }
  }
  // L2 residency hint for the ring's copies of Q when a sizable part of Q fits the
  // L2 (c2 / c3: P1 and P2 of an iteration read mostly the same columns); env
  // ALNNLS_L2_FRAC overrides (A/B; 0 disables)
  LoopArgs b = a;
  {
    // measured at c2 / c3 (Q = 134 MB): fraction 0 84.6 / 97.1 us per iteration,
    // 0.3-0.5 80.8 / 92.2, 0.7 81.7 / 94.8, 1.0 84.6
    const double qbytes = 8.0 * (double)a.m * (double)a.m;
    double f = 50e6 / qbytes;
    if (f > 1.0) f = 1.0;
    if (f < 0.25) f = 0.0;
    if (const char* e = getenv("ALNNLS_L2_FRAC")) f = atof(e);
    b.l2_frac = (float)f;
  }
  if (a.zero_start) {  // x = 0, g = q (nqp.hpp:224-225), zeroed padding and barrier words
    const size_t m = (size_t)a.m;
    if (cudaError_t e2 = cudaMemsetAsync(a.gP, 0, sizeof(double) * (m + 8), stream)) return e2;
    if (cudaError_t e2 = cudaMemsetAsync(a.dC, 0, sizeof(double) * (m + 8), stream)) return e2;
    if (cudaError_t e2 = cudaMemsetAsync(a.x, 0, sizeof(double) * m, stream)) return e2;
    if (cudaError_t e2 = cudaMemcpyAsync(a.g, a.q, sizeof(double) * m, cudaMemcpyDeviceToDevice,
                                         stream))
      return e2;
    if (cudaError_t e2 = cudaMemsetAsync(a.bar, 0, 2 * sizeof(unsigned int), stream)) return e2;
  }
  return launch_loop(nqp_loop_kernel<true>, nqp_loop_kernel<false>, b, num_ctas, stream, which);
}

// ---- standalone masked GEMV (masked_matvec / matvec / residual / warm start) ------------
namespace {
__global__ void __launch_bounds__(kLoopThreads, 1)
    masked_gemv_kernel(const double* M, uint64_t ld, int rows, int rows_per_cta, int blocked,
                       const uint32_t* list, const double* vals, int len, double* y,
                       const int* dlen) {
  extern __shared__ __align__(128) uint8_t smem[];
  if (dlen) len = *dlen;
  const int row0 = blockIdx.x * rows_per_cta;
  const int nrows = max(0, min(rows - row0, rows_per_cta));
  RowRing ring;
  if (blocked) {
    // M is a blocked m x m matrix (m = rows, block rows = rows_per_cta)
    ring_setup(ring, smem, kRingSmemBytes, nrows, rows_per_cta, kWarps);
    gemv_rows(ring, M + (size_t)blockIdx.x * rows_per_cta * rows, rows_per_cta, true, row0, nrows,
              list, vals, len, y);
  } else {
    ring_setup(ring, smem, kRingSmemBytes, nrows, ring_seg(nrows), kWarps);
    gemv_rows(ring, M + row0, ld, false, row0, nrows, list, vals, len, y);
  }
}

cudaError_t gemv_launch(const double* M, uint64_t ld, int rows, int rpc, int blocked,
                        const uint32_t* list, const double* vals, int len, double* y,
                        cudaStream_t stream, const int* dlen = nullptr) {
  if (cudaError_t e = smem_optin(masked_gemv_kernel, (int)nqp_loop_smem_bytes())) return e;
  if (rows <= 0) return cudaSuccess;
  if (rpc > 352) return cudaErrorInvalidValue;  // 11 consumer warps + 1 producer
  const int grid = (rows + rpc - 1) / rpc;
  masked_gemv_kernel<<<grid, kLoopThreads, nqp_loop_smem_bytes(), stream>>>(M, ld, rows, rpc,
                                                                            blocked, list, vals,
                                                                            len, y, dlen);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_masked_gemv(const double* M, uint64_t ld, int rows, const uint32_t* list,
                               const double* vals, int len, double* y, int sm_count,
                               cudaStream_t stream, const int* dlen) {
  int rpc = (rows + sm_count - 1) / sm_count;
  rpc = (rpc + 3) & ~3;
  if (rpc < 4) rpc = 4;
  return gemv_launch(M, ld, rows, rpc, 0, list, vals, len, y, stream, dlen);
}

namespace {
__global__ void copy_parity_kernel(double* y, const double* x, const double* x_alt,
                                   const LoopCtrl* ctrl, int m) {
  const double* src = ctrl->g_parity ? x_alt : x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
    y[i] = src[i];
}
}  // namespace

cudaError_t launch_copy_parity(double* y, const double* x, const double* x_alt,
                               const LoopCtrl* ctrl, int m, cudaStream_t stream) {
  if (m <= 0) return cudaSuccess;
  copy_parity_kernel<<<(m + 255) / 256 < 148 ? (m + 255) / 256 : 148, 256, 0, stream>>>(
      y, x, x_alt, ctrl, m);
  return cudaGetLastError();
}

cudaError_t launch_masked_gemv_blocked(const double* Qb, int m, int R, const uint32_t* list,
                                       const double* vals, int len, double* y,
                                       cudaStream_t stream) {
  return gemv_launch(Qb, 0, m, R, 1, list, vals, len, y, stream);
}

}  // namespace alnnls

namespace alnnls {
cudaError_t launch_acc_loop(const LoopArgs& a, int num_ctas, cudaStream_t stream, int* which) {
  return launch_loop(acc_loop_kernel<true>, acc_loop_kernel<false>, a, num_ctas, stream, which);
}

cudaError_t launch_frobenius(const double* Qb, int m, int R, double* out, cudaStream_t stream) {
  if (cudaError_t e = smem_optin(frobenius_kernel, (int)nqp_loop_smem_bytes())) return e;
  frobenius_kernel<<<1, kLoopThreads, nqp_loop_smem_bytes(), stream>>>(Qb, m, R, out);
  return cudaGetLastError();
}
}  // namespace alnnls
