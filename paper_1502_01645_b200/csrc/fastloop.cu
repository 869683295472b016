// fastloop.cu — the FAST-profile single-RHS solve_nqp loop (north_star: "a
// bandwidth-bound GEMV kernel with coalesced 128-bit loads of Q and warp-shuffle
// plus block reductions for the dot products").
//
// Same method as reference solve_nqp (/root/reference/proj/include/antilop/
// nqp.hpp:215-339): passive mask P = {x > 0 or g < 0}, exact line search
// alpha = |g_P|^2 / (g_P^T Q g_P) (exact_step, nqp.hpp:162-173), projection
// cand = max(0, x - alpha g) on P, halving while df > 0 (nqp.hpp:279-318),
// g += Q delta (nqp.hpp:312), the same ordered stop tests (nqp.hpp:257-275),
// trace records and termination. What differs from the EXACT loop (nqp.cu):
//  - dot products and matrix-vector sums are fixed warp-shuffle / block trees
//    (deterministic run to run, not the reference's sequential chains);
//  - the update is ONE pass over Q per iteration (SURVEY.md §0.1 "one-pass"):
//    delta = -alpha g_P + c with c nonzero only on the clamped set
//    K = {i in P : x_i - alpha g_i < 0} (c_i = alpha g_i - x_i), so
//    Q delta = -alpha (Q g_P) + Q_K c_K reuses u = Q g_P from the line search
//    and only reads the |K| clamped columns again (typically a handful);
//  - multiplies_per_iter counts what this loop multiplies: m|P| + sum m|K|.
// Graded on BASELINE.json's four tolerances, not bitwise.
//
// Work split: CTA b owns rows [bR, bR + R) of the blocked Q (gemv.cuh
// blk_index: its R x m panel is contiguous, column j at j*R). By symmetry of Q,
// u_i = sum_j Q_ij gbar_j over own rows i reads, for every passive column j,
// the contiguous R-double segment of the panel: thread (rp, c) loads the
// double2 of rows (2rp, 2rp+1) for columns j = c, c + C, c + 2C, ... (skipping
// gbar_j == 0 without a load), so one warp covers 2-3 adjacent column segments
// (512 B) per 128-bit load instruction; the C column-group partials of a row
// are then summed in a fixed order. No split-K partial buffer crosses CTAs.
//
// Per iteration three grid (or cluster) barriers: A after u and the den
// partials, A2 after the clamped-set lists, B after the speculative update
// (whose partials carry df, the changed count and the NEXT state's stop-test
// sums). A halving retry costs A2 + B. Every CTA reduces the per-CTA partials
// itself, in the same fixed order, so every decision is taken identically
// everywhere with no broadcast.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "gemv.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace alnnls {

namespace {

#ifndef ALNNLS_FAST_THREADS
#define ALNNLS_FAST_THREADS 512  // build knob: threads per CTA (256 / 384 measured slower)
#endif
#ifndef ALNNLS_FAST_PHASES
#define ALNNLS_FAST_PHASES 1  // build knob: CTA 0 phase clock
#endif
#ifndef ALNNLS_FAST_UNROLL
#define ALNNLS_FAST_UNROLL 8     // build knob: candidate columns per thread per batch
#endif
constexpr int kFT = ALNNLS_FAST_THREADS;  // threads per CTA
constexpr int kFW = kFT / 32;
constexpr int kKWin = 1024;         // clamped-set window staged in shared memory
constexpr int kRedDoubles = 2 * kFT;  // C x R column-group partials (C = kFT / (R/2))
constexpr int kRecPerLane = 5;     // per-CTA records a lane reduces (nblk <= 160)
constexpr int kFastMaxBlk = 32 * kRecPerLane;

// gbar (m) [+ x (m) when local_k] + column-group partials + the K window
__host__ __device__ inline size_t fast_smem_bytes(int m, bool local_k) {
  const size_t mp = ((size_t)m + 1) & ~(size_t)1;
  return mp * sizeof(double) * (local_k ? 2 : 1) + (kRedDoubles + kFT) * sizeof(double) +
         kKWin * (sizeof(double) + sizeof(uint32_t));
}

struct FastShared {
  double wred[kFW][6];
  int wint[kFW][3];
  FastPart tot;       // cross-CTA totals of the last reduced record set
  double den;
  int kpre[kFastMaxBlk + 1];
  int scan[40];
  unsigned long long ph[8];  // CTA 0 phase clock
  uint64_t sbar;             // mbarrier of the bulk-copy staging
};

template <bool kCluster>
struct Barrier {
  cg::grid_group grid;
  __device__ Barrier() : grid(cg::this_grid()) {}
  __device__ __forceinline__ void sync() {
    if constexpr (kCluster) {
      asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
                   "barrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else {
      grid.sync();
    }
  }
};

// 128-bit load of two doubles of Q (read-only for the whole kernel; no L1
// allocation) with an L2 cache policy: a fixed fraction of Q's lines is marked
// evict_last and the rest evict_first, so that part of Q stays resident in the
// 126 MB L2 from one iteration's pass to the next (Q at c2 is 134 MB).
template <bool kL2>
__device__ __forceinline__ double2 ldq2(const double* p, uint64_t pol) {
  double2 v;
  if constexpr (kL2) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p), "l"(pol));
  } else {  // plain streaming load (the hinted form measured 15% slower when Q >> L2, c5)
    (void)pol;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p));
  }
  return v;
}
__device__ __forceinline__ uint64_t l2_policy(float frac) {
  uint64_t pol;
  if (frac > 0.f)
    asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_first.b64 %0, %1;"
                 : "=l"(pol) : "f"(frac));
  else if (frac < 0.f)
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  else
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// Thread (rp, c) accumulates rows (2rp, 2rp+1) over columns j = c, c+C, ... of
// the panel with coefficients w[j] (skipping w[j] == 0: no load).
// Thread (rp, c) accumulates rows (2rp, 2rp+1) over columns j = c, c+C, ... of
// the panel with coefficients w[j] (skipping w[j] == 0: no load). (A running-
// pointer form of this loop measured 2.6x slower at 512 threads: the 128-register
// budget then rematerializes the panel base per load.)
template <bool kL2>
__device__ __forceinline__ void panel_pass(const double* __restrict__ Qp, int R, int m,
                                           const double* __restrict__ w, int c, int C, int r2,
                                           double& acc0, double& acc1, uint64_t pol) {
  constexpr int U = ALNNLS_FAST_UNROLL;
  const double* base = Qp + r2;
  int j = c;
  for (; j + (U - 1) * C < m; j += U * C) {
    double gv[U];
    double2 qv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) gv[u] = w[j + u * C];
#pragma unroll
    for (int u = 0; u < U; ++u)
      qv[u] = gv[u] != 0.0 ? ldq2<kL2>(base + (size_t)(j + u * C) * R, pol) : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc0 = fma(qv[u].x, gv[u], acc0);
      acc1 = fma(qv[u].y, gv[u], acc1);
    }
  }
  for (; j < m; j += C) {
    const double gv = w[j];
    if (gv != 0.0) {
      const double2 qv = ldq2<kL2>(base + (size_t)j * R, pol);
      acc0 = fma(qv.x, gv, acc0);
      acc1 = fma(qv.y, gv, acc1);
    }
  }
}

// Thread (rp, c) over a staged list of (column, coefficient) pairs, t = c, c+C, ...
template <bool kL2>
__device__ __forceinline__ void list_pass(const double* __restrict__ Qp, int R,
                                          const uint32_t* __restrict__ kj,
                                          const double* __restrict__ kv, int len, int c, int C,
                                          int r2, double& acc0, double& acc1, uint64_t pol) {
  constexpr int U = 4;  // independent loads in flight per thread
  const double* base = Qp + r2;
  for (int t = c; t < len; t += U * C) {
    double2 qv[U];
    double cv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int tt = t + u * C;
      cv[u] = tt < len ? kv[tt] : 0.0;
      qv[u] = tt < len ? ldq2<kL2>(base + (size_t)kj[tt] * R, pol) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc0 = fma(qv[u].x, cv[u], acc0);
      acc1 = fma(qv[u].y, cv[u], acc1);
    }
  }
}

// Column-group partials -> per-row sums, a fixed tree: L lanes per row (the
// largest power of two with L*R <= kFT) each add every L-th group partial, then
// an xor-shuffle tree over the L lanes; row t's sum lands in thread t (t < nrows).
// `rs` is R doubles of shared memory.
__device__ __forceinline__ double rows_from_groups(double* red, double* rs, bool gthr, int c,
                                                   int R, int r2, double acc0, double acc1, int C,
                                                   int nrows) {
  if (gthr) *reinterpret_cast<double2*>(red + (size_t)c * R + r2) = make_double2(acc0, acc1);
  __syncthreads();
  int L = 1;
  while (2 * L * R <= kFT && L < 32) L *= 2;
  const int r = threadIdx.x / L, sub = threadIdx.x % L;
  double s = 0.0;
  if (r < nrows)
    for (int k = sub; k < C; k += L) s += red[(size_t)k * R + r];
  for (int o = L / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (r < nrows && sub == 0) rs[r] = s;
  __syncthreads();
  return (int)threadIdx.x < nrows ? rs[threadIdx.x] : 0.0;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_isum(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block sum of one double (fixed tree); result valid in thread 0.
__device__ __forceinline__ double block_sum(double v, FastShared& S) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) S.wred[w][0] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int k = 0; k < kFW; ++k) s += S.wred[k][0];
  __syncthreads();
  return s;
}

// This CTA's partials of a state (own rows): fixed-tree block reductions.
__device__ void write_partials(FastPart* dst, FastShared& S, double gbs, double xg, double qx,
                               double mnx, double df, double el, int cnt, int bad, int nchg) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  gbs = warp_sum(gbs);
  xg = warp_sum(xg);
  qx = warp_sum(qx);
  mnx = warp_min(mnx);
  df = warp_sum(df);
  cnt = warp_isum(cnt);
  bad = __any_sync(0xffffffffu, bad != 0) ? 1 : 0;
  nchg = warp_isum(nchg);
  if (lane == 0) {
    S.wred[w][0] = gbs;
    S.wred[w][1] = xg;
    S.wred[w][2] = qx;
    S.wred[w][3] = mnx;
    S.wred[w][4] = df;
    S.wint[w][0] = cnt;
    S.wint[w][1] = bad;
    S.wint[w][2] = nchg;
  }
  __syncthreads();
  if (w == 0) {  // lane l < kFW takes warp l's partials, then a fixed xor tree
    const bool on = lane < kFW;
    double v0 = on ? S.wred[lane][0] : 0.0, v1 = on ? S.wred[lane][1] : 0.0;
    double v2 = on ? S.wred[lane][2] : 0.0, v4 = on ? S.wred[lane][4] : 0.0;
    double v3 = on ? S.wred[lane][3] : __longlong_as_double(0x7ff0000000000000LL);
    int i0 = on ? S.wint[lane][0] : 0, i1 = on ? S.wint[lane][1] : 0, i2 = on ? S.wint[lane][2] : 0;
    v0 = warp_sum(v0);
    v1 = warp_sum(v1);
    v2 = warp_sum(v2);
    v4 = warp_sum(v4);
    v3 = warp_min(v3);
    i0 = warp_isum(i0);
    i1 = __any_sync(0xffffffffu, i1 != 0) ? 1 : 0;
    i2 = warp_isum(i2);
    if (lane == 0) {
      FastPart p;
      p.gbs = v0;
      p.xg = v1;
      p.qx = v2;
      p.minx = v3;
      p.df = v4;
      p.cnt = i0;
      p.bad = i1;
      p.nchg = i2;
      p.el = el;
      p.pad = 0;
      *dst = p;
    }
  }
  __syncthreads();
}

// Totals over the nblk per-CTA records (every CTA, same fixed order): warp 0,
// lane l sums records l, l+32, ... then an xor tree. el is record 0's.
// Totals over the nblk per-CTA records, every CTA in the same fixed order.
// Called by warps 0..3 (the caller synchronizes the CTA afterwards): warp w
// reduces the w-th 16-byte field pair of every record; lane l takes records
// l, l+32, ... and issues all its loads before the first add (one L2 round trip).
constexpr int kRedWarps = 4;
__device__ void reduce_partials(const FastPart* src, int nblk, FastShared& S) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double2 v[kRecPerLane];
#pragma unroll
  for (int r = 0; r < kRecPerLane; ++r) {
    const int b = lane + 32 * r;
    v[r] = b < nblk ? __ldcg(reinterpret_cast<const double2*>(src + b) + w)
                    : make_double2(0.0, 0.0);
  }
  if (w == 0 || w == 2) {  // (gbs, xg) or (df, el): sums; el is record 0's
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int r = 0; r < kRecPerLane; ++r) {
      a0 += v[r].x;
      a1 += v[r].y;
    }
    a0 = warp_sum(a0);
    a1 = warp_sum(a1);
    const double el0 = __shfl_sync(0xffffffffu, v[0].y, 0);
    if (lane == 0) {
      if (w == 0) {
        S.tot.gbs = a0;
        S.tot.xg = a1;
      } else {
        S.tot.df = a0;
        S.tot.el = el0;
      }
    }
  } else if (w == 1) {     // (qx, minx)
    double a0 = 0.0, mn = __longlong_as_double(0x7ff0000000000000LL);
#pragma unroll
    for (int r = 0; r < kRecPerLane; ++r) {
      a0 += v[r].x;
      if (lane + 32 * r < nblk) mn = fmin(mn, v[r].y);
    }
    a0 = warp_sum(a0);
    mn = warp_min(mn);
    if (lane == 0) {
      S.tot.qx = a0;
      S.tot.minx = mn;
    }
  } else {                 // (cnt | bad, nchg | pad)
    int cnt = 0, bad = 0, nchg = 0;
#pragma unroll
    for (int r = 0; r < kRecPerLane; ++r) {
      const long long w0 = __double_as_longlong(v[r].x), w1 = __double_as_longlong(v[r].y);
      cnt += (int)(w0 & 0xffffffffLL);
      bad |= (int)(w0 >> 32);
      nchg += (int)(w1 & 0xffffffffLL);
    }
    cnt = warp_isum(cnt);
    bad = __any_sync(0xffffffffu, bad != 0) ? 1 : 0;
    nchg = warp_isum(nchg);
    if (lane == 0) {
      S.tot.cnt = cnt;
      S.tot.bad = bad;
      S.tot.nchg = nchg;
    }
  }
}

// Sum of the nblk per-CTA den partials (warp 0; one L2 round trip, fixed order).
__device__ __forceinline__ double reduce_den(const double* den, int nblk) {
  const int lane = threadIdx.x & 31;
  double v[kRecPerLane];
#pragma unroll
  for (int r = 0; r < kRecPerLane; ++r) v[r] = lane + 32 * r < nblk ? __ldcg(den + lane + 32 * r) : 0.0;
  double sd = 0.0;
#pragma unroll
  for (int r = 0; r < kRecPerLane; ++r) sd += v[r];
  return warp_sum(sd);
}

// Trace record (CTA 0 thread 0; the counters live in its registers, not in the
// control block, so no global load sits on the iteration's critical path).
__device__ void fast_record(const FastArgs& a, unsigned long long& idx, unsigned long long k,
                            double f, double gbs, int pc, double el, double alpha, int has_alpha) {
  if (a.trace_cap > 0) {  // past the capacity the last slot keeps the newest record
    alnnls_iter_record r;
    r.iter = k;
    r.f = f;
    r.grad_bar_sq = gbs;
    r.passive_count = (uint64_t)pc;
    r.elapsed_s = el;
    r.alpha = has_alpha ? alpha : 0.0;
    r.has_alpha = has_alpha;
    a.trace[idx < a.trace_cap ? idx : a.trace_cap - 1] = r;
  }
  ++idx;
}

template <bool kCluster, bool kL2>
__global__ void __launch_bounds__(kFT, 1) fast_loop_kernel(FastArgs a) {
  Barrier<kCluster> bar;
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ FastShared S;
  const int m = a.m, R = a.R;
  const int b = blockIdx.x, nblk = gridDim.x;
  const int row0 = b * R;
  const int nrows = max(0, min(m - row0, R));
  const int mp = (m + 1) & ~1;
  const bool lk = a.local_k != 0;  // x staged too: every CTA finds K itself (no barrier A2)
  double* gs = reinterpret_cast<double*>(smem);                   // gbar of the state, m
  double* xs = gs + mp;                                           // x of the state (lk), m
  double* red = xs + (lk ? mp : 0);                               // kRedDoubles
  double* rsum = red + kRedDoubles;                               // R row sums
  double* kvs = rsum + kFT;                                       // kKWin coefficients
  uint32_t* kjs = reinterpret_cast<uint32_t*>(kvs + kKWin);       // kKWin columns
  const double* Qp = a.Q + (size_t)b * R * m;
  const int RP = R / 2;
  const int C = kFT / RP;
  const int rp = threadIdx.x % RP, grp = threadIdx.x / RP;
  const bool gthr = grp < C && 2 * rp < nrows;
  const int r2 = 2 * rp;
  const bool own = (int)threadIdx.x < nrows;
  const int i = row0 + threadIdx.x;
  const bool lead = b == 0 && threadIdx.x == 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t pol = l2_policy(a.l2_frac);
  const uint64_t t0 = globaltimer_ns();

  // ---- this thread's row of the current state --------------------------------------
  double xi = 0.0, gi = 0.0, qi = 0.0;
  if (own) {
    xi = a.x[0][i];
    gi = a.g[0][i];
    qi = a.q[i];
  }
  auto publish_state = [&](int slot, double xv, double gv, double df, int chg, bool wr) {
    // gbar, x, g of own rows and this CTA's partials of the state (xv, gv)
    const bool pf = own && (xv > 0.0 || gv < 0.0);
    if (own) {
      if (wr) {
        a.x[slot][i] = xv;
        a.g[slot][i] = gv;
      }
      a.gbar[slot][i] = pf ? gv : 0.0;
    }
    const double el = lead ? (double)(globaltimer_ns() - t0) * 1e-9 : 0.0;
    write_partials(a.part[slot] + b, S, pf ? gv * gv : 0.0, own ? xv * gv : 0.0,
                   own ? qi * xv : 0.0,
                   own ? xv : __longlong_as_double(0x7ff0000000000000LL), df, el,
                   pf ? 1 : 0, own && !isfinite(gv) ? 1 : 0, chg);
  };
  // stage gbar (and x) of state `slot` into shared memory with threads [first, kFT)
  // Staging of gbar (and x) of state `slot` into shared memory: ONE thread issues
  // bulk copies (cp.async.bulk, TMA 1D) completing on an mbarrier, so the staging
  // needs no registers and costs one round trip; the other warps meanwhile reduce
  // the partials. (Vectors are padded to even length: the byte counts are
  // multiples of 16.)
  uint32_t sphase = 0;
  if (threadIdx.x == 0) {
    mbar_init(&S.sbar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto stage_issue = [&](int slot) {
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const uint32_t bytes = (uint32_t)mp * 8u;
      mbar_arrive_expect_tx(&S.sbar, lk ? 2u * bytes : bytes);
      constexpr uint32_t kChunk = 65536;
      for (uint32_t off = 0; off < bytes; off += kChunk) {
        const uint32_t nb = bytes - off < kChunk ? bytes - off : kChunk;
        bulk_g2s(reinterpret_cast<uint8_t*>(gs) + off,
                 reinterpret_cast<const uint8_t*>(a.gbar[slot]) + off, nb, &S.sbar);
        if (lk)
          bulk_g2s(reinterpret_cast<uint8_t*>(xs) + off,
                   reinterpret_cast<const uint8_t*>(a.x[slot]) + off, nb, &S.sbar);
      }
    }
  };
  auto stage_wait = [&]() {
    mbar_wait(&S.sbar, sphase);
    sphase ^= 1u;
  };
  int cur = 0;
  publish_state(0, xi, gi, 0.0, 0, false);
  // lead-thread counters (written to the control block at the end)
  unsigned long long n_trace = 0, n_mult = 0, mult_total = 0;
  double min_it = 0.0;
  bar.sync();
  stage_issue(0);
  if (warp < kRedWarps) reduce_partials(a.part[0], nblk, S);
  __syncthreads();
  stage_wait();
  min_it = m ? S.tot.minx : 0.0;  // min(start) (nqp.hpp:237)
  double best_gbs = __longlong_as_double(0x7ff0000000000000LL);
  unsigned long long since_best = 0;
  double el = S.tot.el;
  // CTA 0 thread 0 phase clock (alnnls_get_phase_ns): [0] stop test, [1] Q gbar pass
  // + den partial, [2] barrier A + den, [3] clamped set (+ barrier A2 without lk),
  // [4] Q_K c_K pass, [5] update + partials, [6] barrier B + totals + staging
  if (threadIdx.x < 8) S.ph[threadIdx.x] = 0;
  unsigned long long tmark = globaltimer_ns();
  auto mark = [&](int idx) {
    if (ALNNLS_FAST_PHASES && lead) {
      const unsigned long long t = globaltimer_ns();
      S.ph[idx] += t - tmark;
      tmark = t;
    }
  };

  unsigned long long tsamp = 0;  // k % trace_every, kept incrementally
  for (unsigned long long k = 0;; ++k, tsamp = tsamp + 1 == a.trace_every ? 0 : tsamp + 1) {
    // ===== stop tests on the current state (nqp.hpp:249-275), identical in every CTA ====
    const double gbs = S.tot.gbs;
    const double f = 0.5 * (S.tot.xg + S.tot.qx);
    const int ml = S.tot.cnt;
    int stop = -1;
    if (S.tot.bad || !isfinite(f) || !isfinite(gbs)) {
      stop = 100;  // NumericFailure (nqp.hpp:257-259)
    } else if (ml == 0) {
      stop = ALNNLS_EMPTY_PASSIVE_SET;
    } else if (gbs < a.eps) {
      stop = ALNNLS_GRADIENT_BELOW_EPSILON;
    } else if (k >= a.max_iters) {
      stop = ALNNLS_MAX_ITERS;
    } else if (a.has_time_cap && el >= a.time_cap_s) {
      stop = ALNNLS_TIME_CAP;
    } else if (gbs < best_gbs) {
      best_gbs = gbs;
      since_best = 0;
    } else if (++since_best >= a.stall_window) {
      stop = ALNNLS_STALLED;
    }
    if (stop < 0 && !(gbs != 0.0)) stop = ALNNLS_ZERO_CURVATURE;  // num == 0 (nqp.hpp:167)
    if (stop >= 0) {
      if (lead) {
        if (stop == 100) {
          a.ctrl->numeric_failure = 1;
        } else {
          fast_record(a, n_trace, k, f, gbs, ml, el, 0.0, 0);
          a.ctrl->termination = stop;
          a.ctrl->iterations = k;
          a.ctrl->f_final = f;
          a.ctrl->gbs_final = gbs;
        }
      }
      break;
    }
    mark(0);

    // ===== u = Q gbar over own rows (one streaming pass over the passive columns) =====
    double acc0 = 0.0, acc1 = 0.0;
    if (gthr) panel_pass<kL2>(Qp, R, m, gs, grp, C, r2, acc0, acc1, pol);
    const double ui = rows_from_groups(red, rsum, gthr, grp, R, r2, acc0, acc1, C, nrows);
    {
      const double dn = block_sum(own ? gs[i] * ui : 0.0, S);
      if (threadIdx.x == 0) a.den[b] = dn;
    }
    mark(1);
    bar.sync();  // A
    if (warp == 0) {
      const double sd = reduce_den(a.den, nblk);
      if (lane == 0) S.den = sd;
    }
    __syncthreads();
    mark(2);
    const double den = S.den;
    if (!(den > 0.0)) {  // exact_step returns nullopt (nqp.hpp:171) -> ZeroCurvature
      if (lead) {
        fast_record(a, n_trace, k, f, gbs, ml, el, 0.0, 0);
        a.ctrl->termination = ALNNLS_ZERO_CURVATURE;
        a.ctrl->iterations = k;
        a.ctrl->f_final = f;
        a.ctrl->gbs_final = gbs;
      }
      break;
    }
    double alpha = gbs / den;
    unsigned long long mults = (unsigned long long)m * (unsigned long long)ml;
    const bool pas = own && (xi > 0.0 || gi < 0.0);
    const int nxt = cur ^ 1;
    for (int tries = 0;; ++tries) {
      // ---- clamped set K: x_j - alpha g_j < 0 on P (nqp.hpp:295-296), ascending j ----
      // (on P with g_j > 0; g_j <= 0 never clamps). c_j = alpha g_j - x_j.
      double v0 = 0.0, v1 = 0.0;
      int ktot = 0;
      if (lk) {
        // every CTA scans the staged state: warp w owns a contiguous range, lanes
        // read consecutive entries, a ballot per round keeps ascending order
        const int pw = ((m + kFW - 1) / kFW + 31) & ~31;
        const int j0 = warp * pw, j1 = min(m, j0 + pw);
        int cnt = 0;
        for (int jb = j0; jb < j1; jb += 32) {
          const int j = jb + lane;
          const double gv = j < j1 ? gs[j] : 0.0;
          const bool cl = gv > 0.0 && xs[j] < alpha * gv;
          cnt += __popc(__ballot_sync(0xffffffffu, cl));
        }
        if (lane == 0) S.scan[warp] = cnt;
        __syncthreads();
        if (threadIdx.x == 0) {
          int run = 0;
          for (int w = 0; w < kFW; ++w) {
            const int c = S.scan[w];
            S.scan[w] = run;
            run += c;
          }
          S.scan[kFW] = run;
        }
        __syncthreads();
        ktot = S.scan[kFW];
        mark(3);
        for (int w0 = 0; w0 < ktot; w0 += kKWin) {  // windows of K (one unless |K| > kKWin)
          int pos = S.scan[warp];
          for (int jb = j0; jb < j1 && pos < w0 + kKWin; jb += 32) {
            const int j = jb + lane;
            const double gv = j < j1 ? gs[j] : 0.0;
            const double ag = alpha * gv;
            const bool cl = gv > 0.0 && xs[j] < ag;
            const unsigned bl = __ballot_sync(0xffffffffu, cl);
            const int p = pos + __popc(bl & ((1u << lane) - 1u));
            if (cl && p >= w0 && p < w0 + kKWin) {
              kjs[p - w0] = (uint32_t)j;
              kvs[p - w0] = ag - xs[j];
            }
            pos += __popc(bl);
          }
          __syncthreads();
          if (gthr) {
            list_pass<kL2>(Qp, R, kjs, kvs, min(kKWin, ktot - w0), grp, C, r2, v0, v1, pol);
          }
          __syncthreads();
        }
      } else {
        const double ag = alpha * gi;
        const bool clamp = pas && gi > 0.0 && xi < ag;
        {
          int tot = 0;
          const int pos = block_exclusive_scan(clamp ? 1 : 0, S.scan, &tot);
          if (clamp) {
            a.kl[(size_t)b * R + pos] = (uint32_t)i;
            a.kv[(size_t)b * R + pos] = ag - xi;  // c_i = delta_i + alpha g_i
          }
          if (threadIdx.x == 0) a.kc[b] = tot;
        }
        bar.sync();  // A2
        if (warp == 0) {  // prefix of the per-CTA counts: K in ascending row order
          int run = 0;
          for (int b0 = 0; b0 < nblk; b0 += 32) {
            const int bb = b0 + lane;
            const int v = bb < nblk ? __ldcg(a.kc + bb) : 0;
            int incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int t = __shfl_up_sync(0xffffffffu, incl, o);
              if (lane >= o) incl += t;
            }
            if (bb < nblk) S.kpre[bb] = run + incl - v;
            run += __shfl_sync(0xffffffffu, incl, 31);
          }
          if (lane == 0) S.kpre[nblk] = run;
        }
        __syncthreads();
        mark(3);
        ktot = S.kpre[nblk];
        for (int w0 = 0; w0 < ktot; w0 += kKWin) {
          const int wn = min(kKWin, ktot - w0);
          for (int t = threadIdx.x; t < wn; t += kFT) {
            const int p = w0 + t;
            int lo = 0, hi = nblk - 1;  // last bb with kpre[bb] <= p
            while (lo < hi) {
              const int mid = (lo + hi + 1) >> 1;
              if (S.kpre[mid] <= p) lo = mid;
              else hi = mid - 1;
            }
            const size_t e = (size_t)lo * R + (p - S.kpre[lo]);
            kjs[t] = __ldcg(a.kl + e);
            kvs[t] = __ldcg(a.kv + e);
          }
          __syncthreads();
          if (gthr) {
            list_pass<kL2>(Qp, R, kjs, kvs, wn, grp, C, r2, v0, v1, pol);
          }
          __syncthreads();
        }
      }
      double vi = 0.0;
      if (ktot > 0) {
        vi = rows_from_groups(red, rsum, gthr, grp, R, r2, v0, v1, C, nrows);
        mults += (unsigned long long)m * (unsigned long long)ktot;
      }
      mark(4);
      // ---- speculative update of own rows (nqp.hpp:294-313, one-pass Q delta) ----
      const double gd = fma(-alpha, ui, vi);
      double xn = xi, delta = 0.0;
      bool chg = false;
      if (pas) {
        double c = xi - alpha * gi;  // cand = max(0, x - alpha g)
        if (c < 0.0) c = 0.0;
        delta = c - xi;
        chg = c != xi;
        xn = c;
      }
      const double gn = gi + gd;
      const double dft = chg ? (gi + 0.5 * gd) * delta : 0.0;
      publish_state(nxt, xn, gn, dft, chg ? 1 : 0, true);
      mark(5);
      bar.sync();  // B
      // totals of the new state (warp 0) while the other warps stage it speculatively
      stage_issue(nxt);
      if (warp < kRedWarps) reduce_partials(a.part[nxt], nblk, S);
      __syncthreads();
      stage_wait();
      mark(6);
      el = S.tot.el;
      const int nchg = S.tot.nchg;
      const double df = S.tot.df;
      if (nchg == 0 || df <= 0.0 || tries >= 60) {
        // step taken (or too small to move anything, nqp.hpp:304): record it
        if (lead) {
          if (tsamp == 0) fast_record(a, n_trace, k, f, gbs, ml, el, alpha, 1);
          if (a.mults && a.mults_cap > 0)
            a.mults[n_mult < a.mults_cap ? n_mult : a.mults_cap - 1] = mults;
          ++n_mult;
          mult_total += mults;
        }
        if (nchg != 0) {  // accept: the speculative state becomes current
          if (S.tot.minx < min_it) min_it = S.tot.minx;
          xi = xn;
          gi = gn;
          cur = nxt;
        } else {          // nothing moved: the state (and its totals) stay
          __syncthreads();
          stage_issue(cur);
          if (warp < kRedWarps) reduce_partials(a.part[cur], nblk, S);
          __syncthreads();
          stage_wait();
          if (threadIdx.x == 0) S.tot.el = el;
        }
        break;
      }
      alpha *= 0.5;  // nqp.hpp:317
      __syncthreads();
      stage_issue(cur);  // the rejected state was staged: back to the current one
      stage_wait();
    }
    __syncthreads();
  }
  if (lead) {
    a.ctrl->trace_len = n_trace;
    a.ctrl->mult_len = n_mult;
    a.ctrl->mult_total = mult_total;
    a.ctrl->min_iterate = min_it;
    a.ctrl->g_parity = cur;
    for (int q = 0; q < 7; ++q) a.ctrl->phase_ns[q] = S.ph[q];
  }
}
}  // namespace

namespace {
constexpr size_t kFastSmemCap = 227 * 1024;  // static + dynamic per CTA
// static shared memory of the kernel as compiled (FastShared plus alignment)
size_t fast_static_smem() {
  static size_t v = [] {
    cudaFuncAttributes fa{};
    size_t mx = sizeof(FastShared) + 256;
    if (cudaFuncGetAttributes(&fa, fast_loop_kernel<false, false>) == cudaSuccess && fa.sharedSizeBytes > mx)
      mx = fa.sharedSizeBytes;
    if (cudaFuncGetAttributes(&fa, fast_loop_kernel<true, false>) == cudaSuccess && fa.sharedSizeBytes > mx)
      mx = fa.sharedSizeBytes;
    (void)cudaGetLastError();
    return mx;
  }();
  return v;
}
}

bool fast_loop_supported(int m, int R) {
  if (m < 1 || R < 2 || (R & 1) || R > kFT) return false;  // one thread per own row
  const int nblk = (m + R - 1) / R;
  if (nblk > kFastMaxBlk || nblk > 148) return false;
  if ((kFT / (R / 2)) * R > kRedDoubles) return false;
  return fast_smem_bytes(m, false) + fast_static_smem() <= kFastSmemCap;
}

template <bool kL2>
cudaError_t launch_fast_loop_t(const FastArgs& a0, cudaStream_t stream);

cudaError_t launch_fast_loop(const FastArgs& a0, cudaStream_t stream) {
  // L2 residency hints only when a sizable fraction of Q fits the L2 (c2 / c3: 0.7);
  // env ALNNLS_FAST_L2_FRAC overrides (A/B)
  const double qbytes = 8.0 * (double)a0.m * (double)a0.m;
  double f = 94e6 / qbytes;
  if (f > 1.0) f = 1.0;
  if (const char* e = getenv("ALNNLS_FAST_L2_FRAC")) f = atof(e);
  FastArgs a = a0;
  a.l2_frac = (float)f;
  return f >= 0.3 || f < 0.0 ? launch_fast_loop_t<true>(a, stream)
                              : launch_fast_loop_t<false>(a, stream);
}

template <bool kL2>
cudaError_t launch_fast_loop_t(const FastArgs& a0, cudaStream_t stream) {
  if (!fast_loop_supported(a0.m, a0.R)) return cudaErrorInvalidValue;
  FastArgs args = a0;
  // x staged beside gbar when both fit: the clamped set is then found by every CTA
  // from shared memory, without the extra barrier (m up to ~13k)
  args.local_k = fast_smem_bytes(args.m, true) + fast_static_smem() <= kFastSmemCap ? 1 : 0;
  if (getenv("ALNNLS_FAST_FORCE_A2")) args.local_k = 0;  // test hook: the large-m path

  const int nblk = (args.m + args.R - 1) / args.R;
  const size_t smem = fast_smem_bytes(args.m, args.local_k != 0);
  // opt in once for the largest staging any m can need (the size varies with m)
  const int smax = (int)(kFastSmemCap - fast_static_smem());
  if (cudaError_t e = smem_optin(fast_loop_kernel<false, kL2>, smax)) return e;
  if (cudaError_t e = smem_optin(fast_loop_kernel<true, kL2>, smax)) return e;
  const bool cluster_ok =
      func_attr_once(reinterpret_cast<const void*>(fast_loop_kernel<true, kL2>),
                     cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
  (void)cudaGetLastError();
  if (cluster_ok && nblk <= 16) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(nblk);
    cfg.blockDim = dim3(kFT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = nblk;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, fast_loop_kernel<true, kL2>, &cfg);
    if (e == cudaSuccess && nclusters > 0) {
      e = cudaLaunchKernelEx(&cfg, fast_loop_kernel<true, kL2>, args);
      if (e == cudaSuccess) return e;
    }
    if (getenv("ALNNLS_DEBUG"))
      fprintf(stderr, "fast_loop: cluster %d launch not used (%s, %d clusters)\n", nblk,
              cudaGetErrorString(e), nclusters);
    (void)cudaGetLastError();  // no cluster of this size fits: cooperative grid instead
  }
  void* params[] = {&args};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)fast_loop_kernel<false, kL2>, dim3(nblk), dim3(kFT),
                                              params, smem, stream);
  if (e != cudaSuccess && getenv("ALNNLS_DEBUG"))
    fprintf(stderr, "fast_loop: cooperative %d x %d smem %zu: %s\n", nblk, kFT, smem,
            cudaGetErrorString(e));
  return e;
}

}  // namespace alnnls
