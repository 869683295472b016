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

#include "common.cuh"
#include "gemv.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace alnnls {

namespace {

constexpr int kFT = 512;            // threads per CTA
constexpr int kFW = kFT / 32;
constexpr int kKWin = 1024;         // clamped-set window staged in shared memory
constexpr int kRedDoubles = 1024;   // C x R column-group partials (C = kFT / (R/2))
constexpr int kFastMaxBlk = 256;

__host__ __device__ inline size_t fast_smem_bytes(int m) {
  const size_t mp = ((size_t)m + 1) & ~(size_t)1;
  return mp * sizeof(double) + kRedDoubles * sizeof(double) +
         kKWin * (sizeof(double) + sizeof(uint32_t));
}

struct FastShared {
  double wred[kFW][6];
  int wint[kFW][3];
  FastPart tot;       // cross-CTA totals of the last reduced record set
  double den;
  int kpre[kFastMaxBlk + 1];
  int scan[40];
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

// 128-bit streaming load of two doubles of Q (read-only for the whole kernel;
// no L1 allocation, Q is streamed once per pass).
__device__ __forceinline__ double2 ldq2(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p));
  return v;
}

// Thread (rp, c) accumulates rows (2rp, 2rp+1) over columns j = c, c+C, ... of
// the panel with coefficients w[j] (skipping w[j] == 0: no load).
__device__ __forceinline__ void panel_pass(const double* __restrict__ Qp, int R, int m,
                                           const double* __restrict__ w, int c, int C, int r2,
                                           double& acc0, double& acc1) {
  constexpr int U = 8;
  const double* base = Qp + r2;
  int j = c;
  for (; j + (U - 1) * C < m; j += U * C) {
    double gv[U];
    double2 qv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) gv[u] = w[j + u * C];
#pragma unroll
    for (int u = 0; u < U; ++u)
      qv[u] = gv[u] != 0.0 ? ldq2(base + (size_t)(j + u * C) * R) : make_double2(0.0, 0.0);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc0 = fma(qv[u].x, gv[u], acc0);
      acc1 = fma(qv[u].y, gv[u], acc1);
    }
  }
  for (; j < m; j += C) {
    const double gv = w[j];
    if (gv != 0.0) {
      const double2 qv = ldq2(base + (size_t)j * R);
      acc0 = fma(qv.x, gv, acc0);
      acc1 = fma(qv.y, gv, acc1);
    }
  }
}

// Thread (rp, c) over a staged list of (column, coefficient) pairs, t = c, c+C, ...
__device__ __forceinline__ void list_pass(const double* __restrict__ Qp, int R,
                                          const uint32_t* __restrict__ kj,
                                          const double* __restrict__ kv, int len, int c, int C,
                                          int r2, double& acc0, double& acc1) {
  const double* base = Qp + r2;
  for (int t = c; t < len; t += C) {
    const double2 qv = ldq2(base + (size_t)kj[t] * R);
    acc0 = fma(qv.x, kv[t], acc0);
    acc1 = fma(qv.y, kv[t], acc1);
  }
}

// Column-group partials -> per-row sums: row t (thread t < nrows) adds the C
// partials in ascending group order (fixed).
__device__ __forceinline__ double rows_from_groups(double* red, bool gthr, int c, int R, int r2,
                                                   double acc0, double acc1, int C, int nrows) {
  if (gthr) *reinterpret_cast<double2*>(red + (size_t)c * R + r2) = make_double2(acc0, acc1);
  __syncthreads();
  double s = 0.0;
  if ((int)threadIdx.x < nrows) {
    for (int k = 0; k < C; ++k) s += red[(size_t)k * R + threadIdx.x];
  }
  __syncthreads();
  return s;
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
  if (threadIdx.x == 0) {
    FastPart p;
    p.gbs = p.xg = p.qx = p.df = 0.0;
    p.minx = __longlong_as_double(0x7ff0000000000000LL);
    p.cnt = p.bad = p.nchg = 0;
    for (int k = 0; k < kFW; ++k) {
      p.gbs += S.wred[k][0];
      p.xg += S.wred[k][1];
      p.qx += S.wred[k][2];
      p.minx = fmin(p.minx, S.wred[k][3]);
      p.df += S.wred[k][4];
      p.cnt += S.wint[k][0];
      p.bad |= S.wint[k][1];
      p.nchg += S.wint[k][2];
    }
    p.el = el;
    p.pad = 0;
    *dst = p;
  }
  __syncthreads();
}

// Totals over the nblk per-CTA records (every CTA, same fixed order): warp 0,
// lane l sums records l, l+32, ... then an xor tree. el is record 0's.
__device__ void reduce_partials(const FastPart* src, int nblk, FastShared& S) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double gbs = 0.0, xg = 0.0, qx = 0.0, df = 0.0;
    double mnx = __longlong_as_double(0x7ff0000000000000LL);
    int cnt = 0, bad = 0, nchg = 0;
    for (int b = lane; b < nblk; b += 32) {
      const FastPart* p = src + b;
      gbs += __ldcg(&p->gbs);
      xg += __ldcg(&p->xg);
      qx += __ldcg(&p->qx);
      df += __ldcg(&p->df);
      mnx = fmin(mnx, __ldcg(&p->minx));
      cnt += __ldcg(&p->cnt);
      bad |= __ldcg(&p->bad);
      nchg += __ldcg(&p->nchg);
    }
    gbs = warp_sum(gbs);
    xg = warp_sum(xg);
    qx = warp_sum(qx);
    df = warp_sum(df);
    mnx = warp_min(mnx);
    cnt = warp_isum(cnt);
    bad = __any_sync(0xffffffffu, bad != 0) ? 1 : 0;
    nchg = warp_isum(nchg);
    if (lane == 0) {
      S.tot.gbs = gbs;
      S.tot.xg = xg;
      S.tot.qx = qx;
      S.tot.df = df;
      S.tot.minx = mnx;
      S.tot.cnt = cnt;
      S.tot.bad = bad;
      S.tot.nchg = nchg;
      S.tot.el = __ldcg(&src[0].el);
    }
  }
  __syncthreads();
}

__device__ void fast_record(const FastArgs& a, unsigned long long k, double f, double gbs, int pc,
                            double el, double alpha, int has_alpha) {
  LoopCtrl* c = a.ctrl;
  const unsigned long long idx = c->trace_len;
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
  c->trace_len = idx + 1;
}

template <bool kCluster>
__global__ void __launch_bounds__(kFT, 1) fast_loop_kernel(FastArgs a) {
  Barrier<kCluster> bar;
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ FastShared S;
  const int m = a.m, R = a.R;
  const int b = blockIdx.x, nblk = gridDim.x;
  const int row0 = b * R;
  const int nrows = max(0, min(m - row0, R));
  double* gs = reinterpret_cast<double*>(smem);                   // gbar of the state, m
  double* red = gs + ((m + 1) & ~1);                              // kRedDoubles
  double* kvs = red + kRedDoubles;                                // kKWin coefficients
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
  const uint64_t t0 = globaltimer_ns();

  // ---- this thread's row of the current state --------------------------------------
  double xi = 0.0, gi = 0.0, qi = 0.0;
  if (own) {
    xi = a.x[0][i];
    gi = a.g[0][i];
    qi = a.q[i];
  }
  auto publish_state = [&](int slot, double xs, double gsv, double df, int chg, bool wr) {
    // gbar, x, g of own rows and this CTA's partials of the state (xs, gsv)
    const bool pf = own && (xs > 0.0 || gsv < 0.0);
    if (own && wr) {
      a.x[slot][i] = xs;
      a.g[slot][i] = gsv;
    }
    if (own) a.gbar[slot][i] = pf ? gsv : 0.0;
    const double el = lead ? (double)(globaltimer_ns() - t0) * 1e-9 : 0.0;
    write_partials(a.part[slot] + b, S, pf ? gsv * gsv : 0.0, own ? xs * gsv : 0.0,
                   own ? qi * xs : 0.0,
                   own ? xs : __longlong_as_double(0x7ff0000000000000LL), df, el,
                   pf ? 1 : 0, own && !isfinite(gsv) ? 1 : 0, chg);
  };
  int cur = 0;
  publish_state(0, xi, gi, 0.0, 0, false);
  if (lead) {
    a.ctrl->trace_len = 0;
    a.ctrl->mult_len = 0;
    a.ctrl->mult_total = 0;
    a.ctrl->numeric_failure = 0;
  }
  bar.sync();
  reduce_partials(a.part[0], nblk, S);
  if (lead) a.ctrl->min_iterate = m ? S.tot.minx : 0.0;  // min(start) (nqp.hpp:237)
  double best_gbs = __longlong_as_double(0x7ff0000000000000LL);
  unsigned long long since_best = 0;
  double el = S.tot.el;

  for (unsigned long long k = 0;; ++k) {
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
          fast_record(a, k, f, gbs, ml, el, 0.0, 0);
          a.ctrl->termination = stop;
          a.ctrl->iterations = k;
          a.ctrl->f_final = f;
          a.ctrl->gbs_final = gbs;
        }
      }
      break;
    }

    // ===== u = Q gbar over own rows (one streaming pass over the passive columns) =====
    {
      const double* src = a.gbar[cur];
      for (int e = threadIdx.x; e < m; e += kFT) gs[e] = __ldcg(src + e);
    }
    __syncthreads();
    double acc0 = 0.0, acc1 = 0.0;
    if (gthr) panel_pass(Qp, R, m, gs, grp, C, r2, acc0, acc1);
    const double ui = rows_from_groups(red, gthr, grp, R, r2, acc0, acc1, C, nrows);
    {
      const double dn = block_sum(own ? gs[i] * ui : 0.0, S);
      if (threadIdx.x == 0) a.den[b] = dn;
    }
    bar.sync();  // A
    if (threadIdx.x < 32) {
      double s = 0.0;
      for (int bb = threadIdx.x; bb < nblk; bb += 32) s += __ldcg(a.den + bb);
      s = warp_sum(s);
      if (threadIdx.x == 0) S.den = s;
    }
    __syncthreads();
    const double den = S.den;
    if (!(den > 0.0)) {  // exact_step returns nullopt (nqp.hpp:171) -> ZeroCurvature
      if (lead) {
        fast_record(a, k, f, gbs, ml, el, 0.0, 0);
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
      // ---- clamped set K of own rows: x_i - alpha g_i < 0 on P (nqp.hpp:295-296) ----
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
      if (threadIdx.x < 32) {  // prefix of the per-CTA counts: K in ascending row order
        int run = 0;
        for (int b0 = 0; b0 < nblk; b0 += 32) {
          const int bb = b0 + (int)threadIdx.x;
          const int v = bb < nblk ? __ldcg(a.kc + bb) : 0;
          int incl = v;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if ((int)threadIdx.x >= o) incl += t;
          }
          if (bb < nblk) S.kpre[bb] = run + incl - v;
          run += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (threadIdx.x == 0) S.kpre[nblk] = run;
      }
      __syncthreads();
      const int ktot = S.kpre[nblk];
      double vi = 0.0;
      if (ktot > 0) {
        double v0 = 0.0, v1 = 0.0;
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
          if (gthr) list_pass(Qp, R, kjs, kvs, wn, grp, C, r2, v0, v1);
          __syncthreads();
        }
        vi = rows_from_groups(red, gthr, grp, R, r2, v0, v1, C, nrows);
        mults += (unsigned long long)m * (unsigned long long)ktot;
      }
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
      bar.sync();  // B
      reduce_partials(a.part[nxt], nblk, S);
      el = S.tot.el;
      const int nchg = S.tot.nchg;
      const double df = S.tot.df;
      if (nchg == 0 || df <= 0.0 || tries >= 60) {
        // step taken (or too small to move anything, nqp.hpp:304): record it
        if (lead) {
          if (k % a.trace_every == 0) fast_record(a, k, f, gbs, ml, el, alpha, 1);
          const unsigned long long idx = a.ctrl->mult_len;
          if (a.mults && a.mults_cap > 0) a.mults[idx < a.mults_cap ? idx : a.mults_cap - 1] = mults;
          a.ctrl->mult_len = idx + 1;
          a.ctrl->mult_total += mults;
        }
        if (nchg != 0) {  // accept: the speculative state becomes current
          if (lead && S.tot.minx < a.ctrl->min_iterate) a.ctrl->min_iterate = S.tot.minx;
          xi = xn;
          gi = gn;
          cur = nxt;
        } else {          // nothing moved: the state (and its totals) stay
          __syncthreads();
          reduce_partials(a.part[cur], nblk, S);
          if (threadIdx.x == 0) S.tot.el = el;
        }
        break;
      }
      alpha *= 0.5;  // nqp.hpp:317
    }
    __syncthreads();
  }
  if (lead) a.ctrl->g_parity = cur;
}

}  // namespace

bool fast_loop_supported(int m, int R) {
  if (m < 1 || R < 2 || (R & 1) || R / 2 > kFT) return false;
  const int nblk = (m + R - 1) / R;
  if (nblk > kFastMaxBlk || nblk > 148) return false;
  if ((kFT / (R / 2)) * R > kRedDoubles) return false;
  return fast_smem_bytes(m) + sizeof(FastShared) <= 227 * 1024;
}

cudaError_t launch_fast_loop(const FastArgs& a, cudaStream_t stream) {
  if (!fast_loop_supported(a.m, a.R)) return cudaErrorInvalidValue;
  const int nblk = (a.m + a.R - 1) / a.R;
  const size_t smem = fast_smem_bytes(a.m);
  if (cudaError_t e = smem_optin(fast_loop_kernel<false>, (int)smem)) return e;
  if (cudaError_t e = smem_optin(fast_loop_kernel<true>, (int)smem)) return e;
  const bool cluster_ok =
      func_attr_once(reinterpret_cast<const void*>(fast_loop_kernel<true>),
                     cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess;
  (void)cudaGetLastError();
  FastArgs args = a;
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
    if (cudaOccupancyMaxActiveClusters(&nclusters, fast_loop_kernel<true>, &cfg) == cudaSuccess &&
        nclusters > 0)
      return cudaLaunchKernelEx(&cfg, fast_loop_kernel<true>, args);
    (void)cudaGetLastError();
  }
  void* params[] = {&args};
  return cudaLaunchCooperativeKernel((void*)fast_loop_kernel<false>, dim3(nblk), dim3(kFT), params,
                                     smem, stream);
}

}  // namespace alnnls
