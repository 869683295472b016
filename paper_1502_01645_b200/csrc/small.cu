// small.cu — exact solve_nqp for small m as ONE thread-block cluster whose loop
// state lives in distributed shared memory (reference solve_nqp,
// /root/reference/proj/include/antilop/nqp.hpp:215-339).
//
// Latency, not bandwidth, bounds a small problem (c1: m = 300, Q = 720 KB): the
// general loop kernel (nqp.cu) passes every vector through global memory, so
// each phase of an iteration pays L2 round trips on top of its barrier. Here
// the Q panels stay resident in the row CTAs' shared memory and everything the
// CTAs exchange is published in a per-CTA shared block (SmallPub) that the
// other CTAs of the cluster read directly (DSMEM) after a cluster barrier.
//
// CTA 0 leads (stop test, df check, trace, counters); CTAs 1..C-1 own R rows of
// Q each. Per iteration (four cluster barriers):
//   publish  row CTAs: own passive entries (idx, g, x, q), count, min x, bad   B1
//   P1       row CTAs: gather the passive list, u = Q[:, P] g_P on own rows,
//            publish u at own passive rows; leader, concurrently: gather the
//            list, gbs / x.g / q.x chains, f, stop tests (nqp.hpp:250-275)      B2
//   den      every CTA: gather u, the den chain, alpha (nqp.hpp:162-173) --
//            computed redundantly, bit-identical, so no broadcast is needed;
//            the candidate step and the changed set (nqp.hpp:294-303), also
//            redundantly
//   P2       row CTAs: gd = Q[:, C] delta_C on own rows, publish the df terms
//            of own changed rows                                                 B5
//   df       leader: df chain (nqp.hpp:307), accept or halve                     B6
//   apply    row CTAs: x[C] = cand, g += gd (nqp.hpp:309-313)
// Every sum is one sequential chain in the reference's order (rounded products
// formed in parallel into shared memory, then one thread's dependent DADDs),
// so x, the gradient, every trace record and the multiply counts are bitwise
// the reference's (and the general kernel's).
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace alnnls {

namespace {

constexpr int kST = 384;        // threads per CTA
constexpr int kSR = 64;         // rows per row CTA (max)
constexpr int kSMaxM = 2 * kST; // list capacity (two entries per thread in the block scans)
constexpr size_t kSmallSmemMax = 220 * 1024;  // dynamic; the static SmallPub etc. take the rest of 227 KB

// Published by every CTA; read by the others through DSMEM after a barrier.
struct SmallPub {
  int np;        // row CTA: own passive entries of the current state
  int nc;        // row CTA: own entries of the changed set
  int bad;       // row CTA: a non-finite gradient entry among own rows
  int stop;      // leader: -1 continue, else stop (every CTA leaves the loop)
  int accept;    // leader: the df check's decision for the current candidate
  double minx;   // row CTA: min x over own rows
  double gbs;    // leader: gbs of the current iteration (alpha = gbs / den)
  uint32_t pidx[kSR];
  double pg[kSR], px[kSR], pq[kSR];  // g, x, q at own passive rows
  double pu[kSR];                    // (Q g_bar) at own passive rows
  double cdf[kSR];                   // df terms (g + gd/2) delta at own changed rows
};

__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// s = ((0 + p0) + p1) + ... over n rounded products in shared memory, one thread.
// Two register blocks alternate so the loads of the next block are in flight
// during the current block's dependent DADDs.
__device__ __forceinline__ double chain_smem(const double* __restrict__ p, int n) {
  constexpr int B = 16;
  double s = 0.0;
  int t = 0;
  if (n >= 2 * B) {
    double ra[B], rb[B];
#pragma unroll
    for (int k = 0; k < B; ++k) ra[k] = p[k];
    for (; t + 3 * B <= n; t += 2 * B) {
#pragma unroll
      for (int k = 0; k < B; ++k) rb[k] = p[t + B + k];
#pragma unroll
      for (int k = 0; k < B; ++k) s = xadd(s, ra[k]);
#pragma unroll
      for (int k = 0; k < B; ++k) ra[k] = p[t + 2 * B + k];
#pragma unroll
      for (int k = 0; k < B; ++k) s = xadd(s, rb[k]);
    }
    if (t + 2 * B <= n) {
#pragma unroll
      for (int k = 0; k < B; ++k) rb[k] = p[t + B + k];
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
  for (; t < n; ++t) s = xadd(s, p[t]);
  return s;
}

// Row GEMV over a resident panel (column-major, leading dimension R): thread t
// < nrows runs row t's chain over the list in order (products of a 64-column
// block, then their DADDs). Returns the row's sum.
__device__ __forceinline__ double panel_gemv(const double* __restrict__ Qs, int R, int t,
                                             const uint32_t* __restrict__ idx,
                                             const double* __restrict__ val, int len) {
  const double* q = Qs + t;
  double acc = 0.0;
  int s = 0;
  for (; s + 64 <= len; s += 64) {
    double p[64];
#pragma unroll
    for (int l = 0; l < 64; ++l) p[l] = xmul(q[(size_t)idx[s + l] * R], val[s + l]);
#pragma unroll
    for (int l = 0; l < 64; ++l) acc = xadd(acc, p[l]);
  }
  for (; s < len; ++s) acc = xmac(acc, q[(size_t)idx[s] * R], val[s]);
  return acc;
}

struct SmallCtl {  // leader-only loop state (global copies are written, never read back)
  double best_gbs;
  unsigned long long since_best;
  double f, el;
  double min_iterate;
  unsigned long long trace_len, mult_len, mult_total;
  int stepped;  // an accepted step since the last min_iterate update
};

__device__ void small_record(const LoopArgs& a, SmallCtl& c, unsigned long long k, double f,
                             double gbs, int pc, double el, double alpha, int has_alpha) {
  const unsigned long long i = c.trace_len;
  if (a.trace_cap > 0) {  // past the capacity the last slot keeps the newest record
    alnnls_iter_record r;
    r.iter = k;
    r.f = f;
    r.grad_bar_sq = gbs;
    r.passive_count = (uint64_t)pc;
    r.elapsed_s = el;
    r.alpha = has_alpha ? alpha : 0.0;
    r.has_alpha = has_alpha;
    a.trace[i < a.trace_cap ? i : a.trace_cap - 1] = r;
  }
  c.trace_len = i + 1;
}
// Stepped iteration bookkeeping (nqp.hpp:319-326).
__device__ void small_push(const LoopArgs& a, SmallCtl& c, unsigned long long k, double f,
                           double gbs, int ml, double el, double alpha, unsigned long long mults) {
  if (k % a.trace_every == 0) small_record(a, c, k, f, gbs, ml, el, alpha, 1);
  const unsigned long long i = c.mult_len;
  if (a.mults && i < a.mults_cap) a.mults[i] = mults;
  c.mult_len = i + 1;
  c.mult_total += mults;
}
__device__ void small_stop(const LoopArgs& a, SmallCtl& c, unsigned long long k, double f,
                           double gbs, int ml, double el, int term) {
  small_record(a, c, k, f, gbs, ml, el, 0.0, 0);
  a.ctrl->termination = term;
  a.ctrl->iterations = k;
  a.ctrl->f_final = f;
  a.ctrl->gbs_final = gbs;
}

// Gathers every row CTA's published entries (counts cnt_of(r), values get(r, j))
// into a contiguous list in CTA order; returns the total. Whole CTA.
template <class C, class G>
__device__ int gather_lists(int nblk, int* s_off, C cnt_of, G get) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    int c = lane < nblk ? cnt_of(lane + 1) : 0;
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane < nblk) s_off[lane] = incl - c;
    if (lane == 31) s_off[31] = incl;
  }
  __syncthreads();
  const int total = s_off[31];
  const int nw = blockDim.x >> 5;
  for (int r = warp; r < nblk; r += nw) {
    const int n = (r + 1 < nblk ? s_off[r + 1] : total) - s_off[r];
    for (int j = lane; j < n; j += 32) get(r + 1, j, s_off[r] + j);
  }
  __syncthreads();
  return total;
}

__global__ void __launch_bounds__(kST, 1) nqp_small_kernel(LoopArgs a) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ SmallPub pub;
  __shared__ SmallCtl ctl;
  __shared__ int s_off[32];
  __shared__ int s_scan[40];
  __shared__ double s_den, s_sum[3], s_wmin[kST / 32];
  __shared__ unsigned long long s_ph[8];
  __shared__ int s_clo, s_chi, s_bad;
  __shared__ double s_mn;
  const int rank = (int)cluster.block_rank();
  const int nblk = (int)cluster.num_blocks() - 1;
  const bool leader = rank == 0;
  const int m = a.m, R = a.rows_per_cta;
  const int row0 = leader ? 0 : (rank - 1) * R;
  const int nrows = leader ? 0 : max(0, min(m - row0, R));
  const int tid = threadIdx.x;

  // ---- shared-memory carve-up --------------------------------------------------------
  double* Qs = reinterpret_cast<double*>(smem);  // R x m panel (row CTAs)
  double* base = Qs + (leader ? 0 : (size_t)R * m);
  const int mc = (m + 1) & ~1;
  double* Lg = base;            // passive list: g
  double* Lx = Lg + mc;         //               x
  double* Lq = Lx + mc;         //               q
  double* Lu = Lq + mc;         //               (Q g_bar)
  double* T = Lu + mc;          // products of the current chain
  double* Cd = T + mc;          // changed list: delta
  double* Cc = Cd + mc;         //               candidate x
  double* xl = Cc + mc;         // own rows: x, g, q, gd
  double* gl = xl + kSR;
  double* ql = gl + kSR;
  double* gdl = ql + kSR;
  uint32_t* Li = reinterpret_cast<uint32_t*>(gdl + kSR);  // passive list: row index
  uint32_t* Ci = Li + mc;                                    // changed list: row index
  int* lpos = reinterpret_cast<int*>(Ci + mc);               // own row -> own passive slot

  auto remote = [&](int r) { return cluster.map_shared_rank(&pub, r); };

  // ---- prologue -------------------------------------------------------------------------
  if (!leader) {
    const double2* src = reinterpret_cast<const double2*>(a.Q + (size_t)(rank - 1) * R * m);
    double2* dst = reinterpret_cast<double2*>(Qs);
    for (int e = tid; e < R * m / 2; e += blockDim.x) dst[e] = __ldg(src + e);
    for (int t = tid; t < nrows; t += blockDim.x) {
      xl[t] = a.x[row0 + t];
      gl[t] = a.g[row0 + t];
      ql[t] = __ldg(a.q + row0 + t);
    }
  } else if (tid == 0) {
    a.ctrl->numeric_failure = 0;
    a.ctrl->g_parity = 0;
    ctl.best_gbs = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    ctl.since_best = 0;
    ctl.trace_len = 0;
    ctl.mult_len = 0;
    ctl.mult_total = 0;
    ctl.min_iterate = 0.0;
    ctl.stepped = 1;  // min_iterate starts at min(start) (nqp.hpp:237)
    for (int i = 0; i < 8; ++i) s_ph[i] = 0;
  }
  __syncthreads();
  const uint64_t t0 = globaltimer_ns();
  unsigned long long k = 0;
  uint64_t ph_t = t0;
  auto mark = [&](int i) {
    if (leader && tid == 0) {
      const uint64_t t = globaltimer_ns();
      s_ph[i] += t - ph_t;
      ph_t = t;
    }
  };

  for (;;) {
    // ===== publish: own passive entries (row CTAs) ===========================================
    if (!leader) {
      int f = 0, bad = 0;
      double xi = 0.0, gi = 0.0;
      if (tid < nrows) {
        xi = xl[tid];
        gi = gl[tid];
        f = (xi > 0.0 || gi < 0.0) ? 1 : 0;
        bad = !isfinite(gi);
      }
      int total = 0;
      const int pos = block_exclusive_scan(f, s_scan, &total);
      double mn = tid < nrows ? xi : __longlong_as_double(0x7ff0000000000000LL);
      for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      bad = __syncthreads_or(bad);
      if ((tid & 31) == 0) s_wmin[tid >> 5] = mn;
      if (tid < nrows) {
        lpos[tid] = f ? pos : -1;
        if (f) {
          pub.pidx[pos] = (uint32_t)(row0 + tid);
          pub.pg[pos] = gi;
          pub.px[pos] = xi;
          pub.pq[pos] = ql[tid];
        }
      }
      __syncthreads();
      if (tid == 0) {
        double m2 = s_wmin[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m2 = fmin(m2, s_wmin[w]);
        pub.np = total;
        pub.bad = bad;
        pub.minx = m2;
      }
    }
    cluster_barrier();  // B1
    mark(4);

    // ===== gather the passive list; P1 (row CTAs) || stop test (leader) =======================
    const int ml = gather_lists(
        nblk, s_off, [&](int r) { return remote(r)->np; },
        [&](int r, int j, int at) {
          const SmallPub* p = remote(r);
          Li[at] = p->pidx[j];
          Lg[at] = p->pg[j];
          Lx[at] = p->px[j];
          Lq[at] = p->pq[j];
        });
    if (!leader) {
      if (tid < nrows) {
        const double u = panel_gemv(Qs, R, tid, Li, Lg, ml);  // u = Q g_bar, own rows
        if (lpos[tid] >= 0) pub.pu[lpos[tid]] = u;
      }
    } else {
      // gbs: g^2 on the mask; dot(x, grad): x g; dot(q, x): q x (terms off the mask
      // are exact zeros: x = 0 there, g >= 0)
      if (tid >= 32 && tid < 64) {  // the row CTAs' flags and minima, one lane each
        const int r = tid - 32 + 1;
        int bad = 0;
        double mn = __longlong_as_double(0x7ff0000000000000LL);
        if (r <= nblk) {
          bad = remote(r)->bad;
          mn = remote(r)->minx;
        }
        for (int o = 16; o > 0; o >>= 1) {
          bad |= __shfl_xor_sync(0xffffffffu, bad, o);
          mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        }
        if (tid == 32) {
          s_bad = bad;
          s_mn = mn;
        }
      }
      for (int t = tid; t < ml; t += blockDim.x) {
        T[t] = xmul(Lg[t], Lg[t]);
        Lu[t] = xmul(Lx[t], Lg[t]);
        Cd[t] = xmul(Lq[t], Lx[t]);
      }
      __syncthreads();
      const int warp = tid >> 5;
      double r3 = 0.0;
      if ((tid & 31) == 0 && warp < 3) r3 = chain_smem(warp == 0 ? T : (warp == 1 ? Lu : Cd), ml);
      if ((tid & 31) == 0 && warp < 3) s_sum[warp] = r3;
      __syncthreads();
      if (tid == 0) {
        const double gbs = s_sum[0];
        const double f = xmul(0.5, xadd(s_sum[1], s_sum[2]));
        const double el = (double)(globaltimer_ns() - t0) * 1e-9;
        const int bad = s_bad;
        const double mn = s_mn;
        if (ctl.stepped) {  // min over the iterate after each stepped iteration (nqp.hpp:321-324)
          if (k == 0) ctl.min_iterate = m ? mn : 0.0;
          else if (m && mn < ctl.min_iterate) ctl.min_iterate = mn;
          ctl.stepped = 0;
        }
        int stop = -1;
        if (bad || !isfinite(f) || !isfinite(gbs)) {
          stop = 100;  // NumericFailure (nqp.hpp:257-259)
        } else if (ml == 0) {
          stop = ALNNLS_EMPTY_PASSIVE_SET;
        } else if (gbs < a.eps) {
          stop = ALNNLS_GRADIENT_BELOW_EPSILON;
        } else if (k >= a.max_iters) {
          stop = ALNNLS_MAX_ITERS;
        } else if (a.has_time_cap && el >= a.time_cap_s) {
          stop = ALNNLS_TIME_CAP;
        } else if (gbs < ctl.best_gbs) {
          ctl.best_gbs = gbs;
          ctl.since_best = 0;
        } else if (++ctl.since_best >= a.stall_window) {
          stop = ALNNLS_STALLED;
        }
        if (stop < 0 && !(gbs != 0.0)) stop = ALNNLS_ZERO_CURVATURE;  // num == 0 (nqp.hpp:167)
        if (stop == 100) a.ctrl->numeric_failure = 1;
        else if (stop >= 0) small_stop(a, ctl, k, f, gbs, ml, el, stop);
        ctl.f = f;
        ctl.el = el;
        pub.gbs = gbs;
        pub.stop = stop;
      }
    }
    cluster_barrier();  // B2
    mark(0);
    if (remote(0)->stop >= 0) break;

    // ===== den (every CTA, redundantly): gather u, the den chain, alpha ====================
    const double gbs = remote(0)->gbs;
    gather_lists(
        nblk, s_off, [&](int r) { return remote(r)->np; },
        [&](int r, int j, int at) { Lu[at] = remote(r)->pu[j]; });
    for (int t = tid; t < ml; t += blockDim.x) T[t] = xmul(Lg[t], Lu[t]);
    __syncthreads();
    if (tid == 0) s_den = chain_smem(T, ml);
    __syncthreads();
    const double den = s_den;
    mark(1);
    if (!(den > 0.0)) {
      if (leader && tid == 0) small_stop(a, ctl, k, ctl.f, gbs, ml, ctl.el, ALNNLS_ZERO_CURVATURE);
      break;
    }
    double alpha = xdiv(gbs, den);
    unsigned long long mults = (unsigned long long)m * (unsigned long long)ml;
    int tries = 0;
    bool moved = false;
    for (;;) {
      // ---- candidate step and changed set (every CTA, redundantly; nqp.hpp:294-303) ----
      int f0 = 0, f1 = 0;
      double c0 = 0.0, c1 = 0.0;
      const int e0 = 2 * tid, e1 = 2 * tid + 1;
      if (e0 < ml) {
        double xi = xsub(Lx[e0], xmul(alpha, Lg[e0]));  // x - (alpha g), nqp.hpp:296
        if (xi < 0.0) xi = 0.0;
        c0 = xi;
        f0 = xi != Lx[e0];
      }
      if (e1 < ml) {
        double xi = xsub(Lx[e1], xmul(alpha, Lg[e1]));
        if (xi < 0.0) xi = 0.0;
        c1 = xi;
        f1 = xi != Lx[e1];
      }
      int cl = 0;
      int pos = block_exclusive_scan(f0 + f1, s_scan, &cl);
      if (tid == 0) {
        s_clo = 0;
        s_chi = 0;
      }
      __syncthreads();
      if (f0) {
        Ci[pos] = Li[e0];
        Cd[pos] = xsub(c0, Lx[e0]);
        Cc[pos] = c0;
        ++pos;
      }
      if (f1) {
        Ci[pos] = Li[e1];
        Cd[pos] = xsub(c1, Lx[e1]);
        Cc[pos] = c1;
      }
      __syncthreads();
      if (cl == 0) break;  // nothing moved (nqp.hpp:304)
      mults += (unsigned long long)m * (unsigned long long)cl;
      // ---- P2 (row CTAs): gd = Q[:, C] delta_C on own rows; df terms of own changed rows ----
      if (!leader) {
        // own rows' slice [clo, chi) of the ascending changed list: the entries
        // below row0 and below row0 + nrows, counted by warp ballots
        for (int j0 = 0; j0 < cl; j0 += blockDim.x) {
          const int j = j0 + tid;
          const uint32_t i = j < cl ? Ci[j] : 0xffffffffu;
          const int lo = __popc(__ballot_sync(0xffffffffu, i < (uint32_t)row0));
          const int hi = __popc(__ballot_sync(0xffffffffu, i < (uint32_t)(row0 + nrows)));
          if ((tid & 31) == 0) {
            if (lo) atomicAdd(&s_clo, lo);
            if (hi) atomicAdd(&s_chi, hi);
          }
        }
        if (tid < nrows) gdl[tid] = panel_gemv(Qs, R, tid, Ci, Cd, cl);
        __syncthreads();
        const int clo = s_clo, nc = s_chi - s_clo;
        for (int j = tid; j < nc; j += blockDim.x) {
          const int t = (int)Ci[clo + j] - row0;
          pub.cdf[j] = xmul(xadd(gl[t], xmul(0.5, gdl[t])), Cd[clo + j]);  // nqp.hpp:307
        }
        if (tid == 0) pub.nc = nc;
      }
      cluster_barrier();  // B5
      mark(2);
      if (leader) {
        const int n = gather_lists(
            nblk, s_off, [&](int r) { return remote(r)->nc; },
            [&](int r, int j, int at) { T[at] = remote(r)->cdf[j]; });
        if (tid == 0) {
          const double df = chain_smem(T, n);
          pub.accept = (df <= 0.0 || tries >= 60) ? 1 : 0;
        }
      }
      cluster_barrier();  // B6
      mark(3);
      if (remote(0)->accept) {
        moved = true;
        break;
      }
      alpha = xmul(alpha, 0.5);  // nqp.hpp:317
      ++tries;
    }
    // ===== apply (nqp.hpp:309-313) and the step's bookkeeping ================================
    if (moved && !leader) {
      if (tid < nrows) gl[tid] = xadd(gl[tid], gdl[tid]);
      __syncthreads();
      const int clo = s_clo, nc = s_chi - s_clo;
      for (int j = tid; j < nc; j += blockDim.x) xl[(int)Ci[clo + j] - row0] = Cc[clo + j];
    }
    if (leader && tid == 0) {
      small_push(a, ctl, k, ctl.f, gbs, ml, ctl.el, alpha, mults);
      if (moved) ctl.stepped = 1;
    }
    ++k;
    __syncthreads();
  }
  // ---- epilogue: the final iterate and gradient of own rows, the leader's counters ---------
  if (leader && tid == 0) {
    a.ctrl->trace_len = ctl.trace_len;
    a.ctrl->mult_len = ctl.mult_len;
    a.ctrl->mult_total = ctl.mult_total;
    a.ctrl->min_iterate = ctl.min_iterate;
    for (int i = 0; i < 8; ++i) a.ctrl->phase_ns[i] = s_ph[i];
  }
  if (!leader)
    for (int t = tid; t < nrows; t += blockDim.x) {
      a.x[row0 + t] = xl[t];
      a.g[row0 + t] = gl[t];
    }
  cluster_barrier();  // no CTA leaves while another may still read its shared memory
}

size_t small_smem_bytes(int m, int R) {
  const size_t mc = (size_t)((m + 1) & ~1);
  return (size_t)R * m * 8 + 7 * mc * 8 + 4 * kSR * 8 + 2 * mc * 4 + kSR * 4 + 64;
}

}  // namespace

bool nqp_small_fits(int m, int R, int num_ctas) {
  return m >= 1 && m <= kSMaxM && R <= kSR && R % 2 == 0 && num_ctas >= 2 && num_ctas <= 16 &&
         small_smem_bytes(m, R) <= kSmallSmemMax;
}

// Launches the small-m cluster loop; cudaErrorNotSupported when the shape does not
// fit it or no cluster of that size can be placed (the caller takes the general loop).
cudaError_t launch_nqp_small(const LoopArgs& a, int num_ctas, cudaStream_t stream) {
#ifdef ALNNLS_NO_SMALL
  return cudaErrorNotSupported;
#endif
  if (!nqp_small_fits(a.m, a.rows_per_cta, num_ctas)) return cudaErrorNotSupported;
  const size_t smem = small_smem_bytes(a.m, a.rows_per_cta);
  // one opt-in at the largest size: function attributes are per (kernel, device), so a
  // per-shape value would be overwritten by the next smaller shape's
  if (cudaError_t e = smem_optin(nqp_small_kernel, (int)kSmallSmemMax)) return e;
  if (func_attr_once(reinterpret_cast<const void*>(nqp_small_kernel),
                     cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
    (void)cudaGetLastError();
    return cudaErrorNotSupported;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(num_ctas);
  cfg.blockDim = dim3(kST);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = num_ctas;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, nqp_small_kernel, &cfg) != cudaSuccess ||
      nclusters <= 0) {
    (void)cudaGetLastError();
    return cudaErrorNotSupported;
  }
  LoopArgs args = a;
  return cudaLaunchKernelEx(&cfg, nqp_small_kernel, args);
}

}  // namespace alnnls
