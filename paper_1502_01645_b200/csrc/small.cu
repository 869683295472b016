// small.cu — exact solve_nqp for small m as ONE thread-block cluster whose loop
// state lives in distributed shared memory (reference solve_nqp,
// /root/reference/proj/include/antilop/nqp.hpp:215-339).
//
// Latency, not bandwidth, bounds a small problem (c1: m = 300, Q = 720 KB): the
// general loop kernel (nqp.cu) passes every vector through global memory, so
// each phase of an iteration pays L2 round trips on top of its barrier. Here
// the Q panels stay resident in the row CTAs' shared memory and everything the
// CTAs exchange is pushed with remote stores into the shared memory of the CTAs
// that need it (DSMEM) before a cluster barrier, so no CTA waits on a remote
// load after one.
//
// CTA 0 leads (stop test, df check, trace, counters); CTAs 1..C-1 own R rows of
// Q each. Per iteration (two cluster barriers):
//   publish  row CTAs: own passive entries (idx, g, x, q), count, min x, bad,
//            and the df terms of the pending step                              B1
//   P1       row CTAs: gather the passive list, u = Q[:, P] g_P on own rows,
//            publish u at own passive rows; leader, concurrently: gather the
//            list, gbs / x.g / q.x chains, f, stop tests (nqp.hpp:250-275),
//            and the df chain of the pending step (nqp.hpp:307): a rejection
//            rolls the step back and halves it (nqp.hpp:316-317)              B2
//   den      every CTA: gather u, the den chain, alpha (nqp.hpp:162-173) --
//            computed redundantly, bit-identical, so no broadcast is needed;
//            the candidate step and the changed set (nqp.hpp:294-303), also
//            redundantly
//   P2       row CTAs: gd = Q[:, C] delta_C on own rows, the df terms of own
//            changed rows, then the step is applied speculatively
//            (x[C] = cand, g += gd, nqp.hpp:309-313; x and g kept for a rollback)
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
constexpr size_t kSmallSmemMax = 220 * 1024;  // dynamic; the static SmallBox etc. take the rest of 227 KB

// Filled by the other CTAs with remote (DSMEM) stores before a cluster barrier:
// every CTA pushes what the others need, so nothing is fetched across the
// cluster after a barrier (a push costs no round trip; a pull costs one or two).
struct SmallBox {
  int np[16];       // passive count of row CTA r + 1 (the segment Sidx.. of r)
  int nc[16];       // leader: changed count of row CTA r + 1 (the segment Sdf of r)
  int bad[16];      // leader: a non-finite gradient entry among row CTA r + 1's rows
  double minx[16];  // leader: min x over row CTA r + 1's rows
  int act;          // from the leader: continue / stop / roll back (SmallAct)
  double gbs;       // from the leader: gbs of the current iteration (alpha = gbs / den)
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

// Offsets of the row CTAs' segments in the concatenated list (exclusive scan of the
// counts, total in off[31]). Warp 0; the caller synchronises.
__device__ __forceinline__ void seg_offsets(const int* cnt, int nblk, int* off) {
  const int lane = threadIdx.x & 31;
  const int c = lane < nblk ? cnt[lane] : 0;
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane < nblk) off[lane] = incl - c;
  if (lane == 31) off[31] = incl;
}

enum SmallAct { kSmallCont = 0, kSmallStop = 1, kSmallRollback = 2 };

__global__ void __launch_bounds__(kST, 1) nqp_small_kernel(LoopArgs a) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ SmallBox box;
  __shared__ SmallCtl ctl;
  __shared__ int s_offP[32], s_offC[32], s_cntP[16];
  __shared__ int s_scan[40];
  __shared__ double s_den, s_sum[4], s_wmin[kST / 32];
  __shared__ unsigned long long s_ph[8];
  __shared__ int s_clo, s_chi, s_bad;
  __shared__ double s_mn;
  const int rank = (int)cluster.block_rank();
  const int C = (int)cluster.num_blocks();
  const int nblk = C - 1;
  const bool leader = rank == 0;
  const int m = a.m, R = a.rows_per_cta;
  const int row0 = leader ? 0 : (rank - 1) * R;
  const int nrows = leader ? 0 : max(0, min(m - row0, R));
  const int tid = threadIdx.x;
  const int ns = nblk * R;  // segmented arrays: row CTA r's segment at (r - 1) * R

  // ---- shared-memory carve-up (small_smem_bytes) ----------------------------------------
  // the layout is identical in every CTA (the leader leaves the panel unused): remote
  // stores address another CTA's arrays at this CTA's offsets
  double* Qs = reinterpret_cast<double*>(smem);  // R x m panel (row CTAs)
  double* base = Qs + (size_t)R * m;
  const int mc = (m + 1) & ~1;
  // passive lists (g, x, q, row index) of the current and the previous state: set p
  // at base + p * mc (g), + (2 + p) * mc (x), + (4 + p) * mc (q); indices at Li0 + p * mc
  double* Lu = base + 6 * mc;  // (Q g_bar) on the passive list
  double* T = Lu + mc;         // products of the current chain
  double* Cd = T + mc;         // changed list: delta
  double* Cc = Cd + mc;        //               candidate x
  double* Sg = Cc + mc;        // pushed segments: g, x, q, u at passive rows, df terms
  double* Sx = Sg + ns;
  double* Sq = Sx + ns;
  double* Su = Sq + ns;
  double* Sdf = Su + ns;
  double* xl = Sdf + ns;       // own rows: x, g, q, gd, and x, g before the pending step
  double* gl = xl + kSR;
  double* ql = gl + kSR;
  double* gdl = ql + kSR;
  double* xs = gdl + kSR;
  double* gs = xs + kSR;
  uint32_t* Li0 = reinterpret_cast<uint32_t*>(gs + kSR);
  uint32_t* Ci = Li0 + 2 * mc;   // changed list: row index
  uint32_t* Sidx = Ci + mc;      // pushed segments: row index
  int* lpos = reinterpret_cast<int*>(Sidx + ns);  // own row -> own passive slot
  uint32_t* pidx = reinterpret_cast<uint32_t*>(lpos + kSR);  // own passive entries (staging)

  // the same object in CTA r's shared memory (a DSMEM address)
  auto at = [&](auto* p, int r) { return cluster.map_shared_rank(p, r); };

  // ---- prologue -------------------------------------------------------------------------
  if (!leader) {
    const double2* src = reinterpret_cast<const double2*>(a.Q + (size_t)(rank - 1) * R * m);
    double2* dst = reinterpret_cast<double2*>(Qs);
    for (int e = tid; e < R * m / 2; e += blockDim.x) dst[e] = __ldg(src + e);
    for (int t = tid; t < nrows; t += blockDim.x) {
      const double qi = __ldg(a.q + row0 + t);
      xl[t] = a.zero_start ? 0.0 : a.x[row0 + t];  // x = 0, grad = q (nqp.hpp:224-225)
      gl[t] = a.zero_start ? qi : a.g[row0 + t];
      ql[t] = qi;
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
  }
  if (tid < 8) s_ph[tid] = 0;
  __syncthreads();
  const uint64_t t0 = globaltimer_ns();
  uint64_t ph_t = t0;
  auto mark = [&](int i) {
    if (leader && tid == 0) {
      const uint64_t t = globaltimer_ns();
      s_ph[i] += t - ph_t;
      ph_t = t;
    }
  };

  unsigned long long k = 0;  // iteration whose stop test runs next
  int lp = 0;                // list set of the current state
  // the pending (applied, df not yet checked) step; identical in every CTA
  bool pend = false;
  unsigned long long pk = 0, pmults = 0;
  double palpha = 0.0, pgbs = 0.0;
  int ptries = 0, pml = 0;

  for (;;) {
    // ===== publish: own passive entries of the current state, pushed to every CTA ==========
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
        if (f) pidx[pos] = (uint32_t)tid;
      }
      __syncthreads();
      const int sb = (rank - 1) * R;
      for (int e = tid; e < total * C; e += blockDim.x) {  // entry j to CTA d
        const int d = e / total, j = e - d * total;
        const int t = (int)pidx[j];
        *at(Sidx + sb + j, d) = (uint32_t)(row0 + t);
        *at(Sg + sb + j, d) = gl[t];
        *at(Sx + sb + j, d) = xl[t];
        *at(Sq + sb + j, d) = ql[t];
      }
      if (tid < C) *at(&box.np[rank - 1], tid) = total;
      if (tid == 0) {
        double m2 = s_wmin[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m2 = fmin(m2, s_wmin[w]);
        *at(&box.bad[rank - 1], 0) = bad;
        *at(&box.minx[rank - 1], 0) = m2;
      }
    }
    cluster_barrier();  // B1
    mark(4);

    // ===== the passive list (local: concatenate the pushed segments) ========================
    uint32_t* const Lic = Li0 + lp * mc;
    double* const Lgc = base + lp * mc;
    double* const Lxc = base + (2 + lp) * mc;
    double* const Lqc = base + (4 + lp) * mc;
    if (tid < 32) seg_offsets(box.np, nblk, s_offP);
    if (tid < nblk) s_cntP[tid] = box.np[tid];  // kept: box.np may be overwritten before den
    __syncthreads();
    const int ml = s_offP[31];
    for (int e = tid; e < ns; e += blockDim.x) {
      const int r = e / R, j = e - r * R;
      if (j < s_cntP[r]) {
        const int o = s_offP[r] + j;
        Lic[o] = Sidx[e];
        Lgc[o] = Sg[e];
        Lxc[o] = Sx[e];
        Lqc[o] = Sq[e];
      }
    }
    __syncthreads();
    mark(5);
    // ===== P1 (row CTAs) || stop test + the pending step's df (leader) =======================
    if (!leader) {
      const uint64_t tg = globaltimer_ns();
      if (tid < nrows) {
        const double u = panel_gemv(Qs, R, tid, Lic, Lgc, ml);  // u = Q g_bar, own rows
        const int lpt = lpos[tid];
        if (lpt >= 0)
          for (int d = 0; d < C; ++d) *at(Su + (rank - 1) * R + lpt, d) = u;
      }
      if (rank == 1 && tid == 0) s_ph[7] += globaltimer_ns() - tg;
    } else {
      int nd = 0;
      if (pend) {  // the pending step's df terms, pushed by the row CTAs in their P2
        if (tid < 32) seg_offsets(box.nc, nblk, s_offC);
        __syncthreads();
        nd = s_offC[31];
        for (int e = tid; e < ns; e += blockDim.x) {
          const int r = e / R, j = e - r * R;
          if (j < box.nc[r]) Cc[s_offC[r] + j] = Sdf[e];
        }
      }
      if (tid >= 32 && tid < 64) {  // the row CTAs' flags and minima
        const int r = tid - 32;
        int bad = r < nblk ? box.bad[r] : 0;
        double mn = r < nblk ? box.minx[r] : __longlong_as_double(0x7ff0000000000000LL);
        for (int o = 16; o > 0; o >>= 1) {
          bad |= __shfl_xor_sync(0xffffffffu, bad, o);
          mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        }
        if (tid == 32) {
          s_bad = bad;
          s_mn = mn;
        }
      }
      // gbs: g^2 on the mask; dot(x, grad): x g; dot(q, x): q x (terms off the mask
      // are exact zeros: x = 0 there, g >= 0)
      for (int t = tid; t < ml; t += blockDim.x) {
        T[t] = xmul(Lgc[t], Lgc[t]);
        Lu[t] = xmul(Lxc[t], Lgc[t]);
        Cd[t] = xmul(Lqc[t], Lxc[t]);
      }
      __syncthreads();
      const int warp = tid >> 5;
      if ((tid & 31) == 0 && warp < 4) {  // four concurrent chains
        const double* p = warp == 0 ? T : (warp == 1 ? Lu : (warp == 2 ? Cd : Cc));
        s_sum[warp] = chain_smem(p, warp == 3 ? nd : ml);
      }
      __syncthreads();
      if (tid == 0) {
        int act = kSmallCont;
        double gbs = 0.0;
        if (pend && !(s_sum[3] <= 0.0 || ptries >= 60)) {
          act = kSmallRollback;  // df > 0: halve the pending step (nqp.hpp:316-317)
        } else {
          if (pend) {  // the pending step is final: its bookkeeping (nqp.hpp:319-326)
            small_push(a, ctl, pk, ctl.f, pgbs, pml, ctl.el, palpha, pmults);
            ctl.stepped = 1;
          }
          gbs = s_sum[0];
          const double f = xmul(0.5, xadd(s_sum[1], s_sum[2]));
          const double el = (double)(globaltimer_ns() - t0) * 1e-9;
          if (ctl.stepped) {  // min over the iterate after each stepped iteration
            if (k == 0) ctl.min_iterate = m ? s_mn : 0.0;
            else if (m && s_mn < ctl.min_iterate) ctl.min_iterate = s_mn;
            ctl.stepped = 0;
          }
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
          act = stop >= 0 ? kSmallStop : kSmallCont;
        }
        s_bad = act;  // reused: broadcast below
        s_mn = gbs;
      }
      __syncthreads();
      if (tid < C) {  // the decision and gbs to every CTA
        *at(&box.act, tid) = s_bad;
        *at(&box.gbs, tid) = s_mn;
      }
      mark(6);
    }
    cluster_barrier();  // B2
    mark(0);
    const int act = box.act;
    if (act == kSmallStop) break;

    unsigned long long kstep, mults;
    double alpha, gbs;
    int tries, mlc;
    if (act == kSmallRollback) {  // back to the state before the pending step
      lp ^= 1;
      if (!leader)
        for (int t = tid; t < nrows; t += blockDim.x) {
          xl[t] = xs[t];
          gl[t] = gs[t];
        }
      kstep = pk;
      alpha = xmul(palpha, 0.5);
      tries = ptries + 1;
      mults = pmults;
      gbs = pgbs;
      mlc = pml;
    } else {
      // ===== den (every CTA, redundantly): u from the pushed segments, the den chain ======
      gbs = box.gbs;
      for (int e = tid; e < ns; e += blockDim.x) {
        const int r = e / R, j = e - r * R;
        if (j < s_cntP[r]) {
          const int o = s_offP[r] + j;
          T[o] = xmul(Lgc[o], Su[e]);  // g_bar * (Q g_bar) in list order
        }
      }
      __syncthreads();
      if (tid == 0) s_den = chain_smem(T, ml);
      __syncthreads();
      const double den = s_den;
      mark(1);
      if (!(den > 0.0)) {
        if (leader && tid == 0)
          small_stop(a, ctl, k, ctl.f, gbs, ml, ctl.el, ALNNLS_ZERO_CURVATURE);
        break;
      }
      kstep = k;
      alpha = xdiv(gbs, den);
      tries = 0;
      mults = (unsigned long long)m * (unsigned long long)ml;
      mlc = ml;
    }
    // ===== candidate step and changed set (every CTA, redundantly; nqp.hpp:294-303) ==========
    const uint32_t* Lis = Li0 + lp * mc;
    const double* Lgs = base + lp * mc;
    const double* Lxs = base + (2 + lp) * mc;
    int f0 = 0, f1 = 0;
    double c0 = 0.0, c1 = 0.0;
    const int e0 = 2 * tid, e1 = 2 * tid + 1;
    if (e0 < mlc) {
      double xi = xsub(Lxs[e0], xmul(alpha, Lgs[e0]));  // x - (alpha g), nqp.hpp:296
      if (xi < 0.0) xi = 0.0;
      c0 = xi;
      f0 = xi != Lxs[e0];
    }
    if (e1 < mlc) {
      double xi = xsub(Lxs[e1], xmul(alpha, Lgs[e1]));
      if (xi < 0.0) xi = 0.0;
      c1 = xi;
      f1 = xi != Lxs[e1];
    }
    int cl = 0;
    int pos = block_exclusive_scan(f0 + f1, s_scan, &cl);
    if (tid == 0) {
      s_clo = 0;
      s_chi = 0;
    }
    if (f0) {
      Ci[pos] = Lis[e0];
      Cd[pos] = xsub(c0, Lxs[e0]);
      Cc[pos] = c0;
      ++pos;
    }
    if (f1) {
      Ci[pos] = Lis[e1];
      Cd[pos] = xsub(c1, Lxs[e1]);
      Cc[pos] = c1;
    }
    __syncthreads();
    if (cl == 0) {  // nothing moved (nqp.hpp:304): the step is final, the state unchanged
      if (leader && tid == 0) small_push(a, ctl, kstep, ctl.f, gbs, mlc, ctl.el, alpha, mults);
      pend = false;
      k = kstep + 1;
      continue;
    }
    mults += (unsigned long long)m * (unsigned long long)cl;
    // ===== P2 (row CTAs): gd = Q[:, C] delta_C on own rows; df terms; speculative apply =====
    if (!leader) {
      // own rows' slice [clo, chi) of the ascending changed list: the entries below
      // row0 and below row0 + nrows, counted by warp ballots
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
      for (int j = tid; j < nc; j += blockDim.x) {  // the df terms, pushed to the leader
        const int t = (int)Ci[clo + j] - row0;
        *at(Sdf + (rank - 1) * R + j, 0) =
            xmul(xadd(gl[t], xmul(0.5, gdl[t])), Cd[clo + j]);  // nqp.hpp:307
      }
      if (tid == 0) *at(&box.nc[rank - 1], 0) = nc;
      __syncthreads();
      // apply now (nqp.hpp:309-313); the df check runs during the next P1, and a
      // rejection restores x and g from xs / gs
      if (tid < nrows) {
        xs[tid] = xl[tid];
        gs[tid] = gl[tid];
        gl[tid] = xadd(gl[tid], gdl[tid]);
      }
      __syncthreads();
      for (int j = tid; j < nc; j += blockDim.x) xl[(int)Ci[clo + j] - row0] = Cc[clo + j];
      __syncthreads();
    }
    mark(2);
    pend = true;
    pk = kstep;
    palpha = alpha;
    ptries = tries;
    pmults = mults;
    pgbs = gbs;
    pml = mlc;
    k = kstep + 1;
    lp ^= 1;
  }
  // ---- epilogue: the final iterate and gradient of own rows, the leader's counters ---------
  if (rank == 1 && tid == 0) a.ctrl->phase_ns[7] = s_ph[7];
  if (leader && tid == 0) {
    a.ctrl->trace_len = ctl.trace_len;
    a.ctrl->mult_len = ctl.mult_len;
    a.ctrl->mult_total = ctl.mult_total;
    a.ctrl->min_iterate = ctl.min_iterate;
    for (int i = 0; i < 7; ++i) a.ctrl->phase_ns[i] = s_ph[i];
  }
  if (!leader)
    for (int t = tid; t < nrows; t += blockDim.x) {
      a.x[row0 + t] = xl[t];
      a.g[row0 + t] = gl[t];
    }
  cluster_barrier();  // no CTA leaves while another may still write its shared memory
}

size_t small_smem_bytes(int m, int R, int nblk) {
  const size_t mc = (size_t)((m + 1) & ~1), ns = (size_t)nblk * R;
  return (size_t)R * m * 8 + 10 * mc * 8 + 5 * ns * 8 + 6 * kSR * 8 + 3 * mc * 4 + ns * 4 +
         2 * kSR * 4 + 64;
}

}  // namespace

bool nqp_small_fits(int m, int R, int num_ctas) {
  return m >= 1 && m <= kSMaxM && R <= kSR && R % 2 == 0 && num_ctas >= 2 && num_ctas <= 17 &&
         num_ctas - 1 <= 16 && small_smem_bytes(m, R, num_ctas - 1) <= kSmallSmemMax;
}

// Launches the small-m cluster loop; cudaErrorNotSupported when the shape does not
// fit it or no cluster of that size can be placed (the caller takes the general loop).
cudaError_t launch_nqp_small(const LoopArgs& a, int num_ctas, cudaStream_t stream) {
#ifdef ALNNLS_NO_SMALL
  return cudaErrorNotSupported;
#endif
  if (!nqp_small_fits(a.m, a.rows_per_cta, num_ctas)) return cudaErrorNotSupported;
  const size_t smem = small_smem_bytes(a.m, a.rows_per_cta, num_ctas - 1);
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
