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
//   P2   row CTAs: gd = Q[:, C] delta_C (nqp.hpp:305)                       -> barrier
//   F/U  row CTAs: g_next = g + gd on own rows (ping-pong buffer, so doing it
//        before the decision is safe); vector CTA: df chain (nqp.hpp:307),
//        accept -> x[C] = cand, next passive mask from g + gd, trace record;
//        reject -> alpha/2 and a new C (nqp.hpp:316-317)                    -> barrier
//
// Every sum is one sequential chain in the reference order: the vector CTA
// forms the rounded products in parallel into shared memory and one thread
// runs the dependent DADD chain, so the trajectory is bitwise the reference's.
#include <cooperative_groups.h>

#include "common.cuh"
#include "gemv.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace alnnls {

namespace {

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
// Double-buffered register prefetch with 16-byte shared loads keeps the
// dependent DADD (8 cycles on B200) the only thing on the critical path.
__device__ __forceinline__ double smem_chain(double s, const double* __restrict__ p, int n) {
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
  const int CH = min(1024, (int)(sbuf_bytes / (2 * K * sizeof(double))) & ~1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = (len + CH - 1) / CH;
  auto produce = [&](int c, int buf, int first_thread) {
    const int b0 = c * CH;
    const int cnt = min(CH, len - b0);
    double* dst = sbuf + (size_t)buf * K * CH;
    for (int i = (int)threadIdx.x - first_thread; i < cnt; i += blockDim.x - first_thread)
#pragma unroll
      for (int k = 0; k < K; ++k) dst[(size_t)k * CH + i] = prod(k, b0 + i);
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

// Passive mask P = {i : x_i > 0 || g_i < 0}, ascending (nqp.hpp:149-157), with
// g_i = gcur_i (+ gd_i when `gd` is given: the incremental update of
// nqp.hpp:313 evaluated on the fly). Writes mask, gP, xP, qP and min(x).
__device__ void leader_build_mask(const LoopArgs& a, LeaderState& L, const double* gcur,
                                  const double* gd, double* min_x) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  int bad = 0, base = 0;
  double mn = __longlong_as_double(0x7ff0000000000000LL);
  for (int s0 = 0; s0 < a.m; s0 += kSuper) {
    double xv[kU], gv[kU], qv[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const int i = s0 + k * kLoopThreads + threadIdx.x;
      xv[k] = 0.0;
      gv[k] = 0.0;
      qv[k] = 0.0;
      if (i < a.m) {
        xv[k] = a.x[i];
        gv[k] = __ldcg(gcur + i);
        if (gd) gv[k] = xadd(gv[k], __ldcg(gd + i));
        qv[k] = __ldg(a.q + i);
      }
    }
    unsigned sel = 0, wp[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const bool valid = s0 + k * kLoopThreads + (int)threadIdx.x < a.m;
      const bool f = valid && (xv[k] > 0.0 || gv[k] < 0.0);
      if (valid) {
        if (!isfinite(gv[k])) bad = 1;
        mn = fmin(mn, xv[k]);
      }
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
        a.mask[pos] = (uint32_t)(s0 + k * kLoopThreads + threadIdx.x);
        a.gP[pos] = gv[k];
        a.xP[pos] = xv[k];
        a.qP[pos] = qv[k];
      }
    }
    base += total;
    __syncthreads();
  }
  for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  if (lane == 0) L.red[warp] = mn;
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    for (int w = 1; w < kWarps; ++w) mn = fmin(mn, L.red[w]);
    *min_x = mn;
    a.ctrl->mask_len = base;
    L.nonfinite = bad;
  }
  __syncthreads();
}

// Candidate step on the mask and the changed set C (nqp.hpp:294-303).
__device__ void leader_build_changed(const LoopArgs& a, LeaderState& L, int ml, double alpha) {
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
        xv[k] = a.xP[t];
        gv[k] = a.gP[t];
        iv[k] = a.mask[t];
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
  if (idx < a.trace_cap) {
    alnnls_iter_record r;
    r.iter = k;
    r.f = f;
    r.grad_bar_sq = gbs;
    r.passive_count = (uint64_t)pc;
    r.elapsed_s = elapsed;
    r.alpha = has_alpha ? alpha : 0.0;
    r.has_alpha = has_alpha;
    a.trace[idx] = r;
  }
  c->trace_len = idx + 1;
}

// Stepped-iteration bookkeeping (nqp.hpp:319-326). Vector CTA thread 0.
__device__ void finish_step(const LoopArgs& a, LeaderState& L, unsigned long long k, int ml,
                            double min_x) {
  if (a.m && min_x < a.ctrl->min_iterate) a.ctrl->min_iterate = min_x;
  if (k % a.trace_every == 0) write_record(a, k, L.f, L.gbs, ml, L.elapsed, L.alpha, 1);
  const unsigned long long idx = a.ctrl->mult_len;
  if (a.mults && idx < a.mults_cap) a.mults[idx] = L.mults;
  a.ctrl->mult_len = idx + 1;
  a.ctrl->mult_total += L.mults;
}

__device__ void stop_final(const LoopArgs& a, LeaderState& L, unsigned long long k, int ml,
                           int term) {
  write_record(a, k, L.f, L.gbs, ml, L.elapsed, 0.0, 0);
  a.ctrl->termination = term;
  a.ctrl->iterations = k;
  a.ctrl->f_final = L.f;
  a.ctrl->gbs_final = L.gbs;
}

__global__ void __launch_bounds__(kLoopThreads, 1) nqp_loop_kernel(LoopArgs a) {
  // cooperative-groups grid barrier (1.2 us measured; a nanosleep-backoff
  // barrier in common.cuh measured slower here)
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ LeaderState L;
  __shared__ double s_min_x;
  const bool leader = blockIdx.x == 0;
  const int R = a.rows_per_cta;
  const int blk = (int)blockIdx.x - 1;
  const int row0 = leader ? 0 : blk * R;
  const int nrows = leader ? 0 : max(0, min(a.m - row0, R));
  const double* qblk = a.Q + (size_t)(leader ? 0 : blk) * R * a.m;
  RowRing ring;
  if (!leader) ring_setup(ring, smem, kRingSmemBytes, nrows, R, kWarps);
  double* sbuf = reinterpret_cast<double*>(smem);
  volatile LoopCtrl* vc = a.ctrl;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* gbuf[2] = {a.g, a.g_alt};
  int par = 0;

  const uint64_t t0 = globaltimer_ns();
  if (leader) {
    if (threadIdx.x == 0) {
      a.ctrl->trace_len = 0;
      a.ctrl->mult_len = 0;
      a.ctrl->mult_total = 0;
      a.ctrl->numeric_failure = 0;
      a.ctrl->stop = 0;
      a.ctrl->g_parity = 0;
      L.best_gbs = __longlong_as_double(0x7ff0000000000000LL);  // +inf
      L.since_best = 0;
      L.t_mark = t0;
      for (int i = 0; i < 8; ++i) L.ph[i] = 0;
    }
    leader_build_mask(a, L, gbuf[0], nullptr, &s_min_x);
    if (threadIdx.x == 0) a.ctrl->min_iterate = a.m ? s_min_x : 0.0;  // nqp.hpp:237
    __threadfence();
  }
  grid.sync();

  for (unsigned long long k = 0;; ++k) {
    const int ml = vc->mask_len;
    // ---- P1 (row CTAs) || stop-test chains (vector CTA) ----------------------------------
    if (!leader) {
      gemv_rows(ring, qblk, R, true, row0, nrows, a.mask, a.gP, ml, a.u);
    } else {
      const double *gP = a.gP, *xP = a.xP, *qP = a.qP;
      leader_chains<3>(sbuf, kRingSmemBytes, L, ml, [&](int c, int t) {
        // gbs: g_i^2; dot(x, grad): x_i g_i; dot(q, x): q_i x_i (terms off the
        // mask are exact zeros since x_i = 0 there)
        return c == 0 ? xmul(gP[t], gP[t]) : (c == 1 ? xmul(xP[t], gP[t]) : xmul(qP[t], xP[t]));
      });
      if (threadIdx.x == 0) {
        L.gbs = L.res[0];
        const double f = xmul(0.5, xadd(L.res[1], L.res[2]));
        const double gbs = L.gbs;
        const double elapsed = (double)(globaltimer_ns() - t0) * 1e-9;
        L.f = f;
        L.elapsed = elapsed;
        L.mults = 0;
        L.tries = 0;
        int stop = -1;
        if (L.nonfinite || !isfinite(f) || !isfinite(gbs)) {
          a.ctrl->numeric_failure = 1;
          stop = 100;
        } else if (ml == 0) {
          stop = ALNNLS_EMPTY_PASSIVE_SET;
        } else if (gbs < a.eps) {
          stop = ALNNLS_GRADIENT_BELOW_EPSILON;
        } else if (k >= a.max_iters) {
          stop = ALNNLS_MAX_ITERS;
        } else if (a.has_time_cap && elapsed >= a.time_cap_s) {
          stop = ALNNLS_TIME_CAP;
        } else if (gbs < L.best_gbs) {
          L.best_gbs = gbs;
          L.since_best = 0;
        } else if (++L.since_best >= a.stall_window) {
          stop = ALNNLS_STALLED;
        }
        if (stop < 0 && !(gbs != 0.0)) stop = ALNNLS_ZERO_CURVATURE;  // num == 0 (nqp.hpp:167)
        if (stop >= 0 && stop != 100) stop_final(a, L, k, ml, stop);
        a.ctrl->stop = stop >= 0 ? 1 : 0;
        phase_mark(L, 0);  // [0] stop-test chains
        __threadfence();
      }
    }
    grid.sync();
    if (leader && threadIdx.x == 0) phase_mark(L, 1);  // [1] rest of P1 + barrier
    if (vc->stop) break;

    // ---- D/C: den chain, alpha, changed set (vector CTA) --------------------------------
    if (leader) {
      const double *gP = a.gP, *u = a.u;
      const uint32_t* mask = a.mask;
      leader_chains<1>(sbuf, kRingSmemBytes, L, ml,
                       [&](int, int t) { return xmul(gP[t], __ldcg(u + mask[t])); });
      if (threadIdx.x == 0) {
        const double den = L.res[0];
        L.mults += (unsigned long long)a.m * (unsigned long long)ml;
        if (!(den > 0.0)) {
          stop_final(a, L, k, ml, ALNNLS_ZERO_CURVATURE);
          L.alpha = -1.0;
        } else {
          L.alpha = xdiv(L.gbs, den);
        }
        phase_mark(L, 2);  // [2] den chain
      }
      __syncthreads();
      const bool zc = L.alpha < 0.0;
      if (!zc) leader_build_changed(a, L, ml, L.alpha);
      if (threadIdx.x == 0) {
        a.ctrl->state = zc ? kStateStop : (a.ctrl->chg_len == 0 ? kStateNoMove : kStateP2);
        phase_mark(L, 3);  // [3] changed set
        __threadfence();
      }
    }
    grid.sync();
    int state = vc->state;
    if (state == kStateStop) break;

    // ---- halving loop: P2, then the df decision -----------------------------------------
    while (state == kStateP2) {
      const int cl = vc->chg_len;
      if (!leader) gemv_rows(ring, qblk, R, true, row0, nrows, a.chg, a.dC, cl, a.gd);
      grid.sync();
      if (!leader) {
        // speculative U on own rows: g_next = g + gd (nqp.hpp:313); harmless if rejected
        const double* gc = gbuf[par];
        double* gn = gbuf[par ^ 1];
        for (int t = threadIdx.x; t < nrows; t += blockDim.x) {
          const int i = row0 + t;
          gn[i] = xadd(gc[i], a.gd[i]);
        }
      } else {
        if (threadIdx.x == 0) phase_mark(L, 4);  // [4] barrier + P2 + barrier
        const double *gC = a.gC, *dC = a.dC, *gd = a.gd;
        const uint32_t* chg = a.chg;
        leader_chains<1>(sbuf, kRingSmemBytes, L, cl, [&](int, int t) {
          return xmul(xadd(gC[t], xmul(0.5, __ldcg(gd + chg[t]))), dC[t]);
        });
        if (threadIdx.x == 0) {
          const double df = L.res[0];
          const int accept = (df <= 0.0 || L.tries >= 60) ? 1 : 0;  // nqp.hpp:308
          a.ctrl->accept = accept;
          if (!accept) {
            L.alpha = xmul(L.alpha, 0.5);  // nqp.hpp:317
            ++L.tries;
          }
          phase_mark(L, 5);  // [5] df chain
        }
        __syncthreads();
        if (a.ctrl->accept) {
          // x[C] = cand (nqp.hpp:309-311); x is private to the vector CTA
          for (int t = threadIdx.x; t < cl; t += blockDim.x) a.x[a.chg[t]] = a.candC[t];
          __syncthreads();
          leader_build_mask(a, L, gbuf[par], a.gd, &s_min_x);
          if (threadIdx.x == 0) {
            finish_step(a, L, k, ml, s_min_x);
            a.ctrl->state = kStateNext;
          }
        } else {
          leader_build_changed(a, L, ml, L.alpha);
          if (threadIdx.x == 0)
            a.ctrl->state = a.ctrl->chg_len == 0 ? kStateNoMove : kStateP2;  // nqp.hpp:304
        }
        if (threadIdx.x == 0) {
          phase_mark(L, 6);  // [6] update + next mask
          __threadfence();
        }
      }
      grid.sync();
      if (leader && threadIdx.x == 0) phase_mark(L, 7);  // [7] final barrier
      state = vc->state;
      if (state == kStateNext) par ^= 1;
    }
    if (state == kStateNoMove) {
      // no coordinate moved: x and g are unchanged, so the mask lists stay valid
      if (leader && threadIdx.x == 0) {
        finish_step(a, L, k, ml, a.ctrl->min_iterate);
        a.ctrl->mask_len = ml;
        __threadfence();
      }
      grid.sync();
    }
  }
  if (leader && threadIdx.x == 0) {
    a.ctrl->g_parity = par;
    for (int i = 0; i < 8; ++i) a.ctrl->phase_ns[i] = L.ph[i];
  }
}

}  // namespace

size_t nqp_loop_smem_bytes() { return kRingSmemBytes; }

// Rows per block of the blocked Q: the vector CTA takes one SM, the row
// blocks share the rest.
int nqp_rows_per_cta(int m, int sm_count) {
  const int nb = sm_count > 1 ? sm_count - 1 : 1;
  int r = (m + nb - 1) / nb;
  r = (r + 3) & ~3;
  if (r < 4) r = 4;
  return r;
}

cudaError_t launch_nqp_loop(const LoopArgs& a, int num_ctas, cudaStream_t stream) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(nqp_loop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)nqp_loop_smem_bytes());
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  LoopArgs args = a;
  void* params[] = {&args};
  return cudaLaunchCooperativeKernel((void*)nqp_loop_kernel, dim3(num_ctas), dim3(kLoopThreads),
                                     params, nqp_loop_smem_bytes(), stream);
}

// ---- standalone masked GEMV (masked_matvec / matvec / residual / warm start) ------------
namespace {
__global__ void __launch_bounds__(kLoopThreads, 1)
    masked_gemv_kernel(const double* M, uint64_t ld, int rows, int rows_per_cta, int blocked,
                       const uint32_t* list, const double* vals, int len, double* y) {
  extern __shared__ __align__(128) uint8_t smem[];
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
                        cudaStream_t stream) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(masked_gemv_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)nqp_loop_smem_bytes());
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  if (rows <= 0) return cudaSuccess;
  if (rpc > 352) return cudaErrorInvalidValue;  // 11 consumer warps + 1 producer
  const int grid = (rows + rpc - 1) / rpc;
  masked_gemv_kernel<<<grid, kLoopThreads, nqp_loop_smem_bytes(), stream>>>(M, ld, rows, rpc,
                                                                            blocked, list, vals,
                                                                            len, y);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_masked_gemv(const double* M, uint64_t ld, int rows, const uint32_t* list,
                               const double* vals, int len, double* y, int sm_count,
                               cudaStream_t stream) {
  int rpc = (rows + sm_count - 1) / sm_count;
  rpc = (rpc + 3) & ~3;
  if (rpc < 4) rpc = 4;
  return gemv_launch(M, ld, rows, rpc, 0, list, vals, len, y, stream);
}

cudaError_t launch_masked_gemv_blocked(const double* Qb, int m, int R, const uint32_t* list,
                                       const double* vals, int len, double* y,
                                       cudaStream_t stream) {
  return gemv_launch(Qb, 0, m, R, 1, list, vals, len, y, stream);
}

}  // namespace alnnls
