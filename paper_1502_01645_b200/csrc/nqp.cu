// nqp.cu — exact device-resident projected-gradient loop (K4-K6).
//
// Restates reference solve_nqp (/root/reference/proj/include/antilop/nqp.hpp:
// 215-339) as ONE persistent cooperative kernel: no host round trip per
// iteration; the passive mask, step, halving decision, stop tests, stall
// counter, trace records and multiply counts all live in device memory.
//
// Per iteration (grid = one CTA per SM, each CTA owns a contiguous row block):
//   M  leader CTA: passive mask (ballot-free chunked compaction, ascending),
//      gbs / x.g / q.x chains (three threads, concurrently), f, stop tests
//   P1 all CTAs:   u = Q[:, P] g_P, one exact chain per row (gemv.cuh)
//   D  leader:     den chain -> alpha = gbs / den  (exact_step, nqp.hpp:162-173)
//   C  leader:     cand = max(0, x - alpha g) on P, changed set (ascending)
//   P2 all CTAs:   gd = Q[:, C] delta_C
//   F  leader:     df chain, accept or halve (nqp.hpp:293-318)
//   U  all CTAs:   g += gd on own rows; leader x[C] = cand, min_iterate
// Every chain is sequential in the reference index order with rounded
// product then rounded sum, so the trajectory is bitwise the reference's.
#include <cooperative_groups.h>

#include "common.cuh"
#include "gemv.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace alnnls {

namespace {

constexpr int kLoopThreads = 512;

struct LeaderState {
  double best_gbs;
  unsigned long long since_best;
  double gbs, f, xg, qx;
  double elapsed;
  unsigned long long mults;
  int nonfinite;
  int scan[40];
};

__device__ __forceinline__ void chunk(int len, int& lo, int& hi) {
  const int nt = blockDim.x;
  const int per = (len + nt - 1) / nt;
  lo = min(len, (int)threadIdx.x * per);
  hi = min(len, lo + per);
}

// Passive mask P = {i : x_i > 0 || g_i < 0}, ascending (nqp.hpp:149-157), plus
// the per-position products of the gbs / x.g / q.x chains (nqp.hpp:251-254).
__device__ void leader_mask(const LoopArgs& a, LeaderState& L) {
  int lo, hi;
  chunk(a.m, lo, hi);
  int cnt = 0, bad = 0;
  for (int i = lo; i < hi; ++i) {
    const double xi = __ldcg(a.x + i), gi = __ldcg(a.g + i);
    if (!isfinite(gi) || !isfinite(xi)) bad = 1;
    if (xi > 0.0 || gi < 0.0) ++cnt;
  }
  int total;
  int off = block_exclusive_scan(cnt, L.scan, &total);
  for (int i = lo; i < hi; ++i) {
    const double xi = __ldcg(a.x + i), gi = __ldcg(a.g + i);
    if (xi > 0.0 || gi < 0.0) {
      a.mask[off] = (uint32_t)i;
      a.gP[off] = gi;
      a.prod0[off] = xmul(gi, gi);
      a.prod1[off] = xmul(xi, gi);            // dot(x, grad) term
      a.prod2[off] = xmul(__ldg(a.q + i), xi);  // dot(q, x) term
      ++off;
    }
  }
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    a.ctrl->mask_len = total;
    L.nonfinite = bad;
  }
  // Three independent sequential chains in three different warps.
  if (threadIdx.x == 0) L.gbs = chain_sum(a.prod0, total);
  if (threadIdx.x == 32) L.xg = chain_sum(a.prod1, total);
  if (threadIdx.x == 64) L.qx = chain_sum(a.prod2, total);
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

__global__ void __launch_bounds__(kLoopThreads, 1) nqp_loop_kernel(LoopArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ LeaderState L;
  const bool leader = blockIdx.x == 0;
  const int row0 = blockIdx.x * a.rows_per_cta;
  const int nrows = max(0, min(a.m - row0, a.rows_per_cta));
  RowRing ring;
  ring_setup(ring, smem, kRingSmemBytes, nrows);
  volatile LoopCtrl* vc = a.ctrl;

  const uint64_t t0 = globaltimer_ns();
  if (leader) {
    // min_iterate starts at min(x) (nqp.hpp:237)
    if (threadIdx.x == 0) {
      double mn = a.m ? a.x[0] : 0.0;
      for (int i = 1; i < a.m; ++i) mn = a.x[i] < mn ? a.x[i] : mn;
      a.ctrl->min_iterate = mn;
      a.ctrl->trace_len = 0;
      a.ctrl->mult_len = 0;
      a.ctrl->mult_total = 0;
      a.ctrl->numeric_failure = 0;
      a.ctrl->stop = 0;
      L.best_gbs = __longlong_as_double(0x7ff0000000000000LL);  // +inf
      L.since_best = 0;
    }
    __syncthreads();
  }

  for (unsigned long long k = 0;; ++k) {
    // ---- M: mask, chains, stop tests (leader) ---------------------------------
    if (leader) {
      leader_mask(a, L);
      if (threadIdx.x == 0) {
        const double f = xmul(0.5, xadd(L.xg, L.qx));
        const double gbs = L.gbs;
        const double elapsed = (double)(globaltimer_ns() - t0) * 1e-9;
        const int ml = a.ctrl->mask_len;
        L.f = f;
        L.elapsed = elapsed;
        L.mults = 0;
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
        if (stop >= 0) {
          if (stop != 100) {
            write_record(a, k, f, gbs, ml, elapsed, 0.0, 0);
            a.ctrl->termination = stop;
            a.ctrl->iterations = k;
            a.ctrl->f_final = f;
            a.ctrl->gbs_final = gbs;
          }
          a.ctrl->stop = 1;
        }
        __threadfence();
      }
    }
    grid.sync();
    if (vc->stop) break;
    const int ml = vc->mask_len;

    // ---- P1: u = Q[:, P] g_P -----------------------------------------------------
    gemv_rows(ring, a.Q, a.ldq, row0, nrows, a.mask, a.gP, ml, a.u);
    grid.sync();

    // ---- D: den chain, alpha ----------------------------------------------------
    if (leader) {
      int lo, hi;
      chunk(ml, lo, hi);
      for (int t = lo; t < hi; ++t) a.prod0[t] = xmul(a.gP[t], __ldcg(a.u + a.mask[t]));
      __syncthreads();
      if (threadIdx.x == 0) {
        const double den = chain_sum(a.prod0, ml);
        L.mults += (unsigned long long)a.m * (unsigned long long)ml;
        if (!(den > 0.0)) {
          write_record(a, k, L.f, L.gbs, ml, L.elapsed, 0.0, 0);
          a.ctrl->termination = ALNNLS_ZERO_CURVATURE;
          a.ctrl->iterations = k;
          a.ctrl->f_final = L.f;
          a.ctrl->gbs_final = L.gbs;
          a.ctrl->stop = 1;
        } else {
          a.ctrl->alpha = xdiv(L.gbs, den);
        }
        __threadfence();
      }
    }
    grid.sync();
    if (vc->stop) break;

    // ---- halving loop -----------------------------------------------------------
    bool moved = false;
    for (int tries = 0;; ++tries) {
      if (leader) {  // C: candidate step and changed set
        const double alpha = a.ctrl->alpha;
        int lo, hi;
        chunk(ml, lo, hi);
        int cnt = 0;
        for (int t = lo; t < hi; ++t) {
          const uint32_t i = a.mask[t];
          const double xi0 = __ldcg(a.x + i);
          double xi = xsub(xi0, xmul(alpha, a.gP[t]));
          if (xi < 0.0) xi = 0.0;
          if (xi != xi0) ++cnt;
        }
        int total;
        int off = block_exclusive_scan(cnt, L.scan, &total);
        for (int t = lo; t < hi; ++t) {
          const uint32_t i = a.mask[t];
          const double xi0 = __ldcg(a.x + i);
          double xi = xsub(xi0, xmul(alpha, a.gP[t]));
          if (xi < 0.0) xi = 0.0;
          if (xi != xi0) {
            a.chg[off] = i;
            a.candC[off] = xi;
            a.dC[off] = xsub(xi, xi0);
            a.gC[off] = a.gP[t];
            ++off;
          }
        }
        if (threadIdx.x == 0) {
          a.ctrl->chg_len = total;
          if (total > 0) L.mults += (unsigned long long)a.m * (unsigned long long)total;
          __threadfence();
        }
      }
      grid.sync();
      const int cl = vc->chg_len;
      if (cl == 0) break;  // nqp.hpp:304

      // ---- P2: gd = Q[:, C] delta_C ----
      gemv_rows(ring, a.Q, a.ldq, row0, nrows, a.chg, a.dC, cl, a.gd);
      grid.sync();

      if (leader) {  // F: df chain, accept or halve
        int lo, hi;
        chunk(cl, lo, hi);
        for (int t = lo; t < hi; ++t) {
          const double gdi = __ldcg(a.gd + a.chg[t]);
          a.prod0[t] = xmul(xadd(a.gC[t], xmul(0.5, gdi)), a.dC[t]);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          const double df = chain_sum(a.prod0, cl);
          const int acc = (df <= 0.0 || tries >= 60) ? 1 : 0;
          a.ctrl->accept = acc;
          if (!acc) a.ctrl->alpha = xmul(a.ctrl->alpha, 0.5);
          __threadfence();
        }
      }
      grid.sync();
      if (vc->accept) {
        moved = true;
        break;
      }
    }

    // ---- U: apply the step ------------------------------------------------------
    if (moved) {
      for (int t = threadIdx.x; t < nrows; t += blockDim.x) {
        const int i = row0 + t;
        a.g[i] = xadd(a.g[i], __ldcg(a.gd + i));
      }
      if (leader) {
        const int cl = a.ctrl->chg_len;
        for (int t = threadIdx.x; t < cl; t += blockDim.x) a.x[a.chg[t]] = a.candC[t];
      }
    }
    if (leader) {
      __syncthreads();
      // min_iterate = min(min_iterate, min(x)) (nqp.hpp:323-326); order-independent.
      double mn = __longlong_as_double(0x7ff0000000000000LL);
      for (int i = threadIdx.x; i < a.m; i += blockDim.x) mn = fmin(mn, a.x[i]);
      for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      __shared__ double red[kLoopThreads / 32];
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mn;
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mn = fmin(mn, red[w]);
        if (a.m && mn < a.ctrl->min_iterate) a.ctrl->min_iterate = mn;
        if (k % a.trace_every == 0)
          write_record(a, k, L.f, L.gbs, a.ctrl->mask_len, L.elapsed, a.ctrl->alpha, 1);
        const unsigned long long ml_idx = a.ctrl->mult_len;
        if (a.mults && ml_idx < a.mults_cap) a.mults[ml_idx] = L.mults;
        a.ctrl->mult_len = ml_idx + 1;
        a.ctrl->mult_total += L.mults;
        __threadfence();
      }
    }
    grid.sync();
  }
}

}  // namespace

size_t nqp_loop_smem_bytes() { return kRingSmemBytes; }

int nqp_rows_per_cta(int m, int sm_count) {
  int r = (m + sm_count - 1) / sm_count;
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

// ---- standalone masked GEMV (masked_matvec / matvec / residual) --------------------
namespace {
__global__ void __launch_bounds__(kLoopThreads, 1)
    masked_gemv_kernel(const double* M, uint64_t ld, int rows, int rows_per_cta,
                       const uint32_t* list, const double* vals, int len, double* y) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int row0 = blockIdx.x * rows_per_cta;
  const int nrows = max(0, min(rows - row0, rows_per_cta));
  RowRing ring;
  ring_setup(ring, smem, kRingSmemBytes, nrows);
  gemv_rows(ring, M, ld, row0, nrows, list, vals, len, y);
}
}  // namespace

cudaError_t launch_masked_gemv(const double* M, uint64_t ld, int rows, const uint32_t* list,
                               const double* vals, int len, double* y, int sm_count,
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
  const int rpc = nqp_rows_per_cta(rows, sm_count);
  const int grid = (rows + rpc - 1) / rpc;
  masked_gemv_kernel<<<grid, kLoopThreads, nqp_loop_smem_bytes(), stream>>>(M, ld, rows, rpc, list,
                                                                            vals, len, y);
  return cudaGetLastError();
}

}  // namespace alnnls
