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
#include "common.cuh"
#include "kernels.cuh"

namespace alnnls {

namespace {

constexpr int kBT = 256;          // threads per batched CTA
constexpr int kMaxCols = 16;      // NB upper bound (columns per CTA)
constexpr size_t kBatchSmem = 5 * 256 * kMaxCols * sizeof(double);  // V, U, C, X, G

enum ColPhase { kIdle = 0, kNeedP1 = 1, kNeedP2 = 2 };

struct ColState {
  int phase[kMaxCols];
  int col[kMaxCols];
  unsigned long long k[kMaxCols];
  int tries[kMaxCols];
  int cl[kMaxCols];
  int ml[kMaxCols];
  double alpha[kMaxCols];
  double f[kMaxCols], gbs[kMaxCols];
  double best[kMaxCols];
  unsigned long long since[kMaxCols];
  unsigned long long mults[kMaxCols];
  int queue_done;
};

// Layout: V[j * NB + b] etc. (row-major over the m rows, NB columns).
struct BatchSmem {
  double* V;  // GEMM input: g_bar (P1) or delta (P2), 0 off the mask / changed set
  double* U;  // GEMM output: Q g_bar or Q delta
  double* C;  // candidate x
  double* X;  // iterate
  double* G;  // maintained gradient
};

__device__ void finish_col(const BatchArgs& a, ColState& S, const BatchSmem& sm, int NB, int b,
                           int term, int numeric) {
  const int lane = threadIdx.x & 31;
  const int c = S.col[b];
  for (int i = lane; i < a.m; i += 32) a.Y[(size_t)c * a.m + i] = sm.X[i * NB + b];
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
__device__ bool mask_phase(const BatchArgs& a, ColState& S, const BatchSmem& sm, int NB, int b) {
  const int lane = threadIdx.x & 31;
  const double* q = a.QB + (size_t)S.col[b] * a.m;
  int cnt = 0, bad = 0;
  for (int i = lane; i < a.m; i += 32) {
    const double xi = sm.X[i * NB + b], gi = sm.G[i * NB + b];
    const bool p = xi > 0.0 || gi < 0.0;
    cnt += p;
    if (!isfinite(gi)) bad = 1;
    sm.V[i * NB + b] = p ? gi : 0.0;  // g_bar
  }
  for (int o = 16; o > 0; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  __syncwarp();
  // lanes 0, 1, 2: the three chains in ascending index order; terms off the
  // mask are exact zeros (g_bar = 0, x = 0) and are skipped
  double s = 0.0;
  if (lane < 3) {
    for (int i = 0; i < a.m; ++i) {
      const double gb = sm.V[i * NB + b];
      const double xi = sm.X[i * NB + b];
      if (lane == 0) {
        if (gb != 0.0) s = xadd(s, xmul(gb, gb));
      } else if (lane == 1) {
        if (xi != 0.0) s = xadd(s, xmul(xi, sm.G[i * NB + b]));
      } else {
        if (xi != 0.0) s = xadd(s, xmul(__ldg(q + i), xi));
      }
    }
  }
  const double gbs = __shfl_sync(0xffffffffu, s, 0);
  const double xg = __shfl_sync(0xffffffffu, s, 1);
  const double qx = __shfl_sync(0xffffffffu, s, 2);
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
  if (stop >= 0) finish_col(a, S, sm, NB, b, stop == 100 ? 0 : stop, stop == 100);
  return stop >= 0;
}

// Candidate step and changed set with the column's alpha (nqp.hpp:294-303):
// C = candidate x, V = delta (0 off the changed set). Returns |changed|.
__device__ int cand_phase(const BatchArgs& a, ColState& S, const BatchSmem& sm, int NB, int b) {
  const int lane = threadIdx.x & 31;
  const double alpha = S.alpha[b];
  int cnt = 0;
  for (int i = lane; i < a.m; i += 32) {
    const double xi = sm.X[i * NB + b], gi = sm.G[i * NB + b];
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
    sm.C[i * NB + b] = c;
    sm.V[i * NB + b] = d;
  }
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  __syncwarp();
  return cnt;
}

// Loads the next RHS from the queue into slot b and runs its first stop test
// (repeats while columns stop immediately). One warp.
__device__ void refill(const BatchArgs& a, ColState& S, const BatchSmem& sm, int NB, int b) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    int c = 0;
    if (lane == 0) c = atomicAdd(a.next_col, 1);
    c = __shfl_sync(0xffffffffu, c, 0);
    if (c >= a.ncols) {
      for (int i = lane; i < a.m; i += 32) sm.V[i * NB + b] = 0.0;  // idle slots feed zeros
      if (lane == 0) S.phase[b] = kIdle;
      __syncwarp();
      return;
    }
    const double* q = a.QB + (size_t)c * a.m;
    for (int i = lane; i < a.m; i += 32) {
      sm.X[i * NB + b] = 0.0;
      sm.G[i * NB + b] = __ldg(q + i);  // x = 0, grad = q (nqp.hpp:224-225)
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
    if (!mask_phase(a, S, sm, NB, b)) return;
  }
}

template <int NB>
__global__ void __launch_bounds__(kBT, 1) batched_nqp_kernel(BatchArgs a) {
  extern __shared__ __align__(16) double bsm[];
  __shared__ ColState S;
  const int m = a.m;
  BatchSmem sm;
  sm.V = bsm;
  sm.U = bsm + (size_t)m * NB;
  sm.C = bsm + 2 * (size_t)m * NB;
  sm.X = bsm + 3 * (size_t)m * NB;
  sm.G = bsm + 4 * (size_t)m * NB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = kBT / 32;
  for (int b = warp; b < NB; b += nwarps) refill(a, S, sm, NB, b);
  __syncthreads();
  constexpr int RPT = 16 / NB;  // rows per thread
  for (;;) {
    // any active column?
    int active = 0;
    for (int b = 0; b < NB; ++b) active |= S.phase[b] != kIdle;
    if (!active) break;
    // ---- one exact chain GEMM pass: U = Q V (ascending j per output) ----
    double acc[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) acc[t] = 0.0;
    for (int j = 0; j < m; ++j) {
      const double* vrow = sm.V + (size_t)j * NB;
      bool any = false;
      for (int b = 0; b < NB; ++b) any |= vrow[b] != 0.0;
      if (!any) continue;  // all-zero input row: every product is an exact +-0
      const double* qc = a.Q + (size_t)j * m;
      double vb[NB];
#pragma unroll
      for (int b = 0; b < NB; b += 2) {
        const double2 t = *reinterpret_cast<const double2*>(vrow + b);
        vb[b] = t.x;
        vb[b + 1] = t.y;
      }
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
        const int i = threadIdx.x + r * kBT;
        const double qv = i < m ? __ldg(qc + i) : 0.0;
#pragma unroll
        for (int b = 0; b < NB; ++b) acc[r * NB + b] = xmac(acc[r * NB + b], qv, vb[b]);
      }
    }
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int i = threadIdx.x + r * kBT;
      if (i < m) {
#pragma unroll
        for (int b = 0; b < NB; ++b) sm.U[(size_t)i * NB + b] = acc[r * NB + b];
      }
    }
    __syncthreads();
    // ---- per-column state machines ----
    for (int b = warp; b < NB; b += nwarps) {
      const int ph = S.phase[b];
      if (ph == kIdle) continue;
      if (ph == kNeedP1) {
        // den = g_bar . (Q g_bar) over the mask (exact_step, nqp.hpp:166-172)
        double den = 0.0;
        if (lane == 0) {
          for (int i = 0; i < m; ++i) {
            const double gb = sm.V[i * NB + b];
            if (gb != 0.0) den = xadd(den, xmul(gb, sm.U[i * NB + b]));
          }
        }
        den = __shfl_sync(0xffffffffu, den, 0);
        if (!(den > 0.0)) {
          finish_col(a, S, sm, NB, b, ALNNLS_ZERO_CURVATURE, 0);
          refill(a, S, sm, NB, b);
          continue;
        }
        if (lane == 0) {
          S.alpha[b] = xdiv(S.gbs[b], den);
          S.tries[b] = 0;
          S.mults[b] += (unsigned long long)m * (unsigned long long)S.ml[b];
        }
        __syncwarp();
      } else {  // kNeedP2: gd = Q delta in U; df chain (nqp.hpp:307)
        double df = 0.0;
        if (lane == 0) {
          for (int i = 0; i < m; ++i) {
            const double d = sm.V[i * NB + b];
            if (d != 0.0) df = xadd(df, xmul(xadd(sm.G[i * NB + b], xmul(0.5, sm.U[i * NB + b])), d));
          }
        }
        df = __shfl_sync(0xffffffffu, df, 0);
        const bool accept = df <= 0.0 || S.tries[b] >= 60;
        if (accept) {  // x[C] = cand, grad += gd (nqp.hpp:309-313)
          for (int i = lane; i < m; i += 32) {
            sm.X[i * NB + b] = sm.C[i * NB + b];
            sm.G[i * NB + b] = xadd(sm.G[i * NB + b], sm.U[i * NB + b]);
          }
          if (lane == 0) ++S.k[b];
          __syncwarp();
          if (mask_phase(a, S, sm, NB, b)) refill(a, S, sm, NB, b);
          continue;
        }
        if (lane == 0) {
          S.alpha[b] = xmul(S.alpha[b], 0.5);  // nqp.hpp:317
          ++S.tries[b];
        }
        __syncwarp();
      }
      // candidate step with the current alpha
      const int cl = cand_phase(a, S, sm, NB, b);
      if (lane == 0) S.cl[b] = cl;
      if (cl == 0) {  // nothing moved (nqp.hpp:304): next iteration on the same state
        if (lane == 0) ++S.k[b];
        __syncwarp();
        if (mask_phase(a, S, sm, NB, b)) refill(a, S, sm, NB, b);
        continue;
      }
      if (lane == 0) {
        S.mults[b] += (unsigned long long)m * (unsigned long long)cl;
        S.phase[b] = kNeedP2;
      }
      __syncwarp();
    }
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
// columns of A in ascending order (matvec, linalg.hpp:182-186; zero x_j terms are
// exact no-ops), then s += r_i^2 in ascending i. One CTA owns 64 right-hand sides
// and walks all row tiles in order, so each column's s is a single chain.
constexpr int kRT = 32;   // rows per tile
constexpr int kRC = 64;   // columns per CTA
constexpr int kRK = 16;   // k slab
__global__ void __launch_bounds__(256) residual_batched_kernel(const double* A, uint64_t lda, int d,
                                                               int n, const double* X,
                                                               const double* B, uint64_t ldb,
                                                               int ncols,
                                                               alnnls_column_result* res) {
  __shared__ double As[kRK][kRT];
  __shared__ double Xs[kRK][kRC + 1];
  __shared__ double Cs[kRT][kRC + 1];
  const int c0 = blockIdx.x * kRC;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 2 x 4 outputs per thread
  double ssum = 0.0;  // thread t < kRC: the running chain of column c0 + t
  for (int i0 = 0; i0 < d; i0 += kRT) {
    double acc[2][4];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;
    for (int k0 = 0; k0 < n; k0 += kRK) {
      for (int e = threadIdx.x; e < kRK * kRT; e += blockDim.x) {
        const int kk = e / kRT, r = e % kRT;
        const int i = i0 + r, kcol = k0 + kk;
        As[kk][r] = (i < d && kcol < n) ? __ldg(A + (size_t)kcol * lda + i) : 0.0;
      }
      for (int e = threadIdx.x; e < kRK * kRC; e += blockDim.x) {
        const int c = e / kRK, kk = e % kRK;
        const int col = c0 + c, kcol = k0 + kk;
        Xs[kk][c] = (col < ncols && kcol < n) ? __ldg(X + (size_t)col * n + kcol) : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < kRK; ++kk) {
        double av[2], xv[4];
#pragma unroll
        for (int r = 0; r < 2; ++r) av[r] = As[kk][tx + 16 * r];
#pragma unroll
        for (int c = 0; c < 4; ++c) xv[c] = Xs[kk][ty + 16 * c];
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (xv[c] != 0.0) acc[r][c] = xmac(acc[r][c], av[r], xv[c]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 2; ++r)
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
  const int rpt = (m + kBT - 1) / kBT;
  return rpt <= 1 ? 16 : (rpt <= 2 ? 8 : (rpt <= 4 ? 4 : 0));
}

cudaError_t launch_batched(const BatchArgs& a, int sm_count, cudaStream_t stream) {
  const int NB = batched_cols_per_cta(a.m);
  if (NB == 0) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(batched_nqp_kernel<16>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBatchSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(batched_nqp_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)kBatchSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(batched_nqp_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)kBatchSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const size_t smem = 5 * (size_t)a.m * NB * sizeof(double);
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
