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

constexpr int kBT = 512;          // threads per batched CTA (one warp per column at NB = 16)
constexpr int kMaxCols = 16;      // NB upper bound (columns per CTA)

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
};

// GEMM operands V, U are row-major m x ld with ld = NB + 2: the GEMM reads a
// row of V with 16-byte broadcasts, and the padding keeps a warp's per-column
// walk (lane = row) to 4-way bank sharing. The per-column state (candidate C,
// iterate X, gradient G, linear term q) lives in contiguous column panels, so
// the per-column walks are conflict-free.
struct BatchSmem {
  double* V;  // GEMM input: g_bar (P1) or delta (P2), 0 off the mask / changed set
  double* U;  // GEMM output: Q g_bar or Q delta
  int ld;
  int m;
  double* C;  // candidate x   (panel b at C + b * m)
  double* X;  // iterate
  double* G;  // maintained gradient
  double* q;  // linear term
  __device__ double& v(int i, int b) const { return V[i * ld + b]; }
  __device__ double& u(int i, int b) const { return U[i * ld + b]; }
  __device__ double* c(int b) const { return C + b * m; }
  __device__ double* x(int b) const { return X + b * m; }
  __device__ double* g(int b) const { return G + b * m; }
  __device__ double* qc(int b) const { return q + b * m; }
};

__host__ __device__ constexpr int batch_ld(int nb) { return nb + 2; }
size_t batch_smem_bytes(int m, int nb) {
  return ((size_t)2 * m * batch_ld(nb) + (size_t)4 * m * nb) * sizeof(double);
}

// s = ((0 + t(i0)) + t(i1)) + ... over i ascending, skipping the terms with
// use == false (exact zeros in the reference chain). The terms of the next 8
// indices are loaded and multiplied while the current 8 are added, so only the
// DADD latency is on the chain.
template <class F>
__device__ __forceinline__ double col_chain(int m, F term) {
  double s = 0.0;
  double t[8];
  bool use[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    use[k] = false;
    t[k] = 0.0;
    if (k < m) t[k] = term(k, use[k]);
  }
  for (int i0 = 0; i0 < m; i0 += 8) {
    double tn[8];
    bool un[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      un[k] = false;
      tn[k] = 0.0;
      if (i0 + 8 + k < m) tn[k] = term(i0 + 8 + k, un[k]);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (use[k]) s = xadd(s, t[k]);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      t[k] = tn[k];
      use[k] = un[k];
    }
  }
  return s;
}

// Strided product chain: sum of a[i*sa] * b[i*sb] over i with u[i*su] != 0.
__device__ __forceinline__ double prod_chain(int m, const double* a, int sa, const double* b, int sb,
                                             const double* u, int su) {
  return col_chain(m, [&](int i, bool& use) {
    use = u[i * su] != 0.0;
    return xmul(a[i * sa], b[i * sb]);
  });
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
  int cnt = 0, bad = 0;
  for (int i = lane; i < a.m; i += 32) {
    const double xi = xb[i], gi = gb[i];
    const bool p = xi > 0.0 || gi < 0.0;
    cnt += p;
    if (!isfinite(gi)) bad = 1;
    sm.v(i, b) = p ? gi : 0.0;  // g_bar
  }
  for (int o = 16; o > 0; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  __syncwarp();
  // lanes 0, 1, 2 run the three chains side by side (one code path, per-lane
  // operands), each in ascending index order; terms off the mask are exact
  // zeros (g_bar = 0, x = 0) and are skipped. q.x uses x*q (same product bits).
  double s = 0.0;
  if (lane < 3) {
    const double* pa = lane == 0 ? &sm.v(0, b) : xb;
    const int sa = lane == 0 ? sm.ld : 1;
    const double* pb = lane == 0 ? &sm.v(0, b) : (lane == 1 ? gb : sm.qc(b));
    const int sb = lane == 0 ? sm.ld : 1;
    s = prod_chain(a.m, pa, sa, pb, sb, pa, sa);
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
  if (stop >= 0) finish_col(a, S, sm, b, stop == 100 ? 0 : stop, stop == 100);
  return stop >= 0;
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

template <int NB>
__global__ void __launch_bounds__(kBT, 1) batched_nqp_kernel(BatchArgs a) {
  extern __shared__ __align__(16) double bsm[];
  __shared__ ColState S;
  const int m = a.m;
  constexpr int LD = batch_ld(NB);
  BatchSmem sm;
  sm.ld = LD;
  sm.m = m;
  sm.V = bsm;
  sm.U = bsm + (size_t)m * LD;
  sm.C = bsm + 2 * (size_t)m * LD;
  sm.X = sm.C + (size_t)m * NB;
  sm.G = sm.X + (size_t)m * NB;
  sm.q = sm.G + (size_t)m * NB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int nwarps = kBT / 32;
  for (int b = warp; b < NB; b += nwarps) refill(a, S, sm, b);
  __syncthreads();
  // GEMM thread mapping: GROUPS groups of CG columns; rows i = trow + r * ROWT
  constexpr int CG = NB < 8 ? NB : 8;
  constexpr int GROUPS = NB / CG;
  constexpr int ROWT = kBT / GROUPS;
  constexpr int RPT = (4096 / NB + ROWT - 1) / ROWT;  // rows per thread at the largest m (4096/NB)
  const int grp = threadIdx.x / ROWT, trow = threadIdx.x % ROWT;
  for (;;) {
    // any active column?
    int active = 0;
    for (int b = 0; b < NB; ++b) active |= S.phase[b] != kIdle;
    if (!active) break;
    // ---- one exact chain GEMM pass: U = Q V (ascending j per output). Off-mask
    // entries of V are 0 and their +-0 products are exact no-ops (idle slots too).
    double acc[RPT * CG];
#pragma unroll
    for (int t = 0; t < RPT * CG; ++t) acc[t] = 0.0;
    constexpr int JB = 8;  // Q columns whose loads are in flight together (L2 latency)
    for (int j0 = 0; j0 < m; j0 += JB) {
      double qv[RPT][JB];
#pragma unroll
      for (int u = 0; u < JB; ++u) {
        const double* qc = a.Q + (size_t)(j0 + u) * m;
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          const int i = trow + r * ROWT;
          qv[r][u] = (j0 + u < m && i < m) ? __ldg(qc + i) : 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < JB; ++u) {
        const int j = j0 + u;
        if (j >= m) break;
        const double* vrow = sm.V + (size_t)j * LD + grp * CG;
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
    }
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int i = trow + r * ROWT;
      if (i < m) {
        double* urow = sm.U + (size_t)i * LD + grp * CG;
#pragma unroll
        for (int b = 0; b < CG; b += 2)
          *reinterpret_cast<double2*>(urow + b) = make_double2(acc[r * CG + b], acc[r * CG + b + 1]);
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
        if (lane == 0) den = prod_chain(m, &sm.v(0, b), LD, &sm.u(0, b), LD, &sm.v(0, b), LD);
        den = __shfl_sync(0xffffffffu, den, 0);
        if (!(den > 0.0)) {
          finish_col(a, S, sm, b, ALNNLS_ZERO_CURVATURE, 0);
          refill(a, S, sm, b);
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
        const double* gb = sm.g(b);
        if (lane == 0) {
          df = col_chain(m, [&](int i, bool& use) {
            const double dd = sm.v(i, b);
            use = dd != 0.0;
            return xmul(xadd(gb[i], xmul(0.5, sm.u(i, b))), dd);
          });
        }
        df = __shfl_sync(0xffffffffu, df, 0);
        const bool accept = df <= 0.0 || S.tries[b] >= 60;
        if (accept) {  // x[C] = cand, grad += gd (nqp.hpp:309-313)
          double* xb = sm.x(b);
          double* gw = sm.g(b);
          const double* cb = sm.c(b);
          for (int i = lane; i < m; i += 32) {
            xb[i] = cb[i];
            gw[i] = xadd(gw[i], sm.u(i, b));
          }
          if (lane == 0) ++S.k[b];
          __syncwarp();
          if (mask_phase(a, S, sm, b)) refill(a, S, sm, b);
          continue;
        }
        if (lane == 0) {
          S.alpha[b] = xmul(S.alpha[b], 0.5);  // nqp.hpp:317
          ++S.tries[b];
        }
        __syncwarp();
      }
      // candidate step with the current alpha
      const int cl = cand_phase(a, S, sm, b);
      if (lane == 0) S.cl[b] = cl;
      if (cl == 0) {  // nothing moved (nqp.hpp:304): next iteration on the same state
        if (lane == 0) ++S.k[b];
        __syncwarp();
        if (mask_phase(a, S, sm, b)) refill(a, S, sm, b);
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
  // shared memory holds 5 m x NB panels; the GEMM covers m <= 4096 / NB rows
  return m <= 256 ? 16 : (m <= 512 ? 8 : (m <= 1024 ? 4 : 0));
}

cudaError_t launch_batched(const BatchArgs& a, int sm_count, cudaStream_t stream) {
  const int NB = batched_cols_per_cta(a.m);
  if (NB == 0) return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    const int mx = (int)batch_smem_bytes(1024, 4);  // the largest configuration
    cudaError_t e = cudaFuncSetAttribute(batched_nqp_kernel<16>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(batched_nqp_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(batched_nqp_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    if (e != cudaSuccess) return e;
    attr = true;
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
