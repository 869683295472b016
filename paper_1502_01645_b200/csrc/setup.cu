// setup.cu — K1-K3 (Gram over [A | b] with the cosine rescale fused into the
// epilogue) and K7 helpers (unscale, residual), all reference-order exact.
//
// Reference: gram (linalg.hpp:160-174), transpose_matvec + negate
// (nnls.hpp:133-134), rescale (nnls.hpp:41-83), unscale (nnls.hpp:87-96),
// residual_norm_sq (nnls.hpp:115-123).
//
// K1 is a register-tiled SIMT SYRK over the augmented matrix [A | b]: every
// output (i <= j) is ONE chain over k ascending of rounded products
// (__dmul_rn then __dadd_rn), exactly the reference's `s += ci[k]*cj[k]`. The
// b column makes column n of the output A^T b bitwise (products commute,
// same k order). On B200 the DMUL+DADD pair issues at the DFMA rate
// (measured: 36 TFLOP/s useful vs 34 DFMA, 37 DMMA), so the exact profile is
// not capped at half of the fp64 peak. The epilogue writes Q = H/(D_i D_j)
// (Q_ii = 1) and q = (-h)/D directly: H is never materialised.
#include "common.cuh"
#include "gemv.cuh"
#include "kernels.cuh"

namespace alnnls {

namespace {

constexpr int BM = 128;           // output tile (square)
constexpr int BK = 16;            // k slab
constexpr int TM = 8;             // per-thread register tile TM x TM
constexpr int NT = (BM / TM) * (BM / TM);  // 256 threads
constexpr int LDS = BM + 1;       // padded smem row (doubles): conflict-free stores

__device__ __forceinline__ const double* col_ptr(const SetupArgs& s, int c) {
  if (c < s.n) return s.A + (size_t)c * s.lda;
  if (c == s.n && s.b) return s.b;
  return nullptr;
}

// Upper-triangular tile index -> (ti, tj), ti <= tj.
__device__ __forceinline__ void tri_tile(int t, int nt, int& ti, int& tj) {
  // rows of the upper triangle: tj-major enumeration
  int j = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((j + 1) * (j + 2) / 2 <= t) ++j;
  while (j * (j + 1) / 2 > t) --j;
  tj = j;
  ti = t - j * (j + 1) / 2;
  (void)nt;
}

constexpr size_t kSyrkSmem = 2 * 2 * BK * LDS * sizeof(double);

__global__ void __launch_bounds__(NT, 1) syrk_exact_kernel(SetupArgs s, int mode, int na) {
  extern __shared__ __align__(16) double syrk_sm[];
  auto As = reinterpret_cast<double(*)[BK][LDS]>(syrk_sm);
  auto Bs = reinterpret_cast<double(*)[BK][LDS]>(syrk_sm + 2 * BK * LDS);
  const int ntile = (na + BM - 1) / BM;
  int ti, tj;
  tri_tile(blockIdx.x, ntile, ti, tj);
  const int i0 = ti * BM, j0 = tj * BM;
  const int tx = threadIdx.x % (BM / TM), ty = threadIdx.x / (BM / TM);

  // loader mapping: element e = threadIdx.x + r*NT, col = e / BK, kk = e % BK
  const double* pa[8];
  const double* pb[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int e = threadIdx.x + r * NT;
    pa[r] = col_ptr(s, i0 + e / BK);
    pb[r] = col_ptr(s, j0 + e / BK);
  }
  double ra[8], rb[8];
  auto gload = [&](int k0) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int kk = (threadIdx.x + r * NT) % BK;
      const int k = k0 + kk;
      ra[r] = (pa[r] && k < s.d) ? __ldg(pa[r] + k) : 0.0;
      rb[r] = (pb[r] && k < s.d) ? __ldg(pb[r] + k) : 0.0;
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int e = threadIdx.x + r * NT;
      As[buf][e % BK][e / BK] = ra[r];
      Bs[buf][e % BK][e / BK] = rb[r];
    }
  };

  double acc[TM][TM];
#pragma unroll
  for (int r = 0; r < TM; ++r)
#pragma unroll
    for (int c = 0; c < TM; ++c) acc[r][c] = 0.0;

  const int nk = (s.d + BK - 1) / BK;
  gload(0);
  sstore(0);
  __syncthreads();
  for (int kb = 0; kb < nk; ++kb) {
    const int buf = kb & 1;
    if (kb + 1 < nk) gload((kb + 1) * BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      double a[TM], b[TM];
#pragma unroll
      for (int r = 0; r < TM; ++r) a[r] = As[buf][kk][tx + r * (BM / TM)];
#pragma unroll
      for (int c = 0; c < TM; ++c) b[c] = Bs[buf][kk][ty + c * (BM / TM)];
#pragma unroll
      for (int r = 0; r < TM; ++r)
#pragma unroll
        for (int c = 0; c < TM; ++c) acc[r][c] = xmac(acc[r][c], a[r], b[c]);
    }
    if (kb + 1 < nk) {
      sstore(buf ^ 1);
      __syncthreads();
    }
  }

  // epilogue
#pragma unroll
  for (int r = 0; r < TM; ++r) {
    const int i = i0 + tx + r * (BM / TM);
#pragma unroll
    for (int c = 0; c < TM; ++c) {
      const int j = j0 + ty + c * (BM / TM);
      if (i > j || i >= s.n || j > s.n) continue;
      const double v = acc[r][c];
      if (j == s.n) {  // column n: (A^T b)_i, h = -(A^T b) (nnls.hpp:133-134)
        if (!s.b) continue;
        const double h = -v;
        if (mode == 0) {
          if (s.hvec) s.hvec[i] = h;
        } else {
          const int pi = s.pos[i];
          if (pi >= 0) s.q[pi] = xdiv(h, s.scale[pi]);  // nnls.hpp:79
        }
        continue;
      }
      if (mode == 0) {
        s.H[(size_t)j * s.n + i] = v;
        s.H[(size_t)i * s.n + j] = v;
      } else {
        const int pi = s.pos[i], pj = s.pos[j];
        if (pi < 0 || pj < 0) continue;
        if (i == j) {
          s.Q[blk_index(pi, pi, s.m, s.qR)] = 1.0;  // nnls.hpp:72
        } else {
          // nnls.hpp:75: H(ja, jb) / (scale[a] * scale[b]) with a < b
          const double qv = xdiv(v, xmul(s.scale[pi], s.scale[pj]));
          s.Q[blk_index(pi, pj, s.m, s.qR)] = qv;
          s.Q[blk_index(pj, pi, s.m, s.qR)] = qv;
        }
      }
    }
  }
}

// H_ii chain per column (identical to the SYRK diagonal chain).
__global__ void gram_diag_kernel(SetupArgs s) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= s.n) return;
  const double* p = s.A + (size_t)c * s.lda;
  double acc = 0.0;
  int k = 0;
  constexpr int B = 8;
  for (; k + B <= s.d; k += B) {
    double v[B];
#pragma unroll
    for (int t = 0; t < B; ++t) v[t] = __ldg(p + k + t);
#pragma unroll
    for (int t = 0; t < B; ++t) acc = xmac(acc, v[t], v[t]);
  }
  for (; k < s.d; ++k) {
    const double v = __ldg(p + k);
    acc = xmac(acc, v, v);
  }
  s.diag[c] = acc;
}

// rescale bookkeeping (nnls.hpp:53-63): retained ascending, D = sqrt(H_ii).
__global__ void retained_kernel(const double* diag, int n, int* pos, double* scale,
                                uint32_t* retained, int* m_out, int* neg_flag) {
  __shared__ int scan[40];
  const int nt = blockDim.x;
  const int per = (n + nt - 1) / nt;
  const int lo = min(n, (int)threadIdx.x * per), hi = min(n, lo + per);
  int cnt = 0, neg = 0;
  for (int i = lo; i < hi; ++i) {
    const double dg = diag[i];
    if (!(dg >= 0.0)) neg = 1;
    if (dg != 0.0) ++cnt;
  }
  int total;
  int off = block_exclusive_scan(cnt, scan, &total);
  for (int i = lo; i < hi; ++i) {
    const double dg = diag[i];
    if (dg != 0.0) {
      pos[i] = off;
      retained[off] = (uint32_t)i;
      scale[off] = __dsqrt_rn(dg);
      ++off;
    } else {
      pos[i] = -1;
    }
  }
  neg = __syncthreads_or(neg);
  if (threadIdx.x == 0) {
    *m_out = total;
    if (neg_flag) *neg_flag = neg;
  }
}

// Q from an explicit H (alnnls_rescale): one thread per output entry.
__global__ void rescale_from_h_kernel(const double* H, const double* h, int n, const int* pos,
                                      const double* scale, double* Q, int m, int qR, double* q) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  if (i >= n || j >= n || i > j) return;
  const int pi = pos[i], pj = pos[j];
  if (pi < 0 || pj < 0) return;
  if (i == j) {
    Q[blk_index(pi, pi, m, qR)] = 1.0;
    q[pi] = xdiv(h[i], scale[pi]);
    return;
  }
  const double v = xdiv(H[(size_t)j * n + i], xmul(scale[pi], scale[pj]));
  Q[blk_index(pi, pj, m, qR)] = v;
  Q[blk_index(pj, pi, m, qR)] = v;
}

__global__ void unscale_kernel(const double* y, const double* scale, const uint32_t* retained,
                               int m, double* x) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a < m) x[retained[a]] = xdiv(y[a], scale[a]);
}

// r_i = ax_i - b_i; prod_i = r_i*r_i in parallel; then one ordered chain.
__global__ void residual_kernel(const double* ax, const double* b, int d, double* prod,
                                double* out) {
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const double r = xsub(ax[i], b[i]);
    prod[i] = xmul(r, r);
  }
  __syncthreads();
  if (threadIdx.x == 0) *out = chain_sum(prod, d);
}

__global__ void support_kernel(const double* x, int n, uint32_t* list, double* vals, int* len) {
  __shared__ int scan[40];
  const int nt = blockDim.x;
  const int per = (n + nt - 1) / nt;
  const int lo = min(n, (int)threadIdx.x * per), hi = min(n, lo + per);
  int cnt = 0;
  for (int i = lo; i < hi; ++i) cnt += (x[i] != 0.0);
  int total;
  int off = block_exclusive_scan(cnt, scan, &total);
  for (int i = lo; i < hi; ++i) {
    if (x[i] != 0.0) {
      list[off] = (uint32_t)i;
      vals[off] = x[i];
      ++off;
    }
  }
  if (threadIdx.x == 0) *len = total;
}

// y_j = sum_i M[i, j] v_i, one ascending chain per column (linalg.hpp:209-219).
__global__ void coldot_kernel(const double* M, uint64_t ld, int rows, int cols, const double* v,
                              double* y) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  const double* p = M + (size_t)c * ld;
  double acc = 0.0;
  int k = 0;
  constexpr int B = 8;
  for (; k + B <= rows; k += B) {
    double a[B], w[B];
#pragma unroll
    for (int t = 0; t < B; ++t) {
      a[t] = __ldg(p + k + t);
      w[t] = __ldg(v + k + t);
    }
#pragma unroll
    for (int t = 0; t < B; ++t) acc = xmac(acc, a[t], w[t]);
  }
  for (; k < rows; ++k) acc = xmac(acc, __ldg(p + k), __ldg(v + k));
  y[c] = acc;
}

__global__ void add_kernel(const double* y, const double* q, double* g, int m) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) g[i] = xadd(y[i], q[i]);
}

__global__ void check_finite_kernel(const double* p, uint64_t rows, uint64_t cols, uint64_t ld,
                                    int* flag) {
  const uint64_t total = rows * cols;
  int bad = 0;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = e / rows, r = e % rows;
    if (!isfinite(p[c * ld + r])) bad = 1;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) *flag = 1;
}

__global__ void copy_pad_kernel(const double* src, uint64_t ld_src, double* dst, uint64_t ld_dst,
                                uint64_t rows, uint64_t cols) {
  const uint64_t total = rows * cols;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = e / rows, r = e % rows;
    dst[c * ld_dst + r] = src[c * ld_src + r];
  }
}

// column-major (ld) <-> blocked layout; one thread per element
__global__ void to_blocked_kernel(const double* src, uint64_t ld, int m, int R, double* dst,
                                  int dir) {
  const uint64_t total = (uint64_t)m * m;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = e / m, i = e % m;
    if (dir == 0)
      dst[blk_index(i, j, m, R)] = src[j * ld + i];
    else
      dst[j * ld + i] = src[blk_index(i, j, m, R)];
  }
}

}  // namespace

cudaError_t launch_to_blocked(const double* src, uint64_t ld, int m, int R, double* dst,
                              cudaStream_t stream) {
  if (m <= 0) return cudaSuccess;
  to_blocked_kernel<<<148 * 8, 256, 0, stream>>>(src, ld, m, R, dst, 0);
  return cudaGetLastError();
}

cudaError_t launch_from_blocked(const double* src, int m, int R, double* dst, uint64_t ld,
                                cudaStream_t stream) {
  if (m <= 0) return cudaSuccess;
  to_blocked_kernel<<<148 * 8, 256, 0, stream>>>(src, ld, m, R, dst, 1);
  return cudaGetLastError();
}

cudaError_t launch_gram_diag(const SetupArgs& s, cudaStream_t stream) {
  if (s.n <= 0) return cudaSuccess;
  gram_diag_kernel<<<(s.n + 127) / 128, 128, 0, stream>>>(s);
  return cudaGetLastError();
}

cudaError_t launch_retained(const SetupArgs& s, cudaStream_t stream) {
  retained_kernel<<<1, 1024, 0, stream>>>(s.diag, s.n, s.pos, s.scale, s.retained, s.m_out,
                                          nullptr);
  return cudaGetLastError();
}

cudaError_t launch_syrk(const SetupArgs& s, int mode, cudaStream_t stream) {
  const int na = s.n + (s.b ? 1 : 0);
  const int nt = (na + BM - 1) / BM;
  const int tiles = nt * (nt + 1) / 2;
  if (tiles == 0) return cudaSuccess;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(syrk_exact_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSyrkSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  syrk_exact_kernel<<<tiles, NT, kSyrkSmem, stream>>>(s, mode, na);
  return cudaGetLastError();
}

cudaError_t launch_rescale_from_h(const double* H, const double* h, int n, const int* pos,
                                  const double* scale, double* Q, int m, int qR, double* q,
                                  cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  dim3 grid((n + 127) / 128, n);
  rescale_from_h_kernel<<<grid, 128, 0, stream>>>(H, h, n, pos, scale, Q, m, qR, q);
  return cudaGetLastError();
}

cudaError_t launch_unscale(const double* y, const double* scale, const uint32_t* retained, int m,
                           double* x, int n, cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(x, 0, sizeof(double) * (n > 0 ? n : 1), stream);
  if (e != cudaSuccess || m <= 0) return e;
  unscale_kernel<<<(m + 255) / 256, 256, 0, stream>>>(y, scale, retained, m, x);
  return cudaGetLastError();
}

cudaError_t launch_residual(const double* ax, const double* b, int d, double* prod, double* out,
                            cudaStream_t stream) {
  residual_kernel<<<1, 1024, 0, stream>>>(ax, b, d, prod, out);
  return cudaGetLastError();
}

cudaError_t launch_support(const double* x, int n, uint32_t* list, double* vals, int* len,
                           cudaStream_t stream) {
  support_kernel<<<1, 1024, 0, stream>>>(x, n, list, vals, len);
  return cudaGetLastError();
}

cudaError_t launch_coldot(const double* M, uint64_t ld, int rows, int cols, const double* v,
                          double* y, cudaStream_t stream) {
  if (cols <= 0) return cudaSuccess;
  coldot_kernel<<<(cols + 127) / 128, 128, 0, stream>>>(M, ld, rows, cols, v, y);
  return cudaGetLastError();
}

cudaError_t launch_add(const double* y, const double* q, double* g, int m, cudaStream_t stream) {
  if (m <= 0) return cudaSuccess;
  add_kernel<<<(m + 255) / 256, 256, 0, stream>>>(y, q, g, m);
  return cudaGetLastError();
}

cudaError_t launch_check_finite(const double* p, uint64_t rows, uint64_t cols, uint64_t ld,
                                int* flag, cudaStream_t stream) {
  if (rows * cols == 0) return cudaSuccess;
  uint64_t blocks = (rows * cols + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  check_finite_kernel<<<(unsigned)blocks, 256, 0, stream>>>(p, rows, cols, ld, flag);
  return cudaGetLastError();
}

cudaError_t launch_copy_pad(const double* src, uint64_t ld_src, double* dst, uint64_t ld_dst,
                            uint64_t rows, uint64_t cols, cudaStream_t stream) {
  if (rows * cols == 0) return cudaSuccess;
  uint64_t blocks = (rows * cols + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  copy_pad_kernel<<<(unsigned)blocks, 256, 0, stream>>>(src, ld_src, dst, ld_dst, rows, cols);
  return cudaGetLastError();
}

}  // namespace alnnls
