// dmma.cu — FAST profile setup: the Gram (and A^T B for batched right-hand
// sides) on the fp64 tensor cores (mma.sync m16n8k8 f64, DMMA; B200 measured
// 37 TFLOP/s vs 18.5 for the exact DMUL+DADD chains).
//
// DMMA accumulates each k8 group with its own internal ordering and fused
// products, so the results are not the reference's bit pattern (that is what
// the EXACT profile is for); they are within the north-star tolerances
// (tests/test_gpu_fast.py). Everything downstream of the Gram (rescale
// epilogue, loop, unscale, residual) is the same code as EXACT.
//
// Kernel: 128 x 128 output tiles (upper triangle for the Gram, the full grid for
// A^T B), 256 threads = 8 warps as 2 (M) x 4 (N), warp tile 64 x 32 = 4 x 4
// m16n8k8 accumulators; k slabs of 16 staged by cp.async (16 B chunks) through
// a 4-deep ring. Shared tiles are [column][k] with the 16 B chunk index XOR-
// swizzled by 2 (column & 3), so both fragment loads are bank-conflict-free.
#include "common.cuh"
#include "gemv.cuh"
#include "kernels.cuh"

namespace alnnls {

namespace {

constexpr int TB = 128;      // output tile
constexpr int TK = 16;       // k slab (two m16n8k8 steps)
constexpr int TT = 256;      // threads
constexpr int TSTAGES = 4;
constexpr int kTileDoubles = TB * TK;  // one operand slab
constexpr size_t kDmmaSmem = (size_t)TSTAGES * 2 * kTileDoubles * sizeof(double);  // 128 KB

__device__ __forceinline__ void tri_tile_u(int t, int& ti, int& tj) {
  int j = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((j + 1) * (j + 2) / 2 <= t) ++j;
  while (j * (j + 1) / 2 > t) --j;
  tj = j;
  ti = t - j * (j + 1) / 2;
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void dmma(double (&c)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

// element (col r, k) of a swizzled [TB][TK] slab
// The XOR pattern spreads the 4 rows x 4 k of a half-warp's fragment load over all
// 32 banks: ((r & 3) << 1) maps the two 16 B chunks a row contributes to 8 distinct
// chunks (an (r & 7) pattern left the rows r and r ^ 1 on the same banks: 2-way
// conflicts on every fragment load, 207.6 M in the c2 capture).
__device__ __forceinline__ int swz(int r, int k) {
  return r * TK + ((((k >> 1) ^ ((r & 3) << 1))) << 1) + (k & 1);
}

// Output element (i, j) of the Gram / A^T B with the same epilogues as the
// exact kernel (setup.cu syrk_exact_kernel).
__device__ __forceinline__ void store_out(const SetupArgs& s, int mode, int i, int j, double v) {
  if (mode == 2) {  // q_b of RHS column j (nnls.hpp:79, :133-134)
    if (i >= s.n || j >= s.nrhs) return;
    const int pi = s.pos[i];
    if (pi >= 0) s.QB[(size_t)j * s.m + pi] = xdiv(-v, s.scale[pi]);
    return;
  }
  if (i > j || j >= s.n) return;
  if (mode == 0) {
    s.H[(size_t)j * s.n + i] = v;
    s.H[(size_t)i * s.n + j] = v;
    return;
  }
  const int pi = s.pos[i], pj = s.pos[j];
  if (pi < 0 || pj < 0) return;
  if (i == j) {
    s.Q[blk_index(pi, pi, s.m, s.qR)] = 1.0;  // nnls.hpp:72
  } else {
    const double qv = xdiv(v, xmul(s.scale[pi], s.scale[pj]));  // nnls.hpp:75
    s.Q[blk_index(pi, pj, s.m, s.qR)] = qv;
    s.Q[blk_index(pj, pi, s.m, s.qR)] = qv;
  }
}

__global__ void __launch_bounds__(TT, 1) syrk_dmma_kernel(SetupArgs s, int mode) {
  extern __shared__ __align__(128) double dm_sm[];
  double* As = dm_sm;                              // [TSTAGES][TB*TK]
  double* Bs = dm_sm + TSTAGES * kTileDoubles;     // [TSTAGES][TB*TK]
  int ti, tj;
  if (mode == 2) {
    const int nti = (s.n + TB - 1) / TB;
    ti = blockIdx.x % nti;
    tj = blockIdx.x / nti;
  } else {
    tri_tile_u(blockIdx.x, ti, tj);
  }
  const int i0 = ti * TB, j0 = tj * TB;
  const double* Bop = mode == 2 ? s.B : s.A;
  const uint64_t ldb = mode == 2 ? s.ldb : s.lda;
  const int nb = mode == 2 ? s.nrhs : s.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;  // warp tile rows wm*64, cols wn*32
  const int g = lane >> 2, t = lane & 3;

  // loader: chunk e = tid + p*TT (p < 4) of a slab: column e >> 3, k pair (e & 7)
  const double* pa[4];
  const double* pb[4];
  int dst[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int e = tid + p * TT, r = e >> 3, c = e & 7;
    pa[p] = i0 + r < s.n ? s.A + (size_t)(i0 + r) * s.lda + 2 * c : nullptr;
    pb[p] = j0 + r < nb ? Bop + (size_t)(j0 + r) * ldb + 2 * c : nullptr;
    dst[p] = swz(r, 2 * c);
  }
  const int nk = (s.d + TK - 1) / TK;
  auto issue = [&](int kb) {
    const int st = kb % TSTAGES;
    const int k0 = kb * TK;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int c = (tid + p * TT) & 7;
      const int left = s.d - (k0 + 2 * c);  // valid doubles in this pair
      const uint32_t bytes = left >= 2 ? 16u : (left == 1 ? 8u : 0u);
      cp_async16(As + st * kTileDoubles + dst[p], pa[p] && bytes ? pa[p] + k0 : s.A,
                 pa[p] ? bytes : 0u);
      cp_async16(Bs + st * kTileDoubles + dst[p], pb[p] && bytes ? pb[p] + k0 : s.A,
                 pb[p] ? bytes : 0u);
    }
  };

  double acc[4][4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.0;

#pragma unroll
  for (int p = 0; p < TSTAGES - 1; ++p) {
    if (p < nk) issue(p);
    cp_commit();
  }
  for (int kb = 0; kb < nk; ++kb) {
    cp_wait<TSTAGES - 2>();
    __syncthreads();
    if (kb + TSTAGES - 1 < nk) issue(kb + TSTAGES - 1);
    cp_commit();
    const double* as = As + (kb % TSTAGES) * kTileDoubles;
    const double* bs = Bs + (kb % TSTAGES) * kTileDoubles;
#pragma unroll
    for (int ks = 0; ks < TK; ks += 8) {
      double af[4][4], bf[4][2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        const int r = wm * 64 + mi * 16 + g;
        af[mi][0] = as[swz(r, ks + t)];
        af[mi][1] = as[swz(r + 8, ks + t)];
        af[mi][2] = as[swz(r, ks + t + 4)];
        af[mi][3] = as[swz(r + 8, ks + t + 4)];
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const int r = wn * 32 + ni * 8 + g;
        bf[ni][0] = bs[swz(r, ks + t)];
        bf[ni][1] = bs[swz(r, ks + t + 4)];
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], af[mi], bf[ni]);
    }
  }
  cp_wait<0>();

#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int i = i0 + wm * 64 + mi * 16 + g + (c >> 1) * 8;
        const int j = j0 + wn * 32 + ni * 8 + 2 * t + (c & 1);
        if (i < s.n) store_out(s, mode, i, j, acc[mi][ni][c]);
      }
}

}  // namespace

bool syrk_dmma_supported(const SetupArgs& s, int mode) {
  const uint64_t ldb = mode == 2 ? s.ldb : s.lda;
  const void* b = mode == 2 ? static_cast<const void*>(s.B) : static_cast<const void*>(s.A);
  return (s.lda % 2 == 0) && (ldb % 2 == 0) && (reinterpret_cast<uintptr_t>(s.A) % 16 == 0) &&
         (reinterpret_cast<uintptr_t>(b) % 16 == 0);
}

cudaError_t launch_syrk_dmma(const SetupArgs& s, int mode, cudaStream_t stream) {
  const int nt = (s.n + TB - 1) / TB;
  const int tiles = mode == 2 ? nt * ((s.nrhs + TB - 1) / TB) : nt * (nt + 1) / 2;
  if (tiles == 0) return cudaSuccess;
  if (!syrk_dmma_supported(s, mode)) return cudaErrorInvalidValue;
  if (cudaError_t e = smem_optin(syrk_dmma_kernel, (int)kDmmaSmem)) return e;
  syrk_dmma_kernel<<<tiles, TT, kDmmaSmem, stream>>>(s, mode);
  return cudaGetLastError();
}

}  // namespace alnnls
