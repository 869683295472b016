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
#include <cuda.h>

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


// ===== v2: TMA-fed, stream-K persistent DMMA Gram / A^T B (north_star: "DMMA tensor
// cores fed by TMA-staged shared-memory tiles") =====================================
// Operand slabs (128 columns x 16 k of A, and of A or B) arrive by
// cp.async.bulk.tensor.2d (TMA, UTMALDG) with the hardware 128-byte swizzle
// (element (r, k) at r*128 + (((k>>1) ^ (r&7)) << 4) + (k&1)*8 bytes): the
// m16n8k8 fragment loads of a warp then touch every bank exactly twice (two
// wavefronts for 256 bytes, conflict-free), and out-of-range rows / columns are
// zero-filled by the TMA unit (ragged shapes need no special code).
// Schedule: persistent CTAs, one per SM; the (tile, k-slab) units are split into
// equal contiguous ranges (stream-K), so no wave is ragged. A tile cut between
// CTAs is finished by the CTA holding its first slab (k = 0), which processes it
// LAST in its range, by then the later CTAs (which hold the rest at the START of
// their ranges) have published their partial accumulators; it adds them in CTA
// order (a fixed order: deterministic run to run).
// Pipeline: kStages slab pairs in shared memory, full/empty mbarriers; thread 0
// (also a consumer) refills the stage every warp has released.
constexpr int kStages2 = 6;  // 6 x 32 KB; the 128 KB epilogue tile reuses them
constexpr uint32_t kSlabBytes = TB * TK * sizeof(double);  // 16 KB per operand slab
constexpr size_t kDmma2Smem = (size_t)kStages2 * 2 * kSlabBytes + 1024;  // + alignment slack

struct TmaArgs {
  CUtensorMap mapA;  // A: dims {d, n}, box {16, 128}
  CUtensorMap mapB;  // B (mode 2) or A again
  int tiles;         // output tiles (upper triangle, or the full grid in mode 2)
  int tile_lo;       // first tile of the launch (a contiguous range of the tile order)
  int nk;            // k slabs per tile
  int nti;           // tile rows (mode 2 grid decode)
  double* ws;        // [grid][128*128] partial tiles of cut tiles
  int* flags;        // [grid] partial published (zeroed before the launch)
  int accumulate;    // mode 0: bit 0: H += result instead of H = result; bit 1: write
                     // only the upper triangle H(i <= j) (no strided mirror stores)
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ int swz128(int r, int k) {  // double index in a TMA 128B-swizzled slab
  return r * TK + ((((k >> 1) ^ (r & 7))) << 1) + (k & 1);
}

__device__ __forceinline__ void tile_coords(int mode, int t, int nti, int& ti, int& tj) {
  if (mode == 2) {
    ti = t % nti;
    tj = t / nti;
  } else {
    tri_tile_u(t, ti, tj);
  }
}

__global__ void __launch_bounds__(TT, 1)
    syrk_tma_kernel(const __grid_constant__ TmaArgs ta, SetupArgs s, int mode) {
  extern __shared__ uint8_t dm2_raw[];
  // 1024-byte aligned (the 128B swizzle atom), by offsetting the shared array itself so
  // the compiler keeps the shared state space (LDS, not generic loads)
  double* sm = reinterpret_cast<double*>(dm2_raw + ((1024u - (smem_u32(dm2_raw) & 1023u)) & 1023u));
  __shared__ __align__(8) uint64_t full[kStages2];
  __shared__ __align__(8) uint64_t empty[kStages2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;
  const int g = lane >> 2, t = lane & 3;
  const int sg = (g >> 1) | ((g & 1) << 2);  // slab row of fragment row g (see the loads)
  const long long U = (long long)ta.tiles * ta.nk;
  const int G = gridDim.x, c = blockIdx.x;
  const long long u0 = U * c / G, u1 = U * (c + 1) / G;
  if (tid == 0) {
    for (int st = 0; st < kStages2; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], TT / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  auto slabA = [&](int st) { return sm + (size_t)st * 2 * (TB * TK); };
  auto slabB = [&](int st) { return sm + (size_t)st * 2 * (TB * TK) + TB * TK; };
  double* tile_s = sm;  // epilogue staging [128 j][128 i] over the (drained) stages
  long long q = 0;      // units consumed by this CTA (stage / phase counter)
  long long u = u0;
  while (u < u1) {
    // ---- one segment: tile `tile`, slabs [kb0, kb1) ----
    const int tile = (int)(u / ta.nk), kb0 = (int)(u % ta.nk);
    const long long tstart = (long long)tile * ta.nk, tend = tstart + ta.nk;
    const int kb1 = (int)((tend < u1 ? tend : u1) - tstart);
    const int len = kb1 - kb0;
    int ti, tj;
    tile_coords(mode, tile + ta.tile_lo, ta.nti, ti, tj);
    auto issue = [&](long long qq, int kb) {  // thread 0: load slab kb as unit qq
      const int st = (int)(qq % kStages2);
      const long long round = qq / kStages2;
      if (round >= 1) mbar_wait(&empty[st], (uint32_t)((round - 1) & 1));
      mbar_arrive_expect_tx(&full[st], 2 * kSlabBytes);
      tma_load_2d(slabA(st), &ta.mapA, kb * TK, ti * TB, &full[st]);
      tma_load_2d(slabB(st), &ta.mapB, kb * TK, tj * TB, &full[st]);
    };
    if (tid == 0)
      for (int k = 0; k < len && k < kStages2 - 1; ++k) issue(q + k, kb0 + k);
    double acc[4][4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[a][b][e] = 0.0;
    for (int k = 0; k < len; ++k, ++q) {
      if (tid == 0 && k + kStages2 - 1 < len) issue(q + kStages2 - 1, kb0 + k + kStages2 - 1);
      const int st = (int)(q % kStages2);
      mbar_wait(&full[st], (uint32_t)((q / kStages2) & 1));
      const double* as = slabA(st);
      const double* bs = slabB(st);
      // Fragment loads, conflict-free 128-bit: the k8 step's positions (t, t + 4) take
      // k = ks + 2t and ks + 2t + 1 (adjacent: one LDS.128 per row), and fragment row
      // g reads slab row sg = (g >> 1) | ((g & 1) << 2) of its 8-row group, so the 8
      // lanes of each quarter-warp land on 8 distinct 16-byte chunks of the 128B
      // swizzle (the natural mapping put two lanes on each chunk: 2x wavefronts,
      // 207.6 M bank conflicts per c2 Gram). The epilogue undoes the row map.
#pragma unroll
      for (int ks = 0; ks < TK; ks += 8) {
        double af[4][4], bf[4][2];
        const int kk = ks + 2 * t;
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
          const int r = wm * 64 + mi * 16 + sg;
          const double2 lo = *reinterpret_cast<const double2*>(as + swz128(r, kk));
          const double2 hi = *reinterpret_cast<const double2*>(as + swz128(r + 8, kk));
          af[mi][0] = lo.x;
          af[mi][2] = lo.y;
          af[mi][1] = hi.x;
          af[mi][3] = hi.y;
        }
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
          const int r = wn * 32 + ni * 8 + sg;
          const double2 v = *reinterpret_cast<const double2*>(bs + swz128(r, kk));
          bf[ni][0] = v.x;
          bf[ni][1] = v.y;
        }
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], af[mi], bf[ni]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    u = tstart + kb1;
    // ---- epilogue: the stages are drained; stage the tile through shared memory ----
    __syncthreads();
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int cn = 2 * t + (e & 1);  // fragment column -> B slab row
          const int il = wm * 64 + mi * 16 + sg + (e >> 1) * 8;
          const int jl = wn * 32 + ni * 8 + ((cn >> 1) | ((cn & 1) << 2));
          tile_s[jl * TB + il] = acc[mi][ni][e];
        }
    __syncthreads();
    const bool first = tstart >= u0;  // this CTA holds slab 0 of the tile: it finishes it
    if (!first) {                     // publish the partial for the finisher (previous CTA)
      double2* wsl = reinterpret_cast<double2*>(ta.ws + (size_t)c * TB * TB);
      const double2* t2 = reinterpret_cast<const double2*>(tile_s);
      for (int e = tid; e < TB * TB / 2; e += TT) wsl[e] = t2[e];
      __threadfence();
      __syncthreads();
      if (tid == 0) atomicExch(ta.flags + c, 1);
    } else {
      // later CTAs holding the rest of the tile, added in CTA order (deterministic)
      for (int c2 = c + 1; c2 < G && U * c2 / G < tend; ++c2) {
        if (tid == 0)
          while (atomicAdd(ta.flags + c2, 0) == 0) {
          }
        __syncthreads();
        __threadfence();
        const double2* w2 = reinterpret_cast<const double2*>(ta.ws + (size_t)c2 * TB * TB);
        double2* t2 = reinterpret_cast<double2*>(tile_s);
        constexpr int kU = 8;  // 8 independent 16-byte loads in flight per thread
        for (int e = tid; e < TB * TB / 2; e += kU * TT) {
          double2 v[kU];
#pragma unroll
          for (int k2 = 0; k2 < kU; ++k2) v[k2] = __ldcg(w2 + e + k2 * TT);
#pragma unroll
          for (int k2 = 0; k2 < kU; ++k2) {
            double2 o = t2[e + k2 * TT];
            o.x += v[k2].x;
            o.y += v[k2].y;
            t2[e + k2 * TT] = o;
          }
        }
        __syncthreads();
      }
      const int i0 = ti * TB, j0 = tj * TB;
      for (int e = tid; e < TB * TB; e += TT) {
        const int i = i0 + (e & (TB - 1)), j = j0 + e / TB;
        if (i >= s.n) continue;
        const double v = tile_s[e];
        if (mode == 0 && ta.accumulate) {
          if (i <= j && j < s.n) {
            const double w = (ta.accumulate & 1) ? s.H[(size_t)j * s.n + i] + v : v;
            s.H[(size_t)j * s.n + i] = w;
            if (i != j && !(ta.accumulate & 2)) s.H[(size_t)i * s.n + j] = w;
          }
        } else {
          store_out(s, mode, i, j, v);
        }
      }
    }
    __syncthreads();  // the staging area is stage memory again
  }
}

}  // namespace

bool syrk_dmma_supported(const SetupArgs& s, int mode) {
  const uint64_t ldb = mode == 2 ? s.ldb : s.lda;
  const void* b = mode == 2 ? static_cast<const void*>(s.B) : static_cast<const void*>(s.A);
  return (s.lda % 2 == 0) && (ldb % 2 == 0) && (reinterpret_cast<uintptr_t>(s.A) % 16 == 0) &&
         (reinterpret_cast<uintptr_t>(b) % 16 == 0);
}

namespace {
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    (void)cudaGetLastError();
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}
// ===== FAST batched residuals: ||A x_j - b_j||^2 for every column on the fp64 tensor
// cores (nnls.hpp:95-105 per column; the EXACT profile keeps the reference-ordered
// residual_batched_kernel of batched.cu) ================================================
// A CTA owns RN = 64 columns: their x (n <= 256 entries each) stay in shared memory
// as the DMMA B operand for the CTA's whole life, and A streams through in 128-row
// tiles, k slabs of 32 by 16-byte cp.async from L2 (A is read once per CTA: 41 MB at
// c4, L2-resident). 8 warps as 4 (rows) x 2 (columns), warp tile 32 x 32 = 2 x 4
// m16n8k8 accumulators. After a tile's last slab each thread subtracts its b entries,
// squares, and adds into its own per-column sums (tiles in ascending row order); the
// lanes of a column, then the four row warps, are summed in a fixed order at the end
// (deterministic run to run). Strides RLDA / ldx = 4 mod 16 doubles keep both fragment
// loads bank-conflict-free.
constexpr int RM = 128, RN = 64, RKS = 32, RLDA = RM + 4;
__host__ __device__ constexpr int res_ldx(int n) { return (n + RKS - 1) / RKS * RKS + 4; }
size_t res_dmma_smem(int n) {
  return ((size_t)RN * res_ldx(n) + 2 * (size_t)RKS * RLDA) * sizeof(double);
}

__global__ void __launch_bounds__(TT, 1)
residual_dmma_kernel(const double* __restrict__ A, uint64_t lda, int d, int n,
                     const double* __restrict__ X, const double* __restrict__ B, uint64_t ldb,
                     int ncols, alnnls_column_result* res) {
  extern __shared__ __align__(128) double dm_sm[];
  const int ldx = res_ldx(n);
  double* Xs = dm_sm;                       // [RN][ldx]: x of column c at Xs[c * ldx + k]
  double* As = dm_sm + (size_t)RN * ldx;    // [2][RKS][RLDA]: A(i0 + r, k0 + kk) at [kk][r]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = warp >> 1, wc = warp & 1;
  const int g = lane >> 2, t = lane & 3;
  const int c0 = blockIdx.x * RN;
  const int nks = (n + RKS - 1) / RKS;
  const int ntile = (d + RM - 1) / RM;
  const int nslab = ntile * nks;

  // slab q = tile * nks + ks: 2048 16-byte chunks, 8 per thread
  auto issue = [&](int q) {
    const int i0 = (q / nks) * RM, k0 = (q % nks) * RKS;
    double* dst = As + (size_t)(q & 1) * RKS * RLDA;
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      const int e = tid + p * TT, kk = e >> 6, r = (e & 63) * 2;
      const int left = d - (i0 + r);
      const uint32_t bytes = (k0 + kk < n && left > 0) ? (left >= 2 ? 16u : 8u) : 0u;
      cp_async16(dst + kk * RLDA + r, bytes ? A + (size_t)(k0 + kk) * lda + i0 + r : A, bytes);
    }
  };
  issue(0);
  cp_commit();
  for (int e = tid; e < RN * ldx; e += TT) {
    const int c = e / ldx, k = e - c * ldx;
    Xs[e] = (c0 + c < ncols && k < n) ? X[(size_t)(c0 + c) * n + k] : 0.0;
  }

  double acc[2][4][4];
  double csum[4][2];
#pragma unroll
  for (int ni = 0; ni < 4; ++ni) csum[ni][0] = csum[ni][1] = 0.0;
  const double* xw = Xs + (size_t)(wc * 32 + g) * ldx + t;
  for (int q = 0; q < nslab; ++q) {
    const int ks = q % nks;
    if (ks == 0) {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[mi][ni][c] = 0.0;
    }
    cp_wait<0>();
    __syncthreads();  // slab q landed; every warp is done with slab q - 1's buffer
    if (q + 1 < nslab) issue(q + 1);
    cp_commit();
    const double* as = As + (size_t)(q & 1) * RKS * RLDA + wr * 32 + g;
    const double* xs = xw + ks * RKS;
#pragma unroll
    for (int k8 = 0; k8 < RKS; k8 += 8) {
      double af[2][4], bf[4][2];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        af[mi][0] = as[(k8 + t) * RLDA + mi * 16];
        af[mi][1] = as[(k8 + t) * RLDA + mi * 16 + 8];
        af[mi][2] = as[(k8 + t + 4) * RLDA + mi * 16];
        af[mi][3] = as[(k8 + t + 4) * RLDA + mi * 16 + 8];
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        bf[ni][0] = xs[(size_t)ni * 8 * ldx + k8];
        bf[ni][1] = xs[(size_t)ni * 8 * ldx + k8 + 4];
      }
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni], af[mi], bf[ni]);
    }
    if (ks == nks - 1) {  // the tile is complete: (A x - b)^2 into the column sums
      const int i0 = (q / nks) * RM + wr * 32 + g;
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const int col = c0 + wc * 32 + ni * 8 + 2 * t + cc;
          if (col < ncols) {
            const double* bp = B + (size_t)col * ldb;
            double bv[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) {  // rows i0, i0 + 8, i0 + 16, i0 + 24
              const int i = i0 + 8 * h;
              bv[h] = i < d ? __ldg(bp + i) : 0.0;
            }
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const int i = i0 + 8 * h;
              const double df = acc[h >> 1][ni][(h & 1) * 2 + cc] - bv[h];
              if (i < d) csum[ni][cc] += df * df;
            }
          }
        }
    }
  }
  // lanes of a column (same t, g = 0..7), then the four row warps, in a fixed order
#pragma unroll
  for (int ni = 0; ni < 4; ++ni)
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      double v = csum[ni][cc];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      csum[ni][cc] = v;
    }
  __syncthreads();
  double* red = As;  // [4][RN]
  if (g == 0) {
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) red[wr * RN + wc * 32 + ni * 8 + 2 * t + cc] = csum[ni][cc];
  }
  __syncthreads();
  if (tid < RN && c0 + tid < ncols)
    res[c0 + tid].residual_sq = ((red[tid] + red[RN + tid]) + red[2 * RN + tid]) + red[3 * RN + tid];
}

// rows x cols column-major fp64 (ld doubles): box 16 rows (k) x 128 columns, 128B swizzle
bool make_map(CUtensorMap* m, const double* p, uint64_t rows, uint64_t cols, uint64_t ld) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {rows, cols};
  const cuuint64_t strides[1] = {ld * sizeof(double)};
  const cuuint32_t box[2] = {TK, TB};
  const cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(p), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

size_t syrk_dmma_ws_doubles(int sm_count) { return (size_t)sm_count * TB * TB + 64; }

cudaError_t launch_syrk_dmma(const SetupArgs& s, int mode, cudaStream_t stream, int accumulate,
                             int tile_lo, int tile_hi) {
  const int nt = (s.n + TB - 1) / TB;
  const int all = mode == 2 ? nt * ((s.nrhs + TB - 1) / TB) : nt * (nt + 1) / 2;
  if (tile_hi < 0 || tile_hi > all) tile_hi = all;
  if (tile_lo < 0) tile_lo = 0;
  const int tiles = tile_hi - tile_lo;
  if (tiles <= 0) return cudaSuccess;
  if ((tile_lo != 0 || tile_hi != all) && !(s.dm_ws && s.dm_flags && s.dm_ctas > 0))
    return cudaErrorInvalidValue;  // tile ranges: v2 only
  if (!syrk_dmma_supported(s, mode)) return cudaErrorInvalidValue;
  if (s.dm_ws && s.dm_flags && s.dm_ctas > 0) {
    TmaArgs ta{};
    const uint64_t ldb = mode == 2 ? s.ldb : s.lda;
    if (make_map(&ta.mapA, s.A, (uint64_t)s.d, (uint64_t)s.n, s.lda) &&
        make_map(&ta.mapB, mode == 2 ? s.B : s.A, (uint64_t)s.d,
                 (uint64_t)(mode == 2 ? s.nrhs : s.n), ldb)) {
      ta.tiles = tiles;
      ta.tile_lo = tile_lo;
      ta.nk = (s.d + TK - 1) / TK;
      ta.nti = nt;
      ta.ws = s.dm_ws;
      ta.flags = s.dm_flags;
      ta.accumulate = accumulate;
      // every SM even for few tiles (stream-K splits their k ranges); no CTA without
      // a unit (a finisher waits on every later CTA whose range starts in its tile)
      const long long units = (long long)tiles * ta.nk;
      const int grid = units < s.dm_ctas ? (int)units : s.dm_ctas;
      if (cudaError_t e = smem_optin(syrk_tma_kernel, (int)kDmma2Smem)) return e;
      cudaError_t e = cudaMemsetAsync(s.dm_flags, 0, sizeof(int) * grid, stream);
      if (e != cudaSuccess) return e;
      // all CTAs must be co-resident (finishers wait on later CTAs): one per SM
      void* args[] = {&ta, const_cast<SetupArgs*>(&s), &mode};
      return cudaLaunchCooperativeKernel((const void*)syrk_tma_kernel, dim3(grid), dim3(TT), args,
                                         kDmma2Smem, stream);
    }
  }
  if (accumulate) return cudaErrorInvalidValue;  // v1 has no accumulate epilogue
  if (cudaError_t e = smem_optin(syrk_dmma_kernel, (int)kDmmaSmem)) return e;
  syrk_dmma_kernel<<<tiles, TT, kDmmaSmem, stream>>>(s, mode);
  return cudaGetLastError();
}

// FAST residuals on the tensor cores when the shape fits (x block resident in shared
// memory, 16-byte cp.async sources); false: the caller uses the reference-ordered kernel.
bool residual_dmma_supported(const double* A, uint64_t lda, int d, int n, int ncols) {
  return n >= 1 && n <= 256 && d >= 1 && ncols >= 1 && (lda % 2) == 0 &&
         (reinterpret_cast<uintptr_t>(A) % 16) == 0;
}

cudaError_t launch_residual_batched_dmma(const double* A, uint64_t lda, int d, int n,
                                         const double* X, const double* B, uint64_t ldb,
                                         int ncols, alnnls_column_result* res,
                                         cudaStream_t stream) {
  if (!residual_dmma_supported(A, lda, d, n, ncols)) return cudaErrorInvalidValue;
  if (cudaError_t e = smem_optin(residual_dmma_kernel, (int)res_dmma_smem(256))) return e;
  residual_dmma_kernel<<<(ncols + RN - 1) / RN, TT, res_dmma_smem(n), stream>>>(
      A, lda, d, n, X, B, ldb, ncols, res);
  return cudaGetLastError();
}

}  // namespace alnnls
