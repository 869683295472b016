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
// same k order). DMUL, DADD and DFMA each issue at 64 lanes/clk/SM on B200,
// so one DMUL + one DADD per product caps the exact profile at 18.5 TFLOP/s
// useful, half the 37 TFLOP/s DMMA peak (profiles/r01_fp64_probe.txt). The
// epilogue writes Q = H/(D_i D_j)
// (Q_ii = 1) and q = (-h)/D directly: H is never materialised.
#include "common.cuh"
#include "gemv.cuh"
#include "kernels.cuh"

namespace alnnls {

namespace {

constexpr int BM = 128;   // output tile (square)
#ifndef ALNNLS_SYRK_BK
#define ALNNLS_SYRK_BK 16
#endif
constexpr int BK = ALNNLS_SYRK_BK;  // k slab
#ifndef ALNNLS_SYRK_TC
#define ALNNLS_SYRK_TC 4
#endif
constexpr int TC = ALNNLS_SYRK_TC;       // thread tile 8 rows x TC cols
#ifndef ALNNLS_SYRK_HALF
#define ALNNLS_SYRK_HALF 0  // build knob: a CTA takes half a tile (64 of its 128 rows), two CTAs
                            // per SM (bitwise; c2 setup 9.25 -> 9.55 ms measured, so off)
#endif
constexpr int BMR = ALNNLS_SYRK_HALF ? BM / 2 : BM;  // rows of one piece of a tile
constexpr int PPT = BM / BMR;                         // pieces per tile
constexpr int NT = BMR * BM / (8 * TC);  // TC=4: 512 threads (4 warps per scheduler), 256 for halves
constexpr int CPS = 512 / NT;            // CTAs per SM
constexpr int TS = BM * BM;              // doubles of one tile's chain states
constexpr int TSP = BMR * BM;            // ... of one piece's ([8*TC][NT])
constexpr int LDS = BM + 2;   // padded smem row (doubles): 16B-aligned rows, <=2-way store conflicts
constexpr int LDSA = BMR + 2; // the A operand's slab rows (a piece's rows)
// thread tile 8 rows x TC cols: rows 2tx+(r&1)+32(r>>1), cols 2ty+(c&1)+(256/TC)(c>>1)
// (each 16B shared load of a row pair is conflict-free across the 16 tx lanes)

// Upper-triangular tile index -> (ti, tj), ti <= tj (tj-major enumeration).
__device__ __forceinline__ void tri_tile(int t, int& ti, int& tj) {
  int j = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
  while ((j + 1) * (j + 2) / 2 <= t) ++j;
  while (j * (j + 1) / 2 > t) --j;
  tj = j;
  ti = t - j * (j + 1) / 2;
}

#ifndef ALNNLS_SYRK_STAGES
#define ALNNLS_SYRK_STAGES 3
#endif
constexpr int kStages = ALNNLS_SYRK_STAGES;  // cp.async slab ring depth
constexpr size_t kSyrkSmem = (size_t)kStages * BK * (LDSA + LDS) * sizeof(double);

__device__ __forceinline__ void cp_async8(void* dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Output tile t -> (ti, tj): upper-triangular tiles of A^T A (modes 0/1), the
// full grid of A^T B (mode 2).
__device__ __forceinline__ void tile_of(const SetupArgs& s, int mode, int t, int& ti, int& tj) {
  if (mode == 2) {
    const int nti = (s.n + BM - 1) / BM;
    ti = t % nti;
    tj = t / nti;
  } else {
    tri_tile(t, ti, tj);
  }
}

// k slabs [kb0, kb1) of output tile (ti, tj). The 32 accumulators of each
// thread start from +0, or from a partial chain state `pin` ([8*TC][NT]) that
// another CTA left after slabs [0, kb0); they end in the epilogue, or are
// stored to `pout` for the CTA that continues the chain. Either way every
// output is ONE chain over k ascending, bit for bit the same as one CTA doing
// all slabs.
__device__ __forceinline__ void syrk_piece(const SetupArgs& s, int mode, double* smem, int ti, int tj,
                                           int piece, int kb0, int kb1, const double* pin,
                                           double* pout) {
  auto As = reinterpret_cast<double(*)[BK][LDSA]>(smem);
  auto Bs = reinterpret_cast<double(*)[BK][LDS]>(smem + kStages * BK * LDSA);
  const int i0 = ti * BM + piece * BMR, j0 = tj * BM;
  constexpr int TXN = BMR / 8;  // thread columns of the row dimension
  const int tx = threadIdx.x % TXN, ty = threadIdx.x / TXN;
  const double* Bop = mode == 2 ? s.B : s.A;
  const uint64_t ldb = mode == 2 ? s.ldb : s.lda;
  const int nb = mode == 2 ? s.nrhs : s.n;

  // loader: element e = tid + r*NT (r < LPT) of a BK x BM slab: column e/BK, row k0 + e%BK.
  // Out-of-range elements are zero-filled (src-size 0): adding +0 to a chain is exact
  // (s + (+0) == s, and s is never -0).
  constexpr int LPTA = BK * BMR / NT, LPTB = BK * BM / NT;
  const double* pa[LPTA];
  const double* pb[LPTB];
#pragma unroll
  for (int r = 0; r < LPTA; ++r) {
    const int ca = i0 + (threadIdx.x + r * NT) / BK;
    pa[r] = ca < s.n ? s.A + (size_t)ca * s.lda : nullptr;
  }
#pragma unroll
  for (int r = 0; r < LPTB; ++r) {
    const int cb = j0 + (threadIdx.x + r * NT) / BK;
    pb[r] = cb < nb ? Bop + (size_t)cb * ldb : nullptr;
  }
  auto issue = [&](int kb) {
    const int buf = (kb - kb0) % kStages;
    const int k0 = kb * BK;
#pragma unroll
    for (int r = 0; r < LPTA; ++r) {
      const int e = threadIdx.x + r * NT;
      const int kk = e % BK, k = k0 + kk;
      const bool va = pa[r] && k < s.d;
      cp_async8(&As[buf][kk][e / BK], va ? pa[r] + k : s.A, va ? 8u : 0u);
    }
#pragma unroll
    for (int r = 0; r < LPTB; ++r) {
      const int e = threadIdx.x + r * NT;
      const int kk = e % BK, k = k0 + kk;
      const bool vb = pb[r] && k < s.d;
      cp_async8(&Bs[buf][kk][e / BK], vb ? pb[r] + k : s.A, vb ? 8u : 0u);
    }
  };

  double acc[8][TC];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < TC; ++c)
      acc[r][c] = pin ? __ldcg(pin + (size_t)(r * TC + c) * NT + threadIdx.x) : 0.0;

  __syncthreads();  // the previous piece's last slab buffers are no longer read
#pragma unroll
  for (int p = 0; p < kStages - 1; ++p) {
    if (kb0 + p < kb1) issue(kb0 + p);
    cp_async_commit();
  }
  for (int kb = kb0; kb < kb1; ++kb) {
    cp_async_wait<kStages - 2>();  // slab kb has landed (this thread's copies)
    __syncthreads();               // ... everyone's; and slab kb-1's buffer is free
    if (kb + kStages - 1 < kb1) issue(kb + kStages - 1);
    cp_async_commit();
    const int buf = (kb - kb0) % kStages;
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      double a[8], b[TC];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const double2 v = *reinterpret_cast<const double2*>(&As[buf][kk][2 * tx + (BMR / 4) * h]);
        a[2 * h] = v.x;
        a[2 * h + 1] = v.y;
      }
#pragma unroll
      for (int h = 0; h < TC / 2; ++h) {
        const double2 v = *reinterpret_cast<const double2*>(&Bs[buf][kk][2 * ty + (256 / TC) * h]);
        b[2 * h] = v.x;
        b[2 * h + 1] = v.y;
      }
      // each output: one chain over k ascending, rounded product then rounded sum
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        double p[TC];
#pragma unroll
        for (int c = 0; c < TC; ++c) p[c] = xmul(a[r], b[c]);
#pragma unroll
        for (int c = 0; c < TC; ++c) acc[r][c] = xadd(acc[r][c], p[c]);
      }
    }
  }
  cp_async_wait<0>();

  if (pout) {  // hand the chain states to the CTA that finishes this tile
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < TC; ++c) pout[(size_t)(r * TC + c) * NT + threadIdx.x] = acc[r][c];
    return;
  }
  // epilogue: upper triangle only, mirrored (exact symmetry, linalg.hpp:169-170)
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = i0 + 2 * tx + (r & 1) + (BMR / 4) * (r >> 1);
#pragma unroll
    for (int c = 0; c < TC; ++c) {
      const int j = j0 + 2 * ty + (c & 1) + (256 / TC) * (c >> 1);
      const double v = acc[r][c];
      if (mode == 2) {  // q_b of RHS column j: (-(A^T b_j))_{j_b} / D_b (nnls.hpp:79, :133-134)
        if (i >= s.n || j >= s.nrhs) continue;
        const int pi = s.pos[i];
        if (pi >= 0) s.QB[(size_t)j * s.m + pi] = xdiv(-v, s.scale[pi]);
        continue;
      }
      if (i > j || j >= s.n) continue;
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

// Small n (few 128 x 128 tiles; e.g. the c4 Gram, n = 256: 3 tiles for 148 SMs):
// 32 x 32 output tiles, 64 threads, 4 x 4 outputs per thread, every output ONE
// ascending-k chain (rounded product, then rounded sum; zero-filled k beyond d
// add +0, an exact no-op). The next 32-k slab is loaded into registers while the
// current one is multiplied. Modes 0 (H) and 1 (fused rescale), same epilogue
// as syrk_piece.
constexpr int SB = 32, SK = 32, ST = 64;
__global__ void __launch_bounds__(ST) syrk_small_kernel(SetupArgs s, int mode) {
  __shared__ double As[2][SK][SB + 1];
  __shared__ double Bs[2][SK][SB + 1];
  int ti, tj;
  tri_tile(blockIdx.x, ti, tj);
  const int i0 = ti * SB, j0 = tj * SB;
  const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;  // rows tx + 8 r, columns ty + 8 c
  double ra[16], rb[16];
  auto fetch = [&](int k0) {  // element e = tid + 64 u: column e / SK, k = k0 + e % SK
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = threadIdx.x + ST * u, col = e / SK, k = k0 + e % SK;
      const bool kv = k < s.d;
      ra[u] = kv && i0 + col < s.n ? __ldg(s.A + (size_t)(i0 + col) * s.lda + k) : 0.0;
      rb[u] = kv && j0 + col < s.n ? __ldg(s.A + (size_t)(j0 + col) * s.lda + k) : 0.0;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int e = threadIdx.x + ST * u;
      As[buf][e % SK][e / SK] = ra[u];
      Bs[buf][e % SK][e / SK] = rb[u];
    }
  };
  double acc[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[r][c] = 0.0;
  const int nk = (s.d + SK - 1) / SK;
  fetch(0);
  stash(0);
  __syncthreads();
  for (int kb = 0; kb < nk; ++kb) {
    const int buf = kb & 1;
    if (kb + 1 < nk) fetch((kb + 1) * SK);
#pragma unroll
    for (int kk = 0; kk < SK; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) a[r] = As[buf][kk][tx + 8 * r];
#pragma unroll
      for (int c = 0; c < 4; ++c) b[c] = Bs[buf][kk][ty + 8 * c];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        double p[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) p[c] = xmul(a[r], b[c]);
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = xadd(acc[r][c], p[c]);
      }
    }
    if (kb + 1 < nk) stash(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = i0 + tx + 8 * r, j = j0 + ty + 8 * c;
      const double v = acc[r][c];
      if (i > j || j >= s.n) continue;
      if (mode == 0) {
        s.H[(size_t)j * s.n + i] = v;
        s.H[(size_t)i * s.n + j] = v;
      } else {
        const int pi = s.pos[i], pj = s.pos[j];
        if (pi < 0 || pj < 0) continue;
        if (i == j) {
          s.Q[blk_index(pi, pi, s.m, s.qR)] = 1.0;  // nnls.hpp:72
        } else {
          const double qv = xdiv(v, xmul(s.scale[pi], s.scale[pj]));  // nnls.hpp:75
          s.Q[blk_index(pi, pj, s.m, s.qR)] = qv;
          s.Q[blk_index(pj, pi, s.m, s.qR)] = qv;
        }
      }
    }
}

// One CTA per output tile.
__global__ void __launch_bounds__(NT, CPS) syrk_exact_kernel(SetupArgs s, int mode) {
  extern __shared__ __align__(16) double syrk_sm[];
  int ti, tj;
  tile_of(s, mode, blockIdx.x / PPT, ti, tj);
  syrk_piece(s, mode, syrk_sm, ti, tj, blockIdx.x % PPT, 0, (s.d + BK - 1) / BK, nullptr, nullptr);
}

// Stream-K: one persistent CTA per SM takes an equal contiguous share of the
// (tile, k-slab) sequence, so the last wave is not partly idle. A tile split
// between CTA c-1 and CTA c is continued from c-1's chain states: CTA c-1 does
// its trailing partial tile FIRST and publishes it (flag, release), and CTA c
// takes its leading partial tile LAST (acquire), so nobody waits in practice.
// Requires every CTA's share to span at least two tiles (checked on the host)
// and co-residency (cooperative launch).
__global__ void __launch_bounds__(NT, CPS) syrk_streamk_kernel(SetupArgs s, int mode, int tiles) {
  extern __shared__ __align__(16) double syrk_sm[];
  const int nk = (s.d + BK - 1) / BK;
  // units: (piece, k slab); a tile is PPT pieces of BMR rows
  const long long total = (long long)tiles * PPT * nk;
  const long long per = (total + gridDim.x - 1) / gridDim.x;
  const long long u0 = (long long)blockIdx.x * per;
  const long long u1 = min(total, u0 + per);
  if (u0 >= u1) return;
  const int t0 = (int)(u0 / nk), k0 = (int)(u0 % nk);
  const int t1 = (int)((u1 - 1) / nk), k1 = (int)((u1 - 1) % nk) + 1;
  double* my_part = s.sk_part + (size_t)blockIdx.x * TSP;
  int ti, tj;
  // piece chain states carried in from earlier row blocks / out to later ones
  // (row-block continuation, s.tpin / s.tpout, [tiles][PPT][8*TC][NT]; nullptr: none)
  auto tin = [&](int p) { return s.tpin ? s.tpin + (size_t)p * TSP : nullptr; };
  auto tout = [&](int p) { return s.tpout ? s.tpout + (size_t)p * TSP : nullptr; };
  // 1. trailing partial piece: slabs [0, k1) of t1, handed to the next CTA
  if (k1 < nk) {
    tile_of(s, mode, t1 / PPT, ti, tj);
    syrk_piece(s, mode, syrk_sm, ti, tj, t1 % PPT, 0, k1, tin(t1), my_part);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(s.sk_flag + blockIdx.x), "r"(1u)
                   : "memory");
    }
  }
  // 2. whole pieces
  const int full_lo = k0 == 0 ? t0 : t0 + 1;
  const int full_hi = k1 == nk ? t1 : t1 - 1;
  for (int t = full_lo; t <= full_hi; ++t) {
    tile_of(s, mode, t / PPT, ti, tj);
    syrk_piece(s, mode, syrk_sm, ti, tj, t % PPT, 0, nk, tin(t), tout(t));
  }
  // 3. leading partial piece: slabs [k0, nk) of t0, continuing CTA blockIdx-1's chains
  if (k0 > 0) {
    if (threadIdx.x == 0) {
      unsigned v = 0;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(s.sk_flag + blockIdx.x - 1)
                     : "memory");
      } while (v == 0);
    }
    __syncthreads();
    tile_of(s, mode, t0 / PPT, ti, tj);
    syrk_piece(s, mode, syrk_sm, ti, tj, t0 % PPT, k0, nk,
               s.sk_part + (size_t)(blockIdx.x - 1) * TSP, tout(t0));
  }
}
// q_b = h(j_b) / D_b with h = -(A^T b) (nnls.hpp:79, :133-134); atb = A^T b.
__global__ void q_from_atb_kernel(const double* atb, const int* pos, const double* scale, int n,
                                  double* q, double* hvec) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const double h = -atb[j];
  if (hvec) hvec[j] = h;
  if (q) {
    const int p = pos[j];
    if (p >= 0) q[p] = xdiv(h, scale[p]);
  }
}

// Column chains over A (K1 diagonal + K2): for each column c of a 32-column
// group, diag_c = sum_k A[k,c]^2 (bitwise the SYRK diagonal / gram (c,c)
// chain, linalg.hpp:168) and atb_c = sum_k A[k,c] b[k] (transpose_matvec,
// linalg.hpp:215), each ONE chain in ascending k. Warps 1..7 stream k-tiles
// of the 32 columns with coalesced loads into a double-buffered shared tile
// (transposed to [column][k]); lane c of warp 0 runs column c's chains.
constexpr int kCcKT = 224;                 // k per stage (7 loader warps x 32)
constexpr int kCcLD = kCcKT + 1;           // odd stride: 2-wavefront reads
constexpr size_t kColChainSmem = (2 * 32 * kCcLD + 2 * kCcKT) * sizeof(double);

__global__ void __launch_bounds__(256, 1)
    colchain_kernel(const double* A, uint64_t lda, int d, int n, const double* b, double* diag,
                    double* atb, const double* atb0) {
  extern __shared__ __align__(16) double cc_sm[];
  double* tile = cc_sm;                    // [2][32][kCcLD]
  double* btile = cc_sm + 2 * 32 * kCcLD;  // [2][kCcKT]
  const int c0 = blockIdx.x * 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nst = (d + kCcKT - 1) / kCcKT;
  auto load = [&](int st, int buf) {
    const int kk = (warp - 1) * 32 + lane;
    const int k = st * kCcKT + kk;
    double* t = tile + (size_t)buf * 32 * kCcLD;
#pragma unroll 8
    for (int c = 0; c < 32; ++c) {
      const int col = c0 + c;
      t[c * kCcLD + kk] = (k < d && col < n) ? __ldg(A + (size_t)col * lda + k) : 0.0;
    }
    if (b) btile[buf * kCcKT + kk] = k < d ? __ldg(b + k) : 0.0;
  };
  // atb0: A^T b chain states after earlier row blocks (host-buffer overlap)
  double sd = 0.0, sb = atb0 && c0 + lane < n ? atb0[c0 + lane] : 0.0;
  if (warp > 0) load(0, 0);
  __syncthreads();
  for (int st = 0; st < nst; ++st) {
    const int buf = st & 1;
    if (warp == 0) {
      const double* t = tile + (size_t)buf * 32 * kCcLD + lane * kCcLD;
      const double* bt = btile + buf * kCcKT;
      // zero padding past d is exact (s + (+0) == s; s is never -0)
#pragma unroll 8
      for (int kk = 0; kk < kCcKT; ++kk) {
        const double v = t[kk];
        sd = xmac(sd, v, v);
        if (b) sb = xmac(sb, v, bt[kk]);
      }
    } else if (st + 1 < nst) {
      load(st + 1, buf ^ 1);
    }
    __syncthreads();
  }
  if (warp == 0 && c0 + lane < n) {
    if (diag) diag[c0 + lane] = sd;
    if (atb) atb[c0 + lane] = sb;
  }
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
                                double* out, double s0) {
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const double r = xsub(ax[i], b[i]);
    prod[i] = xmul(r, r);
  }
  __syncthreads();
  if (threadIdx.x == 0) *out = chain_sum_from(s0, prod, d);
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

// Device-side checks of NqpProblem (nqp.hpp:37-41) and the warm start
// (nqp.hpp:227-230) for the device-pointer entries. kind 0: exact symmetry of the
// m x m matrix (ld), kind 1: every entry >= 0 (NaN fails).
__global__ void check_matrix_kernel(const double* p, uint64_t rows, uint64_t cols, uint64_t ld,
                                    int kind, int* flag) {
  const uint64_t total = rows * cols;
  int bad = 0;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = e / rows, r = e % rows;
    const double v = p[c * ld + r];
    if (kind == 0) {
      if (r < c && !(v == p[r * ld + c])) bad = 1;
    } else if (!(v >= 0.0)) {
      bad = 1;
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) *flag = 1;
}

// Packed upper triangle of a symmetric n x n column-major matrix: entry (i, j),
// i <= j, at j (j + 1) / 2 + i. dir 0 packs, dir 1 unpacks and mirrors (the
// c5 allreduce moves n (n + 1) / 2 doubles instead of n^2).
__global__ void pack_upper_kernel(double* H, uint64_t n, double* P, int dir) {
  const uint64_t total = n * n;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = e / n, i = e % n;
    const uint64_t a = i <= j ? i : j, c = i <= j ? j : i;
    const uint64_t pidx = c * (c + 1) / 2 + a;
    if (dir == 0) {
      if (i <= j) P[pidx] = H[e];
    } else {
      H[e] = P[pidx];
    }
  }
}

// C[:, j] = matvec(A, H[:, j]) in the reference's order (linalg.hpp:179-188: the
// column sweep y[i] += M(i, t) v[t], t ascending, is per row one chain of
// rounded products then rounded sums). One thread per output (i, j); a block
// covers 256 consecutive rows of one column, so A's column t is read coalesced
// and H(t, j) is a broadcast.
__global__ void matmat_kernel(const double* __restrict__ A, uint64_t lda, int rows, int inner,
                              const double* __restrict__ H, uint64_t ldh, double* C, uint64_t ldc) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t j = blockIdx.y;
  if (i >= rows) return;
  const double* h = H + j * ldh;
  double s = 0.0;
  for (int t = 0; t < inner; ++t) s = xmac(s, A[(uint64_t)t * lda + i], __ldg(h + t));
  C[j * ldc + i] = s;
}

// dst (cols x rows, ld_dst) = src^T (src rows x cols, ld_src), 32 x 32 tiles through
// shared memory (both sides coalesced). Pure data movement: no arithmetic.
__global__ void transpose_kernel(const double* __restrict__ src, uint64_t ld_src, int rows,
                                 int cols, double* __restrict__ dst, uint64_t ld_dst) {
  __shared__ double tile[32][33];
  const int r0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int r = r0 + threadIdx.x, c = c0 + k;
    if (r < rows && c < cols) tile[k][threadIdx.x] = src[(uint64_t)c * ld_src + r];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int c = c0 + threadIdx.x, r = r0 + k;  // dst column r, row c
    if (r < rows && c < cols) dst[(uint64_t)r * ld_dst + c] = tile[threadIdx.x][k];
  }
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
  if (cudaError_t e = smem_optin(colchain_kernel, (int)kColChainSmem)) return e;
  colchain_kernel<<<(s.n + 31) / 32, 256, kColChainSmem, stream>>>(
      s.A, s.lda, s.d, s.n, s.b, s.diag, s.b ? s.hvec_scratch : nullptr, nullptr);
  return cudaGetLastError();
}

cudaError_t launch_atb_chain(const double* A, uint64_t lda, int rows, int n, const double* b,
                             const double* atb0, double* atb, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  if (cudaError_t e = smem_optin(colchain_kernel, (int)kColChainSmem)) return e;
  colchain_kernel<<<(n + 31) / 32, 256, kColChainSmem, stream>>>(A, lda, rows, n, b, nullptr, atb,
                                                                 atb0);
  return cudaGetLastError();
}

cudaError_t launch_q_from_atb(const SetupArgs& s, int mode, cudaStream_t stream) {
  if (!s.b || s.n <= 0) return cudaSuccess;
  q_from_atb_kernel<<<(s.n + 255) / 256, 256, 0, stream>>>(s.hvec_scratch, s.pos, s.scale, s.n,
                                                           mode == 1 ? s.q : nullptr,
                                                           mode == 0 ? s.hvec : nullptr);
  return cudaGetLastError();
}

cudaError_t launch_retained(const SetupArgs& s, cudaStream_t stream) {
  retained_kernel<<<1, 1024, 0, stream>>>(s.diag, s.n, s.pos, s.scale, s.retained, s.m_out,
                                          nullptr);
  return cudaGetLastError();
}

// Row-block continuation (multi-GPU exact Gram): tiles
// [tile_lo, tile_lo + gridDim.x) over the block's rows s.A[0, s.d), starting
// from the chain states `pin` the previous row blocks left (nullptr: start of
// the chains) and ending in `pout` (nullptr: finish, write H). The states of a
// tile are the kernel's thread layout [8*TC][NT]; feeding the row blocks in order
// is the reference's single ascending-k chain per entry.
__global__ void __launch_bounds__(NT, CPS) syrk_rowblock_kernel(SetupArgs s, int tile_lo,
                                                                const double* pin, double* pout) {
  extern __shared__ __align__(16) double syrk_sm[];
  int ti, tj;
  tile_of(s, 0, tile_lo + (int)blockIdx.x / PPT, ti, tj);
  const size_t off = (size_t)blockIdx.x * TSP;  // = (tile - tile_lo) * TS + piece * TSP
  syrk_piece(s, 0, syrk_sm, ti, tj, (int)blockIdx.x % PPT, 0, (s.d + BK - 1) / BK,
             pin ? pin + off : nullptr, pout ? pout + off : nullptr);
}

__global__ void diag_kernel(const double* H, int n, double* diag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) diag[i] = H[(size_t)i * n + i];
}

__global__ void negate_kernel(const double* x, int n, double* y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = -x[i];
}

// Build knob: the 32 x 32-tile SYRK runs when the 128 x 128 tiles number fewer than
// half this many (0 disables it).
#ifndef ALNNLS_SYRK_SMALL
#define ALNNLS_SYRK_SMALL 148
#endif

int syrk_streamk_ctas(const SetupArgs& s, int mode, int sm_count) {
  const int nt = (s.n + BM - 1) / BM;
  const long long tiles = mode == 2 ? (long long)nt * ((s.nrhs + BM - 1) / BM) : (long long)nt * (nt + 1) / 2;
  const long long nk = (s.d + BK - 1) / BK;
  // stream-K only pays when the tile grid leaves a ragged last wave, and needs
  // every share to span >= 2 tiles (one partial tile at each end at most)
  const long long ctas = (long long)sm_count * CPS, pieces = tiles * PPT;
  if (pieces < 2LL * ctas || pieces % ctas == 0 || nk < 2) return 0;
  return (int)ctas;
}

cudaError_t launch_syrk(const SetupArgs& s, int mode, cudaStream_t stream) {
  const int nt = (s.n + BM - 1) / BM;
  const int tiles = mode == 2 ? nt * ((s.nrhs + BM - 1) / BM) : nt * (nt + 1) / 2;
  if (tiles == 0) return cudaSuccess;
  if (cudaError_t e = smem_optin(syrk_exact_kernel, (int)kSyrkSmem)) return e;
  if (cudaError_t e = smem_optin(syrk_streamk_kernel, (int)kSyrkSmem)) return e;
  if (s.sk_part && s.sk_flag && s.sk_ctas > 0) {
    cudaError_t e = cudaMemsetAsync(s.sk_flag, 0, sizeof(int) * s.sk_ctas, stream);
    if (e != cudaSuccess) return e;
    SetupArgs sa = s;
    int md = mode, tl = tiles;
    void* args[] = {&sa, &md, &tl};
    return cudaLaunchCooperativeKernel((const void*)syrk_streamk_kernel, dim3(s.sk_ctas), dim3(NT),
                                       args, kSyrkSmem, stream);
  }
  if (ALNNLS_SYRK_SMALL && mode != 2 && !s.tpin && !s.tpout && 2 * tiles < ALNNLS_SYRK_SMALL) {
    const int nt32 = (s.n + SB - 1) / SB;
    syrk_small_kernel<<<nt32 * (nt32 + 1) / 2, ST, 0, stream>>>(s, mode);
    return cudaGetLastError();
  }
  syrk_exact_kernel<<<tiles * PPT, NT, kSyrkSmem, stream>>>(s, mode);
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
                            cudaStream_t stream, double s0) {
  residual_kernel<<<1, 1024, 0, stream>>>(ax, b, d, prod, out, s0);
  return cudaGetLastError();
}

cudaError_t launch_support(const double* x, int n, uint32_t* list, double* vals, int* len,
                           cudaStream_t stream) {
  support_kernel<<<1, 1024, 0, stream>>>(x, n, list, vals, len);
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

cudaError_t launch_check_matrix(const double* p, uint64_t rows, uint64_t cols, uint64_t ld,
                                int kind, int* flag, cudaStream_t stream) {
  if (rows * cols == 0) return cudaSuccess;
  uint64_t blocks = (rows * cols + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  check_matrix_kernel<<<(unsigned)blocks, 256, 0, stream>>>(p, rows, cols, ld, kind, flag);
  return cudaGetLastError();
}

cudaError_t launch_pack_upper(double* H, uint64_t n, double* P, int dir, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  uint64_t blocks = (n * n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  pack_upper_kernel<<<(unsigned)blocks, 256, 0, stream>>>(H, n, P, dir);
  return cudaGetLastError();
}

cudaError_t launch_matmat(const double* A, uint64_t lda, int rows, int inner, const double* H,
                          uint64_t ldh, int cols, double* C, uint64_t ldc, cudaStream_t stream) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  for (int j0 = 0; j0 < cols; j0 += 65535) {  // gridDim.y limit
    const int nc = cols - j0 < 65535 ? cols - j0 : 65535;
    matmat_kernel<<<dim3((rows + 255) / 256, nc), 256, 0, stream>>>(
        A, lda, rows, inner, H + (uint64_t)j0 * ldh, ldh, C + (uint64_t)j0 * ldc, ldc);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_transpose(const double* src, uint64_t ld_src, int rows, int cols, double* dst,
                             uint64_t ld_dst, cudaStream_t stream) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  for (int c0 = 0; c0 < cols; c0 += 32 * 65535) {  // gridDim.y limit
    const int nc = cols - c0 < 32 * 65535 ? cols - c0 : 32 * 65535;
    transpose_kernel<<<dim3((rows + 31) / 32, (nc + 31) / 32), dim3(32, 8), 0, stream>>>(
        src + (uint64_t)c0 * ld_src, ld_src, rows, nc, dst + c0, ld_dst);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
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

namespace alnnls {
uint64_t gram_tiles(uint64_t n) {
  const uint64_t nt = (n + BM - 1) / BM;
  return nt * (nt + 1) / 2;
}
cudaError_t launch_syrk_rowblock(const SetupArgs& s, int tile_lo, int ntiles, const double* pin,
                                 double* pout, cudaStream_t stream) {
  if (ntiles <= 0) return cudaSuccess;
  if (cudaError_t e = smem_optin(syrk_rowblock_kernel, (int)kSyrkSmem)) return e;
  syrk_rowblock_kernel<<<ntiles * PPT, NT, kSyrkSmem, stream>>>(s, tile_lo, pin, pout);
  return cudaGetLastError();
}
cudaError_t launch_diag(const double* H, int n, double* diag, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  diag_kernel<<<(n + 255) / 256, 256, 0, stream>>>(H, n, diag);
  return cudaGetLastError();
}
cudaError_t launch_negate(const double* x, int n, double* y, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  negate_kernel<<<(n + 255) / 256, 256, 0, stream>>>(x, n, y);
  return cudaGetLastError();
}
}  // namespace alnnls
