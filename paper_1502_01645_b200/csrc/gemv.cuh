// gemv.cuh — exact row-block masked GEMV (K5/K6/K7 building block).
//
// y[i] = sum_{t < len} M[i, list[t]] * vals[t]   for the CTA's rows i in [row0, row0+nrows)
//
// This is reference masked_matvec (linalg.hpp:193-206) restated row-wise: the
// reference sweeps columns in mask order and does y[i] += col[i]*v_j, so each
// y[i] is one chain over the mask in list order. Here one consumer thread owns
// one row and runs exactly that chain (rounded product, then rounded sum), so
// the result is bitwise equal. `vals` is the vector compacted to the list
// (vals[t] = v[list[t]]).
//
// Data movement (B200): a producer warp streams the CTA's column segments
// M[row0 : row0+seg, list[t]] (contiguous in the column-major layout) into a
// deep shared-memory ring with cp.async.bulk (TMA 1D, UBLKCP) completing on
// mbarriers; consumer warps walk the ring. Only the listed columns are read,
// so HBM traffic equals the reference's multiply count x 8 bytes.
#pragma once

#include "common.cuh"

namespace alnnls {

constexpr int kRingCols = 8;    // columns per stage (even: keeps vals 16B aligned)
constexpr int kMaxStages = 64;
constexpr size_t kRingSmemBytes = 200 * 1024;  // dynamic smem of ring-carrying kernels

struct RowRing {
  uint64_t* full;
  uint64_t* empty;
  double* data;   // [S][G][seg]
  double* vals;   // [S][G]
  int S;
  int seg;        // doubles per column segment (nrows rounded up to even)
  int cons_warps; // consumer warps (warps 1..cons_warps)
  uint32_t pos;   // stages issued so far (identical in every thread)
};

__host__ __device__ inline int ring_seg(int nrows) { return (nrows + 1) & ~1; }
__host__ __device__ inline size_t ring_stage_bytes(int seg) {
  return (size_t)kRingCols * seg * 8 + (size_t)kRingCols * 8;
}

// Carves the ring out of `smem` (16B aligned, `bytes` long). Must be called by
// every thread; contains a __syncthreads.
__device__ inline void ring_setup(RowRing& r, uint8_t* smem, size_t bytes, int nrows) {
  r.seg = ring_seg(nrows > 0 ? nrows : 2);
  r.cons_warps = (nrows + 31) / 32;
  if (r.cons_warps < 1) r.cons_warps = 1;
  const size_t sb = ring_stage_bytes(r.seg);
  const size_t hdr = (size_t)kMaxStages * 16;
  int S = (int)((bytes - hdr) / sb);
  if (S > kMaxStages) S = kMaxStages;
  r.S = S;
  r.full = reinterpret_cast<uint64_t*>(smem);
  r.empty = r.full + kMaxStages;
  r.data = reinterpret_cast<double*>(smem + hdr);
  r.vals = r.data + (size_t)S * kRingCols * r.seg;
  r.pos = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&r.full[s], 1);
      mbar_init(&r.empty[s], r.cons_warps);
    }
    fence_mbar_init();
  }
  __syncthreads();
}

// Runs the row-block GEMV over `len` listed columns. Every thread of the CTA
// calls it (idle warps just advance the ring position). Consumers write
// out[row0 + t]. No block barrier inside or at the end.
__device__ inline void gemv_rows(RowRing& r, const double* __restrict__ M, uint64_t ld, int row0,
                                 int nrows, const uint32_t* __restrict__ list,
                                 const double* __restrict__ vals, int len,
                                 double* __restrict__ out) {
  const int nst = (len + kRingCols - 1) / kRingCols;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int seg = r.seg;
  if (warp == 0) {
    // order generic-proxy writes of list/vals (other CTAs, before the grid
    // barrier) before the async-proxy bulk reads issued below
    asm volatile("fence.proxy.async.global;" ::: "memory");
    for (int s = 0; s < nst; ++s) {
      const uint32_t p = r.pos + s;
      const int st = (int)(p % r.S);
      const uint32_t ph = (p / r.S) & 1u;
      const int base = s * kRingCols;
      const int cnt = min(kRingCols, len - base);
      if (lane == 0) {
        mbar_wait(&r.empty[st], ph ^ 1u);
        const uint32_t bytes = (uint32_t)(cnt * seg * 8 + ((cnt + 1) & ~1) * 8);
        mbar_arrive_expect_tx(&r.full[st], bytes);
      }
      __syncwarp();
      double* dst = r.data + (size_t)st * kRingCols * seg;
      if (lane < cnt) {
        const uint32_t j = __ldcg(list + base + lane);
        bulk_g2s(dst + (size_t)lane * seg, M + (size_t)j * ld + row0, (uint32_t)seg * 8,
                 &r.full[st]);
      } else if (lane == 31) {
        bulk_g2s(r.vals + (size_t)st * kRingCols, vals + base, (uint32_t)(((cnt + 1) & ~1) * 8),
                 &r.full[st]);
      }
    }
  } else if (warp <= r.cons_warps) {
    const int t = (warp - 1) * 32 + lane;
    double acc = 0.0;
    for (int s = 0; s < nst; ++s) {
      const uint32_t p = r.pos + s;
      const int st = (int)(p % r.S);
      const uint32_t ph = (p / r.S) & 1u;
      const int cnt = min(kRingCols, len - s * kRingCols);
      mbar_wait(&r.full[st], ph);
      const double* col = r.data + (size_t)st * kRingCols * seg;
      const double* v = r.vals + (size_t)st * kRingCols;
      if (t < nrows) {
#pragma unroll
        for (int l = 0; l < kRingCols; ++l)
          if (l < cnt) acc = xmac(acc, col[l * seg + t], v[l]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&r.empty[st]);
    }
    if (t < nrows) out[row0 + t] = acc;
  }
  r.pos += nst;
}

}  // namespace alnnls
