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
// Data movement (B200): producer warps stream the CTA's column segments into a
// deep shared-memory ring with cp.async.bulk (TMA 1D, UBLKCP) completing on
// mbarriers; consumer warps walk the ring. Only the listed columns are read,
// so HBM traffic equals the reference's multiply count x 8 bytes.
//
// Measured on B200: bulk copies are request-rate bound per SM (~13 ns per
// request per producer group), so (a) several producer warps issue stages
// round-robin, and (b) Q is stored row-block-contiguous ("blocked": the R
// rows of block b for column j at Qb + b*R*m + j*R), which makes a run of
// consecutive mask columns ONE contiguous copy.
#pragma once

#include "common.cuh"

namespace alnnls {

// Producer warps issuing the ring's bulk copies (build knob; 6, 8 and 11 measured
// equal or slower than 4 at c2 and c5).
#ifndef ALNNLS_PRODUCERS
#define ALNNLS_PRODUCERS 4
#endif

// Stages a ring must hold before the stage width drops (build knob). 6 measured
// best at c5 (seg 112 -> 32-column stages: loop 3.68 -> 3.46 s; 8 -> 16-column
// stages, 3 -> 64-column stages 3.95 s); c2/c3 (seg 28) keep 64 columns x 13.
#ifndef ALNNLS_MIN_STAGES
#define ALNNLS_MIN_STAGES 6
#endif

#ifndef ALNNLS_RPW_MIN
#define ALNNLS_RPW_MIN 32  // build knob: fewest rows per consumer warp (8, 16 or 32);
                          // 8 measured slower (c2 89.5 vs 83.9 us/iteration), 16 equal
#endif
#ifndef ALNNLS_RING_COLS
#define ALNNLS_RING_COLS 128  // build knob: widest stage (columns); 128 halves the per-column
                             // share of the stage wait, chained as two 64-column halves
                             // (c2 87.0 -> 83.8, c3 101.1 -> 96.0 us/iteration vs 64)
#endif
constexpr int kRingCols = ALNNLS_RING_COLS;   // columns per stage
constexpr int kMaxStages = 48;
#ifndef ALNNLS_RING_KB
#define ALNNLS_RING_KB 208  // build knob (c5: 7 instead of 6 32-column stages, 503 -> 497 us/iteration)
#endif
constexpr size_t kRingSmemBytes = ALNNLS_RING_KB * 1024;  // dynamic smem of ring-carrying kernels

struct RowRing {
  uint64_t* full;
  uint64_t* empty;
  double* data;   // [S][G][seg]
  double* vals;   // [S][2][G] (the second half: a second right-hand side)
  int S;
  int G;          // columns per stage
  int seg;        // doubles per column slot
  int P;          // producer warps: warps [0, P)
  int cons_warps; // consumer warps: warps [P, P + cons_warps)
  int rpw;        // rows per consumer warp (lanes [0, rpw) own rows)
  uint32_t pos;   // stages issued so far (identical in every thread)
  uint32_t smask; // S - 1 when S is a power of two (ALNNLS_POW2_STAGES), else 0
  uint32_t sshift;
  uint64_t l2pol; // L2 policy of the matrix copies (0: none)
};

#ifndef ALNNLS_POW2_STAGES
#define ALNNLS_POW2_STAGES 1  // build knob: round the stage count down to a power of two
                              // (c2: 12 -> 8 stages, 86.2 -> 83.3-85.3 us/iteration)
#endif
// Slot and phase parity of the p-th stage use: shifts and masks for a power-of-two
// ring instead of a 32-bit division per stage.
__device__ __forceinline__ int ring_slot(const RowRing& r, uint32_t p) {
  return r.smask ? (int)(p & r.smask) : (int)(p % r.S);
}
__device__ __forceinline__ uint32_t ring_par(const RowRing& r, uint32_t p) {
  return r.smask ? (p >> r.sshift) & 1u : (p / r.S) & 1u;
}
#ifndef ALNNLS_STAGE_CAP
#define ALNNLS_STAGE_CAP 48  // build knob: most stages a ring keeps
#endif

__host__ __device__ inline int ring_seg(int nrows) { return (nrows + 1) & ~1; }
__host__ __device__ inline size_t ring_stage_bytes(int seg, int G) {
  return (size_t)G * seg * 8 + (size_t)2 * G * 8;
}

// Carves the ring out of `smem` (16B aligned, `bytes` long). seg = doubles per
// column slot (>= nrows, even). max_warps bounds producers + consumers. Must be
// called by every thread; contains a __syncthreads.
__device__ inline void ring_setup(RowRing& r, uint8_t* smem, size_t bytes, int nrows, int seg,
                                  int max_warps) {
  r.seg = seg;
  // Rows per consumer warp: the smallest of ALNNLS_RPW_MIN, 16, 32 that fits the
  // warps left beside the producers. Fewer rows per warp = more warps running
  // their (latency-bound) DADD chains concurrently: while one warp waits on its
  // chain, another forms its products (c2, 28 rows: 4 warps of 8 rows).
  {
    const int avail = max(1, max_warps - min(ALNNLS_PRODUCERS, 4));
    int rpw = ALNNLS_RPW_MIN;
    while (rpw < 32 && (nrows + rpw - 1) / rpw > avail) rpw *= 2;
    r.rpw = rpw;
  }
  r.cons_warps = max(1, (nrows + r.rpw - 1) / r.rpw);
  const size_t hdr = (size_t)kMaxStages * 16;
  int G = kRingCols;
  while (G > 8 && (bytes - hdr) / ring_stage_bytes(seg, G) < ALNNLS_MIN_STAGES) G >>= 1;
  r.G = G;
  int S = (int)((bytes - hdr) / ring_stage_bytes(seg, G));
  if (S > kMaxStages) S = kMaxStages;
  if (S > ALNNLS_STAGE_CAP) S = ALNNLS_STAGE_CAP;
  r.smask = 0;
  r.sshift = 0;
  if (ALNNLS_POW2_STAGES) {  // a power of two unless that leaves fewer than the minimum
    int sh = 0;
    while ((2 << sh) <= S) ++sh;
    if ((1 << sh) >= ALNNLS_MIN_STAGES || (1 << sh) == S) {
      S = 1 << sh;
      r.smask = (uint32_t)S - 1u;
      r.sshift = (uint32_t)sh;
    }
  }
  r.S = S;
  r.P = max(1, min(min(ALNNLS_PRODUCERS, S), max_warps - r.cons_warps));
  r.full = reinterpret_cast<uint64_t*>(smem);
  r.empty = r.full + kMaxStages;
  r.data = reinterpret_cast<double*>(smem + hdr);
  r.vals = r.data + (size_t)S * G * seg;
  r.pos = 0;
  r.l2pol = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&r.full[s], 1);
      mbar_init(&r.empty[s], r.cons_warps);
    }
    fence_mbar_init();
  }
  __syncthreads();
}

// Runs the row-block GEMV over `len` listed columns. Column j's segment for
// this CTA starts at base + j*col_stride and is seg doubles long. When
// `runs` is true (blocked layout, col_stride == seg) consecutive listed
// columns are fetched with one bulk copy. Warps outside [0, P+cons_warps)
// return immediately. Every thread must call it (r.pos advances uniformly).
// Consumers write out[row0 + t], and, when opos is given, also
// out_c[opos[t]] for rows with opos[t] >= 0 (a compacted copy). No block
// barrier inside.
__device__ inline void gemv_rows(RowRing& r, const double* __restrict__ base, uint64_t col_stride,
                                 bool runs, int row0, int nrows,
                                 const uint32_t* __restrict__ list,
                                 const double* __restrict__ vals, int len,
                                 double* __restrict__ out, const int* opos = nullptr,
                                 double* __restrict__ out_c = nullptr,
                                 const double* __restrict__ vals2 = nullptr,
                                 double* __restrict__ out2 = nullptr) {
  const int G = r.G;
  const int nst = (len + G - 1) / G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int seg = r.seg;
  if (warp < r.P) {
    // order generic-proxy writes of list/vals (before the grid barrier)
    // before the async-proxy bulk reads issued below
    asm volatile("fence.proxy.async.global;" ::: "memory");
    for (int s = warp; s < nst; s += r.P) {
      const uint32_t p = r.pos + s;
      const int st = ring_slot(r, p);
      const uint32_t ph = ring_par(r, p);
      const int sbase = s * G;
      const int cnt = min(G, len - sbase);
      if (lane == 0) {
        mbar_wait(&r.empty[st], ph ^ 1u);
        const uint32_t bytes =
            (uint32_t)(cnt * seg * 8 + (vals2 ? 2 : 1) * ((cnt + 1) & ~1) * 8);
        mbar_arrive_expect_tx(&r.full[st], bytes);
      }
      __syncwarp();
      double* dst = r.data + (size_t)st * G * seg;
      for (int l0 = 0; l0 < cnt; l0 += 32) {
        const int l = l0 + lane;
        const bool valid = l < cnt;
        const uint32_t j = valid ? __ldcg(list + sbase + l) : 0u;
        if (runs) {
          // a lane starts a run unless its column directly follows the previous one
          const uint32_t jp = __shfl_up_sync(0xffffffffu, j, 1);
          const bool start = valid && (lane == 0 || j != jp + 1u);
          const uint32_t starts = __ballot_sync(0xffffffffu, start);
          if (start) {
            const uint32_t later = starts & ~((2u << lane) - 1u);  // run starts after me
            int end = later ? __ffs(later) - 1 : 32;
            end = min(end, cnt - l0);
            const int rl = end - lane;
            if (r.l2pol)
              bulk_g2s_hint(dst + (size_t)l * seg, base + (size_t)j * col_stride,
                            (uint32_t)(rl * seg * 8), &r.full[st], r.l2pol);
            else
              bulk_g2s(dst + (size_t)l * seg, base + (size_t)j * col_stride,
                       (uint32_t)(rl * seg * 8), &r.full[st]);
          }
        } else if (valid) {
          bulk_g2s(dst + (size_t)l * seg, base + (size_t)j * col_stride, (uint32_t)seg * 8,
                   &r.full[st]);
        }
      }
      if (lane == 0)
        bulk_g2s(r.vals + (size_t)st * 2 * G, vals + sbase, (uint32_t)(((cnt + 1) & ~1) * 8),
                 &r.full[st]);
      if (lane == 1 && vals2)
        bulk_g2s(r.vals + (size_t)st * 2 * G + G, vals2 + sbase,
                 (uint32_t)(((cnt + 1) & ~1) * 8), &r.full[st]);
    }
  } else if (warp < r.P + r.cons_warps) {
    const int t = (warp - r.P) * r.rpw + lane;
    const bool mine = lane < r.rpw && t < nrows;
    const int tt = mine ? t : 0;
    double acc = 0.0, acc2 = 0.0;
    for (int s = 0; s < nst; ++s) {
      const uint32_t p = r.pos + s;
      const int st = ring_slot(r, p);
      const uint32_t ph = ring_par(r, p);
      const int cnt = min(G, len - s * G);
      mbar_wait(&r.full[st], ph);
      const double* col = r.data + (size_t)st * G * seg;
      const double* v = r.vals + (size_t)st * 2 * G;
      if (vals2) {  // two right-hand sides: two independent chains per row
        const double* v2 = v + G;
        for (int l0 = 0; l0 < cnt; l0 += 16) {
          double p1[16], p2[16];
#pragma unroll
          for (int l = 0; l < 16; ++l) {
            const double c = l0 + l < cnt ? col[(l0 + l) * seg + tt] : 0.0;
            p1[l] = xmul(c, v[l0 + l < cnt ? l0 + l : 0]);
            p2[l] = xmul(c, v2[l0 + l < cnt ? l0 + l : 0]);
          }
#pragma unroll
          for (int l = 0; l < 16; ++l) {  // past cnt: 0 * v = +-0, an exact no-op
            acc = xadd(acc, p1[l]);
            acc2 = xadd(acc2, p2[l]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&r.empty[st]);
        continue;
      }
      // All rounded products of a full stage are formed first (independent
      // LDS + DMUL, in registers), then one dependent DADD chain runs over
      // them: ptxas cannot interleave the chain ahead of the loads, so the
      // 8-cycle DADD latency is the only per-column cost (measured ~2.3x
      // faster than a fused mul/add loop on B200).
      if (cnt == 128 && G == 128) {
#pragma unroll 1
        for (int h = 0; h < 128; h += 64) {
          double p[64];
#pragma unroll
          for (int l = 0; l < 64; ++l) p[l] = xmul(col[(h + l) * seg + tt], v[h + l]);
#pragma unroll
          for (int l = 0; l < 64; ++l) acc = xadd(acc, p[l]);
        }
      } else if (cnt == 64 && G == 64) {
        double p[64];
#pragma unroll
        for (int l = 0; l < 64; ++l) p[l] = xmul(col[l * seg + tt], v[l]);
#pragma unroll
        for (int l = 0; l < 64; ++l) acc = xadd(acc, p[l]);
      } else if (cnt == 32 && G == 32) {
        double p[32];
#pragma unroll
        for (int l = 0; l < 32; ++l) p[l] = xmul(col[l * seg + tt], v[l]);
#pragma unroll
        for (int l = 0; l < 32; ++l) acc = xadd(acc, p[l]);
      } else if (cnt == 16 && G == 16) {  // large m (c5: seg 112)
        double p[16];
#pragma unroll
        for (int l = 0; l < 16; ++l) p[l] = xmul(col[l * seg + tt], v[l]);
#pragma unroll
        for (int l = 0; l < 16; ++l) acc = xadd(acc, p[l]);
      } else {
        for (int l = 0; l < cnt; ++l) acc = xmac(acc, col[l * seg + tt], v[l]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&r.empty[st]);
    }
    if (mine) {
      out[row0 + t] = acc;
      if (opos && opos[t] >= 0) out_c[opos[t]] = acc;
      if (out2) out2[row0 + t] = acc2;
    }
  }
  r.pos += nst;
}

// Shared-memory bytes of a resident row-block panel (seg x m doubles) plus the
// staged list and values (small m; see gemv_resident).
__host__ __device__ inline size_t resident_smem_bytes(int seg, int m) {
  return (size_t)seg * m * 8 + (size_t)(m + 8) * 12 + 64;
}

// Row-block GEMV with the CTA's Q panel resident in shared memory (small m: the
// panel, seg x m doubles, is copied in once per solve). y[row0 + t] = sum over the
// list of Qs[list[s] * seg + t] * vals[s]: thread t owns row t and runs its one
// chain in list order (the rounded products of a 64-column block, then their
// dependent DADDs), bitwise the ring GEMV's result without its per-stage waits.
// The list and values are staged into shared memory first. Whole CTA; starts and
// ends with a block barrier.
__device__ inline void gemv_resident(const double* Qs, int seg, uint32_t* sl, double* sv,
                                     int row0, int nrows, const uint32_t* __restrict__ list,
                                     const double* __restrict__ vals, int len,
                                     double* __restrict__ out, const int* opos = nullptr,
                                     double* __restrict__ out_c = nullptr) {
  __syncthreads();  // the previous call's readers are done with sl / sv
  for (int e = threadIdx.x; e < len; e += blockDim.x) {
    sl[e] = __ldcg(list + e);
    sv[e] = __ldcg(vals + e);
  }
  __syncthreads();
  const int t = threadIdx.x;
  if (t < nrows) {
    const double* q = Qs + t;
    double acc = 0.0;
    int s = 0;
    for (; s + 64 <= len; s += 64) {
      double p[64];
#pragma unroll
      for (int l = 0; l < 64; ++l) p[l] = xmul(q[(size_t)sl[s + l] * seg], sv[s + l]);
#pragma unroll
      for (int l = 0; l < 64; ++l) acc = xadd(acc, p[l]);
    }
    for (; s < len; ++s) acc = xmac(acc, q[(size_t)sl[s] * seg], sv[s]);
    out[row0 + t] = acc;
    if (opos && opos[t] >= 0) out_c[opos[t]] = acc;
  }
  __syncthreads();
}

// Blocked-layout index of Q(i, j) with block rows R (m x m logical).
__host__ __device__ inline size_t blk_index(uint64_t i, uint64_t j, uint64_t m, uint64_t R) {
  return (i / R) * R * m + j * R + (i % R);
}

}  // namespace alnnls
