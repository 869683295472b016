// Cycles per column of the row-GEMV consumer patterns (data already in shared
// memory, no mbarriers): (a) products of a 64-column stage then its DADD chain;
// (b) two warps alternating stages with a named-barrier hand-off of the sums;
// (c) one warp, products of stage s+1 in the same basic block as the chain of s.
#include <cstdio>
#include "common.cuh"
using namespace alnnls;

constexpr int SEG = 28, G = 64, NST = 64;  // 4096 columns

__global__ void k_a(double* out, long long* cyc) {
  extern __shared__ double sm[];
  double* col = sm;                 // [G][SEG]
  double* v = sm + G * SEG;         // [G]
  for (int e = threadIdx.x; e < G * SEG + G; e += blockDim.x) sm[e] = 1.0 + e * 1e-9;
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int tt = threadIdx.x % SEG;
  double acc = 0.0;
  const long long c0 = clock64();
  for (int s = 0; s < NST; ++s) {
    double p[G];
#pragma unroll
    for (int l = 0; l < G; ++l) p[l] = xmul(col[l * SEG + tt], v[l]);
#pragma unroll
    for (int l = 0; l < G; ++l) acc = xadd(acc, p[l]);
    __syncwarp();
  }
  const long long c1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}

__global__ void k_c(double* out, long long* cyc) {
  extern __shared__ double sm[];
  double* col = sm;
  double* v = sm + G * SEG;
  for (int e = threadIdx.x; e < G * SEG + G; e += blockDim.x) sm[e] = 1.0 + e * 1e-9;
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int tt = threadIdx.x % SEG;
  double acc = 0.0;
  const long long c0 = clock64();
  constexpr int H = 32;  // pipeline unit: products of the next half-stage during the chain
  double pa[H], pb[H];
#pragma unroll
  for (int l = 0; l < H; ++l) pa[l] = xmul(col[l * SEG + tt], v[l]);
  for (int q = 0; q < 2 * NST - 1; q += 2) {
    const int o1 = ((q + 1) & 1) * H;
#pragma unroll
    for (int l = 0; l < H; ++l) {
      pb[l] = xmul(col[(o1 + l) * SEG + tt], v[o1 + l]);
      acc = xadd(acc, pa[l]);
    }
    const int o2 = ((q + 2) & 1) * H;
#pragma unroll
    for (int l = 0; l < H; ++l) {
      pa[l] = xmul(col[(o2 + l) * SEG + tt], v[o2 + l]);
      acc = xadd(acc, pb[l]);
    }
  }
#pragma unroll
  for (int l = 0; l < H; ++l) acc = xadd(acc, pa[l]);
  const long long c1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}

__global__ void k_b(double* out, long long* cyc) {
  extern __shared__ double sm[];
  double* col = sm;
  double* v = sm + G * SEG;
  __shared__ double hand[2][32];
  for (int e = threadIdx.x; e < G * SEG + G; e += blockDim.x) sm[e] = 1.0 + e * 1e-9;
  __syncthreads();
  if (threadIdx.x >= 64) return;
  const int role = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tt = lane % SEG;
  double acc = 0.0;
  const long long c0 = clock64();
  for (int s = role; s < NST; s += 2) {
    double p[G];
#pragma unroll
    for (int l = 0; l < G; ++l) p[l] = xmul(col[l * SEG + tt], v[l]);
    if (s > 0) {
      asm volatile("bar.sync %0, 64;" ::"r"(1 + ((s - 1) & 1)) : "memory");
      acc = hand[(s - 1) & 1][lane];
    }
#pragma unroll
    for (int l = 0; l < G; ++l) acc = xadd(acc, p[l]);
    if (s + 1 < NST) {
      hand[s & 1][lane] = acc;
      asm volatile("bar.arrive %0, 64;" ::"r"(1 + (s & 1)) : "memory");
    }
  }
  const long long c1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 32) *cyc = c1 - c0;  // role 1 ends last
}

// (d) = (c) with a runtime segment stride, a ring of 12 slots indexed modulo,
// and an mbarrier wait (already-complete phase) at every 64-column stage start.
__device__ __forceinline__ bool probe_mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return done != 0;
}
__device__ __forceinline__ bool probe_mbar_test_nc(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity));
  return done != 0;
}
template <bool WAIT, int CSEG, int KIND = 0>
__global__ void k_d(double* out, long long* cyc, int seg_rt, int S) {
  const int seg = CSEG ? CSEG : seg_rt;
  extern __shared__ double sm[];
  __shared__ uint64_t bar[12];
  double* col = sm;
  double* v = sm + G * SEG;
  for (int e = threadIdx.x; e < G * SEG + G; e += blockDim.x) sm[e] = 1.0 + e * 1e-9;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 12; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < 12; ++i) mbar_arrive(&bar[i]);  // phase 0 complete
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int tt = threadIdx.x % seg;
  double acc = 0.0;
  const long long c0 = clock64();
  constexpr int H = 32;
  double pa[H], pb[H];
  mbar_wait(&bar[0], 0);
#pragma unroll
  for (int l = 0; l < H; ++l) pa[l] = xmul(col[l * seg + tt], v[l]);
  for (int q = 0; q < 2 * NST - 1; q += 2) {
    // chunk q+1: second half of stage q/2 (no wait)
    const int o1 = H;
#pragma unroll
    for (int l = 0; l < H; ++l) {
      pb[l] = xmul(col[(o1 + l) * seg + tt], v[o1 + l]);
      acc = xadd(acc, pa[l]);
    }
    // chunk q+2: first half of the next stage: wait for it first
    const int st = ((q + 2) / 2) % S;
    if (WAIT) {
      if (KIND == 0) mbar_wait(&bar[st % 12], 0);
      else while (!probe_mbar_test(&bar[st % 12], 0)) {}
    }
#pragma unroll
    for (int l = 0; l < H; ++l) {
      pa[l] = xmul(col[l * seg + tt], v[l]);
      acc = xadd(acc, pb[l]);
    }
  }
#pragma unroll
  for (int l = 0; l < H; ++l) acc = xadd(acc, pa[l]);
  const long long c1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}

// (i): readiness of stage s+1 tested (non-blocking test_wait) one stage ahead;
// the blocking wait only runs if that test failed.
template <bool NC>
__global__ void k_i(double* out, long long* cyc, int seg, int S) {
  extern __shared__ double sm[];
  __shared__ uint64_t bar[12];
  double* col = sm;
  double* v = sm + G * SEG;
  for (int e = threadIdx.x; e < G * SEG + G; e += blockDim.x) sm[e] = 1.0 + e * 1e-9;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 12; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < 12; ++i) mbar_arrive(&bar[i]);
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int tt = threadIdx.x % seg;
  double acc = 0.0;
  const long long c0 = clock64();
  constexpr int H = 32;
  double pa[H], pb[H];
  mbar_wait(&bar[0], 0);
  bool rnext = probe_mbar_test(&bar[1 % 12], 0);
#pragma unroll
  for (int l = 0; l < H; ++l) pa[l] = xmul(col[l * seg + tt], v[l]);
  for (int q = 0; q < 2 * NST - 1; q += 2) {
    const int sn = ((q + 2) / 2) % S;   // next stage
    const int snn = ((q + 4) / 2) % S;  // the one after: test it now
    const bool rn2 = NC ? probe_mbar_test_nc(&bar[snn % 12], 0) : probe_mbar_test(&bar[snn % 12], 0);
#pragma unroll
    for (int l = 0; l < H; ++l) {
      pb[l] = xmul(col[(H + l) * seg + tt], v[H + l]);
      acc = xadd(acc, pa[l]);
    }
    if (!rnext) mbar_wait(&bar[sn % 12], 0);
    rnext = rn2;
#pragma unroll
    for (int l = 0; l < H; ++l) {
      pa[l] = xmul(col[l * seg + tt], v[l]);
      acc = xadd(acc, pb[l]);
    }
  }
#pragma unroll
  for (int l = 0; l < H; ++l) acc = xadd(acc, pa[l]);
  const long long c1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}


// (o) = (i) with the probe placed AFTER the next half's product loads in program
// order: ptxas hoists register-only DADDs above an mbarrier probe but keeps loads
// below it, so a probe issued before the loads serialises products and chain.
__global__ void k_o(double* out, long long* cyc, int seg, int S) {
  extern __shared__ double sm[];
  __shared__ uint64_t bar[12];
  double* col = sm;
  double* v = sm + G * SEG;
  for (int e = threadIdx.x; e < G * SEG + G; e += blockDim.x) sm[e] = 1.0 + e * 1e-9;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 12; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < 12; ++i) mbar_arrive(&bar[i]);
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int tt = threadIdx.x % seg;
  double acc = 0.0;
  const long long c0 = clock64();
  constexpr int H = 32;
  double pa[H], pb[H];
  mbar_wait(&bar[0], 0);
  bool rnext = probe_mbar_test(&bar[1 % 12], 0);
#pragma unroll
  for (int l = 0; l < H; ++l) pa[l] = xmul(col[l * seg + tt], v[l]);
  for (int s = 0; s < NST; ++s) {
#pragma unroll
    for (int l = 0; l < H; ++l) pb[l] = xmul(col[(H + l) * seg + tt], v[H + l]);
    const bool rn2 = s + 2 < NST ? probe_mbar_test(&bar[((s + 2) % S) % 12], 0) : true;
#pragma unroll
    for (int l = 0; l < H; ++l) acc = xadd(acc, pa[l]);
    if (s + 1 < NST) {
      if (!rnext) mbar_wait(&bar[((s + 1) % S) % 12], 0);
#pragma unroll
      for (int l = 0; l < H; ++l) pa[l] = xmul(col[l * seg + tt], v[l]);
    }
#pragma unroll
    for (int l = 0; l < H; ++l) acc = xadd(acc, pb[l]);
    rnext = rn2;
  }
  const long long c1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}

// (k) = (d) with the per-stage wait replaced by a poll of a plain shared-memory
// flag (what a relay warp that did the mbarrier wait would publish).
__device__ __forceinline__ uint32_t lds_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t lds_volatile(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.volatile.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
template <int KIND>
__global__ void k_k(double* out, long long* cyc, int seg, int S) {
  extern __shared__ double sm[];
  __shared__ uint32_t flag[12];
  double* col = sm;
  double* v = sm + G * SEG;
  for (int e = threadIdx.x; e < G * SEG + G; e += blockDim.x) sm[e] = 1.0 + e * 1e-9;
  if (threadIdx.x < 12) flag[threadIdx.x] = 1;
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int tt = threadIdx.x % seg;
  double acc = 0.0;
  const long long c0 = clock64();
  constexpr int H = 32;
  double pa[H], pb[H];
#pragma unroll
  for (int l = 0; l < H; ++l) pa[l] = xmul(col[l * seg + tt], v[l]);
  for (int q = 0; q < 2 * NST - 1; q += 2) {
#pragma unroll
    for (int l = 0; l < H; ++l) {
      pb[l] = xmul(col[(H + l) * seg + tt], v[H + l]);
      acc = xadd(acc, pa[l]);
    }
    const int st = ((q + 2) / 2) % S;
    if (KIND == 0) { while (lds_acquire(&flag[st % 12]) != 1u) {} }
    else { while (lds_volatile(&flag[st % 12]) != 1u) {} }
#pragma unroll
    for (int l = 0; l < H; ++l) {
      pa[l] = xmul(col[l * seg + tt], v[l]);
      acc = xadd(acc, pb[l]);
    }
  }
#pragma unroll
  for (int l = 0; l < H; ++l) acc = xadd(acc, pa[l]);
  const long long c1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}

// (m) dependent latency of one mbarrier phase check on a completed phase
__global__ void k_m(double* out, long long* cyc, int kind) {
  __shared__ uint64_t bar[2];
  if (threadIdx.x == 0) { mbar_init(&bar[0], 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) mbar_arrive(&bar[0]);
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const long long c0 = clock64();
  uint32_t par = 0;
  for (int i = 0; i < 1000; ++i) {
    if (kind == 0) { par ^= mbar_try_wait(&bar[0], 0) ? 0u : 1u; }
    else { par ^= probe_mbar_test(&bar[0], par) ? 0u : 1u; }
  }
  const long long c1 = clock64();
  out[threadIdx.x] = par;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}


// (n) = (d) with the mbarrier waits batched: before every W-th stage the
// consumer waits for the next W stages at once, then runs them straight-line.
template <int W>
__global__ void k_n(double* out, long long* cyc, int seg, int S) {
  extern __shared__ double sm[];
  __shared__ uint64_t bar[12];
  double* col = sm;
  double* v = sm + G * SEG;
  for (int e = threadIdx.x; e < G * SEG + G; e += blockDim.x) sm[e] = 1.0 + e * 1e-9;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 12; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < 12; ++i) mbar_arrive(&bar[i]);
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int tt = threadIdx.x % seg;
  double acc = 0.0;
  const long long c0 = clock64();
  constexpr int H = 32;
  double pa[H], pb[H];
  for (int w = 0; w < W; ++w) mbar_wait(&bar[w % 12], 0);
#pragma unroll
  for (int l = 0; l < H; ++l) pa[l] = xmul(col[l * seg + tt], v[l]);
  for (int s0 = 0; s0 < NST; s0 += W) {
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const int s = s0 + w;
      if (w == W - 1 && s + 1 < NST)
        for (int x = 0; x < W; ++x) mbar_wait(&bar[((s + 1 + x) % S) % 12], 0);
#pragma unroll
      for (int l = 0; l < H; ++l) {
        pb[l] = xmul(col[(H + l) * seg + tt], v[H + l]);
        acc = xadd(acc, pa[l]);
      }
      if (s + 1 < NST) {
#pragma unroll
        for (int l = 0; l < H; ++l) {
          pa[l] = xmul(col[l * seg + tt], v[l]);
          acc = xadd(acc, pb[l]);
        }
      } else {
#pragma unroll
        for (int l = 0; l < H; ++l) acc = xadd(acc, pb[l]);
      }
    }
  }
  const long long c1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 64 * 8);
  cudaMalloc(&cyc, 8);
  const size_t smem = (G * SEG + G) * 8;
  long long h = 0;
  auto run = [&](auto kern, int threads, const char* name) {
    for (int rep = 0; rep < 3; ++rep) kern<<<1, threads, smem>>>(out, cyc);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-34s %6.2f cycles/column (%lld cycles, %d columns)\n", name, (double)h / (G * NST), h,
           G * NST);
  };
  run(k_a, 32, "(a) products then chain, 1 warp");
  run(k_b, 64, "(b) 2 warps alternating, bar hand-off");
  run(k_c, 32, "(c) 1 warp, products || chain");
  auto rd = [&](auto kern, const char* name) {
    for (int rep = 0; rep < 3; ++rep) kern<<<1, 32, smem>>>(out, cyc, SEG, 12);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-34s %6.2f cycles/column\n", name, (double)h / (G * NST));
  };
  rd(k_d<true, 0>, "(d) runtime seg + mbar waits");
  rd(k_d<false, 0>, "(e) runtime seg, no waits");
  rd(k_d<true, SEG>, "(f) const seg + mbar waits");
  rd(k_d<false, SEG>, "(g) const seg, no waits");
  rd(k_d<true, 0, 1>, "(h) runtime seg + test_wait spin");
  rd(k_i<false>, "(i) test one stage ahead");
  rd(k_i<true>, "(j) test ahead, no memory clobber");
  rd(k_o, "(o) probe after the next loads");
  rd(k_n<2>, "(n2) waits batched per 2 stages");
  rd(k_n<4>, "(n4) waits batched per 4 stages");
  rd(k_n<8>, "(n8) waits batched per 8 stages");
  rd(k_k<0>, "(k) shared flag poll, ld.acquire");
  rd(k_k<1>, "(l) shared flag poll, ld.volatile");
  for (int kind = 0; kind < 2; ++kind) {
    k_m<<<1, 32>>>(out, cyc, kind);
    k_m<<<1, 32>>>(out, cyc, kind);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("(m%d) mbarrier %s dependent latency: %.1f cycles\n", kind, kind ? "test_wait" : "try_wait", h / 1000.0);
  }
  return 0;
}
