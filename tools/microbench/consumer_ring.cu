// Cycles per column of the GEMV consumer over a REAL ring (12 stages of 64
// columns x 28 rows in shared memory, stage index advancing, one mbarrier wait
// per stage on an already-complete phase), so no load is loop-invariant.
//   (p0) production consumer: products of a stage into p[64], then the chain
//   (pU) software-pipelined consumer: units of U columns; while the chain runs
//        over unit i, the products of unit i+1 are formed and the loads of
//        unit i+2 are in flight (registers carried across the stage waits)
#include <cstdio>
#include "common.cuh"
using namespace alnnls;

constexpr int SEG = 28, G = 64, S = 12, NST = 64;

__device__ __forceinline__ const double* stage_col(const double* ring, int s) {
  return ring + (size_t)(s % S) * (G * SEG + 2 * G);
}

__global__ void p0(double* out, long long* cyc, int seg) {
  extern __shared__ double sm[];
  __shared__ uint64_t bar[S];
  for (int e = threadIdx.x; e < S * (G * SEG + 2 * G); e += blockDim.x) sm[e] = 1.0 + e * 1e-9;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < S; ++i) mbar_arrive(&bar[i]);
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int tt = threadIdx.x % seg;
  double acc = 0.0;
  const long long c0 = clock64();
  for (int s = 0; s < NST; ++s) {
    mbar_wait(&bar[s % S], 0);
    const double* col = stage_col(sm, s);
    const double* v = col + G * seg;
    double p[64];
#pragma unroll
    for (int l = 0; l < 64; ++l) p[l] = xmul(col[l * seg + tt], v[l]);
#pragma unroll
    for (int l = 0; l < 64; ++l) acc = xadd(acc, p[l]);
  }
  const long long c1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}

template <int U>
__global__ void pu(double* out, long long* cyc, int seg) {
  extern __shared__ double sm[];
  __shared__ uint64_t bar[S];
  for (int e = threadIdx.x; e < S * (G * SEG + 2 * G); e += blockDim.x) sm[e] = 1.0 + e * 1e-9;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < S; ++i) mbar_arrive(&bar[i]);
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int tt = threadIdx.x % seg;
  constexpr int UPS = G / U;        // units per stage
  const int nu = NST * UPS;         // units
  double acc = 0.0;
  double c[U], v[U], pn[U], pc[U];
  auto load = [&](int unit) {       // issue the loads of `unit` (waits at a stage start)
    const int s = unit / UPS, o = (unit % UPS) * U;
    if (o == 0) mbar_wait(&bar[s % S], 0);
    const double* col = stage_col(sm, s);
    const double* vv = col + G * seg;
#pragma unroll
    for (int l = 0; l < U; ++l) {
      c[l] = col[(o + l) * seg + tt];
      v[l] = vv[o + l];
    }
  };
  const long long c0 = clock64();
  load(0);
#pragma unroll
  for (int l = 0; l < U; ++l) pn[l] = xmul(c[l], v[l]);
  load(1);
  for (int s = 0; s < NST; ++s) {
#pragma unroll
    for (int u = 0; u < UPS; ++u) {
      const int i = s * UPS + u;
#pragma unroll
      for (int l = 0; l < U; ++l) pc[l] = pn[l];
#pragma unroll
      for (int l = 0; l < U; ++l) pn[l] = xmul(c[l], v[l]);   // products of unit i+1
      if (i + 2 < nu) {                                        // loads of unit i+2
        const int s2 = s + (u + 2) / UPS, o2 = ((u + 2) % UPS) * U;
        if (o2 == 0) mbar_wait(&bar[s2 % S], 0);
        const double* col = stage_col(sm, s2);
        const double* vv = col + G * seg;
#pragma unroll
        for (int l = 0; l < U; ++l) {
          c[l] = col[(o2 + l) * seg + tt];
          v[l] = vv[o2 + l];
        }
      }
#pragma unroll
      for (int l = 0; l < U; ++l) acc = xadd(acc, pc[l]);      // chain of unit i
    }
  }
  const long long c1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}


// (r) a relay warp waits on the full mbarriers and publishes each stage on a
// named barrier (id 1 + s % S); the consumer syncs the NEXT stage's named barrier
// (one instruction, no loop, so no basic-block split) before the chain of the
// current one, and runs U-column units with loads two units ahead.
__device__ __forceinline__ void nb_sync(int id) {
  asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
}
__device__ __forceinline__ void nb_arrive(int id) {
  asm volatile("bar.arrive %0, 64;" ::"r"(id) : "memory");
}
template <int U>
__global__ void pr(double* out, long long* cyc, int seg) {
  extern __shared__ double sm[];
  __shared__ uint64_t bar[S];
  for (int e = threadIdx.x; e < S * (G * SEG + 2 * G); e += blockDim.x) sm[e] = 1.0 + e * 1e-9;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < S; ++i) mbar_arrive(&bar[i]);
  __syncthreads();
  __shared__ volatile int synced;  // stages the consumer has synced (stands in for the empty barriers)
  if (threadIdx.x == 0) synced = 0;
  __syncthreads();
  if (threadIdx.x >= 64) return;
  if (threadIdx.x >= 32) {  // relay
    for (int s = 0; s < NST + 2; ++s) {
      while (synced < s - S + 1) {}
      mbar_wait(&bar[s % S], 0);
      nb_arrive(1 + s % S);
    }
    return;
  }
  const int tt = threadIdx.x % seg;
  constexpr int UPS = G / U;
  double acc = 0.0;
  double c[U], v[U], pn[U], pc[U];
  const long long c0 = clock64();
  nb_sync(1);
  nb_sync(2);
  if (threadIdx.x == 0) synced = 2;
  {
    const double* col = stage_col(sm, 0);
    const double* vv = col + G * seg;
#pragma unroll
    for (int l = 0; l < U; ++l) pn[l] = xmul(col[l * seg + tt], vv[l]);
#pragma unroll
    for (int l = 0; l < U; ++l) { c[l] = col[(U + l) * seg + tt]; v[l] = vv[U + l]; }
  }
  for (int s = 0; s < NST; ++s) {
#pragma unroll
    for (int u = 0; u < UPS; ++u) {
#pragma unroll
      for (int l = 0; l < U; ++l) pc[l] = pn[l];
#pragma unroll
      for (int l = 0; l < U; ++l) pn[l] = xmul(c[l], v[l]);   // unit i+1
      {
        const int s2 = s + (u + 2) / UPS, o2 = ((u + 2) % UPS) * U;
        if (o2 == 0) {
          nb_sync(1 + (s2 + 1) % S);                           // one stage ahead
          if (threadIdx.x == 0) synced = s2 + 2;
        }
        const double* col = stage_col(sm, s2);
        const double* vv = col + G * seg;
#pragma unroll
        for (int l = 0; l < U; ++l) { c[l] = col[(o2 + l) * seg + tt]; v[l] = vv[o2 + l]; }
      }
#pragma unroll
      for (int l = 0; l < U; ++l) acc = xadd(acc, pc[l]);      // unit i
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
  const int smem = S * (G * SEG + 2 * G) * 8;
  long long h = 0;
  cudaFuncSetAttribute(p0, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(pu<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(pu<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(pu<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  auto run = [&](auto kern, const char* name) {
    for (int rep = 0; rep < 3; ++rep) kern<<<1, 32, smem>>>(out, cyc, SEG);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-44s %6.2f cycles/column %s\n", name, (double)h / (G * NST),
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  cudaFuncSetAttribute(pr<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(pr<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  auto run2 = [&](auto kern, const char* name) {
    for (int rep = 0; rep < 3; ++rep) kern<<<1, 64, smem>>>(out, cyc, SEG);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-44s %6.2f cycles/column %s\n", name, (double)h / (G * NST),
           e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  run2(pr<16>, "(r16) relay + named barrier, units of 16");
  run2(pr<32>, "(r32) relay + named barrier, units of 32");
  run(p0, "(p0) production: products then chain");
  run(pu<8>, "(p8) pipelined units of 8");
  run(pu<16>, "(p16) pipelined units of 16");
  run(pu<32>, "(p32) pipelined units of 32");
  return 0;
}
