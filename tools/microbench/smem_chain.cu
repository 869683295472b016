// One thread's ordered DADD chain over n products in shared memory: cycles per term
// for the production form (two alternating 16-term register blocks, LDS.128) and
// variants with deeper prefetch. The dependent DADD latency (8.05 cycles) is the floor.
#include <cstdio>
#include "common.cuh"
using namespace alnnls;

// production (nqp.cu smem_chain / small.cu chain_smem)
__device__ __forceinline__ double chain_prod(const double* __restrict__ p, int n) {
  constexpr int B = 16;
  double s = 0.0;
  int t = 0;
  if (n >= 2 * B) {
    double ra[B], rb[B];
#pragma unroll
    for (int k = 0; k < B; ++k) ra[k] = p[k];
    for (; t + 3 * B <= n; t += 2 * B) {
#pragma unroll
      for (int k = 0; k < B; ++k) rb[k] = p[t + B + k];
#pragma unroll
      for (int k = 0; k < B; ++k) s = xadd(s, ra[k]);
#pragma unroll
      for (int k = 0; k < B; ++k) ra[k] = p[t + 2 * B + k];
#pragma unroll
      for (int k = 0; k < B; ++k) s = xadd(s, rb[k]);
    }
    for (; t < n; ++t) s = xadd(s, p[t]);
  }
  return s;
}

// three blocks in rotation: loads two blocks ahead of the chain
template <int B>
__device__ __forceinline__ double chain3(const double* __restrict__ p, int n) {
  double s = 0.0;
  int t = 0;
  if (n >= 3 * B) {
    double ra[B], rb[B], rc[B];
#pragma unroll
    for (int k = 0; k < B; ++k) ra[k] = p[k];
#pragma unroll
    for (int k = 0; k < B; ++k) rb[k] = p[B + k];
    for (; t + 5 * B <= n; t += 3 * B) {
#pragma unroll
      for (int k = 0; k < B; ++k) rc[k] = p[t + 2 * B + k];
#pragma unroll
      for (int k = 0; k < B; ++k) s = xadd(s, ra[k]);
#pragma unroll
      for (int k = 0; k < B; ++k) ra[k] = p[t + 3 * B + k];
#pragma unroll
      for (int k = 0; k < B; ++k) s = xadd(s, rb[k]);
#pragma unroll
      for (int k = 0; k < B; ++k) rb[k] = p[t + 4 * B + k];
#pragma unroll
      for (int k = 0; k < B; ++k) s = xadd(s, rc[k]);
    }
    for (; t < n; ++t) s = xadd(s, p[t]);
  }
  return s;
}

// interleaved: each DADD followed by the load of the term 2B ahead (one register ring)
template <int B>
__device__ __forceinline__ double chain_ring(const double* __restrict__ p, int n) {
  double s = 0.0;
  int t = 0;
  if (n >= B) {
    double r[B];
#pragma unroll
    for (int k = 0; k < B; ++k) r[k] = p[k];
    for (; t + 2 * B <= n; t += B) {
#pragma unroll
      for (int k = 0; k < B; ++k) {
        s = xadd(s, r[k]);
        r[k] = p[t + B + k];
      }
    }
    for (; t < n; ++t) s = xadd(s, p[t]);
  }
  return s;
}

template <int MODE>
__global__ void k(double* out, long long* cyc, int n) {
  extern __shared__ __align__(16) double sm[];
  for (int i = threadIdx.x; i < n + 64; i += blockDim.x) sm[i] = 1.0 + i * 1e-9;
  __syncthreads();
  if (threadIdx.x != 0) return;
  const long long c0 = clock64();
  double s;
  if (MODE == 0) s = chain_prod(sm, n);
  else if (MODE == 1) s = chain3<16>(sm, n);
  else if (MODE == 2) s = chain3<8>(sm, n);
  else if (MODE == 3) s = chain_ring<16>(sm, n);
  else s = chain_ring<32>(sm, n);
  const long long c1 = clock64();
  out[0] = s;
  *cyc = c1 - c0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8);
  const int n = 2900;
  const char* names[] = {"production (2 x 16, LDS.128)", "3 blocks x 16", "3 blocks x 8",
                         "register ring 16", "register ring 32"};
  auto run = [&](auto kern, int mode) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    long long h = 0;
    for (int r = 0; r < 3; ++r) kern<<<1, 32, (n + 64) * 8>>>(out, cyc, n);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-30s %6.2f cycles/term\n", names[mode], (double)h / n);
  };
  run(k<0>, 0);
  run(k<1>, 1);
  run(k<2>, 2);
  run(k<3>, 3);
  run(k<4>, 4);
  return 0;
}
