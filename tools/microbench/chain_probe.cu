// Why does the row-GEMV consumer take ~19 cycles per column? Same loop, pieces added one by one.
#include <cstdio>
#include "common.cuh"
using namespace alnnls;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; } } while (0)

template <int MODE>
__global__ void k(double* out, long long* cyc, int nst) {
  __shared__ __align__(16) double col[64 * 28];
  __shared__ __align__(16) double v[64];
  __shared__ uint64_t bar;
  for (int i = threadIdx.x; i < 64 * 28; i += blockDim.x) col[i] = 1.0 + i * 1e-6;
  for (int i = threadIdx.x; i < 64; i += blockDim.x) v[i] = 0.5 + i * 1e-3;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0 && MODE >= 1) mbar_arrive(&bar);  // complete phase 0
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int tt = threadIdx.x < 28 ? threadIdx.x : 0;
  double acc = 0.0;
  long long t0 = clock64();
  for (int s = 0; s < nst; ++s) {
    if (MODE >= 1) mbar_wait(&bar, 0);
    double pr[64];
#pragma unroll
    for (int l = 0; l < 64; ++l) pr[l] = xmul(col[l * 28 + tt], v[l]);
#pragma unroll
    for (int l = 0; l < 64; ++l) acc = xadd(acc, pr[l]);
    if (MODE >= 2) { __syncwarp(); }
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* out; long long* cyc; CK(cudaMalloc(&out, 256)); CK(cudaMalloc(&cyc, 8));
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k<0><<<1, 64>>>(out, cyc, 46);
      if (mode == 1) k<1><<<1, 64>>>(out, cyc, 46);
      if (mode == 2) k<2><<<1, 64>>>(out, cyc, 46);
      CK(cudaDeviceSynchronize());
    }
    long long c; CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    printf("mode %d: %.2f cycles per column (46 stages x 64)\n", mode, (double)c / (46 * 64));
  }
  return 0;
}
