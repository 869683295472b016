// Ring consumer cost: runtime stride + rotating stages + a real producer warp (arrive only).
#include <cstdio>
#include "common.cuh"
using namespace alnnls;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; } } while (0)

template <int MODE>
__global__ void __launch_bounds__(384, 1) k(double* out, long long* cyc, int nst, int seg, int S, int P) {
  extern __shared__ __align__(16) double sm[];
  __shared__ uint64_t full[48], empty[48];
  double* data = sm;
  double* vb = sm + (size_t)S * 64 * seg;
  for (int i = threadIdx.x; i < S * 64 * seg; i += blockDim.x) data[i] = 1.0 + i * 1e-7;
  for (int i = threadIdx.x; i < S * 64; i += blockDim.x) vb[i] = 0.5 + i * 1e-4;
  if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); } fence_mbar_init(); }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (MODE == 0 && warp < P) {  // producer: wait empty, arrive full
    for (int s = warp; s < nst; s += P) {
      const int st = s % S; const uint32_t ph = (s / S) & 1u;
      if (lane == 0) { mbar_wait(&empty[st], ph ^ 1u); mbar_arrive(&full[st]); }
      __syncwarp();
    }
  } else if (warp == P) {
    const int tt = lane < 28 ? lane : 0;
    double acc = 0.0;
    long long t0 = clock64();
    for (int s = 0; s < nst; ++s) {
      const int st = s % S; const uint32_t ph = (s / S) & 1u;
      if (MODE == 0) mbar_wait(&full[st], ph);
      const double* col = data + (size_t)st * 64 * seg + tt;
      const double* v = vb + st * 64;
      double pr[64];
#pragma unroll
      for (int l = 0; l < 64; ++l) pr[l] = xmul(col[l * seg], v[l]);
#pragma unroll
      for (int l = 0; l < 64; ++l) acc = xadd(acc, pr[l]);
      __syncwarp();
      if (MODE == 0 && lane == 0) mbar_arrive(&empty[st]);
    }
    long long t1 = clock64();
    out[lane] = acc;
    if (lane == 0) cyc[0] = t1 - t0;
  }
}

int main() {
  double* out; long long* cyc; CK(cudaMalloc(&out, 256)); CK(cudaMalloc(&cyc, 8));
  CK(cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000));
  CK(cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000));
  const int seg = 28, S = 12;
  const size_t sm = (size_t)S * 64 * seg * 8 + S * 64 * 8;
  for (int mode = 0; mode < 2; ++mode) for (int P : {1, 4}) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k<0><<<1, 384, sm>>>(out, cyc, 46, seg, S, P);
      else k<1><<<1, 384, sm>>>(out, cyc, 46, seg, S, P);
      CK(cudaDeviceSynchronize());
    }
    long long c; CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    printf("mode %d (0 = with producer/barriers, 1 = no barriers) P=%d: %.2f cycles per column\n", mode, P, (double)c / (46 * 64));
  }
  return 0;
}
