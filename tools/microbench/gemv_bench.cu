// Standalone timing of the production gemv_rows (gemv.cuh) on the blocked layout.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "gemv.cuh"
using namespace alnnls;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void __launch_bounds__(384, 1) k_blocked(const double* Qb, int m, int R, const uint32_t* list, const double* vals, int len, double* y, int maxw) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int row0 = blockIdx.x * R;
  const int nrows = max(0, min(m - row0, R));
  RowRing ring;
  ring_setup(ring, smem, kRingSmemBytes, nrows, R, maxw);
  gemv_rows(ring, Qb + (size_t)blockIdx.x * R * m, R, true, row0, nrows, list, vals, len, y);
}

int main(int argc, char** argv) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  CK(cudaFuncSetAttribute(k_blocked, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRingSmemBytes));
  for (int cfg = 0; cfg < 4; ++cfg) {
    const int m = cfg < 2 ? 4096 : 16384;
    const double dens = (cfg % 2 == 0) ? 0.71 : 1.0;
    int R = (m + 146) / 147; R = (R + 3) & ~3;
    const int nb = (m + R - 1) / R;
    const size_t qsz = (size_t)nb * R * m;
    double *Q, *vals, *y; uint32_t* list;
    CK(cudaMalloc(&Q, qsz * 8)); CK(cudaMemset(Q, 0, qsz * 8));
    CK(cudaMalloc(&vals, (m + 64) * 8)); CK(cudaMemset(vals, 0, (m + 64) * 8));
    CK(cudaMalloc(&y, m * 8)); CK(cudaMalloc(&list, (m + 64) * 4));
    std::vector<uint32_t> hl; srand(7);
    for (int j = 0; j < m; ++j) if ((rand() % 1000) < dens * 1000) hl.push_back(j);
    const int L = hl.size();
    int runs = 0; for (int t = 0; t < L; ++t) if (t == 0 || hl[t] != hl[t-1] + 1) ++runs;
    CK(cudaMemcpy(list, hl.data(), L * 4, cudaMemcpyHostToDevice));
    for (int maxw : {4, 5, 12}) {
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        for (int it = 0; it < 20; ++it) k_blocked<<<nb, 384, kRingSmemBytes>>>(Q, m, R, list, vals, L, y, maxw);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
      }
      cudaEventElapsedTime(&ms, e0, e1);
      const double us = ms * 1e3 / 20;
      printf("m=%5d R=%3d |P|=%5d runs=%5d maxw=%2d : %7.1f us/pass  %6.0f GB/s algorithmic\n", m, R, L, runs, maxw, us, 8.0 * m * L / (us * 1e3));
    }
    cudaFree(Q); cudaFree(vals); cudaFree(y); cudaFree(list);
  }
  return 0;
}
