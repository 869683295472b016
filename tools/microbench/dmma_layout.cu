// Checks the mma.sync m16n8k8 f64 fragment layout assumed by dmma.cuh:
//   A (16x8 row):  a0 (g, t) a1 (g+8, t) a2 (g, t+4) a3 (g+8, t+4)
//   B (8x8 col):   b0 (t, g) b1 (t+4, g)
//   C (16x8):      c0 (g, 2t) c1 (g, 2t+1) c2 (g+8, 2t) c3 (g+8, 2t+1)
// with g = lane / 4, t = lane % 4. Integer-valued inputs make the products exact.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__global__ void k(const double* A, const double* B, double* C) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a0 = A[g * 8 + t], a1 = A[(g + 8) * 8 + t], a2 = A[g * 8 + t + 4], a3 = A[(g + 8) * 8 + t + 4];
  double b0 = B[t * 8 + g], b1 = B[(t + 4) * 8 + g];
  double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3)
      : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  C[g * 8 + 2 * t] = c0;
  C[g * 8 + 2 * t + 1] = c1;
  C[(g + 8) * 8 + 2 * t] = c2;
  C[(g + 8) * 8 + 2 * t + 1] = c3;
}

int main() {
  double hA[128], hB[64], hC[128], ref[128];
  for (int i = 0; i < 128; ++i) hA[i] = (i * 7) % 13 - 6;
  for (int i = 0; i < 64; ++i) hB[i] = (i * 5) % 11 - 5;
  for (int i = 0; i < 16; ++i)
    for (int j = 0; j < 8; ++j) {
      double s = 0;
      for (int kk = 0; kk < 8; ++kk) s += hA[i * 8 + kk] * hB[kk * 8 + j];
      ref[i * 8 + j] = s;
    }
  double *dA, *dB, *dC;
  cudaMalloc(&dA, sizeof hA);
  cudaMalloc(&dB, sizeof hB);
  cudaMalloc(&dC, sizeof hC);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(dA, dB, dC);
  cudaMemcpy(hC, dC, sizeof hC, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < 128; ++i) bad += hC[i] != ref[i];
  printf("dmma m16n8k8 f64 layout: %s (%d mismatches)\n", bad ? "WRONG" : "ok", bad);
  return bad != 0;
}
