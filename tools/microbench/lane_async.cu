// Exact row GEMV at the c2 shape: the production TMA ring (gemv.cuh gemv_rows) vs
// a consumer warp that streams its own rows' elements with per-lane cp.async
// (LDGSTS) and waits with cp.async.wait_group (one instruction, no mbarrier loop,
// so the chain's basic block is not split). Each lane only reads what it copied,
// so there is no cross-lane synchronisation at all. Checks bitwise agreement.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "gemv.cuh"
using namespace alnnls;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void __launch_bounds__(384, 1) k_ring(const double* Qb, int m, int R, const uint32_t* list,
                                                const double* vals, int len, double* y) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int row0 = blockIdx.x * R;
  const int nrows = max(0, min(m - row0, R));
  RowRing ring;
  ring_setup(ring, smem, kRingSmemBytes, nrows, R, 12);
  gemv_rows(ring, Qb + (size_t)blockIdx.x * R * m, R, true, row0, nrows, list, vals, len, y);
}

__device__ __forceinline__ void cp8(void* dst, const void* src, uint32_t n) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(n)
               : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void wait_g() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// MODE 0: per group, products then chain. MODE 1: products of group g+1 formed
// while the chain of group g runs (the wait for g+1 comes first).
template <int G, int D, int MODE>
__global__ void __launch_bounds__(384, 1) k_lane(const double* Qb, int m, int R, const uint32_t* list,
                                                const double* vals, int len, double* y) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint32_t* sl = reinterpret_cast<uint32_t*>(smem);
  double* sv = reinterpret_cast<double*>(smem + (((size_t)len * 4 + 15) & ~15));
  double* buf = sv + ((len + 1) & ~1);  // [(D + 1)][G][32]
  const int row0 = blockIdx.x * R;
  const int nrows = max(0, min(m - row0, R));
  for (int e = threadIdx.x; e < len; e += blockDim.x) {
    sl[e] = list[e];
    sv[e] = vals[e];
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  const int tt = lane < R ? lane : R - 1;
  const double* qb = Qb + (size_t)blockIdx.x * R * m + tt;
  const int ng = (len + G - 1) / G;
  auto issue = [&](int g) {
    double* dst = buf + (size_t)(g % (D + 1)) * G * 32 + lane;
#pragma unroll
    for (int l = 0; l < G; ++l) {
      const int c = g * G + l;
      const bool v = c < len;
      cp8(dst + l * 32, v ? qb + (size_t)sl[c] * R : qb, v ? 8u : 0u);
    }
  };
  for (int g = 0; g < D; ++g) {
    if (g < ng) issue(g);
    commit();
  }
  double acc = 0.0;
  if (MODE == 0) {
    for (int g = 0; g < ng; ++g) {
      wait_g<D - 1>();
      const double* src = buf + (size_t)(g % (D + 1)) * G * 32 + lane;
      double p[G];
#pragma unroll
      for (int l = 0; l < G; ++l) {
        const int c = g * G + l;
        p[l] = xmul(src[l * 32], sv[c < len ? c : 0]);  // past len: 0 * v = +-0, a no-op
      }
      if (g + D < ng) issue(g + D);
      commit();
#pragma unroll
      for (int l = 0; l < G; ++l) acc = xadd(acc, p[l]);
    }
  } else {
    double pa[G], pb[G];
    wait_g<D - 1>();
    {
      const double* src = buf + lane;
#pragma unroll
      for (int l = 0; l < G; ++l) pa[l] = xmul(src[l * 32], sv[l < len ? l : 0]);
    }
    if (D < ng) issue(D);
    commit();
    for (int g = 0; g < ng; g += 2) {
      // group g+1: wait, products, while the chain of g runs
      wait_g<D - 1>();
      {
        const double* src = buf + (size_t)((g + 1) % (D + 1)) * G * 32 + lane;
#pragma unroll
        for (int l = 0; l < G; ++l) {
          const int c = (g + 1) * G + l;
          pb[l] = xmul(src[l * 32], sv[c < len ? c : 0]);
          acc = xadd(acc, pa[l]);
        }
      }
      if (g + 1 + D < ng) issue(g + 1 + D);
      commit();
      if (g + 1 >= ng) break;  // pb is past the end (zeros): done
      wait_g<D - 1>();
      {
        const double* src = buf + (size_t)((g + 2) % (D + 1)) * G * 32 + lane;
#pragma unroll
        for (int l = 0; l < G; ++l) {
          const int c = (g + 2) * G + l;
          pa[l] = xmul(src[l * 32], sv[c < len ? c : 0]);
          acc = xadd(acc, pb[l]);
        }
      }
      if (g + 2 + D < ng) issue(g + 2 + D);
      commit();
    }
  }
  if (lane < nrows) y[row0 + lane] = acc;
}


// L1-prefetch consumer: warps 1..P prefetch (prefetch.global.L1) the CTA's column
// segments D columns ahead of the consumer's published position; warp 0 (the
// consumer) reads Q with plain loads (L1 hits when the prefetch landed) -- no
// mbarrier, no wait, no branch in its loop. Correctness does not depend on the
// prefetch. The list and values are staged in shared memory first.
template <int D, int P, int MODE>
__global__ void __launch_bounds__(384, 1) k_pref(const double* Qb, int m, int R, const uint32_t* list,
                                                const double* vals, int len, double* y) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint32_t* sl = reinterpret_cast<uint32_t*>(smem);
  double* sv = reinterpret_cast<double*>(smem + (((size_t)len * 4 + 15) & ~15));
  __shared__ volatile int progress;
  const int row0 = blockIdx.x * R;
  const int nrows = max(0, min(m - row0, R));
  for (int e = threadIdx.x; e < len; e += blockDim.x) {
    sl[e] = list[e];
    sv[e] = vals[e];
  }
  if (threadIdx.x == 0) progress = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* qb = Qb + (size_t)blockIdx.x * R * m;
  if (warp >= 1 && warp <= P) {
    // prefetcher: columns [pos, progress + D), round-robin over the P warps in 32-column chunks
    int next = (warp - 1) * 32;
    while (next < len) {
      while (next >= progress + D) { }
      const int c = next + lane;
      if (c < len) {
        const char* a = reinterpret_cast<const char*>(qb + (size_t)sl[c] * R);
        asm volatile("prefetch.global.L1 [%0];" ::"l"(a));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(a + 128));
        if (R * 8 > 256) asm volatile("prefetch.global.L1 [%0];" ::"l"(a + 256));
      }
      next += P * 32;
    }
    return;
  }
  if (warp != 0) return;
  const int tt = lane < R ? lane : R - 1;
  const double* q = qb + tt;
  double acc = 0.0;
  int s = 0;
  if (MODE == 0) {  // products of 32 columns, then their chain
    for (; s + 32 <= len; s += 32) {
      double p[32];
#pragma unroll
      for (int l = 0; l < 32; ++l) p[l] = xmul(__ldg(q + (size_t)sl[s + l] * R), sv[s + l]);
#pragma unroll
      for (int l = 0; l < 32; ++l) acc = xadd(acc, p[l]);
      if (lane == 0) progress = s + 32;
    }
  } else {  // pipelined: products of the next 32 while the chain of these runs
    double pa[32], pb[32];
    if (len >= 64) {
#pragma unroll
      for (int l = 0; l < 32; ++l) pa[l] = xmul(__ldg(q + (size_t)sl[l] * R), sv[l]);
      for (; s + 96 <= len; s += 64) {
#pragma unroll
        for (int l = 0; l < 32; ++l) {
          pb[l] = xmul(__ldg(q + (size_t)sl[s + 32 + l] * R), sv[s + 32 + l]);
          acc = xadd(acc, pa[l]);
        }
        if (lane == 0) progress = s + 32;
#pragma unroll
        for (int l = 0; l < 32; ++l) {
          pa[l] = xmul(__ldg(q + (size_t)sl[s + 64 + l] * R), sv[s + 64 + l]);
          acc = xadd(acc, pb[l]);
        }
        if (lane == 0) progress = s + 64;
      }
#pragma unroll
      for (int l = 0; l < 32; ++l) acc = xadd(acc, pa[l]);
      s += 32;
    }
  }
  for (; s < len; ++s) acc = xmac(acc, __ldg(q + (size_t)sl[s] * R), sv[s]);
  if (lane < nrows) y[row0 + lane] = acc;
}

template <class K>
float run(K kern, size_t smem, int nb, const double* Q, int m, int R, const uint32_t* list,
          const double* vals, int L, double* y) {
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    for (int it = 0; it < 20; ++it) kern<<<nb, 384, smem>>>(Q, m, R, list, vals, L, y);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
  }
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1e3f / 20;
}

int main() {
  const int m = 4096;
  int R = (m + 146) / 147;
  R = (R + 3) & ~3;
  const int nb = (m + R - 1) / R;
  const size_t qsz = (size_t)nb * R * m;
  std::vector<double> hq(qsz);
  srand(7);
  for (auto& v : hq) v = (rand() % 20001 - 10000) * 1e-4 + 1e-9 * (rand() % 997);
  std::vector<uint32_t> hl;
  for (int j = 0; j < m; ++j)
    if ((rand() % 1000) < 710) hl.push_back(j);
  const int L = hl.size();
  std::vector<double> hv(L);
  for (auto& v : hv) v = (rand() % 20001 - 10000) * 1e-3;
  double *Q, *vals, *y0, *y1;
  uint32_t* list;
  CK(cudaMalloc(&Q, qsz * 8));
  CK(cudaMemcpy(Q, hq.data(), qsz * 8, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&vals, (L + 64) * 8));
  CK(cudaMemcpy(vals, hv.data(), L * 8, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&list, (L + 64) * 4));
  CK(cudaMemcpy(list, hl.data(), L * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&y0, m * 8));
  CK(cudaMalloc(&y1, m * 8));
  std::vector<double> a(m), b(m);
  const float t0 = run(k_ring, kRingSmemBytes, nb, Q, m, R, list, vals, L, y0);
  CK(cudaMemcpy(a.data(), y0, m * 8, cudaMemcpyDeviceToHost));
  printf("ring (production)      %7.2f us  %6.2f cycles/col  (|P| = %d, R = %d)\n", t0,
         t0 * 1965.0 / L, L, R);
  auto lane = [&](auto kern, int G, int D, const char* name) {
    const size_t smem = (((size_t)L * 4 + 15) & ~15) + ((L + 1) & ~1) * 8 + (size_t)(D + 1) * G * 32 * 8;
    const float t = run(kern, smem, nb, Q, m, R, list, vals, L, y1);
    CK(cudaMemcpy(b.data(), y1, m * 8, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int i = 0; i < m; ++i) bad += memcmp(&a[i], &b[i], 8) != 0;
    printf("%-22s %7.2f us  %6.2f cycles/col  mismatches %d\n", name, t, t * 1965.0 / L, bad);
  };
  auto pref = [&](auto kern, const char* name) {
    const size_t smem = (((size_t)L * 4 + 15) & ~15) + ((L + 1) & ~1) * 8;
    const float t = run(kern, smem, nb, Q, m, R, list, vals, L, y1);
    CK(cudaMemcpy(b.data(), y1, m * 8, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int i = 0; i < m; ++i) bad += memcmp(&a[i], &b[i], 8) != 0;
    printf("%-22s %7.2f us  %6.2f cycles/col  mismatches %d\n", name, t, t * 1965.0 / L, bad);
  };
  pref(k_pref<256, 4, 0>, "pref D256 P4 m0");
  pref(k_pref<512, 4, 0>, "pref D512 P4 m0");
  pref(k_pref<1024, 4, 0>, "pref D1024 P4 m0");
  pref(k_pref<512, 4, 1>, "pref D512 P4 m1");
  pref(k_pref<1024, 8, 1>, "pref D1024 P8 m1");
  pref(k_pref<0, 0, 0>, "no prefetch m0");
  lane(k_lane<16, 8, 0>, 16, 8, "lane G16 D8 m0");
  lane(k_lane<16, 16, 0>, 16, 16, "lane G16 D16 m0");
  lane(k_lane<16, 24, 0>, 16, 24, "lane G16 D24 m0");
  lane(k_lane<32, 12, 0>, 32, 12, "lane G32 D12 m0");
  lane(k_lane<16, 16, 1>, 16, 16, "lane G16 D16 m1");
  lane(k_lane<16, 24, 1>, 16, 24, "lane G16 D24 m1");
  lane(k_lane<32, 12, 1>, 32, 12, "lane G32 D12 m1");
  lane(k_lane<8, 32, 1>, 8, 32, "lane G8 D32 m1");
  return 0;
}
