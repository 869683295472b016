// Consumer-side variants for the exact row GEMV and warp-local smem chains.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "probe_util.cuh"
using namespace alnnls;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}

// warp-local smem chain: lanes form products for round r+1 while all lanes chain round r
template <class F>
__device__ double warp_chain_smem(double* wbuf /*64 doubles*/, int len, F prod) {
  const int lane = threadIdx.x & 31;
  double nxt[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) { const int t = r * 32 + lane; nxt[r] = t < len ? prod(t) : 0.0; }
  wbuf[lane] = nxt[0];
  __syncwarp();
  double s = 0.0;
  int slot = 0;
  for (int base = 0; base < len; base += 32) {
    // rotate prefetch registers
    const double n1 = nxt[1];
    nxt[0] = nxt[1]; nxt[1] = nxt[2]; nxt[2] = nxt[3];
    { const int t = base + 128 + lane; nxt[3] = t < len ? prod(t) : 0.0; }
    wbuf[(slot ^ 1) * 32 + lane] = n1;
    const double* p = wbuf + slot * 32;
    const int cnt = min(32, len - base);
    if (cnt == 32) {
      double v[32];
#pragma unroll
      for (int k = 0; k < 32; k += 2) { const double2 d2 = *reinterpret_cast<const double2*>(p + k); v[k] = d2.x; v[k + 1] = d2.y; }
#pragma unroll
      for (int k = 0; k < 32; ++k) s = xadd(s, v[k]);
    } else {
      for (int k = 0; k < cnt; ++k) s = xadd(s, p[k]);
    }
    __syncwarp();
    slot ^= 1;
  }
  return s;
}

__global__ void chain_ws(const double* a, const double* b, int len, double* out) {
  __shared__ __align__(16) double wbuf[64];
  if (threadIdx.x >= 32) return;
  const double v = warp_chain_smem(wbuf, len, [&](int t) { return xmul(a[t], b[t]); });
  if (threadIdx.x == 0) out[0] = v;
}

// thread-0 chain over a block-filled smem array with double-buffered register prefetch
__global__ void chain_block2(const double* a, const double* b, int len, double* out) {
  extern __shared__ __align__(16) double pbuf[];
  for (int i = threadIdx.x; i < len; i += blockDim.x) pbuf[i] = xmul(a[i], b[i]);
  __syncthreads();
  if (threadIdx.x != 0) return;
  double s = 0.0;
  constexpr int B = 16;
  double cur[B], nx[B];
  int t = 0;
#pragma unroll
  for (int k = 0; k < B; k += 2) { double2 d = *reinterpret_cast<const double2*>(pbuf + k); cur[k] = d.x; cur[k+1] = d.y; }
  for (; t + 2 * B <= len; t += B) {
#pragma unroll
    for (int k = 0; k < B; k += 2) { double2 d = *reinterpret_cast<const double2*>(pbuf + t + B + k); nx[k] = d.x; nx[k+1] = d.y; }
#pragma unroll
    for (int k = 0; k < B; ++k) s = xadd(s, cur[k]);
#pragma unroll
    for (int k = 0; k < B; ++k) cur[k] = nx[k];
  }
  for (int k = 0; k < B && t + k < len; ++k) s = xadd(s, cur[k]);
  for (t += B; t < len; ++t) s = xadd(s, pbuf[t]);
  out[0] = s;
}

// GEMV with bulk-copy ring; consumer variants: 0 = simple, 1 = register pipelined + early test_wait
template <int VAR, int G>
__global__ void __launch_bounds__(512, 1)
    gemv_v(const double* M, uint64_t ld, int rows, int rpc, const uint32_t* list, const double* vals, int len, double* y) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int seg = (rpc + 1) & ~1;
  const size_t stage_b = (size_t)G * seg * 8 + G * 8;
  const int S = min(64, (int)((190 * 1024) / stage_b));
  __shared__ uint64_t full[64], empty[64];
  double* data = reinterpret_cast<double*>(smem);
  const int row0 = blockIdx.x * rpc;
  const int nrows = max(0, min(rows - row0, rpc));
  const int cw = (nrows + 31) / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], cw); } fence_mbar_init(); }
  __syncthreads();
  const int nst = (len + G - 1) / G;
  const size_t sd = stage_b / 8;
  if (warp == 0) {
    for (int s = 0; s < nst; ++s) {
      const int st = s % S; const uint32_t ph = (s / S) & 1u;
      const int base = s * G; const int cnt = min(G, len - base);
      if (lane == 0) { mbar_wait(&empty[st], ph ^ 1u); mbar_arrive_expect_tx(&full[st], (uint32_t)(cnt * seg * 8 + ((cnt + 1) & ~1) * 8)); }
      __syncwarp();
      double* dst = data + st * sd;
      for (int l = lane; l < cnt; l += 32) {
        const uint32_t j = __ldg(list + base + l);
        bulk_g2s(dst + (size_t)l * seg, M + (size_t)j * ld + row0, (uint32_t)seg * 8, &full[st]);
      }
      if (lane == 0) bulk_g2s(dst + (size_t)G * seg, vals + base, (uint32_t)(((cnt + 1) & ~1) * 8), &full[st]);
    }
  } else if (warp <= cw) {
    const int t = (warp - 1) * 32 + lane;
    const int tt = t < nrows ? t : 0;
    double acc = 0.0;
    if (VAR == 0) {
      for (int s = 0; s < nst; ++s) {
        const int st = s % S; const uint32_t ph = (s / S) & 1u;
        const int cnt = min(G, len - s * G);
        mbar_wait(&full[st], ph);
        const double* col = data + st * sd; const double* v = col + G * seg;
        for (int l = 0; l < cnt; ++l) acc = xmac(acc, col[l * seg + tt], v[l]);
        __syncwarp(); if (lane == 0) mbar_arrive(&empty[st]);
      }
    } else {
      for (int s = 0; s < nst; ++s) {
        const int st = s % S; const uint32_t ph = (s / S) & 1u;
        const int cnt = min(G, len - s * G);
        mbar_wait(&full[st], ph);
        const double* col = data + st * sd; const double* v = col + G * seg;
        if (cnt == G) {
          double c0[8], w0[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) c0[k] = col[k * seg + tt];
#pragma unroll
          for (int k = 0; k < 8; k += 2) { double2 d = *reinterpret_cast<const double2*>(v + k); w0[k] = d.x; w0[k+1] = d.y; }
#pragma unroll
          for (int g = 0; g < G / 8; ++g) {
            double c1[8], w1[8];
            if (g + 1 < G / 8) {
#pragma unroll
              for (int k = 0; k < 8; ++k) c1[k] = col[((g + 1) * 8 + k) * seg + tt];
#pragma unroll
              for (int k = 0; k < 8; k += 2) { double2 d = *reinterpret_cast<const double2*>(v + (g + 1) * 8 + k); w1[k] = d.x; w1[k+1] = d.y; }
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) acc = xmac(acc, c0[k], w0[k]);
            if (g + 1 < G / 8) {
#pragma unroll
              for (int k = 0; k < 8; ++k) { c0[k] = c1[k]; w0[k] = w1[k]; }
            }
          }
        } else {
          for (int l = 0; l < cnt; ++l) acc = xmac(acc, col[l * seg + tt], v[l]);
        }
        __syncwarp(); if (lane == 0) mbar_arrive(&empty[st]);
      }
    }
    if (t < nrows) y[row0 + t] = acc;
  }
}

int main() {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  {
    const int len = 3000;
    std::vector<double> h(len); for (int i = 0; i < len; ++i) h[i] = 1.0 + 1e-3 * i;
    double *a, *out; CK(cudaMalloc(&a, len * 8)); CK(cudaMalloc(&out, 8));
    CK(cudaMemcpy(a, h.data(), len * 8, cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(chain_block2, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000));
    for (int v = 0; v < 3; ++v) {
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        for (int it = 0; it < 20; ++it) {
          if (v == 0) chain_ws<<<1, 32>>>(a, a, len, out);
          if (v == 1) chain_block2<<<1, 512, len * 8>>>(a, a, len, out);
          if (v == 2) chain_ws<<<1, 32>>>(a, a, 32, out);
        }
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      }
      cudaEventElapsedTime(&ms, e0, e1);
      printf("chain %s: %.2f us per call (len %d)\n", v == 0 ? "warp-smem" : v == 1 ? "block-smem2" : "empty-ish", ms * 1e3 / 20, v == 2 ? 32 : len);
    }
  }
  for (int cfg = 0; cfg < 2; ++cfg) {
    const int m = cfg == 0 ? 4096 : 16384, len = cfg == 0 ? 3000 : 10000;
    const uint64_t ld = (m + 31) / 32 * 32;
    double *Q, *vals, *y; uint32_t* list;
    CK(cudaMalloc(&Q, ld * m * 8)); CK(cudaMemset(Q, 0, ld * m * 8));
    CK(cudaMalloc(&vals, (len + 64) * 8)); CK(cudaMemset(vals, 0, (len + 64) * 8));
    CK(cudaMalloc(&y, m * 8)); CK(cudaMalloc(&list, (len + 64) * 4));
    std::vector<uint32_t> hl(len); srand(1); int j = 0;
    for (int t = 0; t < len; ++t) { j += 1 + (rand() % 100 < (100LL * (m - len) / len) ? 1 : 0); hl[t] = (uint32_t)std::min(j, m - 1); }
    CK(cudaMemcpy(list, hl.data(), len * 4, cudaMemcpyHostToDevice));
    const double bytes = 8.0 * m * len;
    int rpc = (m + 147) / 148; rpc = (rpc + 3) & ~3; const int grid = (m + rpc - 1) / rpc;
    auto run = [&](auto kern, const char* name) {
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 192 * 1024));
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        for (int it = 0; it < 10; ++it) kern<<<grid, 512, 192 * 1024>>>(Q, ld, m, rpc, list, vals, len, y);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
      }
      cudaEventElapsedTime(&ms, e0, e1);
      printf("gemv m=%d len=%d %-16s: %.1f us/pass, %.0f GB/s\n", m, len, name, ms * 1e3 / 10, bytes / (ms * 1e-3 / 10) / 1e9);
    };
    run(gemv_v<0, 32>, "simple G32");
    run(gemv_v<1, 32>, "pipelined G32");
    run(gemv_v<1, 64>, "pipelined G64");
    run(gemv_v<1, 16>, "pipelined G16");
    cudaFree(Q); cudaFree(vals); cudaFree(y); cudaFree(list);
  }
  return 0;
}
