// Microbenchmarks for the two primitives of the exact NQP loop:
//  (1) sequential DADD chains over products formed in parallel (warp_chain variants)
//  (2) the row-block masked GEMV streaming Q columns (bulk-copy ring vs LDGSTS ring vs LDG)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -I../../paper_1502_01645_b200/csrc
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "probe_util.cuh"
#include "gemv.cuh"

using namespace alnnls;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

// ---------------- chains ----------------
__global__ void chain_warp_shfl(const double* a, const double* b, int len, double* out) {
  if (threadIdx.x >= 32) return;
  const double v = warp_chain(len, [&](int t) { return xmul(a[t], b[t]); });
  if (threadIdx.x == 0) out[0] = v;
}

// shuffle results staged in registers before the adds
__global__ void chain_warp_shfl2(const double* a, const double* b, int len, double* out) {
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  double s = 0.0;
  double nxt = lane < len ? xmul(a[lane], b[lane]) : 0.0;
  for (int base = 0; base < len; base += 32) {
    const double cur = nxt;
    const int tn = base + 32 + lane;
    nxt = tn < len ? xmul(a[tn], b[tn]) : 0.0;
    double v[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = __shfl_sync(0xffffffffu, cur, k);
    const int cnt = min(32, len - base);
    if (cnt == 32) {
#pragma unroll
      for (int k = 0; k < 32; ++k) s = xadd(s, v[k]);
    } else {
      for (int k = 0; k < cnt; ++k) s = xadd(s, v[k]);
    }
  }
  if (lane == 0) out[0] = s;
}

// block forms products into smem chunks (double buffered); thread 0 chains
__global__ void chain_block_smem(const double* a, const double* b, int len, double* out) {
  constexpr int CH = 2048;
  __shared__ double buf[2][CH];
  double s = 0.0;
  const int nch = (len + CH - 1) / CH;
  for (int i = threadIdx.x; i < CH && i < len; i += blockDim.x) buf[0][i] = xmul(a[i], b[i]);
  __syncthreads();
  for (int c = 0; c < nch; ++c) {
    const int cur = c & 1;
    const int base = c * CH;
    const int cnt = min(CH, len - base);
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0) {
        const double* p = buf[cur];
        int t = 0;
        for (; t + 16 <= cnt; t += 16) {
          double v[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) v[k] = p[t + k];
#pragma unroll
          for (int k = 0; k < 16; ++k) s = xadd(s, v[k]);
        }
        for (; t < cnt; ++t) s = xadd(s, p[t]);
      }
    } else {
      const int nb = base + CH;
      for (int i = threadIdx.x - 32; i < CH && nb + i < len; i += blockDim.x - 32)
        buf[cur ^ 1][i] = xmul(a[nb + i], b[nb + i]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = s;
}

// ---------------- GEMV ----------------
__global__ void __launch_bounds__(512, 1)
    gemv_bulk(const double* M, uint64_t ld, int rows, int rpc, const uint32_t* list,
              const double* vals, int len, double* y) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int row0 = blockIdx.x * rpc;
  const int nrows = max(0, min(rows - row0, rpc));
  RowRing ring;
  ring_setup(ring, smem, kRingSmemBytes, nrows, ring_seg(nrows), 12);
  gemv_rows(ring, M + row0, ld, false, row0, nrows, list, vals, len, y);
}

// LDG direct: each consumer thread streams its row's entries with deep register prefetch.
template <int D>
__global__ void __launch_bounds__(512, 1)
    gemv_ldg(const double* M, uint64_t ld, int rows, int rpc, const uint32_t* list,
             const double* vals, int len, double* y) {
  const int row0 = blockIdx.x * rpc;
  const int t = threadIdx.x;
  if (t >= rpc || row0 + t >= rows) return;
  const double* base = M + row0 + t;
  double acc = 0.0;
  double q[D], v[D];
#pragma unroll
  for (int k = 0; k < D; ++k) {
    q[k] = k < len ? __ldg(base + (size_t)__ldg(list + k) * ld) : 0.0;
    v[k] = k < len ? __ldg(vals + k) : 0.0;
  }
  for (int c = 0; c < len; c += D) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const double qk = q[k], vk = v[k];
      const int tn = c + D + k;
      if (tn < len) {
        q[k] = __ldg(base + (size_t)__ldg(list + tn) * ld);
        v[k] = __ldg(vals + tn);
      }
      if (c + k < len) acc = xmac(acc, qk, vk);
    }
  }
  y[row0 + t] = acc;
}

// LDGSTS ring: warps 1..P produce with 16B cp.async, warp 0 consumes (rows <= 32 per CTA)
template <int P>
__global__ void __launch_bounds__(512, 1)
    gemv_ldgsts(const double* M, uint64_t ld, int rows, int rpc, const uint32_t* list,
                const double* vals, int len, double* y) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int G = 32;  // columns per stage
  const int seg = (rpc + 1) & ~1;
  const int stage_d = G * seg + G;
  const int S = min(64, (int)(kRingSmemBytes / 8 / stage_d) - 1);
  double* data = reinterpret_cast<double*>(smem);
  __shared__ uint64_t full[64], empty[64];
  const int row0 = blockIdx.x * rpc;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], P * 32);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int nst = (len + G - 1) / G;
  if (warp >= 1 && warp <= P) {
    const int pt = (warp - 1) * 32 + lane;  // producer thread
    const int chunks = seg / 2;             // 16B chunks per column
    for (int s = (warp - 1); s < nst; s += 0) {
      (void)s;
      break;
    }
    for (int s = 0; s < nst; ++s) {
      const int st = s % S;
      const uint32_t ph = (s / S) & 1u;
      mbar_wait(&empty[st], ph ^ 1u);
      const int base = s * G;
      const int cnt = min(G, len - base);
      double* dst = data + (size_t)st * stage_d;
      for (int e = pt; e < cnt * chunks; e += P * 32) {
        const int l = e / chunks, c = e % chunks;
        const uint32_t j = __ldg(list + base + l);
        const double* src = M + (size_t)j * ld + row0 + 2 * c;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + l * seg + 2 * c)),
                     "l"(src)
                     : "memory");
      }
      if (pt < G / 2 && 2 * pt < cnt) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + G * seg + 2 * pt)),
                     "l"(vals + base + 2 * pt)
                     : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[st]))
                   : "memory");
    }
  } else if (warp == 0) {
    const int t = lane;
    double acc = 0.0;
    for (int s = 0; s < nst; ++s) {
      const int st = s % S;
      const uint32_t ph = (s / S) & 1u;
      mbar_wait(&full[st], ph);
      const double* col = data + (size_t)st * stage_d;
      const double* v = col + G * seg;
      const int cnt = min(G, len - s * G);
      if (t < rpc) {
        if (cnt == G) {
#pragma unroll 8
          for (int l = 0; l < G; ++l) acc = xmac(acc, col[l * seg + t], v[l]);
        } else {
          for (int l = 0; l < cnt; ++l) acc = xmac(acc, col[l * seg + t], v[l]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    if (t < rpc && row0 + t < rows) y[row0 + t] = acc;
  }
}

int main() {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  // chains
  {
    const int len = 3000;
    std::vector<double> h(len);
    for (int i = 0; i < len; ++i) h[i] = 1.0 + 1e-3 * i;
    double *a, *out;
    CK(cudaMalloc(&a, len * 8));
    CK(cudaMalloc(&out, 8));
    CK(cudaMemcpy(a, h.data(), len * 8, cudaMemcpyHostToDevice));
    for (int v = 0; v < 3; ++v) {
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        for (int it = 0; it < 20; ++it) {
          if (v == 0) chain_warp_shfl<<<1, 32>>>(a, a, len, out);
          if (v == 1) chain_warp_shfl2<<<1, 32>>>(a, a, len, out);
          if (v == 2) chain_block_smem<<<1, 512>>>(a, a, len, out);
        }
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
      }
      cudaEventElapsedTime(&ms, e0, e1);
      printf("chain variant %d: %.2f ns/element (len %d, incl. launch)\n", v, ms * 1e6 / 20 / len, len);
    }
  }
  // gemv
  for (int cfg = 0; cfg < 2; ++cfg) {
    const int m = cfg == 0 ? 4096 : 16384;
    const int len = cfg == 0 ? 3000 : 10000;
    const uint64_t ld = (m + 31) / 32 * 32;
    double *Q, *vals, *y;
    uint32_t* list;
    CK(cudaMalloc(&Q, ld * m * 8));
    CK(cudaMemset(Q, 0, ld * m * 8));
    CK(cudaMalloc(&vals, (len + 64) * 8));
    CK(cudaMemset(vals, 0, (len + 64) * 8));
    CK(cudaMalloc(&y, m * 8));
    CK(cudaMalloc(&list, (len + 64) * 4));
    std::vector<uint32_t> hl(len);
    srand(1);
    int j = 0;
    for (int t = 0; t < len; ++t) {
      j += 1 + (rand() % 100 < (100LL * (m - len) / len) ? 1 : 0);
      hl[t] = (uint32_t)std::min(j, m - 1);
    }
    CK(cudaMemcpy(list, hl.data(), len * 4, cudaMemcpyHostToDevice));
    const double bytes = 8.0 * m * len;
    int rpc = (m + 147) / 148;
    rpc = (rpc + 3) & ~3;
    const int grid = (m + rpc - 1) / rpc;
    CK(cudaFuncSetAttribute(gemv_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRingSmemBytes));
    CK(cudaFuncSetAttribute(gemv_ldgsts<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRingSmemBytes));
    CK(cudaFuncSetAttribute(gemv_ldgsts<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRingSmemBytes));
    for (int v = 0; v < 5; ++v) {
      if ((v == 3 || v == 4) && rpc > 32) continue;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        for (int it = 0; it < 10; ++it) {
          if (v == 0) gemv_bulk<<<grid, 512, kRingSmemBytes>>>(Q, ld, m, rpc, list, vals, len, y);
          if (v == 1) gemv_ldg<16><<<grid, 512>>>(Q, ld, m, rpc, list, vals, len, y);
          if (v == 2) gemv_ldg<48><<<grid, 512>>>(Q, ld, m, rpc, list, vals, len, y);
          if (v == 3) gemv_ldgsts<4><<<grid, 512, kRingSmemBytes>>>(Q, ld, m, rpc, list, vals, len, y);
          if (v == 4) gemv_ldgsts<8><<<grid, 512, kRingSmemBytes>>>(Q, ld, m, rpc, list, vals, len, y);
        }
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
      }
      cudaEventElapsedTime(&ms, e0, e1);
      const char* names[] = {"bulk ring", "ldg D16", "ldg D48", "ldgsts P4", "ldgsts P8"};
      printf("gemv m=%d len=%d rpc=%d %-10s: %.1f us/pass, %.0f GB/s\n", m, len, rpc, names[v],
             ms * 1e3 / 10, bytes / (ms * 1e-3 / 10) / 1e9);
    }
    cudaFree(Q);
    cudaFree(vals);
    cudaFree(y);
    cudaFree(list);
  }
  return 0;
}
