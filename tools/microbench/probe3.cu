// TMA request-rate probes: (a) per-column bulk copies from P producer warps,
// (b) blocked Q layout (each CTA's row block contiguous): dense stage copies
// of G consecutive columns (one request), consumer walks only mask columns.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "common.cuh"
using namespace alnnls;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <int P, int G>
__global__ void __launch_bounds__(512, 1)
    gemv_mp(const double* M, uint64_t ld, int rows, int rpc, const uint32_t* list, const double* vals, int len, double* y) {
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
  if (warp >= cw + 1 && warp < cw + 1 + P) {
    const int pw = warp - cw - 1;
    for (int s = pw; s < nst; s += P) {
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
  } else if (warp >= 1 && warp <= cw) {
    const int t = (warp - 1) * 32 + lane; const int tt = t < nrows ? t : 0;
    double acc = 0.0;
    for (int s = 0; s < nst; ++s) {
      const int st = s % S; const uint32_t ph = (s / S) & 1u;
      const int cnt = min(G, len - s * G);
      mbar_wait(&full[st], ph);
      const double* col = data + st * sd; const double* v = col + G * seg;
      for (int l = 0; l < cnt; ++l) acc = xmac(acc, col[l * seg + tt], v[l]);
      __syncwarp(); if (lane == 0) mbar_arrive(&empty[st]);
    }
    if (t < nrows) y[row0 + t] = acc;
  }
}

// producers: LDG.128 into registers, STS into the stage, warp arrive (no TMA)
template <int P, int G>
__global__ void __launch_bounds__(512, 1)
    gemv_ldsts(const double* M, uint64_t ld, int rows, int rpc, const uint32_t* list, const double* vals, int len, double* y) {
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
  const int chunks = seg / 2;  // 16B chunks per column
  if (warp >= cw + 1 && warp < cw + 1 + P) {
    const int pw = warp - cw - 1;
    for (int s = pw; s < nst; s += P) {
      const int st = s % S; const uint32_t ph = (s / S) & 1u;
      const int base = s * G; const int cnt = min(G, len - base);
      const int tot = cnt * chunks;
      constexpr int MAXC = 64;
      double2 r[MAXC / 2 > 0 ? 32 : 1];
      int nl = 0;
      // up to 32 chunks per lane in flight
      for (int e = lane, k = 0; e < tot && k < 32; e += 32, ++k) {
        const int l = e / chunks, c = e % chunks;
        const uint32_t j = __ldg(list + base + l);
        r[k] = __ldg(reinterpret_cast<const double2*>(M + (size_t)j * ld + row0) + c);
        nl = k + 1;
      }
      if (lane == 0) mbar_wait(&empty[st], ph ^ 1u);
      __syncwarp();
      double* dst = data + st * sd;
      for (int e = lane, k = 0; k < nl; e += 32, ++k) {
        const int l = e / chunks, c = e % chunks;
        if (e < tot) reinterpret_cast<double2*>(dst + (size_t)l * seg)[c] = r[k];
      }
      if (lane < cnt) dst[(size_t)G * seg + lane] = __ldg(vals + base + lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[st]);
    }
  } else if (warp >= 1 && warp <= cw) {
    const int t = (warp - 1) * 32 + lane; const int tt = t < nrows ? t : 0;
    double acc = 0.0;
    for (int s = 0; s < nst; ++s) {
      const int st = s % S; const uint32_t ph = (s / S) & 1u;
      const int cnt = min(G, len - s * G);
      mbar_wait(&full[st], ph);
      const double* col = data + st * sd; const double* v = col + G * seg;
      for (int l = 0; l < cnt; ++l) acc = xmac(acc, col[l * seg + tt], v[l]);
      __syncwarp(); if (lane == 0) mbar_arrive(&empty[st]);
    }
    if (t < nrows) y[row0 + t] = acc;
  }
}

// Blocked layout: block c holds rows [c*R, c*R+R) as R x m col-major (column j at offset j*R).
// Stage = G consecutive columns (dense) in one bulk copy; consumer uses mask sub-lists.
template <int G>
__global__ void __launch_bounds__(512, 1)
    gemv_blocked(const double* Mb, int m, int R, const uint32_t* list, const double* vals, const int* stage_t0, int len, double* y) {
  extern __shared__ __align__(128) uint8_t smem[];
  const size_t stage_b = (size_t)G * R * 8;
  const int S = min(64, (int)((180 * 1024) / stage_b));
  __shared__ uint64_t full[64], empty[64];
  double* data = reinterpret_cast<double*>(smem);
  const double* blk = Mb + (size_t)blockIdx.x * R * m;
  const int cw = (R + 31) / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], cw); } fence_mbar_init(); }
  __syncthreads();
  const int nst = (m + G - 1) / G;
  if (warp == 0) {
    if (lane == 0) {
      int p = 0;
      for (int s = 0; s < nst; ++s) {
        if (stage_t0[s + 1] == stage_t0[s]) continue;  // no mask column in this stage
        const int st = p % S; const uint32_t ph = (p / S) & 1u; ++p;
        const int cols = min(G, m - s * G);
        mbar_wait(&empty[st], ph ^ 1u);
        mbar_arrive_expect_tx(&full[st], (uint32_t)(cols * R * 8));
        bulk_g2s(data + (size_t)st * G * R, blk + (size_t)s * G * R, (uint32_t)(cols * R * 8), &full[st]);
      }
    }
  } else if (warp <= cw) {
    const int t = (warp - 1) * 32 + lane; const int tt = t < R ? t : 0;
    double acc = 0.0;
    int p = 0;
    for (int s = 0; s < nst; ++s) {
      const int a = stage_t0[s], b = stage_t0[s + 1];
      if (a == b) continue;
      const int st = p % S; const uint32_t ph = (p / S) & 1u; ++p;
      mbar_wait(&full[st], ph);
      const double* col = data + (size_t)st * G * R - (size_t)s * G * R;
      for (int q = a; q < b; ++q) { const uint32_t j = __ldg(list + q); acc = xmac(acc, col[(size_t)j * R + tt], __ldg(vals + q)); }
      __syncwarp(); if (lane == 0) mbar_arrive(&empty[st]);
    }
    if (t < R) y[blockIdx.x * R + t] = acc;
  }
}

int main() {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  for (int cfg = 0; cfg < 2; ++cfg) {
    const int m = cfg == 0 ? 4096 : 16384, len = cfg == 0 ? 2900 : 10300;
    const uint64_t ld = (m + 31) / 32 * 32;
    double *Q, *vals, *y; uint32_t* list; int* st0;
    CK(cudaMalloc(&Q, ld * m * 8 + (1 << 20))); CK(cudaMemset(Q, 0, ld * m * 8));
    CK(cudaMalloc(&vals, (len + 64) * 8)); CK(cudaMemset(vals, 0, (len + 64) * 8));
    CK(cudaMalloc(&y, m * 8)); CK(cudaMalloc(&list, (len + 64) * 4)); CK(cudaMalloc(&st0, (m + 2) * 4));
    std::vector<uint32_t> hl; srand(1);
    for (int j = 0; j < m && (int)hl.size() < len; ++j) if (rand() % m < len) hl.push_back(j);
    const int L = hl.size();
    CK(cudaMemcpy(list, hl.data(), L * 4, cudaMemcpyHostToDevice));
    const double bytes = 8.0 * m * L;
    int rpc = (m + 147) / 148; rpc = (rpc + 3) & ~3; const int grid = (m + rpc - 1) / rpc;
    auto run = [&](auto kern, const char* name) {
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 192 * 1024));
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        for (int it = 0; it < 10; ++it) kern<<<grid, 512, 192 * 1024>>>(Q, ld, m, rpc, list, vals, L, y);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
      }
      cudaEventElapsedTime(&ms, e0, e1);
      printf("m=%d |P|=%d %-22s: %.1f us/pass, %.0f GB/s (algorithmic)\n", m, L, name, ms * 1e3 / 10, bytes / (ms * 1e-3 / 10) / 1e9);
    };
    run(gemv_mp<1, 32>, "percol P1 G32");
    run(gemv_mp<2, 32>, "percol P2 G32");
    run(gemv_mp<4, 32>, "percol P4 G32");
    run(gemv_mp<8, 16>, "percol P8 G16");
    run(gemv_mp<8, 32>, "percol P8 G32");
    run(gemv_mp<11, 32>, "percol P11 G32");
    run(gemv_mp<4, 64>, "percol P4 G64");
    run(gemv_mp<8, 64>, "percol P8 G64");
    run(gemv_ldsts<8, 32>, "ldg.128->sts P8 G32");
    run(gemv_ldsts<12, 32>, "ldg.128->sts P12 G32");
    for (int G : std::vector<int>{}) {
      std::vector<int> h0(m / G + 2, 0);
      const int nst = (m + G - 1) / G;
      int q = 0;
      for (int s = 0; s <= nst; ++s) { while (q < L && (int)hl[q] < s * G) ++q; h0[s] = q; }
      CK(cudaMemcpy(st0, h0.data(), (nst + 1) * 4, cudaMemcpyHostToDevice));
      auto kb = G == 16 ? gemv_blocked<16> : G == 32 ? gemv_blocked<32> : gemv_blocked<64>;
      CK(cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, 192 * 1024));
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        for (int it = 0; it < 10; ++it) kb<<<grid, 512, 192 * 1024>>>(Q, m, rpc, list, vals, st0, L, y);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
      }
      cudaEventElapsedTime(&ms, e0, e1);
      printf("m=%d |P|=%d blocked dense G%-3d      : %.1f us/pass, %.0f GB/s (algorithmic), %.0f GB/s (read)\n", m, L, G, ms * 1e3 / 10,
             bytes / (ms * 1e-3 / 10) / 1e9, 8.0 * m * rpc * grid / (ms * 1e-3 / 10) / 1e9);
    }
    cudaFree(Q); cudaFree(vals); cudaFree(y); cudaFree(list); cudaFree(st0);
  }
  return 0;
}
