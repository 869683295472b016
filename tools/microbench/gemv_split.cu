// Which side limits the exact row GEMV at c2 shape? Producer-only / consumer-only variants.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "common.cuh"
using namespace alnnls;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

// MODE 0: full; 1: consumer skips MACs; 2: producer skips copies (arrive only); 3: consumer pipelined
template <int MODE>
__global__ void __launch_bounds__(384, 1) k(const double* Qb, int m, int R, const uint32_t* list, const double* vals, int len, double* y, int G, int P) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[48], empty[48], mfull[48];
  const int row0 = blockIdx.x * R;
  const int nrows = max(0, min(m - row0, R));
  const double* base = Qb + (size_t)blockIdx.x * R * m;
  const int seg = R;
  const int S = min(48, (int)((190 * 1024) / ((size_t)G * seg * 8 + G * 8)));
  double* data = reinterpret_cast<double*>(smem);
  double* vb = data + (size_t)S * G * seg;
  const int cw = (nrows + 31) / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) { mbar_init(&full[s], MODE == 7 ? 32 : 1); mbar_init(&empty[s], cw); mbar_init(&mfull[s], 12 - P - cw); } fence_mbar_init(); }
  __syncthreads();
  const int nst = (len + G - 1) / G;
  if (MODE == 7 && warp < P) {
    // cp.async 16B producers on the blocked layout; one warp per stage; completion via
    // cp.async.mbarrier.arrive.noinc (full barrier count = 32 lanes x producing warps)
    const int ch = seg / 2;
    for (int s = warp; s < nst; s += P) {
      const int st = s % S; const uint32_t ph = (s / S) & 1u;
      const int sbase = s * G; const int cnt = min(G, len - sbase);
      uint32_t j0 = lane < cnt ? __ldg(list + sbase + lane) : 0u;
      uint32_t j1 = lane + 32 < cnt ? __ldg(list + sbase + lane + 32) : 0u;
      if (lane == 0) mbar_wait(&empty[st], ph ^ 1u);
      __syncwarp();
      double* dst = data + (size_t)st * G * seg;
      const int tot = cnt * ch;
      for (int e = lane; e < tot; e += 32) {
        const int l = e / ch, c = e - l * ch;
        const uint32_t jv = __shfl_sync(0xffffffffu, l < 32 ? j0 : j1, l & 31);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + (size_t)l * seg + 2 * c)),
                     "l"(base + (size_t)jv * seg + 2 * c) : "memory");
      }
      if (lane < cnt) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(vb + (size_t)st * G + lane)), "l"(vals + sbase + lane) : "memory");
      if (lane + 32 < cnt) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(vb + (size_t)st * G + lane + 32)), "l"(vals + sbase + lane + 32) : "memory");
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[st])) : "memory");
    }
  } else if (MODE == 6 && warp < P) {
    const int ch = seg / 2;  // 16B chunks per column
    for (int s = warp; s < nst; s += P) {
      const int st = s % S; const uint32_t ph = (s / S) & 1u;
      const int sbase = s * G; const int cnt = min(G, len - sbase);
      const int tot = cnt * ch;
      double* dst = data + (size_t)st * G * seg;
      if (lane == 0) mbar_wait(&empty[st], ph ^ 1u);
      __syncwarp();
      for (int e0 = 0; e0 < tot; e0 += 32 * 14) {
        double2 r[14];
#pragma unroll
        for (int k = 0; k < 14; ++k) {
          const int e = e0 + k * 32 + lane;
          if (e < tot) {
            const int l = e / ch, c = e - l * ch;
            const uint32_t j = __ldcg(list + sbase + l);
            r[k] = __ldcg(reinterpret_cast<const double2*>(base + (size_t)j * seg) + c);
          }
        }
#pragma unroll
        for (int k = 0; k < 14; ++k) {
          const int e = e0 + k * 32 + lane;
          if (e < tot) {
            const int l = e / ch, c = e - l * ch;
            reinterpret_cast<double2*>(dst + (size_t)l * seg)[c] = r[k];
          }
        }
      }
      for (int l = lane; l < cnt; l += 32) vb[(size_t)st * G + l] = __ldcg(vals + sbase + l);
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[st]);
    }
  } else if (warp < P) {
    for (int s = warp; s < nst; s += P) {
      const int st = s % S; const uint32_t ph = (s / S) & 1u;
      const int sbase = s * G; const int cnt = min(G, len - sbase);
      if (lane == 0) { mbar_wait(&empty[st], ph ^ 1u); if (MODE == 2 || MODE == 8 || MODE == 10) mbar_arrive(&full[st]); else mbar_arrive_expect_tx(&full[st], (uint32_t)(cnt * seg * 8 + ((cnt + 1) & ~1) * 8)); }
      __syncwarp();
      if (MODE == 2 || MODE == 8 || MODE == 10) continue;
      double* dst = data + (size_t)st * G * seg;
      for (int l0 = 0; l0 < cnt; l0 += 32) {
        const int l = l0 + lane; const bool valid = l < cnt;
        const uint32_t j = valid ? __ldcg(list + sbase + l) : 0u;
        const uint32_t jp = __shfl_up_sync(0xffffffffu, j, 1);
        const bool start = valid && (lane == 0 || j != jp + 1u);
        const uint32_t starts = __ballot_sync(0xffffffffu, start);
        if (start) {
          const uint32_t later = starts & ~((2u << lane) - 1u);
          int end = later ? __ffs(later) - 1 : 32; end = min(end, cnt - l0);
          bulk_g2s(dst + (size_t)l * seg, base + (size_t)j * seg, (uint32_t)((end - lane) * seg * 8), &full[st]);
        }
      }
      if (lane == 0) bulk_g2s(vb + (size_t)st * G, vals + sbase, (uint32_t)(((cnt + 1) & ~1) * 8), &full[st]);
    }
  } else if (MODE == 4 && warp >= P + cw) {
    // multiplier warps: products in place, then arrive on mfull
    const int nm = 12 - P - cw;
    const int mt = (warp - P - cw) * 32 + lane;
    for (int s = 0; s < nst; ++s) {
      const int st = s % S; const uint32_t ph = (s / S) & 1u;
      const int cnt = min(G, len - s * G);
      mbar_wait(&full[st], ph);
      double* col = data + (size_t)st * G * seg; const double* v = vb + (size_t)st * G;
      for (int e = mt; e < cnt * seg; e += nm * 32) { const int l = e / seg; col[e] = xmul(col[e], v[l]); }
      __syncwarp(); if (lane == 0) mbar_arrive(&mfull[st]);
    }
  } else if (warp < P + cw) {
    const int t = (warp - P) * 32 + lane; const int tt = t < nrows ? t : 0;
    double acc = 0.0;
    for (int s = 0; s < nst; ++s) {
      const int st = s % S; const uint32_t ph = (s / S) & 1u;
      const int cnt = min(G, len - s * G);
      if (MODE == 4) {
        mbar_wait(&mfull[st], ph);
        const double* p = data + (size_t)st * G * seg + tt;
        if (cnt == G) {
          double cur[16], nx[16];
#pragma unroll
          for (int l = 0; l < 16; ++l) cur[l] = p[l * seg];
          for (int l0 = 0; l0 < G; l0 += 16) {
            if (l0 + 16 < G) {
#pragma unroll
              for (int l = 0; l < 16; ++l) nx[l] = p[(l0 + 16 + l) * seg];
            }
#pragma unroll
            for (int l = 0; l < 16; ++l) acc = xadd(acc, cur[l]);
#pragma unroll
            for (int l = 0; l < 16; ++l) cur[l] = nx[l];
          }
        } else {
          for (int l = 0; l < cnt; ++l) acc = xadd(acc, p[l * seg]);
        }
        __syncwarp(); if (lane == 0) mbar_arrive(&empty[st]);
        continue;
      }
      mbar_wait(&full[st], ph);
      const double* col = data + (size_t)st * G * seg; const double* v = vb + (size_t)st * G;
      if (MODE != 1) {
        if ((MODE == 9 || MODE == 10) && cnt == 64) {
          // pinned-order shared loads: all 64 issued before any product/add
          const uint32_t cbase = smem_u32(col + tt), vbase = smem_u32(v);
          double c[64], w[64];
#pragma unroll
          for (int l = 0; l < 64; ++l)
            asm volatile("ld.shared.f64 %0, [%1];" : "=d"(c[l]) : "r"(cbase + (uint32_t)(l * seg * 8)));
#pragma unroll
          for (int l = 0; l < 64; l += 2)
            asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(w[l]), "=d"(w[l + 1]) : "r"(vbase + (uint32_t)(l * 8)));
#pragma unroll
          for (int l = 0; l < 64; ++l) acc = xadd(acc, xmul(c[l], w[l]));
        } else if ((MODE == 5 || MODE == 6 || MODE == 7 || MODE == 8) && cnt == 64) {
          double p[64];
#pragma unroll
          for (int l = 0; l < 64; ++l) p[l] = xmul(col[l * seg + tt], v[l]);
#pragma unroll
          for (int l = 0; l < 64; ++l) acc = xadd(acc, p[l]);
        } else if (MODE == 3 && cnt == G) {
          double pc[8], pn[8];
#pragma unroll
          for (int l = 0; l < 8; ++l) pc[l] = xmul(col[l * seg + tt], v[l]);
          for (int l0 = 0; l0 < G; l0 += 8) {
            if (l0 + 8 < G) {
#pragma unroll
              for (int l = 0; l < 8; ++l) pn[l] = xmul(col[(l0 + 8 + l) * seg + tt], v[l0 + 8 + l]);
            }
#pragma unroll
            for (int l = 0; l < 8; ++l) acc = xadd(acc, pc[l]);
#pragma unroll
            for (int l = 0; l < 8; ++l) pc[l] = pn[l];
          }
        } else {
          for (int l0 = 0; l0 < cnt; l0 += 8) {
#pragma unroll
            for (int l = 0; l < 8; ++l) if (l0 + l < cnt) acc = xmac(acc, col[(l0 + l) * seg + tt], v[l0 + l]);
          }
        }
      }
      __syncwarp(); if (lane == 0) mbar_arrive(&empty[st]);
    }
    if (t < nrows) y[row0 + t] = acc;
  }
}

int main(int argc, char** argv) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  const int m = 4096; const double dens = argc > 1 ? atof(argv[1]) : 0.71;
  int R = (m + 146) / 147; R = (R + 3) & ~3; const int nb = (m + R - 1) / R;
  double *Q, *vals, *y; uint32_t* list;
  CK(cudaMalloc(&Q, (size_t)nb * R * m * 8)); CK(cudaMemset(Q, 0, (size_t)nb * R * m * 8));
  CK(cudaMalloc(&vals, (m + 64) * 8)); CK(cudaMemset(vals, 0, (m + 64) * 8));
  CK(cudaMalloc(&y, m * 8)); CK(cudaMalloc(&list, (m + 64) * 4));
  std::vector<uint32_t> hl; srand(7);
  for (int j = 0; j < m; ++j) if ((rand() % 1000) < dens * 1000) hl.push_back(j);
  const int L = hl.size();
  CK(cudaMemcpy(list, hl.data(), L * 4, cudaMemcpyHostToDevice));
  auto run = [&](auto kern, const char* name, int G, int P) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 192 * 1024));
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      for (int it = 0; it < 20; ++it) kern<<<nb, 384, 192 * 1024>>>(Q, m, R, list, vals, L, y, G, P);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-22s G=%2d P=%d: %6.1f us/pass (|P|=%d, chain floor %.1f us)\n", name, G, P, ms * 1e3 / 20, L, L * 8 / 1.9e3);
  };
  for (int G : {64}) for (int P : {1, 2, 3, 4}) {
    run(k<5>, "stage in regs", G, P);
    run(k<8>, "consumer only (regs)", G, P);
  }
  run(k<1>, "no MACs", 64, 4);
  run(k<10>, "consumer only (pinned)", 64, 4);
  run(k<9>, "full pinned", 64, 4);
  return 0;
}
