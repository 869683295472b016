// FP64 microbenchmarks that set the ceilings for the exact and fast profiles:
//  1. dependent DADD chain latency (the den/df/gbs chains and the per-row GEMV chains)
//  2. SIMT throughput of DMUL+DADD pairs (exact profile) and DFMA (fast SIMT)
//  3. DMMA mma.sync f64 throughput (m8n8k4, m16n8k4, m16n8k8, m16n8k16)
//  4. grid-wide barrier cost (cooperative grid.sync and a hand-rolled atomic barrier)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void chain_latency(const double* in, double* out, long long* cyc, int n) {
  double s = 0.0;
  double a = in[0], b = in[1];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    s = __dadd_rn(s, a);
    s = __dadd_rn(s, b);
    s = __dadd_rn(s, a);
    s = __dadd_rn(s, b);
  }
  long long t1 = clock64();
  out[0] = s;
  cyc[0] = t1 - t0;
}

// chain where products come from smem (like the den chain over staged products)
__global__ void chain_smem(const double* in, double* out, long long* cyc, int n) {
  __shared__ double p[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) p[i] = in[i & 1023];
  __syncthreads();
  if (threadIdx.x != 0) return;
  double s = 0.0;
  long long t0 = clock64();
  for (int r = 0; r < n / 4096 + 1; ++r) {
#pragma unroll 16
    for (int i = 0; i < 4096; ++i) s = __dadd_rn(s, p[i]);
  }
  long long t1 = clock64();
  out[0] = s;
  cyc[0] = t1 - t0;
}

template <int MODE>
__global__ void fp64_tput(const double* in, double* out, int n) {
  double a[8], s[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) { a[k] = in[(threadIdx.x + k) & 1023]; s[k] = 0.0; }
  double b = in[5];
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (MODE == 0) s[k] = __dadd_rn(s[k], __dmul_rn(a[k], b));
      else s[k] = __fma_rn(a[k], b, s[k]);
    }
  }
  double t = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) t += s[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

template <int SHAPE>
__global__ void dmma_tput(const double* in, double* out, int n) {
  double acc[4] = {0, 0, 0, 0};
  double a[4], b[2];
#pragma unroll
  for (int k = 0; k < 4; ++k) a[k] = in[(threadIdx.x * 4 + k) & 1023];
  b[0] = in[threadIdx.x & 1023];
  b[1] = in[(threadIdx.x + 7) & 1023];
  for (int i = 0; i < n; ++i) {
    if (SHAPE == 0) {  // m8n8k4: a 1, b 1, c/d 2
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[0]), "+d"(acc[1]) : "d"(a[0]), "d"(b[0]));
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[2]), "+d"(acc[3]) : "d"(a[1]), "d"(b[1]));
    } else if (SHAPE == 1) {  // m16n8k4: a 2, b 1, c/d 4
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(acc[0]), "+d"(acc[1]), "+d"(acc[2]), "+d"(acc[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
    } else if (SHAPE == 2) {  // m16n8k8: a 4, b 2
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(acc[0]), "+d"(acc[1]), "+d"(acc[2]), "+d"(acc[3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc[0] + acc[1] + acc[2] + acc[3];
}

__global__ void coop_barrier(int iters, double* out) {
  cg::grid_group g = cg::this_grid();
  double s = 0;
  for (int i = 0; i < iters; ++i) {
    s += 1.0;
    g.sync();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = s;
}

__device__ unsigned int g_bar_count;
__device__ volatile unsigned int g_bar_gen;

__device__ __forceinline__ void my_grid_sync(unsigned int nblocks, unsigned int& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int want = gen + 1;
    __threadfence();
    unsigned int arrived = atomicAdd(&g_bar_count, 1);
    if (arrived == nblocks - 1) {
      g_bar_count = 0;
      __threadfence();
      atomicExch((unsigned int*)&g_bar_gen, want);
    } else {
      while (true) {
        unsigned int v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&g_bar_gen));
        if (v == want) break;
      }
    }
    gen = want;
  }
  __syncthreads();
}

__global__ void atomic_barrier(int iters, double* out) {
  unsigned int gen = 0;
  if (threadIdx.x == 0) gen = g_bar_gen;
  double s = 0;
  for (int i = 0; i < iters; ++i) {
    s += 1.0;
    my_grid_sync(gridDim.x, gen);
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = s;
}

int main() {
  int dev = 0;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  printf("device %s SMs %d L2 %d MB clock %d kHz\n", prop.name, prop.multiProcessorCount,
         prop.l2CacheSize >> 20, prop.clockRate);
  const int nsm = prop.multiProcessorCount;
  double *d_in, *d_out;
  long long* d_cyc;
  CK(cudaMalloc(&d_in, 1024 * sizeof(double)));
  CK(cudaMalloc(&d_out, 1 << 24));
  CK(cudaMalloc(&d_cyc, sizeof(long long)));
  double h_in[1024];
  for (int i = 0; i < 1024; ++i) h_in[i] = 1.0 + i * 1e-3;
  CK(cudaMemcpy(d_in, h_in, sizeof(h_in), cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;

  // 1. chain latency
  {
    int n = 1 << 16;
    chain_latency<<<1, 1>>>(d_in, d_out, d_cyc, n);
    CK(cudaDeviceSynchronize());
    chain_latency<<<1, 1>>>(d_in, d_out, d_cyc, n);
    CK(cudaDeviceSynchronize());
    long long cyc;
    CK(cudaMemcpy(&cyc, d_cyc, 8, cudaMemcpyDeviceToHost));
    printf("DADD dependent latency: %.2f cycles/add\n", (double)cyc / (4.0 * n));
    chain_smem<<<1, 256>>>(d_in, d_out, d_cyc, 1 << 16);
    CK(cudaDeviceSynchronize());
    chain_smem<<<1, 256>>>(d_in, d_out, d_cyc, 1 << 16);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(&cyc, d_cyc, 8, cudaMemcpyDeviceToHost));
    int reps = (1 << 16) / 4096 + 1;
    printf("DADD chain over smem operands: %.2f cycles/add\n", (double)cyc / (4096.0 * reps));
    cudaEventRecord(e0);
    chain_latency<<<1, 1>>>(d_in, d_out, d_cyc, n);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DADD chain wall: %.3f ns/add\n", ms * 1e6 / (4.0 * n));
  }
  // 2. SIMT throughput
  {
    int n = 4096;
    int blocks = nsm * 8, threads = 256;
    for (int mode = 0; mode < 2; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (mode == 0) fp64_tput<0><<<blocks, threads>>>(d_in, d_out, n);
        else fp64_tput<1><<<blocks, threads>>>(d_in, d_out, n);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
      }
      cudaEventElapsedTime(&ms, e0, e1);
      double prods = (double)blocks * threads * n * 8;
      printf("%s: %.2f Gproducts/s = %.2f TFLOP/s (2 flop/product)\n",
             mode == 0 ? "DMUL+DADD" : "DFMA", prods / ms / 1e6, 2 * prods / ms / 1e9);
    }
  }
  // 3. DMMA throughput
  {
    int n = 4096;
    int blocks = nsm * 8, threads = 256;
    const char* names[3] = {"m8n8k4", "m16n8k4", "m16n8k8"};
    double flops_per_warp_iter[3] = {2.0 * 2 * 8 * 8 * 4, 2.0 * 16 * 8 * 4, 2.0 * 16 * 8 * 8};
    for (int s = 0; s < 3; ++s) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (s == 0) dmma_tput<0><<<blocks, threads>>>(d_in, d_out, n);
        if (s == 1) dmma_tput<1><<<blocks, threads>>>(d_in, d_out, n);
        if (s == 2) dmma_tput<2><<<blocks, threads>>>(d_in, d_out, n);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
      }
      cudaError_t err = cudaGetLastError();
      cudaEventElapsedTime(&ms, e0, e1);
      double fl = (double)blocks * (threads / 32) * n * flops_per_warp_iter[s];
      printf("DMMA %s: %.2f TFLOP/s (%s)\n", names[s], fl / ms / 1e9, cudaGetErrorString(err));
    }
  }
  // 4. barriers
  {
    int iters = 2000;
    int threads = 256;
    void* args[] = {&iters, &d_out};
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      CK(cudaLaunchCooperativeKernel((void*)coop_barrier, nsm, threads, args, 0, 0));
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("cg grid.sync (%d CTAs): %.3f us/barrier\n", nsm, ms * 1e3 / iters);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      CK(cudaLaunchCooperativeKernel((void*)atomic_barrier, nsm, threads, args, 0, 0));
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("atomic grid barrier (%d CTAs): %.3f us/barrier\n", nsm, ms * 1e3 / iters);
  }
  printf("done\n");
  return 0;
}
