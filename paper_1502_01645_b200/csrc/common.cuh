// common.cuh — device helpers shared by the sm_100a kernels.
//
// Exactness rules (SURVEY.md Appendix B rule 12): every reference `s += a*b`
// is __dmul_rn followed by __dadd_rn (never contracted into an FMA; the TUs are
// also built with --fmad=false), every sum is one sequential chain in the
// reference's index order, and no fp64 atomics or tree reductions feed x, g,
// alpha, f or gbs.
#pragma once

#include <cstdint>
#include <mutex>
#include <set>
#include <tuple>
#include <cuda_runtime.h>

namespace alnnls {

constexpr int kMaxThreads = 512;

// cudaFuncSetAttribute once per (kernel, attribute, value, device). Function attributes
// are per device, and one process may drive several devices (one context per
// GPU), so a process-wide "done" flag would leave the second device's launches
// without the shared-memory opt-in. Thread-safe.
inline cudaError_t func_attr_once(const void* func, cudaFuncAttribute attr, int value) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  static std::mutex mu;
  static std::set<std::tuple<const void*, int, int, int>> done;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(func, (int)attr, value, dev);
  if (done.count(key)) return cudaSuccess;
  e = cudaFuncSetAttribute(func, attr, value);
  if (e == cudaSuccess) done.insert(key);
  return e;
}
template <class K>
inline cudaError_t smem_optin(K* kernel, int bytes) {
  return func_attr_once(reinterpret_cast<const void*>(kernel),
                        cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double xdiv(double a, double b) { return __ddiv_rn(a, b); }
// s += a*b in the reference's rounding: rounded product, then rounded sum.
__device__ __forceinline__ double xmac(double s, double a, double b) {
  return __dadd_rn(s, __dmul_rn(a, b));
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_u32(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---- mbarrier + bulk async copy (TMA 1D, sm_90+) ----------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// The retry loop is C++, not a branch inside the asm: a loop hidden in inline
// asm lets lanes leave it at different times with no reconvergence point the
// compiler knows of, and the warp then reaches later warp-synchronous code
// (shuffles, __syncthreads) diverged.
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return done != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// global -> shared bulk copy completing on an mbarrier (UBLKCP in SASS).
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// The same copy with an L2 cache policy (createpolicy): e.g. a fraction of the
// source's lines evict_last, so that part stays in L2 for the next pass.
__device__ __forceinline__ void bulk_g2s_hint(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                              uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;" ::"r"(smem_u32(dst_smem)),
      "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// Bulk prefetch of a global range into L2 (no destination, no completion).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src_gmem, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src_gmem), "r"(bytes) : "memory");
}
// Fraction `frac` of the lines evict_last (the rest evict_first).
__device__ __forceinline__ uint64_t l2_evict_last_fraction(float frac) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_first.b64 %0, %1;"
               : "=l"(pol) : "f"(frac));
  return pol;
}

// ---- block scan (exclusive) of one int per thread -----------------------------
// Returns the exclusive prefix; *total gets the block sum. Uses `scratch`
// (>= 33 ints of shared memory). All threads of the block must call it.
__device__ __forceinline__ int block_exclusive_scan(int v, int* scratch, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) scratch[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int w = lane < nw ? scratch[lane] : 0;
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < nw) scratch[lane] = wi - w;  // exclusive warp offsets
    if (lane == nw - 1) scratch[32] = wi;
  }
  __syncthreads();
  const int res = scratch[wid] + incl - v;
  *total = scratch[32];
  __syncthreads();
  return res;
}

// Sequential sum s = ((0 + p0) + p1) + ... in index order, products already
// rounded. One thread; loads are batched ahead of the dependent DADD chain.
__device__ __forceinline__ double chain_sum_from(double s, const double* __restrict__ p, int len);
__device__ __forceinline__ double chain_sum(const double* __restrict__ p, int len) {
  return chain_sum_from(0.0, p, len);
}
// s = ((s0 + p0) + p1) + ... : continues a chain left by earlier row blocks.
__device__ __forceinline__ double chain_sum_from(double s, const double* __restrict__ p, int len) {
  constexpr int B = 16;
  int t = 0;
  double buf[B];
  for (; t + B <= len; t += B) {
#pragma unroll
    for (int k = 0; k < B; ++k) buf[k] = p[t + k];
#pragma unroll
    for (int k = 0; k < B; ++k) s = xadd(s, buf[k]);
  }
  for (; t < len; ++t) s = xadd(s, p[t]);
  return s;
}

}  // namespace alnnls
