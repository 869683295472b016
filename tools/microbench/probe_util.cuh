// Helpers used only by the microbenchmarks (not by the product kernels).
#pragma once
#include "common.cuh"

namespace alnnls {

// Warp-cooperative sequential chain: s = ((0 + p(0)) + p(1)) + ... + p(len-1).
// Lanes compute the products of a 32-element round in parallel (rounded
// exactly like the reference, inside `prod`), then every lane runs the same
// dependent DADD chain over the round via shuffles, so only the adds are
// serial (8-cycle DADD latency per element on B200). Rounds are prefetched
// kDepth ahead to hide L2 latency. Must be called by all 32 lanes of a warp;
// the result is returned in every lane.
template <int kDepth = 4, class F>
__device__ __forceinline__ double warp_chain(int len, F prod) {
  const int lane = threadIdx.x & 31;
  double p[kDepth];
#pragma unroll
  for (int r = 0; r < kDepth; ++r) {
    const int t = r * 32 + lane;
    p[r] = t < len ? prod(t) : 0.0;
  }
  double s = 0.0;
  for (int base = 0; base < len; base += 32 * kDepth) {
#pragma unroll
    for (int r = 0; r < kDepth; ++r) {
      const int rb = base + r * 32;
      const double cur = p[r];
      const int tn = rb + 32 * kDepth + lane;
      p[r] = tn < len ? prod(tn) : 0.0;  // refill this slot for the next sweep
      const int cnt = len - rb;
      if (cnt >= 32) {
#pragma unroll
        for (int k = 0; k < 32; ++k) s = xadd(s, __shfl_sync(0xffffffffu, cur, k));
      } else if (cnt > 0) {
        for (int k = 0; k < cnt; ++k) s = xadd(s, __shfl_sync(0xffffffffu, cur, k));
      }
    }
  }
  return s;
}

}  // namespace alnnls
