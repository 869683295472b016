// Standalone timing of the vector-CTA phases of nqp_loop_kernel (one CTA, no row CTAs).
#include "../../paper_1502_01645_b200/csrc/nqp.cu"
#include <cstdio>
#include <vector>
using namespace alnnls;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void __launch_bounds__(384, 1) vec_kernel(LoopArgs a, unsigned long long* t, int reps) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ LeaderState L;
  __shared__ double mn;
  double* sbuf = reinterpret_cast<double*>(smem);
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    unsigned long long t0 = globaltimer_ns();
    leader_build_mask(a, L, a.g, a.gd, &mn);
    unsigned long long t1 = globaltimer_ns();
    const int ml = a.ctrl->mask_len;
    leader_build_changed(a, L, ml, 0.01);
    unsigned long long t2 = globaltimer_ns();
    const double *gP = a.gP, *xP = a.xP, *qP = a.qP;
    leader_chains<3>(sbuf, kRingSmemBytes, L, ml, [&](int c, int tt) {
      return c == 0 ? xmul(gP[tt], gP[tt]) : (c == 1 ? xmul(xP[tt], gP[tt]) : xmul(qP[tt], xP[tt]));
    });
    unsigned long long t3 = globaltimer_ns();
    const double* u = a.u; const uint32_t* mask = a.mask;
    leader_chains<1>(sbuf, kRingSmemBytes, L, ml, [&](int, int tt) { return xmul(gP[tt], __ldcg(u + mask[tt])); });
    unsigned long long t4 = globaltimer_ns();
    if (threadIdx.x == 0 && r == reps - 1) { t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; t[3] = t4 - t3; t[4] = ml; t[5] = a.ctrl->chg_len; }
  }
}

int main() {
  const int m = 4096; const size_t mp = 4096 + 64;
  std::vector<double> hx(mp, 0.0), hg(mp), hq(mp);
  srand(3);
  for (int i = 0; i < m; ++i) { hx[i] = (rand() % 10 < 5) ? (rand() % 1000) * 1e-3 : 0.0; hg[i] = ((rand() % 2000) - 1000) * 1e-3; hq[i] = hg[i]; }
  auto dalloc = [&](size_t n) { double* p; CK(cudaMalloc(&p, n * 8)); CK(cudaMemset(p, 0, n * 8)); return p; };
  LoopArgs a{};
  a.m = m;
  a.x = dalloc(mp); a.g = dalloc(mp); a.g_alt = dalloc(mp); a.u = dalloc(mp); a.gd = dalloc(mp);
  a.q = dalloc(mp); a.gP = dalloc(mp); a.dC = dalloc(mp); a.candC = dalloc(mp); a.gC = dalloc(mp);
  a.xP = dalloc(mp); a.qP = dalloc(mp);
  uint32_t *mk, *ch; CK(cudaMalloc(&mk, mp * 4)); CK(cudaMalloc(&ch, mp * 4)); a.mask = mk; a.chg = ch;
  LoopCtrl* c; CK(cudaMalloc(&c, sizeof(LoopCtrl))); CK(cudaMemset(c, 0, sizeof(LoopCtrl))); a.ctrl = c;
  CK(cudaMemcpy(a.x, hx.data(), mp * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(a.g, hg.data(), mp * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy((void*)a.q, hq.data(), mp * 8, cudaMemcpyHostToDevice));
  unsigned long long* t; CK(cudaMalloc(&t, 64));
  CK(cudaFuncSetAttribute(vec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRingSmemBytes));
  for (int it = 0; it < 3; ++it) vec_kernel<<<1, 384, kRingSmemBytes>>>(a, t, 5);
  CK(cudaDeviceSynchronize());
  unsigned long long h[6]; CK(cudaMemcpy(h, t, 48, cudaMemcpyDeviceToHost));
  printf("m=%d |P|=%llu |C|=%llu  build_mask %.2f us  build_changed %.2f us  3 chains %.2f us  den chain %.2f us\n",
         m, h[4], h[5], h[0] * 1e-3, h[1] * 1e-3, h[2] * 1e-3, h[3] * 1e-3);
  return 0;
}
