// capi.cu — the C ABI (include/alnnls.h): context, device buffers, host-side
// validation with the reference's error semantics, and the orchestration of
// the sm_100a kernels for solve_nnls / solve_nqp and the dense helpers.
//
// Validation mirrors the reference preconditions (linalg.hpp:22-24, :42-52,
// :74-85; nqp.hpp:35-41, :84-98, :227-230; nnls.hpp:43-56, :131) so that the
// same inputs fail with the same category (EINVAL / ERANGE / ENUMERIC).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <initializer_list>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/alnnls.h"
#include "kernels.cuh"

using namespace alnnls;

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

}  // namespace

struct alnnls_ctx {
  int device = 0;
  int sm_count = 0;
  int cc_major = 0, cc_minor = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // H2D of the host-buffer entries (overlapped uploads)
  cudaEvent_t ev[6] = {};
  cudaEvent_t up[16] = {};            // row-block upload events (kMaxUpBlocks)
  cudaStream_t bstream[2] = {};       // batched host pipeline: alternating solve streams (lazy)
  cudaEvent_t bev[8] = {};            // its per-chunk events: [2c] q ready, [2c+1] chunk solved
  std::string err;

  DevBuf A, b, Q, q, x, g, y_out, u, gd, mask, gP, chg, dC, candC, gC, prod0, prod1, prod2;
  DevBuf diag, pos, scale, retained, mscalar, trace, mults, ctrl, list, vals, ax, resid, flag, H,
      hvec, start, bcols, X, x_alt, mask2, gP2, xP2, qP2, part, resb, yb, qb, uP, gdC, skp, skf,
      ay, axn, aw, avy, apc, tst, fgb0, fgb1, fpart, fden, fkl, fkv, fkc, dmws, dmfl, nvt,
      nht, nwt, nv, nw, nh, qfrag, bcnt;

  // last solve
  bool last_nnls = false;
  uint64_t last_n = 0, last_m = 0;
  uint64_t qR = 4;   // block rows of the blocked Q (gemv.cuh)
  alnnls_summary last{};
  std::vector<uint64_t> dropped_h;
  bool have_setup = false;
  int g_parity = 0;
  int solver = 0;  // 0: solve_nqp loop; 1: accelerated baseline (set by the *_accelerated entries)
  unsigned long long phase_ns[8] = {};
  uint64_t launches = 0;
  int loop_kernel = 0;  // ALNNLS_LOOP_* of the last solve
  cudaEvent_t timer[2] = {};
  // pinned host copies read after one stream sync (deferred NQP control block,
  // the residual), so a solve needs no host round trip between the loop and its finish
  struct Pinned {
    LoopCtrl hc;
    double hres;
    int hm;
  };
  Pinned* pin = nullptr;
  uint64_t nqp_tcap = 0, nqp_mcap = 0, nqp_m = 0;
  int nqp_record_mults = 0;
};

namespace {

int set_err(alnnls_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

int cuda_fail(alnnls_ctx* c, cudaError_t e, const char* where) {
  const int code = (e == cudaErrorMemoryAllocation) ? ALNNLS_ENOMEM : ALNNLS_ECUDA;
  return set_err(c, code, std::string(where) + ": " + cudaGetErrorString(e));
}

// Every launch_* wrapper launches exactly one of our kernels: count them (the
// benchmark reports the number of our kernels in its timed region).
#define CK(call)                                                        \
  do {                                                                  \
    if (std::strncmp(#call, "launch_", 7) == 0) ++ctx->launches;        \
    cudaError_t e__ = (call);                                           \
    if (e__ != cudaSuccess) return cuda_fail(ctx, e__, #call);          \
  } while (0)

template <class T>
T* ensure(alnnls_ctx* ctx, DevBuf& b, size_t count, int* st) {
  const size_t bytes = sizeof(T) * (count + 4);
  if (b.bytes < bytes) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    cudaError_t e = cudaMalloc(&b.p, bytes);
    if (e != cudaSuccess) {
      *st = cuda_fail(ctx, e, "cudaMalloc");
      return nullptr;
    }
    b.bytes = bytes;
  }
  return static_cast<T*>(b.p);
}

#define ENSURE(T, buf, count)                      \
  ensure<T>(ctx, ctx->buf, (size_t)(count), &st__); \
  if (st__ != ALNNLS_OK) return st__

uint64_t round_up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

// device trace / multiply-count capacity caps (records): 4 Mi trace records
// (192 MiB) and 16 Mi multiply counts (128 MiB)
constexpr uint64_t kTraceCapMax = (uint64_t)1 << 22;
constexpr uint64_t kMultCapMax = (uint64_t)1 << 24;

// doubles of a blocked m x m matrix with block rows R (gemv.cuh blk_index)
uint64_t blocked_size(uint64_t m, uint64_t R) { return round_up(m, R) * m; }

// vector length padded to the loop kernel tile (512 threads x 8) plus slack
uint64_t vec_pad(uint64_t m) { return round_up(m > 0 ? m : 1, 4096) + 64; }

bool all_finite(const double* p, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(p[i])) return false;
  return true;
}

struct Resolved {
  double eps;
  uint64_t max_iters;
  uint64_t trace_every;
};

// SolverConfig::resolve_epsilon / resolve_max_iters (nqp.hpp:84-98).
int resolve(alnnls_ctx* ctx, const alnnls_config* cfg, uint64_t m, Resolved* r) {
  if (cfg->has_epsilon) {
    if (!(cfg->epsilon > 0.0)) return set_err(ctx, ALNNLS_EINVAL, "SolverConfig: epsilon must be > 0");
    r->eps = cfg->epsilon;
  } else {
    r->eps = 1e-10 * (double)m;
  }
  if (cfg->has_max_iters) {
    if (cfg->max_iters < 1) return set_err(ctx, ALNNLS_EINVAL, "SolverConfig: max_iters must be >= 1");
    r->max_iters = cfg->max_iters;
  } else {
    r->max_iters = 5 * m;
  }
  r->trace_every = cfg->trace_every > 0 ? cfg->trace_every : 1;
  if (cfg->profile != ALNNLS_PROFILE_EXACT && cfg->profile != ALNNLS_PROFILE_FAST)
    return set_err(ctx, ALNNLS_EINVAL, "alnnls_config: unknown profile");
  return ALNNLS_OK;
}

int check_ctx(alnnls_ctx* ctx) {
  if (!ctx) return ALNNLS_EINVAL;
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
  return ALNNLS_OK;
}

// ---- the device-resident NQP solve on ctx->Q / ctx->q (already uploaded) ------
// x0: nullptr -> start at 0 (g = q); otherwise device start vector (validated).
// solver 0: solve_nqp (nqp.hpp:215-339); 1: solve_accelerated (accelerated.hpp:21-117).
int collect_nqp(alnnls_ctx* ctx, alnnls_summary* out);

// defer: return right after the launches with the control block's copy enqueued;
// the caller enqueues more work, synchronises once and calls collect_nqp.
int run_nqp(alnnls_ctx* ctx, uint64_t m, const Resolved& r, const alnnls_config* cfg,
            const double* dstart, alnnls_summary* out, int solver = 0, bool defer = false) {
  int st__ = ALNNLS_OK;
  const double* Q = static_cast<const double*>(ctx->Q.p);
  const double* q = static_cast<const double*>(ctx->q.p);
  // vector buffers are padded to the loop kernel's 4096-element tiles
  const uint64_t mp = vec_pad(m);
  double* x = ENSURE(double, x, mp);
  double* g = ENSURE(double, g, mp);
  double* u = ENSURE(double, u, mp);
  double* gd = ENSURE(double, gd, mp);
  uint32_t* mask = ENSURE(uint32_t, mask, mp);
  double* gP = ENSURE(double, gP, mp);
  uint32_t* chg = ENSURE(uint32_t, chg, mp);
  double* dC = ENSURE(double, dC, mp);
  double* candC = ENSURE(double, candC, mp);
  double* gC = ENSURE(double, gC, mp);
  double* g_alt = ENSURE(double, prod1, mp);
  double* xP = ENSURE(double, prod2, mp);
  double* qP = ENSURE(double, prod0, mp);
  double* x_alt = ENSURE(double, x_alt, mp);
  uint32_t* mask2 = ENSURE(uint32_t, mask2, mp);
  double* gP2 = ENSURE(double, gP2, mp);
  double* xP2 = ENSURE(double, xP2, mp);
  double* qP2 = ENSURE(double, qP2, mp);
  double* uP = ENSURE(double, uP, mp);
  double* gdC = ENSURE(double, gdC, mp);
  // per row-CTA partials: cnt (int), badv (int), minx (double)
  double* part = ENSURE(double, part, 3 * 160);
  int* cnt = reinterpret_cast<int*>(part);
  int* badv = cnt + 160;
  double* minx = part + 160;
  LoopCtrl* ctrl = ENSURE(LoopCtrl, ctrl, 2);  // [1] holds the grid-barrier words
  unsigned int* bar = reinterpret_cast<unsigned int*>(ctrl + 1);
  // The reference's trace grows as needed; the device buffers are sized up front
  // from max_iters, capped (overflow-safe) so an "unlimited" max_iters cannot wrap
  // or exhaust HBM. Past the cap the last slot always holds the newest record
  // (so the final record survives) and trace_len / mult_len are clamped.
  const uint64_t tcap = std::min(r.max_iters / r.trace_every, kTraceCapMax - 2) + 2;
  alnnls_iter_record* trace = ENSURE(alnnls_iter_record, trace, tcap);
  uint64_t mcap = 0;
  uint64_t* mults = nullptr;
  if (cfg->record_multiplies) {
    mcap = std::min(r.max_iters, kMultCapMax - 1) + 1;
    mults = ENSURE(uint64_t, mults, mcap);
  }
  cudaStream_t s = ctx->stream;
  // the exact loop from 0 initialises x, g and its scratch itself (launch_nqp_loop):
  // for a small problem the cluster kernel does it in its prologue, so no extra
  // stream operations precede the launch
  const int R0 = (int)ctx->qR;
  const bool fast_loop = solver == 0 && cfg->profile == ALNNLS_PROFILE_FAST &&
                         fast_loop_supported((int)m, R0);
  const bool zero_start = solver == 0 && !fast_loop && !dstart;
  if (!zero_start) {
    CK(cudaMemsetAsync(gP, 0, sizeof(double) * (m + 8), s));
    CK(cudaMemsetAsync(dC, 0, sizeof(double) * (m + 8), s));
  }
  if (!dstart) {
    if (!zero_start) {
      CK(cudaMemsetAsync(x, 0, sizeof(double) * m, s));
      CK(cudaMemcpyAsync(g, q, sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
    }
  } else {
    // g = matvec(Q, start) + q (nqp.hpp:231-233); skipping x_j == 0 columns is exact.
    CK(cudaMemcpyAsync(x, dstart, sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
    uint32_t* list = ENSURE(uint32_t, list, m);
    double* vals = ENSURE(double, vals, m + 8);
    int* len = ENSURE(int, mscalar, 4);
    CK(launch_support(x, (int)m, list, vals, len, s));
    int hlen = 0;
    CK(cudaMemcpyAsync(&hlen, len, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    CK(launch_masked_gemv_blocked(Q, (int)m, (int)ctx->qR, list, vals, hlen, u, s));
    CK(launch_add(u, q, g, (int)m, s));
  }
  LoopArgs a{};
  a.Q = Q;
  a.ldq = 0;
  a.q = q;
  a.m = (int)m;
  a.x = x;
  a.g = g;
  a.u = u;
  a.gd = gd;
  a.mask = mask;
  a.gP = gP;
  a.chg = chg;
  a.dC = dC;
  a.candC = candC;
  a.gC = gC;
  a.g_alt = g_alt;
  a.xP = xP;
  a.qP = qP;
  a.x_alt = x_alt;
  a.mask2 = mask2;
  a.gP2 = gP2;
  a.xP2 = xP2;
  a.qP2 = qP2;
  a.uP = uP;
  a.gdC = gdC;
  a.cnt = cnt;
  a.badv = badv;
  a.minx = minx;
  a.eps = r.eps;
  a.max_iters = r.max_iters;
  a.has_time_cap = cfg->has_time_cap;
  a.time_cap_s = cfg->time_cap_s;
  a.stall_window = cfg->stall_window;
  a.trace_every = r.trace_every;
  a.trace = trace;
  a.trace_cap = tcap;
  a.mults = mults;
  a.mults_cap = mcap;
  a.ctrl = ctrl;
  a.bar = bar;
  if (!zero_start) CK(cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned int), ctx->stream));
  a.zero_start = zero_start ? 1 : 0;
  a.rows_per_cta = (int)ctx->qR;
  a.resident = solver == 0 && nqp_resident_fits((int)m, a.rows_per_cta) ? 1 : 0;
  if (a.rows_per_cta > 352)
    return set_err(ctx, ALNNLS_EINVAL, "solve_nqp: dimension too large for one GPU row split");
  const int nctas = 1 + (int)((m + a.rows_per_cta - 1) / a.rows_per_cta);
  if (solver == 1) {
    if (m > 46340) return set_err(ctx, ALNNLS_EINVAL, "solve_accelerated: m too large");
    a.y = ENSURE(double, ay, mp);
    a.xn = ENSURE(double, axn, mp);
    a.w = ENSURE(double, aw, mp);
    a.vy = ENSURE(double, avy, mp);
    a.pcnt = ENSURE(int, apc, 160);
    a.restart = cfg->nesterov_restart != 0;
    CK(cudaMemsetAsync(a.y, 0, sizeof(double) * m, s));
    double* nrm = ENSURE(double, resid, 2);
    CK(launch_frobenius(Q, (int)m, (int)ctx->qR, nrm, s));  // M = ||Q||_F (accelerated.hpp:27)
    double hn = 0.0;
    CK(cudaMemcpyAsync(&hn, nrm, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    a.alpha = 1.0 / hn;  // :83 (host IEEE division, same rounding)
  }
  // FAST profile: the one-pass bandwidth-bound loop (fastloop.cu) when its
  // shared-memory staging fits (m up to ~26k); otherwise the exact loop.
  const bool fast = solver == 0 && cfg->profile == ALNNLS_PROFILE_FAST &&
                    fast_loop_supported((int)m, a.rows_per_cta);
  FastArgs fa{};
  if (fast) {
    const int nblk = (int)((m + a.rows_per_cta - 1) / a.rows_per_cta);
    fa.Q = Q;
    fa.m = (int)m;
    fa.R = a.rows_per_cta;
    fa.q = q;
    fa.x[0] = x;
    fa.x[1] = x_alt;
    fa.g[0] = g;
    fa.g[1] = g_alt;
    fa.gbar[0] = ENSURE(double, fgb0, mp);
    fa.gbar[1] = ENSURE(double, fgb1, mp);
    FastPart* fp = ENSURE(FastPart, fpart, 2 * nblk);
    fa.part[0] = fp;
    fa.part[1] = fp + nblk;
    fa.den = ENSURE(double, fden, nblk);
    fa.kl = ENSURE(uint32_t, fkl, (size_t)nblk * a.rows_per_cta);
    fa.kv = ENSURE(double, fkv, (size_t)nblk * a.rows_per_cta);
    fa.kc = ENSURE(int, fkc, nblk);
    fa.eps = a.eps;
    fa.max_iters = a.max_iters;
    fa.has_time_cap = a.has_time_cap;
    fa.time_cap_s = a.time_cap_s;
    fa.stall_window = a.stall_window;
    fa.trace_every = a.trace_every;
    fa.trace = trace;
    fa.trace_cap = tcap;
    fa.mults = mults;
    fa.mults_cap = mcap;
    fa.ctrl = ctrl;
    CK(cudaMemsetAsync(ctrl, 0, sizeof(LoopCtrl), s));
  }
  CK(cudaEventRecord(ctx->ev[2], s));
  if (fast) {
    CK(launch_fast_loop(fa, s));
    ctx->loop_kernel = ALNNLS_LOOP_FAST;
  } else if (solver == 1) {
    CK(launch_acc_loop(a, nctas, s, &ctx->loop_kernel));
  } else {
    CK(launch_nqp_loop(a, nctas, s, &ctx->loop_kernel));
  }
  CK(cudaEventRecord(ctx->ev[3], s));
  if (!ctx->pin) CK(cudaMallocHost(&ctx->pin, sizeof(alnnls_ctx::Pinned)));
  CK(cudaMemcpyAsync(&ctx->pin->hc, ctrl, sizeof(LoopCtrl), cudaMemcpyDeviceToHost, s));
  ctx->nqp_tcap = tcap;
  ctx->nqp_mcap = mcap;
  ctx->nqp_m = m;
  ctx->nqp_record_mults = cfg->record_multiplies;
  if (defer) return ALNNLS_OK;
  CK(cudaStreamSynchronize(s));
  return collect_nqp(ctx, out);
}

// Fills the summary from the control block run_nqp copied (after a stream sync).
int collect_nqp(alnnls_ctx* ctx, alnnls_summary* out) {
  const LoopCtrl& hc = ctx->pin->hc;
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]);
  out->t_loop_s = ms * 1e-3;
  out->termination = hc.termination;
  out->numeric_failure = hc.numeric_failure;
  out->iterations = hc.iterations;
  out->trace_len = std::min<uint64_t>(hc.trace_len, ctx->nqp_tcap);
  out->mult_len = ctx->nqp_record_mults ? std::min<uint64_t>(hc.mult_len, ctx->nqp_mcap) : 0;
  out->multiplies_total = hc.mult_total;
  out->min_iterate = hc.min_iterate;
  out->f_final = hc.f_final;
  out->gbs_final = hc.gbs_final;
  out->m = ctx->nqp_m;
  ctx->g_parity = hc.g_parity;
  for (int i = 0; i < 8; ++i) ctx->phase_ns[i] = hc.phase_ns[i];
  if (hc.numeric_failure)
    return set_err(ctx, ALNNLS_ENUMERIC, "solve_nqp: non-finite objective or gradient");
  return ALNNLS_OK;
}

// ---- setup on device A (lda) and b: rescale(gram(A), -A^T b) -> ctx->Q, q ----
// profile FAST forms the Gram on the fp64 tensor cores (dmma.cu); EXACT (and
// FAST when the operands are not 16-byte aligned) uses the bitwise chain SYRK.
// Scratch of the stream-K exact SYRK (setup.cu syrk_streamk_kernel), when the
// shape uses it.
int streamk_buffers(alnnls_ctx* ctx, SetupArgs& sa, int mode) {
  int st__ = ALNNLS_OK;
  sa.sk_ctas = syrk_streamk_ctas(sa, mode, ctx->sm_count);
  sa.sk_part = nullptr;
  sa.sk_flag = nullptr;
  if (sa.sk_ctas > 0) {
    sa.sk_part = ENSURE(double, skp, (size_t)sa.sk_ctas * ALNNLS_GRAM_TILE_DOUBLES);
    sa.sk_flag = ENSURE(int, skf, sa.sk_ctas);
  }
  return ALNNLS_OK;
}

// Workspace of the TMA stream-K DMMA Gram (dmma.cu syrk_tma_kernel): one partial
// 128 x 128 tile and one flag per persistent CTA.
int dmma_buffers(alnnls_ctx* ctx, SetupArgs& sa) {
  int st__ = ALNNLS_OK;
  sa.dm_ctas = ctx->sm_count;
  sa.dm_ws = ENSURE(double, dmws, syrk_dmma_ws_doubles(ctx->sm_count));
  sa.dm_flags = ENSURE(int, dmfl, ctx->sm_count + 4);
  return ALNNLS_OK;
}

int run_setup(alnnls_ctx* ctx, uint64_t d, uint64_t n, const double* dA, uint64_t lda,
              const double* db, uint64_t* m_out, int profile = ALNNLS_PROFILE_EXACT) {
  int st__ = ALNNLS_OK;
  int rc_sk = ALNNLS_OK;
  cudaStream_t s = ctx->stream;
  SetupArgs sa{};
  sa.A = dA;
  sa.lda = lda;
  sa.b = db;
  sa.d = (int)d;
  sa.n = (int)n;
  sa.diag = ENSURE(double, diag, n);
  sa.pos = ENSURE(int, pos, n);
  sa.scale = ENSURE(double, scale, n);
  sa.retained = ENSURE(uint32_t, retained, n);
  sa.m_out = ENSURE(int, mscalar, 4);
  sa.hvec_scratch = ENSURE(double, hvec, n);
  CK(launch_gram_diag(sa, s));
  CK(launch_retained(sa, s));
  if (!ctx->pin) CK(cudaMallocHost(&ctx->pin, sizeof(alnnls_ctx::Pinned)));
  CK(cudaMemcpyAsync(&ctx->pin->hm, sa.m_out, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaEventRecord(ctx->ev[5], s));  // the count has landed in pinned memory
  // The retained count m is only known on the device. Speculate m = n (no zero
  // column, the usual case) and queue the Gram + rescale right behind the count,
  // so the host's read of m overlaps the Gram; if a column was dropped, the Gram
  // is redone for the real m (the speculative one wrote Q in the wrong layout).
  auto gram = [&](uint64_t m) -> int {
    const uint64_t mm = m > 0 ? m : 1;
    ctx->qR = (uint64_t)nqp_rows_per_cta((int)mm, ctx->sm_count);
    sa.Q = ENSURE(double, Q, blocked_size(mm, ctx->qR));
    sa.m = (int)m;
    sa.qR = (int)ctx->qR;
    sa.q = ENSURE(double, q, vec_pad(m));
    if (m > 0) {
      if (profile == ALNNLS_PROFILE_FAST && syrk_dmma_supported(sa, 1)) {
        if (int rc = dmma_buffers(ctx, sa)) return rc;
        CK(launch_syrk_dmma(sa, 1, s));
      } else {
        if ((rc_sk = streamk_buffers(ctx, sa, 1))) return rc_sk;
        CK(launch_syrk(sa, 1, s));
      }
      CK(launch_q_from_atb(sa, 1, s));
    }
    return ALNNLS_OK;
  };
  if (int rc = gram(n)) return rc;
  CK(cudaEventSynchronize(ctx->ev[5]));  // waits for the count, not for the Gram
  const uint64_t m = (uint64_t)ctx->pin->hm;
  if (m != n)
    if (int rc = gram(m)) return rc;
  *m_out = m;
  ctx->have_setup = true;
  return ALNNLS_OK;
}

// nnls.hpp:129-144 on device-resident A (lda, 16B-aligned, lda even) and b.
int run_nnls(alnnls_ctx* ctx, uint64_t d, uint64_t n, const double* dA, uint64_t lda,
             const double* db, const alnnls_config* cfg, alnnls_summary* out, int solver = 0) {
  int st__ = ALNNLS_OK;
  cudaStream_t s = ctx->stream;
  alnnls_summary sum{};
  CK(cudaEventRecord(ctx->ev[0], s));
  uint64_t m = 0;
  int rc = run_setup(ctx, d, n, dA, lda, db, &m, cfg->profile);
  if (rc) return rc;
  CK(cudaEventRecord(ctx->ev[1], s));
  ctx->last_nnls = true;
  ctx->last_n = n;
  ctx->last_m = m;
  double* y = ENSURE(double, y_out, m);
  if (m > 0) {
    Resolved r;
    rc = resolve(ctx, cfg, m, &r);  // solve_nqp validates its config (nqp.hpp:220-221)
    if (rc) return rc;
    rc = run_nqp(ctx, m, r, cfg, nullptr, &sum, solver | ctx->solver, /*defer=*/true);
    if (rc) {
      if (out) *out = sum;
      ctx->last = sum;
      return rc;
    }
    CK(launch_copy_parity(y, static_cast<double*>(ctx->x.p), static_cast<double*>(ctx->x_alt.p),
                          static_cast<LoopCtrl*>(ctx->ctrl.p), (int)m, s));
  } else {
    // detail::empty_solve_result (nnls.hpp:107-113)
    alnnls_iter_record rec{};
    alnnls_iter_record* tr = ENSURE(alnnls_iter_record, trace, 2);
    CK(cudaMemcpyAsync(tr, &rec, sizeof(rec), cudaMemcpyHostToDevice, s));
    sum.termination = ALNNLS_EMPTY_PASSIVE_SET;
    sum.trace_len = 1;
    sum.min_iterate = 0.0;
    sum.iterations = 0;
    CK(cudaEventRecord(ctx->ev[2], s));
    CK(cudaEventRecord(ctx->ev[3], s));
  }
  // K7: unscale + residual recomputed from A and b (nnls.hpp:141-142)
  double* xn = ENSURE(double, X, n);
  CK(launch_unscale(y, static_cast<double*>(ctx->scale.p), static_cast<uint32_t*>(ctx->retained.p),
                    (int)m, xn, (int)n, s));
  uint32_t* list = ENSURE(uint32_t, list, n);
  double* vals = ENSURE(double, vals, n + 8);
  int* len = ENSURE(int, mscalar, 4);
  CK(launch_support(xn, (int)n, list, vals, len, s));
  double* ax = ENSURE(double, ax, d);
  double* pr = ENSURE(double, bcols, d + 8);
  double* res = ENSURE(double, resid, 2);
  // the support length stays on the device: no host round trip before the residual
  CK(launch_masked_gemv(dA, lda, (int)d, list, vals, (int)n, ax, ctx->sm_count, s, len));
  CK(launch_residual(ax, db, (int)d, pr, res, s));
  CK(cudaEventRecord(ctx->ev[4], s));
  if (!ctx->pin) CK(cudaMallocHost(&ctx->pin, sizeof(alnnls_ctx::Pinned)));
  CK(cudaMemcpyAsync(&ctx->pin->hres, res, sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));  // the one host sync after the setup's
  const double hres = ctx->pin->hres;
  if (m > 0) {
    rc = collect_nqp(ctx, &sum);
    if (rc) {
      if (out) *out = sum;
      ctx->last = sum;
      return rc;
    }
  }
  float t01 = 0, t23 = 0, t34 = 0, t04 = 0;
  cudaEventElapsedTime(&t01, ctx->ev[0], ctx->ev[1]);
  cudaEventElapsedTime(&t23, ctx->ev[2], ctx->ev[3]);
  cudaEventElapsedTime(&t34, ctx->ev[3], ctx->ev[4]);
  cudaEventElapsedTime(&t04, ctx->ev[0], ctx->ev[4]);
  sum.t_setup_s = t01 * 1e-3;
  sum.t_loop_s = t23 * 1e-3;
  sum.t_finish_s = t34 * 1e-3;
  sum.t_total_s = t04 * 1e-3;
  sum.residual_sq = hres;
  sum.n = n;
  sum.m = m;
  sum.n_dropped = n - m;
  ctx->last = sum;
  if (out) *out = sum;
  return ALNNLS_OK;
}

// Uploads host A (d x n, ld d) into ctx->A with an even, 32B-friendly ld.
int upload_matrix(alnnls_ctx* ctx, DevBuf& buf, uint64_t rows, uint64_t cols, const double* h,
                  uint64_t* ld_out) {
  int st__ = ALNNLS_OK;
  const uint64_t ld = round_up(rows, 4);
  double* dst = ensure<double>(ctx, buf, ld * cols, &st__);
  if (st__) return st__;
  CK(cudaMemcpy2DAsync(dst, ld * sizeof(double), h, rows * sizeof(double), rows * sizeof(double),
                       cols, cudaMemcpyHostToDevice, ctx->stream));
  *ld_out = ld;
  return ALNNLS_OK;
}

int copy_out(alnnls_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return ALNNLS_OK;
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return ALNNLS_OK;
}

// The reference validates finiteness when a DenseMatrix / Vector is built
// (linalg.hpp:42-52, :84). The host-buffer entries upload first and run that
// check on the device over the copies (one flag per operand, reported in the
// reference's construction order), instead of a single-threaded host scan.
struct FiniteArg {
  const double* p;
  uint64_t rows, cols, ld;
  const char* msg;
};
int device_check_finite(alnnls_ctx* ctx, std::initializer_list<FiniteArg> args) {
  int st__ = ALNNLS_OK;
  const size_t k = args.size();
  int* flag = ENSURE(int, flag, 4);
  CK(cudaMemsetAsync(flag, 0, sizeof(int) * k, ctx->stream));
  int i = 0;
  for (const FiniteArg& a : args) {
    CK(launch_check_finite(a.p, a.rows, a.cols, a.ld, flag + i, ctx->stream));
    ++i;
  }
  int hf[4] = {0, 0, 0, 0};
  if (int rc = copy_out(ctx, hf, flag, sizeof(int) * k)) return rc;
  i = 0;
  for (const FiniteArg& a : args) {
    if (hf[i]) return set_err(ctx, ALNNLS_EINVAL, a.msg);
    ++i;
  }
  return ALNNLS_OK;
}

// Host-buffer solve_nnls with the upload of A overlapped with the Gram: A is
// copied in row blocks on the copy stream, and each block's Gram contribution
// is computed as soon as it lands by continuing every tile's chain states over
// its rows (stream-K SYRK with tpin/tpout; A^T b chains likewise), so the
// result is bitwise the one-shot Gram. Blocks grow geometrically: the first is
// small (the only upload not hidden), later ones ~1.75x the previous, since a
// row's Gram work takes ~1.8x its PCIe upload time. The finiteness check runs
// after the last block (results are discarded on failure, as if validated first).
constexpr int kMaxUpBlocks = 16;  // ctx->up
// FAST (DMMA) Gram work per row is shorter than its upload, so only the last
// block's Gram is exposed: equal blocks, as many as the events allow.
int upload_blocks_equal(uint64_t d, uint64_t* edges) {
  uint64_t nb = d / 256;
  if (nb > (uint64_t)kMaxUpBlocks) nb = kMaxUpBlocks;
  if (nb < 1) nb = 1;
  const uint64_t sz = (d / nb + 15) / 16 * 16;
  int k = 0;
  edges[0] = 0;
  for (uint64_t r = 0; r < d && k < kMaxUpBlocks; r += sz) {
    const uint64_t r1 = (k == kMaxUpBlocks - 1 || r + sz >= d) ? d : r + sz;
    edges[++k] = r1;
    if (r1 == d) break;
  }
  return k;
}
// FAST row blocks: a geometric series shrinking by 0.7, from ~30% of d down to
// >= 256 rows (the last block's Gram is what stays exposed after the copy).
int upload_blocks_shrinking(uint64_t d, uint64_t* edges) {
  int nb = 0;
  uint64_t r = 0;
  edges[0] = 0;
  double frac = 0.3;
  while (r < d && nb < kMaxUpBlocks) {
    uint64_t sz = (uint64_t)(frac * (double)d);
    sz = (sz + 15) / 16 * 16;
    if (sz < 256) sz = 256;
    uint64_t r1 = r + sz;
    if (nb == kMaxUpBlocks - 1 || r1 + 128 >= d) r1 = d;
    edges[++nb] = r1;
    r = r1;
    frac *= 0.7;
  }
  return nb;
}
int upload_blocks(uint64_t d, uint64_t* edges) {
  uint64_t sz = d / 32 < 256 ? 256 : (d / 32 + 15) / 16 * 16;
  int nb = 0;
  uint64_t r = 0;
  edges[0] = 0;
  while (r < d && nb < kMaxUpBlocks) {
    uint64_t r1 = r + sz;
    if (nb == kMaxUpBlocks - 1 || r1 + sz / 2 >= d) r1 = d;  // fold a small remainder in
    edges[++nb] = r1;
    r = r1;
    sz = (sz * 7 / 4 + 15) / 16 * 16;
  }
  return nb;
}

int run_nnls_overlapped(alnnls_ctx* ctx, uint64_t d, uint64_t n, const double* A, const double* b,
                        const alnnls_config* cfg, alnnls_summary* out) {
  int st__ = ALNNLS_OK;
  cudaStream_t s = ctx->stream, cs = ctx->copy_stream;
  const uint64_t lda = round_up(d, 4);
  double* dA = ENSURE(double, A, lda * n);
  double* db = ENSURE(double, b, d);
  const uint64_t T = gram_tiles(n);
  const uint64_t TD = ALNNLS_GRAM_TILE_DOUBLES;
  const bool fast = cfg->profile == ALNNLS_PROFILE_FAST;
  double* H = ENSURE(double, H, n * n);
  double* st_buf = fast ? nullptr : ENSURE(double, tst, 2 * T * TD);  // ping-pong tile chain states
  double* hb = ENSURE(double, hvec, 2 * n + 8);       // ping-pong A^T b chain states
  CK(cudaEventRecord(ctx->ev[0], s));
  CK(cudaStreamWaitEvent(cs, ctx->ev[0], 0));
  CK(cudaMemcpyAsync(db, b, sizeof(double) * d, cudaMemcpyHostToDevice, cs));
  const double* pin = nullptr;
  const double* hin = nullptr;
  uint64_t edges[kMaxUpBlocks + 1];
  // Row blocks growing ~1.75x (the 2D copy of a row block moves one short segment
  // per column: larger segments copy faster). EXACT continues every tile's chain
  // over each block (bitwise the one-shot Gram); FAST accumulates each block's DMMA
  // Gram into the upper triangle of H (rescale reads only that). Measured at c2
  // (tools/e2e_probe2.py, setup + upload): FAST growing 6.89 ms, shrinking 7.69,
  // equal 7.88; column blocks with per-block tile ranges 8.7 (the late tile
  // columns hold most of the Gram: small launches). Knob ALNNLS_FAST_UPLOAD=1|2.
  static const int fast_sched = getenv("ALNNLS_FAST_UPLOAD") ? atoi(getenv("ALNNLS_FAST_UPLOAD")) : 0;
  const int nblk = fast && fast_sched == 1 ? upload_blocks_shrinking(d, edges)
                   : fast && fast_sched == 2 ? upload_blocks_equal(d, edges)
                                            : upload_blocks(d, edges);
  for (int k = 0; k < nblk; ++k) {
    const uint64_t r0 = edges[k], r1 = edges[k + 1];
    CK(cudaMemcpy2DAsync(dA + r0, lda * sizeof(double), A + r0, d * sizeof(double),
                         (r1 - r0) * sizeof(double), n, cudaMemcpyHostToDevice, cs));
    CK(cudaEventRecord(ctx->up[k], cs));
    CK(cudaStreamWaitEvent(s, ctx->up[k], 0));
    const bool last = k == nblk - 1;
    SetupArgs sa{};
    sa.A = dA + r0;
    sa.lda = lda;
    sa.d = (int)(r1 - r0);
    sa.n = (int)n;
    sa.H = H;
    double* pout = last || fast ? nullptr : st_buf + (size_t)(k & 1) * T * TD;
    if (fast) {
      if (int rc = dmma_buffers(ctx, sa)) return rc;
      CK(launch_syrk_dmma(sa, 0, s, (k > 0 ? 1 : 0) | 2));  // H(upper) (+)= A_blk^T A_blk
    } else {
      sa.tpin = pin;
      sa.tpout = pout;
      if (int rc = streamk_buffers(ctx, sa, 0)) return rc;
      if (sa.sk_ctas > 0) {
        CK(launch_syrk(sa, 0, s));  // stream-K over all tiles, chains continued
      } else {
        CK(launch_syrk_rowblock(sa, 0, (int)T, pin, pout, s));
      }
    }
    double* hout = hb + (size_t)(k & 1) * (n + 4);
    CK(launch_atb_chain(dA + r0, lda, (int)(r1 - r0), (int)n, db + r0, hin, hout, s));
    pin = pout;
    hin = hout;
  }
  if (int rc = device_check_finite(ctx, {{dA, d, n, lda, "DenseMatrix: non-finite entry"},
                                         {db, d, 1, d, "Vector: non-finite entry"}}))
    return rc;
  // rescale from the finished H and A^T b, loop, unscale, residual
  alnnls_summary sum{};
  {
    const double* atb = hin;
    SetupArgs sa{};
    sa.n = (int)n;
    sa.diag = ENSURE(double, diag, n);
    sa.pos = ENSURE(int, pos, n);
    sa.scale = ENSURE(double, scale, n);
    sa.retained = ENSURE(uint32_t, retained, n);
    sa.m_out = ENSURE(int, mscalar, 4);
    double* h = ENSURE(double, bcols, n + 8);
    CK(launch_diag(H, (int)n, sa.diag, s));
    CK(launch_negate(atb, (int)n, h, s));
    CK(launch_retained(sa, s));
    int hm = 0;
    CK(cudaMemcpyAsync(&hm, sa.m_out, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const uint64_t m = (uint64_t)hm;
    const uint64_t mm = m > 0 ? m : 1;
    ctx->qR = (uint64_t)nqp_rows_per_cta((int)mm, ctx->sm_count);
    double* Q = ENSURE(double, Q, blocked_size(mm, ctx->qR));
    double* q = ENSURE(double, q, vec_pad(m));
    if (m > 0) CK(launch_rescale_from_h(H, h, (int)n, sa.pos, sa.scale, Q, (int)m, (int)ctx->qR, q, s));
    ctx->have_setup = true;
    CK(cudaEventRecord(ctx->ev[1], s));
    ctx->last_nnls = true;
    ctx->last_n = n;
    ctx->last_m = m;
    double* y = ENSURE(double, y_out, mm);
    if (m > 0) {
      Resolved r;
      if (int rc = resolve(ctx, cfg, m, &r)) return rc;
      if (int rc = run_nqp(ctx, m, r, cfg, nullptr, &sum, ctx->solver, /*defer=*/true)) {
        if (out) *out = sum;
        ctx->last = sum;
        return rc;
      }
      CK(launch_copy_parity(y, static_cast<double*>(ctx->x.p),
                            static_cast<double*>(ctx->x_alt.p),
                            static_cast<LoopCtrl*>(ctx->ctrl.p), (int)m, s));
    } else {
      alnnls_iter_record rec{};
      alnnls_iter_record* tr = ENSURE(alnnls_iter_record, trace, 2);
      CK(cudaMemcpyAsync(tr, &rec, sizeof(rec), cudaMemcpyHostToDevice, s));
      sum.termination = ALNNLS_EMPTY_PASSIVE_SET;
      sum.trace_len = 1;
      CK(cudaEventRecord(ctx->ev[2], s));
      CK(cudaEventRecord(ctx->ev[3], s));
    }
    double* xn = ENSURE(double, X, n);
    CK(launch_unscale(y, sa.scale, sa.retained, (int)m, xn, (int)n, s));
    uint32_t* list = ENSURE(uint32_t, list, n);
    double* vals = ENSURE(double, vals, n + 8);
    int* len = ENSURE(int, mscalar, 4);
    CK(launch_support(xn, (int)n, list, vals, len, s));
    double* ax = ENSURE(double, ax, d);
    double* pr = ENSURE(double, resid, d + 8);
    double* res = ENSURE(double, flag, 8);  // doubles in the flag buffer (ints there are done)
    CK(launch_masked_gemv(dA, lda, (int)d, list, vals, (int)n, ax, ctx->sm_count, s, len));
    CK(launch_residual(ax, db, (int)d, pr, res, s));
    CK(cudaEventRecord(ctx->ev[4], s));
    if (!ctx->pin) CK(cudaMallocHost(&ctx->pin, sizeof(alnnls_ctx::Pinned)));
    CK(cudaMemcpyAsync(&ctx->pin->hres, res, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const double hres = ctx->pin->hres;
    if (m > 0) {
      if (int rc = collect_nqp(ctx, &sum)) {
        if (out) *out = sum;
        ctx->last = sum;
        return rc;
      }
    }
    float t01 = 0, t23 = 0, t34 = 0, t04 = 0;
    cudaEventElapsedTime(&t01, ctx->ev[0], ctx->ev[1]);
    cudaEventElapsedTime(&t23, ctx->ev[2], ctx->ev[3]);
    cudaEventElapsedTime(&t34, ctx->ev[3], ctx->ev[4]);
    cudaEventElapsedTime(&t04, ctx->ev[0], ctx->ev[4]);
    sum.t_setup_s = t01 * 1e-3;  // includes the overlapped upload
    sum.t_loop_s = t23 * 1e-3;
    sum.t_finish_s = t34 * 1e-3;
    sum.t_total_s = t04 * 1e-3;
    sum.residual_sq = hres;
    sum.n = n;
    sum.m = m;
    sum.n_dropped = n - m;
  }
  ctx->last = sum;
  if (out) *out = sum;
  return ALNNLS_OK;
}

}  // namespace

extern "C" {

int alnnls_abi_version(void) { return ALNNLS_ABI_VERSION; }

void alnnls_config_default(alnnls_config* cfg) {
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->stall_window = 50;
  cfg->trace_every = 1;
  cfg->profile = ALNNLS_PROFILE_EXACT;
  cfg->record_multiplies = 1;
}

int alnnls_create(alnnls_ctx** out, int device) {
  if (!out) return ALNNLS_EINVAL;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count <= device || device < 0)
    return ALNNLS_ENODEV;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return ALNNLS_ENODEV;
  if (prop.major != 10) return ALNNLS_ENODEV;  // sm_100a code only
  auto* c = new alnnls_ctx();
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  c->cc_major = prop.major;
  c->cc_minor = prop.minor;
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return ALNNLS_ENODEV;
  }
  for (auto& e : c->ev) cudaEventCreate(&e);
  for (auto& e : c->up) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking);
  *out = c;
  return ALNNLS_OK;
}

void alnnls_destroy(alnnls_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  DevBuf* bufs[] = {&ctx->A,      &ctx->b,     &ctx->Q,       &ctx->q,     &ctx->x,    &ctx->g,
                    &ctx->y_out,  &ctx->u,     &ctx->gd,      &ctx->mask,  &ctx->gP,   &ctx->chg,
                    &ctx->dC,     &ctx->candC, &ctx->gC,      &ctx->prod0, &ctx->prod1, &ctx->prod2,
                    &ctx->diag,   &ctx->pos,   &ctx->scale,   &ctx->retained, &ctx->mscalar,
                    &ctx->trace,  &ctx->mults, &ctx->ctrl,    &ctx->list,  &ctx->vals, &ctx->ax,
                    &ctx->resid,  &ctx->flag,  &ctx->H,       &ctx->hvec,  &ctx->start, &ctx->bcols,
                    &ctx->X,      &ctx->x_alt, &ctx->mask2,   &ctx->gP2,   &ctx->xP2,  &ctx->qP2,
                    &ctx->part,   &ctx->resb,  &ctx->yb,      &ctx->qb,   &ctx->uP,   &ctx->gdC,
                    &ctx->skp,    &ctx->skf,   &ctx->ay,      &ctx->axn,   &ctx->aw,
                    &ctx->avy,    &ctx->apc,   &ctx->tst,   &ctx->fgb0,  &ctx->fgb1,
                    &ctx->fpart,  &ctx->fden,  &ctx->fkl,   &ctx->fkv,   &ctx->fkc,
                    &ctx->dmws,   &ctx->dmfl,  &ctx->nvt,   &ctx->nht,   &ctx->nwt,
                    &ctx->nv,     &ctx->nw,    &ctx->nh,    &ctx->qfrag, &ctx->bcnt};
  for (DevBuf* b : bufs)
    if (b->p) cudaFree(b->p);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : ctx->up)
    if (e) cudaEventDestroy(e);
  for (auto& e : ctx->bev)
    if (e) cudaEventDestroy(e);
  for (auto& t : ctx->bstream)
    if (t) cudaStreamDestroy(t);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->pin) cudaFreeHost(ctx->pin);
  delete ctx;
}

const char* alnnls_last_error(const alnnls_ctx* ctx) { return ctx ? ctx->err.c_str() : "no context"; }

int alnnls_device_info(alnnls_ctx* ctx, int* sm_count, int* cc_major, int* cc_minor) {
  if (!ctx) return ALNNLS_EINVAL;
  if (sm_count) *sm_count = ctx->sm_count;
  if (cc_major) *cc_major = ctx->cc_major;
  if (cc_minor) *cc_minor = ctx->cc_minor;
  return ALNNLS_OK;
}

int alnnls_solve_nnls_device(alnnls_ctx* ctx, uint64_t d, uint64_t n, const double* dA,
                             uint64_t lda, const double* db, const alnnls_config* cfg,
                             alnnls_summary* out) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!cfg || !dA || !db) return set_err(ctx, ALNNLS_EINVAL, "solve_nnls: null argument");
  if (d < 1 || n < 1) return set_err(ctx, ALNNLS_EINVAL, "DenseMatrix: rows and cols must be >= 1");
  if (lda < d) return set_err(ctx, ALNNLS_EINVAL, "solve_nnls: lda < rows");
  int st__ = ALNNLS_OK;
  int* flag = ENSURE(int, flag, 1);
  CK(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
  CK(launch_check_finite(dA, d, n, lda, flag, ctx->stream));
  CK(launch_check_finite(db, d, 1, d, flag, ctx->stream));
  int hf = 0;
  if ((rc = copy_out(ctx, &hf, flag, sizeof(int)))) return rc;
  if (hf) return set_err(ctx, ALNNLS_EINVAL, "DenseMatrix: non-finite entry");
  // the bulk-copy GEMV on A needs an even lda and 16B-aligned columns
  if ((lda & 1) || (reinterpret_cast<uintptr_t>(dA) & 15)) {
    const uint64_t ld = round_up(d, 4);
    double* dst = ENSURE(double, A, ld * n);
    CK(launch_copy_pad(dA, lda, dst, ld, d, n, ctx->stream));
    dA = dst;
    lda = ld;
  }
  return run_nnls(ctx, d, n, dA, lda, db, cfg, out);
}

int alnnls_solve_nnls(alnnls_ctx* ctx, uint64_t d, uint64_t n, const double* A, const double* b,
                      const alnnls_config* cfg, alnnls_summary* out) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!cfg || !A || !b) return set_err(ctx, ALNNLS_EINVAL, "solve_nnls: null argument");
  if (d < 1 || n < 1) return set_err(ctx, ALNNLS_EINVAL, "DenseMatrix: rows and cols must be >= 1");
  // large problems: overlap the upload of A with the Gram (row blocks)
  if (d >= 4096 && n >= 1024 && n <= 46340 && d * n >= (uint64_t)1 << 24)
    return run_nnls_overlapped(ctx, d, n, A, b, cfg, out);
  int st__ = ALNNLS_OK;
  uint64_t lda = 0;
  if ((rc = upload_matrix(ctx, ctx->A, d, n, A, &lda))) return rc;
  double* db = ENSURE(double, b, d);
  CK(cudaMemcpyAsync(db, b, sizeof(double) * d, cudaMemcpyHostToDevice, ctx->stream));
  double* dA = static_cast<double*>(ctx->A.p);
  if ((rc = device_check_finite(ctx, {{dA, d, n, lda, "DenseMatrix: non-finite entry"},
                                      {db, d, 1, d, "Vector: non-finite entry"}})))
    return rc;
  return run_nnls(ctx, d, n, dA, lda, db, cfg, out);
}

int alnnls_solve_nqp_device(alnnls_ctx* ctx, uint64_t m, const double* dQ, uint64_t ldq,
                            const double* dq, const double* dstart, const alnnls_config* cfg,
                            alnnls_summary* out) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!cfg || !dQ || !dq) return set_err(ctx, ALNNLS_EINVAL, "solve_nqp: null argument");
  if (m < 1) return set_err(ctx, ALNNLS_EINVAL, "DenseMatrix: rows and cols must be >= 1");
  if (ldq < m) return set_err(ctx, ALNNLS_EINVAL, "solve_nqp: ldq < m");
  int st__ = ALNNLS_OK;
  {
    // the reference's construction-time checks, in its order, on the device copies:
    // finite Q and q (linalg.hpp:42-52, :84), symmetric Q (nqp.hpp:37-41); after the
    // config (nqp.hpp:219-222): a finite, nonnegative start (nqp.hpp:227-230)
    int* flag = ENSURE(int, flag, 8);
    CK(cudaMemsetAsync(flag, 0, sizeof(int) * 5, ctx->stream));
    CK(launch_check_finite(dQ, m, m, ldq, flag + 0, ctx->stream));
    CK(launch_check_finite(dq, m, 1, m, flag + 1, ctx->stream));
    CK(launch_check_matrix(dQ, m, m, ldq, 0, flag + 2, ctx->stream));
    if (dstart) {
      CK(launch_check_finite(dstart, m, 1, m, flag + 3, ctx->stream));
      CK(launch_check_matrix(dstart, m, 1, m, 1, flag + 4, ctx->stream));
    }
    int hf[5] = {0, 0, 0, 0, 0};
    if ((rc = copy_out(ctx, hf, flag, sizeof(hf)))) return rc;
    if (hf[0]) return set_err(ctx, ALNNLS_EINVAL, "DenseMatrix: non-finite entry");
    if (hf[1]) return set_err(ctx, ALNNLS_EINVAL, "Vector: non-finite entry");
    if (hf[2]) return set_err(ctx, ALNNLS_EINVAL, "NqpProblem: Q must be symmetric");
    Resolved r0;
    if ((rc = resolve(ctx, cfg, m, &r0))) return rc;
    if (hf[3]) return set_err(ctx, ALNNLS_EINVAL, "Vector: non-finite entry");
    if (hf[4]) return set_err(ctx, ALNNLS_EINVAL, "solve_nqp: start must be nonnegative");
  }
  Resolved r;
  if ((rc = resolve(ctx, cfg, m, &r))) return rc;
  ctx->qR = (uint64_t)nqp_rows_per_cta((int)m, ctx->sm_count);
  double* Qd = ENSURE(double, Q, blocked_size(m, ctx->qR));
  CK(launch_to_blocked(dQ, ldq, (int)m, (int)ctx->qR, Qd, ctx->stream));
  double* qd = ENSURE(double, q, vec_pad(m));
  CK(cudaMemcpyAsync(qd, dq, sizeof(double) * m, cudaMemcpyDeviceToDevice, ctx->stream));
  ctx->last_nnls = false;
  ctx->last_n = m;
  ctx->last_m = m;
  alnnls_summary sum{};
  rc = run_nqp(ctx, m, r, cfg, dstart, &sum, ctx->solver);
  sum.n = m;
  ctx->last = sum;
  if (out) *out = sum;
  return rc;
}

int alnnls_solve_nqp(alnnls_ctx* ctx, uint64_t m, const double* Q, const double* q,
                     const double* start, const alnnls_config* cfg, alnnls_summary* out) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!cfg || !Q || !q) return set_err(ctx, ALNNLS_EINVAL, "solve_nqp: null argument");
  if (m < 1) return set_err(ctx, ALNNLS_EINVAL, "DenseMatrix: rows and cols must be >= 1");
  if (!all_finite(Q, m * m)) return set_err(ctx, ALNNLS_EINVAL, "DenseMatrix: non-finite entry");
  if (!all_finite(q, m)) return set_err(ctx, ALNNLS_EINVAL, "Vector: non-finite entry");
  for (uint64_t j = 0; j < m; ++j)  // NqpProblem (nqp.hpp:37-41)
    for (uint64_t i = 0; i < j; ++i)
      if (!(Q[j * m + i] == Q[i * m + j]))
        return set_err(ctx, ALNNLS_EINVAL, "NqpProblem: Q must be symmetric");
  Resolved r;
  if ((rc = resolve(ctx, cfg, m, &r))) return rc;
  if (start) {
    if (!all_finite(start, m)) return set_err(ctx, ALNNLS_EINVAL, "Vector: non-finite entry");
    for (uint64_t i = 0; i < m; ++i)  // nqp.hpp:227-230
      if (!(start[i] >= 0.0))
        return set_err(ctx, ALNNLS_EINVAL, "solve_nqp: start must be nonnegative");
  }
  int st__ = ALNNLS_OK;
  uint64_t ld = 0;
  (void)ld;
  double* Qtmp = ENSURE(double, H, m * m);
  CK(cudaMemcpyAsync(Qtmp, Q, sizeof(double) * m * m, cudaMemcpyHostToDevice, ctx->stream));
  ctx->qR = (uint64_t)nqp_rows_per_cta((int)m, ctx->sm_count);
  double* Qd = ENSURE(double, Q, blocked_size(m, ctx->qR));
  CK(launch_to_blocked(Qtmp, m, (int)m, (int)ctx->qR, Qd, ctx->stream));
  double* qd = ENSURE(double, q, vec_pad(m));
  CK(cudaMemcpyAsync(qd, q, sizeof(double) * m, cudaMemcpyHostToDevice, ctx->stream));
  double* ds = nullptr;
  if (start) {
    ds = ENSURE(double, start, m);
    CK(cudaMemcpyAsync(ds, start, sizeof(double) * m, cudaMemcpyHostToDevice, ctx->stream));
  }
  ctx->last_nnls = false;
  ctx->last_n = m;
  ctx->last_m = m;
  alnnls_summary sum{};
  rc = run_nqp(ctx, m, r, cfg, ds, &sum, ctx->solver);
  sum.n = m;
  sum.t_total_s = sum.t_loop_s;
  ctx->last = sum;
  if (out) *out = sum;
  return rc;
}

int alnnls_get_x(alnnls_ctx* ctx, double* x, uint64_t len) {
  if (!ctx || !x) return ALNNLS_EINVAL;
  const uint64_t n = ctx->last_nnls ? ctx->last_n : ctx->last_m;
  if (len < n) return set_err(ctx, ALNNLS_ECAPACITY, "get_x: buffer too small");
  const void* src = ctx->last_nnls ? ctx->X.p : (ctx->g_parity ? ctx->x_alt.p : ctx->x.p);
  return copy_out(ctx, x, src, sizeof(double) * n);
}

int alnnls_get_inner_x(alnnls_ctx* ctx, double* y, uint64_t len) {
  if (!ctx || !y) return ALNNLS_EINVAL;
  if (len < ctx->last_m) return set_err(ctx, ALNNLS_ECAPACITY, "get_inner_x: buffer too small");
  return copy_out(ctx, y,
                  ctx->last_nnls ? ctx->y_out.p : (ctx->g_parity ? ctx->x_alt.p : ctx->x.p),
                  sizeof(double) * ctx->last_m);
}

int alnnls_get_final_grad(alnnls_ctx* ctx, double* g, uint64_t len) {
  if (!ctx || !g) return ALNNLS_EINVAL;
  if (len < ctx->last_m) return set_err(ctx, ALNNLS_ECAPACITY, "get_final_grad: buffer too small");
  return copy_out(ctx, g, ctx->g_parity ? ctx->prod1.p : ctx->g.p, sizeof(double) * ctx->last_m);
}

int alnnls_get_trace(alnnls_ctx* ctx, alnnls_iter_record* rec, uint64_t cap) {
  if (!ctx || !rec) return ALNNLS_EINVAL;
  // never past what the device buffer holds (trace_len is clamped by run_nqp too)
  const uint64_t n = std::min<uint64_t>(ctx->last.trace_len,
                                        ctx->trace.bytes / sizeof(alnnls_iter_record));
  if (cap < n) return set_err(ctx, ALNNLS_ECAPACITY, "get_trace: buffer too small");
  return copy_out(ctx, rec, ctx->trace.p, sizeof(alnnls_iter_record) * n);
}

int alnnls_get_multiplies(alnnls_ctx* ctx, uint64_t* mults, uint64_t cap) {
  if (!ctx || !mults) return ALNNLS_EINVAL;
  const uint64_t n = std::min<uint64_t>(ctx->last.mult_len, ctx->mults.bytes / sizeof(uint64_t));
  if (cap < n) return set_err(ctx, ALNNLS_ECAPACITY, "get_multiplies: buffer too small");
  return copy_out(ctx, mults, ctx->mults.p, sizeof(uint64_t) * n);
}

int alnnls_timer_start(alnnls_ctx* ctx) {
  if (!ctx) return ALNNLS_EINVAL;
  if (!ctx->timer[0]) {
    cudaEventCreate(&ctx->timer[0]);
    cudaEventCreate(&ctx->timer[1]);
  }
  CK(cudaEventRecord(ctx->timer[0], ctx->stream));
  return ALNNLS_OK;
}

int alnnls_timer_stop(alnnls_ctx* ctx, double* seconds) {
  if (!ctx || !seconds) return ALNNLS_EINVAL;
  CK(cudaEventRecord(ctx->timer[1], ctx->stream));
  CK(cudaEventSynchronize(ctx->timer[1]));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, ctx->timer[0], ctx->timer[1]));
  *seconds = ms * 1e-3;
  return ALNNLS_OK;
}

uint64_t alnnls_launch_count(const alnnls_ctx* ctx) { return ctx ? ctx->launches : 0; }
int alnnls_last_loop_kernel(const alnnls_ctx* ctx) { return ctx ? ctx->loop_kernel : 0; }

int alnnls_get_phase_ns(alnnls_ctx* ctx, uint64_t* ns, uint64_t cap) {
  if (!ctx || !ns) return ALNNLS_EINVAL;
  for (uint64_t i = 0; i < cap && i < 8; ++i) ns[i] = ctx->phase_ns[i];
  return ALNNLS_OK;
}

int alnnls_get_scale(alnnls_ctx* ctx, double* scale, uint64_t cap) {
  if (!ctx || !scale) return ALNNLS_EINVAL;
  if (cap < ctx->last_m) return set_err(ctx, ALNNLS_ECAPACITY, "get_scale: buffer too small");
  return copy_out(ctx, scale, ctx->scale.p, sizeof(double) * ctx->last_m);
}

int alnnls_get_retained(alnnls_ctx* ctx, uint64_t* idx, uint64_t cap) {
  if (!ctx || !idx) return ALNNLS_EINVAL;
  const uint64_t m = ctx->last_m;
  if (cap < m) return set_err(ctx, ALNNLS_ECAPACITY, "get_retained: buffer too small");
  std::vector<uint32_t> tmp(m);
  int rc = copy_out(ctx, tmp.data(), ctx->retained.p, sizeof(uint32_t) * m);
  for (uint64_t i = 0; i < m; ++i) idx[i] = tmp[i];
  return rc;
}

int alnnls_get_dropped(alnnls_ctx* ctx, uint64_t* idx, uint64_t cap) {
  if (!ctx || !idx) return ALNNLS_EINVAL;
  const uint64_t n = ctx->last_n, m = ctx->last_m;
  if (cap < n - m) return set_err(ctx, ALNNLS_ECAPACITY, "get_dropped: buffer too small");
  std::vector<int> pos(n);
  int rc = copy_out(ctx, pos.data(), ctx->pos.p, sizeof(int) * n);
  uint64_t k = 0;
  for (uint64_t i = 0; i < n; ++i)
    if (pos[i] < 0) idx[k++] = i;
  return rc;
}

int alnnls_setup(alnnls_ctx* ctx, uint64_t d, uint64_t n, const double* A, const double* b,
                 alnnls_summary* out) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!A || !b) return set_err(ctx, ALNNLS_EINVAL, "setup: null argument");
  if (d < 1 || n < 1) return set_err(ctx, ALNNLS_EINVAL, "DenseMatrix: rows and cols must be >= 1");
  if (!all_finite(A, d * n) || !all_finite(b, d))
    return set_err(ctx, ALNNLS_EINVAL, "DenseMatrix: non-finite entry");
  int st__ = ALNNLS_OK;
  uint64_t lda = 0;
  if ((rc = upload_matrix(ctx, ctx->A, d, n, A, &lda))) return rc;
  double* db = ENSURE(double, b, d);
  CK(cudaMemcpyAsync(db, b, sizeof(double) * d, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaEventRecord(ctx->ev[0], ctx->stream));
  uint64_t m = 0;
  if ((rc = run_setup(ctx, d, n, static_cast<double*>(ctx->A.p), lda, db, &m))) return rc;
  CK(cudaEventRecord(ctx->ev[1], ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  float ms = 0;
  cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
  ctx->last_nnls = true;
  ctx->last_n = n;
  ctx->last_m = m;
  ctx->last = alnnls_summary{};
  ctx->last.n = n;
  ctx->last.m = m;
  ctx->last.n_dropped = n - m;
  ctx->last.t_setup_s = ms * 1e-3;
  if (out) *out = ctx->last;
  return ALNNLS_OK;
}

int alnnls_get_Q(alnnls_ctx* ctx, double* Q, uint64_t cap) {
  if (!ctx || !Q) return ALNNLS_EINVAL;
  const uint64_t m = ctx->last_m;
  if (cap < m * m) return set_err(ctx, ALNNLS_ECAPACITY, "get_Q: buffer too small");
  if (m == 0) return ALNNLS_OK;
  int st__ = ALNNLS_OK;
  double* tmp = ENSURE(double, H, m * m);
  CK(launch_from_blocked(static_cast<double*>(ctx->Q.p), (int)m, (int)ctx->qR, tmp, m,
                         ctx->stream));
  return copy_out(ctx, Q, tmp, sizeof(double) * m * m);
}

int alnnls_get_q(alnnls_ctx* ctx, double* q, uint64_t cap) {
  if (!ctx || !q) return ALNNLS_EINVAL;
  if (cap < ctx->last_m) return set_err(ctx, ALNNLS_ECAPACITY, "get_q: buffer too small");
  return copy_out(ctx, q, ctx->q.p, sizeof(double) * ctx->last_m);
}

int alnnls_rescale(alnnls_ctx* ctx, uint64_t n, const double* H, const double* h,
                   alnnls_summary* out) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!H || !h || n < 1) return set_err(ctx, ALNNLS_EINVAL, "rescale: bad argument");
  for (uint64_t j = 0; j < n; ++j)  // nnls.hpp:45-49
    for (uint64_t i = 0; i < j; ++i)
      if (!(H[j * n + i] == H[i * n + j]))
        return set_err(ctx, ALNNLS_EINVAL, "rescale: H must be symmetric");
  for (uint64_t i = 0; i < n; ++i)  // nnls.hpp:55
    if (!(H[i * n + i] >= 0.0)) return set_err(ctx, ALNNLS_EINVAL, "rescale: negative diagonal entry");
  int st__ = ALNNLS_OK;
  cudaStream_t s = ctx->stream;
  double* dH = ENSURE(double, H, n * n);
  double* dh = ENSURE(double, hvec, n);
  CK(cudaMemcpyAsync(dH, H, sizeof(double) * n * n, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dh, h, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  std::vector<double> diag(n);
  for (uint64_t i = 0; i < n; ++i) diag[i] = H[i * n + i];
  double* ddiag = ENSURE(double, diag, n);
  CK(cudaMemcpyAsync(ddiag, diag.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
  SetupArgs sa{};
  sa.n = (int)n;
  sa.diag = ddiag;
  sa.pos = ENSURE(int, pos, n);
  sa.scale = ENSURE(double, scale, n);
  sa.retained = ENSURE(uint32_t, retained, n);
  sa.m_out = ENSURE(int, mscalar, 4);
  CK(launch_retained(sa, s));
  int hm = 0;
  if ((rc = copy_out(ctx, &hm, sa.m_out, sizeof(int)))) return rc;
  const uint64_t m = (uint64_t)hm;
  const uint64_t mm = m > 0 ? m : 1;
  ctx->qR = (uint64_t)nqp_rows_per_cta((int)mm, ctx->sm_count);
  double* Qd = ENSURE(double, Q, blocked_size(mm, ctx->qR));
  double* qd = ENSURE(double, q, vec_pad(m));
  CK(launch_rescale_from_h(dH, dh, (int)n, sa.pos, sa.scale, Qd, (int)m, (int)ctx->qR, qd, s));
  CK(cudaStreamSynchronize(s));
  ctx->last_nnls = true;
  ctx->last_n = n;
  ctx->last_m = m;
  ctx->last = alnnls_summary{};
  ctx->last.n = n;
  ctx->last.m = m;
  ctx->last.n_dropped = n - m;
  if (out) *out = ctx->last;
  return ALNNLS_OK;
}

int alnnls_gram(alnnls_ctx* ctx, uint64_t d, uint64_t n, const double* A, double* H) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!A || !H || d < 1 || n < 1) return set_err(ctx, ALNNLS_EINVAL, "gram: bad argument");
  int st__ = ALNNLS_OK;
  uint64_t lda = 0;
  if ((rc = upload_matrix(ctx, ctx->A, d, n, A, &lda))) return rc;
  double* dH = ENSURE(double, H, n * n);
  SetupArgs sa{};
  sa.A = static_cast<double*>(ctx->A.p);
  sa.lda = lda;
  sa.b = nullptr;
  sa.d = (int)d;
  sa.n = (int)n;
  sa.H = dH;
  if ((rc = streamk_buffers(ctx, sa, 0))) return rc;
  CK(launch_syrk(sa, 0, ctx->stream));
  return copy_out(ctx, H, dH, sizeof(double) * n * n);
}

int alnnls_transpose_matvec(alnnls_ctx* ctx, uint64_t rows, uint64_t cols, const double* M,
                            const double* v, double* y) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!M || !v || !y || rows < 1 || cols < 1)
    return set_err(ctx, ALNNLS_EINVAL, "transpose_matvec: bad argument");
  int st__ = ALNNLS_OK;
  uint64_t ld = 0;
  if ((rc = upload_matrix(ctx, ctx->A, rows, cols, M, &ld))) return rc;
  double* dv = ENSURE(double, b, rows);
  double* dy = ENSURE(double, ax, cols);
  CK(cudaMemcpyAsync(dv, v, sizeof(double) * rows, cudaMemcpyHostToDevice, ctx->stream));
  CK(launch_atb_chain(static_cast<double*>(ctx->A.p), ld, (int)rows, (int)cols, dv, nullptr, dy,
                      ctx->stream));
  return copy_out(ctx, y, dy, sizeof(double) * cols);
}

int alnnls_masked_matvec(alnnls_ctx* ctx, uint64_t rows, uint64_t cols, const double* M,
                         const double* v, const uint64_t* mask, uint64_t mask_len, double* y,
                         uint64_t* multiply_count) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!M || !v || !y || rows < 1 || cols < 1 || (mask_len && !mask))
    return set_err(ctx, ALNNLS_EINVAL, "masked_matvec: bad argument");
  for (uint64_t t = 0; t < mask_len; ++t)  // linalg.hpp:199
    if (mask[t] >= cols) return set_err(ctx, ALNNLS_ERANGE, "masked_matvec: mask index out of range");
  int st__ = ALNNLS_OK;
  uint64_t ld = 0;
  if ((rc = upload_matrix(ctx, ctx->A, rows, cols, M, &ld))) return rc;
  std::vector<uint32_t> lst(mask_len + 1);
  std::vector<double> vv(mask_len + 2, 0.0);
  for (uint64_t t = 0; t < mask_len; ++t) {
    lst[t] = (uint32_t)mask[t];
    vv[t] = v[mask[t]];
  }
  uint32_t* dl = ENSURE(uint32_t, list, mask_len + 1);
  double* dvals = ENSURE(double, vals, mask_len + 8);
  double* dy = ENSURE(double, ax, rows);
  CK(cudaMemcpyAsync(dl, lst.data(), sizeof(uint32_t) * (mask_len + 1), cudaMemcpyHostToDevice,
                     ctx->stream));
  CK(cudaMemcpyAsync(dvals, vv.data(), sizeof(double) * (mask_len + 2), cudaMemcpyHostToDevice,
                     ctx->stream));
  CK(launch_masked_gemv(static_cast<double*>(ctx->A.p), ld, (int)rows, dl, dvals, (int)mask_len,
                        dy, ctx->sm_count, ctx->stream));
  rc = copy_out(ctx, y, dy, sizeof(double) * rows);
  if (rc == ALNNLS_OK && multiply_count) *multiply_count += rows * mask_len;
  return rc;
}

int alnnls_matvec(alnnls_ctx* ctx, uint64_t rows, uint64_t cols, const double* M,
                  const double* v, double* y) {
  std::vector<uint64_t> all(cols);
  for (uint64_t j = 0; j < cols; ++j) all[j] = j;
  return alnnls_masked_matvec(ctx, rows, cols, M, v, all.data(), cols, y, nullptr);
}

}  // extern "C"

namespace {

// K8 pipeline on device A (d x n, lda) and B (d x nrhs, ldb): per column bitwise
// solve_nnls(A, B[:, j], cfg). X (n x nrhs, ld n) and per-column results.
//
// hB != nullptr (the host-buffer entry): dB is only allocated, and the columns of the host
// B are uploaded in kHostChunks column chunks on the copy stream. Each chunk's finiteness
// check and q formation wait for its own upload only, and the chunks' solves run on two
// alternating streams, so the second chunk's upload hides under the first chunk's solve
// and its persistent CTAs take over the SMs as the first chunk's CTAs retire (columns
// are independent: the per-column results are those of the one-launch path). The first
// chunk is a quarter of the columns: its upload is what stays exposed, its solve is
// longer than the rest of the upload. *bad_b reports a non-finite B (checked after the
// fact; the caller discards the results, as if the DenseMatrix had been validated first).
constexpr int kHostChunks = 2;
int run_batched(alnnls_ctx* ctx, uint64_t d, uint64_t n, const double* dA, uint64_t lda,
                uint64_t nrhs, const double* dB, uint64_t ldb, const alnnls_config* cfg,
                double* dX, alnnls_column_result* cols, alnnls_summary* out,
                const double* hB = nullptr, int* bad_b = nullptr) {
  int st__ = ALNNLS_OK;
  cudaStream_t s = ctx->stream, cs = ctx->copy_stream;
  alnnls_summary sum{};
  // column chunks [edge[c], edge[c + 1])
  uint64_t edge[kHostChunks + 1] = {0, nrhs, nrhs};
  int nch = 1;
  // ALNNLS_BATCH_OVERLAP_MIN: the smallest batch that is chunked (default 64 columns per
  // SM: below it the upload is short and the extra launch's tail is not); 0 turns it off
  const char* omin = getenv("ALNNLS_BATCH_OVERLAP_MIN");
  const uint64_t min_cols = omin ? (uint64_t)atoll(omin) : (uint64_t)64 * ctx->sm_count;
  if (hB && min_cols > 0 && nrhs >= min_cols && nrhs >= 64) {
    nch = 2;
    edge[1] = (nrhs / 4 + 15) / 16 * 16;
  }
  if (nch > 1 && !ctx->bstream[0]) {
    for (auto& t : ctx->bstream) CK(cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking));
    for (auto& e : ctx->bev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  CK(cudaEventRecord(ctx->ev[0], s));
  int* bflag = nullptr;
  // chunk c's upload on the copy stream (a pageable B makes the call block: chunk c + 1 is
  // therefore enqueued after chunk c's launches, which then run under it)
  auto upload_chunk = [&](int c) -> int {
    const uint64_t c0 = edge[c], cnt = edge[c + 1] - c0;
    CK(cudaMemcpy2DAsync(const_cast<double*>(dB) + c0 * ldb, ldb * sizeof(double), hB + c0 * d,
                         d * sizeof(double), d * sizeof(double), cnt, cudaMemcpyHostToDevice, cs));
    CK(cudaEventRecord(ctx->up[c], cs));
    return ALNNLS_OK;
  };
  if (hB) {
    int* fl = ENSURE(int, flag, 4);
    bflag = fl + 1;
    CK(cudaMemsetAsync(bflag, 0, sizeof(int), s));
    CK(cudaStreamWaitEvent(cs, ctx->ev[0], 0));
    if (int urc = upload_chunk(0)) return urc;
  }
  uint64_t m = 0;
  int rc = run_setup(ctx, d, n, dA, lda, nullptr, &m, cfg->profile);  // the shared Gram, once
  if (rc) return rc;
  alnnls_column_result* dres = ENSURE(alnnls_column_result, resb, nrhs);
  std::vector<alnnls_column_result> init(nrhs);
  for (auto& r : init) {  // empty_solve_result (nnls.hpp:107-113) when every column is dropped
    std::memset(&r, 0, sizeof(r));
    r.termination = ALNNLS_EMPTY_PASSIVE_SET;
  }
  CK(cudaMemcpyAsync(dres, init.data(), sizeof(alnnls_column_result) * nrhs,
                     cudaMemcpyHostToDevice, s));
  double* Y = ENSURE(double, yb, (m ? m : 1) * nrhs);
  Resolved r{};
  bool wide = false;
  std::vector<alnnls_column_result> wres;
  double wide_loop_s = 0.0;
  double* Qc = nullptr;
  double* QB = nullptr;
  int* counter = nullptr;
  BatchArgs ba{};
  const bool dmma_q = m > 0 && cfg->profile == ALNNLS_PROFILE_FAST;
  if (m > 0) {
    if ((rc = resolve(ctx, cfg, m, &r))) return rc;  // solve_nqp validates its config
    // m > 1024 does not fit the batched kernel's shared-memory state: those columns go one
    // at a time through the single-RHS device loop on the shared blocked Q (same per-column
    // results as solve_nnls; any m that entry takes)
    wide = batched_cols_per_cta((int)m) == 0;
    if (!wide) {
      Qc = ENSURE(double, H, m * m);
      CK(launch_from_blocked(static_cast<double*>(ctx->Q.p), (int)m, (int)ctx->qR, Qc, m, s));
    } else {
      wres.resize(nrhs);
    }
    QB = ENSURE(double, qb, m * nrhs);
    counter = ENSURE(int, bcnt, kHostChunks);
    CK(cudaMemsetAsync(counter, 0, sizeof(int) * kHostChunks, s));
    ba.Q = Qc;
    ba.m = (int)m;
    ba.eps = r.eps;
    ba.max_iters = r.max_iters;
    ba.stall_window = cfg->stall_window;
    ba.fast = cfg->profile == ALNNLS_PROFILE_FAST;
    ba.total_cols = (int)nrhs;
    // FAST, m <= 256: Q re-laid in DMMA fragment order for the tensor-core passes
    ba.Qf = nullptr;
    if (ba.fast && m <= 256) {
      double* qf = ENSURE(double, qfrag, (size_t)((m + 15) & ~15) * 256);
      ba.Qf = qf;
      if (nch > 1) {  // once, before the chunks' launches on two streams read it
        CK(launch_qfrag(ba, s));
        ba.qf_ready = 1;
      }
    }
  }
  for (int c = 0; c < nch; ++c) {
    const uint64_t c0 = edge[c], cnt = edge[c + 1] - c0;
    if (hB) {
      CK(cudaStreamWaitEvent(s, ctx->up[c], 0));
      CK(launch_check_finite(dB + c0 * ldb, d, cnt, ldb, bflag, s));
    }
    cudaStream_t ts = nch > 1 && !wide ? ctx->bstream[c & 1] : s;
    if (m > 0) {
      SetupArgs sa{};
      sa.A = dA;
      sa.lda = lda;
      sa.d = (int)d;
      sa.n = (int)n;
      sa.pos = static_cast<int*>(ctx->pos.p);
      sa.scale = static_cast<double*>(ctx->scale.p);
      sa.m = (int)m;
      sa.B = dB + c0 * ldb;
      sa.ldb = ldb;
      sa.nrhs = (int)cnt;
      sa.QB = QB + c0 * m;
      // q_j = (-(A^T b_j))[retained] / D for every column of the chunk
      if (dmma_q && syrk_dmma_supported(sa, 2)) {
        if ((rc = dmma_buffers(ctx, sa))) return rc;
        CK(launch_syrk_dmma(sa, 2, s));
      } else {
        if ((rc = streamk_buffers(ctx, sa, 2))) return rc;
        CK(launch_syrk(sa, 2, s));
      }
    }
    if (c == 0) {
      CK(cudaEventRecord(ctx->ev[1], s));
      CK(cudaEventRecord(ctx->ev[2], s));
    }
    if (nch > 1) {
      CK(cudaEventRecord(ctx->bev[2 * c], s));
      CK(cudaStreamWaitEvent(ts, ctx->bev[2 * c], 0));
    }
    if (m > 0 && wide) {
      double* qv = ENSURE(double, q, vec_pad(m));
      for (uint64_t j = c0; j < c0 + cnt; ++j) {
        CK(cudaMemcpyAsync(qv, QB + j * m, sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
        alnnls_summary cs{};
        rc = run_nqp(ctx, m, r, cfg, nullptr, &cs, 0, /*defer=*/true);
        if (rc) return rc;
        CK(launch_copy_parity(Y + j * m, static_cast<double*>(ctx->x.p),
                              static_cast<double*>(ctx->x_alt.p),
                              static_cast<LoopCtrl*>(ctx->ctrl.p), (int)m, s));
        CK(cudaStreamSynchronize(s));
        rc = collect_nqp(ctx, &cs);
        if (rc && rc != ALNNLS_ENUMERIC) return rc;  // a NumericFailure column is a result
        wide_loop_s += cs.t_loop_s;
        alnnls_column_result& w = wres[j];
        w.termination = cs.numeric_failure ? 0 : cs.termination;
        w.numeric_failure = cs.numeric_failure;
        w.iterations = cs.iterations;
        w.residual_sq = 0.0;
        w.f_final = cs.f_final;
        w.gbs_final = cs.gbs_final;
        w.multiplies_total = cs.multiplies_total;
      }
      CK(cudaMemcpyAsync(dres + c0, wres.data() + c0, sizeof(alnnls_column_result) * cnt,
                         cudaMemcpyHostToDevice, s));
      CK(cudaEventRecord(ctx->ev[2], s));  // run_nqp re-records ev[2] / ev[3] per column
    } else if (m > 0) {
      BatchArgs bc = ba;
      bc.QB = QB + c0 * m;
      bc.ncols = (int)cnt;
      bc.Y = Y + c0 * m;
      bc.res = dres + c0;
      bc.next_col = counter + c;
      CK(launch_batched(bc, ctx->sm_count, ts));
    }
    if (nch == 1) CK(cudaEventRecord(ctx->ev[3], s));
    CK(launch_unscale_batched(Y + c0 * m, (int)m, static_cast<double*>(ctx->scale.p),
                              static_cast<uint32_t*>(ctx->retained.p), dX + c0 * n, (int)n,
                              (int)cnt, ts));
    if (cfg->profile == ALNNLS_PROFILE_FAST &&
        residual_dmma_supported(dA, lda, (int)d, (int)n, (int)cnt)) {
      CK(launch_residual_batched_dmma(dA, lda, (int)d, (int)n, dX + c0 * n, dB + c0 * ldb, ldb,
                                      (int)cnt, dres + c0, ts));
    } else {
      CK(launch_residual_batched(dA, lda, (int)d, (int)n, dX + c0 * n, dB + c0 * ldb, ldb,
                                 (int)cnt, dres + c0, ts));
    }
    if (nch > 1) CK(cudaEventRecord(ctx->bev[2 * c + 1], ts));
    if (hB && c + 1 < nch)
      if (int urc = upload_chunk(c + 1)) return urc;
  }
  if (nch > 1) {  // join: the chunked loop time includes each chunk's unscale and residual
    for (int c = 0; c < nch; ++c) CK(cudaStreamWaitEvent(s, ctx->bev[2 * c + 1], 0));
    CK(cudaEventRecord(ctx->ev[3], s));
  }
  CK(cudaEventRecord(ctx->ev[4], s));
  if (cols) {
    CK(cudaMemcpyAsync(cols, dres, sizeof(alnnls_column_result) * nrhs, cudaMemcpyDeviceToHost, s));
  }
  int hbad = 0;
  if (hB) CK(cudaMemcpyAsync(&hbad, bflag, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (bad_b) *bad_b = hbad;
  float t01 = 0, t23 = 0, t34 = 0, t04 = 0;
  cudaEventElapsedTime(&t01, ctx->ev[0], ctx->ev[1]);
  cudaEventElapsedTime(&t23, ctx->ev[2], ctx->ev[3]);
  cudaEventElapsedTime(&t34, ctx->ev[3], ctx->ev[4]);
  cudaEventElapsedTime(&t04, ctx->ev[0], ctx->ev[4]);
  sum.t_setup_s = t01 * 1e-3;
  sum.t_loop_s = wide ? wide_loop_s : t23 * 1e-3;
  sum.t_finish_s = t34 * 1e-3;
  sum.t_total_s = t04 * 1e-3;
  sum.n = n;
  sum.m = m;
  sum.n_dropped = n - m;
  if (cols) {
    for (uint64_t j = 0; j < nrhs; ++j) {
      sum.multiplies_total += cols[j].multiplies_total;
      sum.iterations += cols[j].iterations;  // total iterations over all columns
      if (cols[j].numeric_failure) sum.numeric_failure = 1;
    }
  }
  ctx->last = sum;
  if (out) *out = sum;
  return ALNNLS_OK;
}

}  // namespace

extern "C" {

int alnnls_solve_nnls_batched_device(alnnls_ctx* ctx, uint64_t d, uint64_t n, const double* dA,
                                     uint64_t nrhs, const double* dB, const alnnls_config* cfg,
                                     double* dX, alnnls_column_result* cols, alnnls_summary* out) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!cfg || !dA || !dB || !dX) return set_err(ctx, ALNNLS_EINVAL, "solve_nnls_batched: null argument");
  if (d < 1 || n < 1 || nrhs < 1)
    return set_err(ctx, ALNNLS_EINVAL, "DenseMatrix: rows and cols must be >= 1");
  int st__ = ALNNLS_OK;
  int* flag = ENSURE(int, flag, 1);
  CK(cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
  CK(launch_check_finite(dA, d, n, d, flag, ctx->stream));
  CK(launch_check_finite(dB, d, nrhs, d, flag, ctx->stream));
  int hf = 0;
  if ((rc = copy_out(ctx, &hf, flag, sizeof(int)))) return rc;
  if (hf) return set_err(ctx, ALNNLS_EINVAL, "DenseMatrix: non-finite entry");
  return run_batched(ctx, d, n, dA, d, nrhs, dB, d, cfg, dX, cols, out);
}

int alnnls_solve_nnls_batched(alnnls_ctx* ctx, uint64_t d, uint64_t n, const double* A,
                              uint64_t nrhs, const double* B, const alnnls_config* cfg, double* X,
                              alnnls_column_result* cols, alnnls_summary* out) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!cfg || !A || !B || !X) return set_err(ctx, ALNNLS_EINVAL, "solve_nnls_batched: null argument");
  if (d < 1 || n < 1 || nrhs < 1)
    return set_err(ctx, ALNNLS_EINVAL, "DenseMatrix: rows and cols must be >= 1");
  int st__ = ALNNLS_OK;
  uint64_t lda = 0, ldb = 0;
  if ((rc = upload_matrix(ctx, ctx->A, d, n, A, &lda))) return rc;
  if ((rc = device_check_finite(
           ctx, {{static_cast<double*>(ctx->A.p), d, n, lda, "DenseMatrix: non-finite entry"}})))
    return rc;
  ldb = round_up(d, 4);
  double* dB = ENSURE(double, bcols, ldb * nrhs);
  double* dX = ENSURE(double, X, n * nrhs);
  int bad_b = 0;
  rc = run_batched(ctx, d, n, static_cast<double*>(ctx->A.p), lda, nrhs, dB, ldb, cfg, dX, cols,
                   out, B, &bad_b);  // uploads B in column chunks under the solves
  if (rc) return rc;
  if (bad_b) return set_err(ctx, ALNNLS_EINVAL, "DenseMatrix: non-finite entry");
  return copy_out(ctx, X, dX, sizeof(double) * n * nrhs);
}

// ---- multi-GPU exact setup by row blocks ----------------------------------------------

uint64_t alnnls_gram_tiles(uint64_t n) { return gram_tiles(n); }

int alnnls_gram_rowblock_device(alnnls_ctx* ctx, uint64_t rows, uint64_t n, const double* dA,
                                uint64_t lda, uint64_t tile_lo, uint64_t tile_hi,
                                const double* dpin, double* dpout, double* dH) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!dA || rows < 1 || n < 1 || lda < rows || tile_hi < tile_lo || tile_hi > gram_tiles(n) ||
      (!dpout && !dH))
    return set_err(ctx, ALNNLS_EINVAL, "gram_rowblock: bad argument");
  SetupArgs sa{};
  sa.A = dA;
  sa.lda = lda;
  sa.d = (int)rows;
  sa.n = (int)n;
  sa.H = dH;
  CK(launch_syrk_rowblock(sa, (int)tile_lo, (int)(tile_hi - tile_lo), dpin, dpout, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return ALNNLS_OK;
}

int alnnls_gram_partial_device(alnnls_ctx* ctx, uint64_t rows, uint64_t n, const double* dA,
                               uint64_t lda, const double* db, int profile, double* dH,
                               double* datb) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!dA || !dH || rows < 1 || n < 1 || lda < rows || (db && !datb))
    return set_err(ctx, ALNNLS_EINVAL, "gram_partial: bad argument");
  if (profile != ALNNLS_PROFILE_EXACT && profile != ALNNLS_PROFILE_FAST)
    return set_err(ctx, ALNNLS_EINVAL, "gram_partial: unknown profile");
  int st__ = ALNNLS_OK;
  SetupArgs sa{};
  sa.A = dA;
  sa.lda = lda;
  sa.b = nullptr;
  sa.d = (int)rows;
  sa.n = (int)n;
  sa.H = dH;
  if (profile == ALNNLS_PROFILE_FAST && syrk_dmma_supported(sa, 0)) {
    if ((rc = dmma_buffers(ctx, sa))) return rc;
    CK(launch_syrk_dmma(sa, 0, ctx->stream));
  } else {
    if ((rc = streamk_buffers(ctx, sa, 0))) return rc;
    CK(launch_syrk(sa, 0, ctx->stream));
  }
  if (db) CK(launch_atb_chain(dA, lda, (int)rows, (int)n, db, nullptr, datb, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return ALNNLS_OK;
}

int alnnls_atb_rowblock_device(alnnls_ctx* ctx, uint64_t rows, uint64_t n, const double* dA,
                               uint64_t lda, const double* db, const double* dpin, double* dout) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!dA || !db || !dout || rows < 1 || n < 1 || lda < rows)
    return set_err(ctx, ALNNLS_EINVAL, "atb_rowblock: bad argument");
  CK(launch_atb_chain(dA, lda, (int)rows, (int)n, db, dpin, dout, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return ALNNLS_OK;
}

int alnnls_solve_nnls_gram_device(alnnls_ctx* ctx, uint64_t n, const double* dH,
                                  const double* dAtb, const alnnls_config* cfg,
                                  alnnls_summary* out) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!dH || !dAtb || !cfg || n < 1) return set_err(ctx, ALNNLS_EINVAL, "solve_nnls_gram: bad argument");
  int st__ = ALNNLS_OK;
  cudaStream_t s = ctx->stream;
  alnnls_summary sum{};
  CK(cudaEventRecord(ctx->ev[0], s));
  // rescale (nnls.hpp:41-83) from H and h = -A^T b
  SetupArgs sa{};
  sa.n = (int)n;
  sa.diag = ENSURE(double, diag, n);
  sa.pos = ENSURE(int, pos, n);
  sa.scale = ENSURE(double, scale, n);
  sa.retained = ENSURE(uint32_t, retained, n);
  sa.m_out = ENSURE(int, mscalar, 4);
  double* h = ENSURE(double, hvec, n);
  CK(launch_diag(dH, (int)n, sa.diag, s));
  CK(launch_negate(dAtb, (int)n, h, s));
  CK(launch_retained(sa, s));
  int hm = 0;
  CK(cudaMemcpyAsync(&hm, sa.m_out, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const uint64_t m = (uint64_t)hm;
  const uint64_t mm = m > 0 ? m : 1;
  ctx->qR = (uint64_t)nqp_rows_per_cta((int)mm, ctx->sm_count);
  double* Q = ENSURE(double, Q, blocked_size(mm, ctx->qR));
  double* q = ENSURE(double, q, vec_pad(m));
  if (m > 0)
    CK(launch_rescale_from_h(dH, h, (int)n, sa.pos, sa.scale, Q, (int)m, (int)ctx->qR, q, s));
  ctx->have_setup = true;
  CK(cudaEventRecord(ctx->ev[1], s));
  ctx->last_nnls = true;
  ctx->last_n = n;
  ctx->last_m = m;
  double* y = ENSURE(double, y_out, mm);
  if (m > 0) {
    Resolved r;
    if ((rc = resolve(ctx, cfg, m, &r))) return rc;
    rc = run_nqp(ctx, m, r, cfg, nullptr, &sum);
    if (rc) {
      if (out) *out = sum;
      ctx->last = sum;
      return rc;
    }
    CK(cudaMemcpyAsync(y, ctx->g_parity ? ctx->x_alt.p : ctx->x.p, sizeof(double) * m,
                       cudaMemcpyDeviceToDevice, s));
  } else {
    alnnls_iter_record rec{};
    alnnls_iter_record* tr = ENSURE(alnnls_iter_record, trace, 2);
    CK(cudaMemcpyAsync(tr, &rec, sizeof(rec), cudaMemcpyHostToDevice, s));
    sum.termination = ALNNLS_EMPTY_PASSIVE_SET;
    sum.trace_len = 1;
    CK(cudaEventRecord(ctx->ev[2], s));
    CK(cudaEventRecord(ctx->ev[3], s));
  }
  double* xn = ENSURE(double, X, n);
  CK(launch_unscale(y, sa.scale, sa.retained, (int)m, xn, (int)n, s));
  CK(cudaEventRecord(ctx->ev[4], s));
  CK(cudaStreamSynchronize(s));
  float t01 = 0, t23 = 0, t34 = 0, t04 = 0;
  cudaEventElapsedTime(&t01, ctx->ev[0], ctx->ev[1]);
  cudaEventElapsedTime(&t23, ctx->ev[2], ctx->ev[3]);
  cudaEventElapsedTime(&t34, ctx->ev[3], ctx->ev[4]);
  cudaEventElapsedTime(&t04, ctx->ev[0], ctx->ev[4]);
  sum.t_setup_s = t01 * 1e-3;
  sum.t_loop_s = t23 * 1e-3;
  sum.t_finish_s = t34 * 1e-3;
  sum.t_total_s = t04 * 1e-3;
  sum.n = n;
  sum.m = m;
  sum.n_dropped = n - m;
  ctx->last = sum;
  if (out) *out = sum;
  return ALNNLS_OK;
}

int alnnls_residual_rowblock_device(alnnls_ctx* ctx, uint64_t rows, uint64_t n, const double* dA,
                                    uint64_t lda, const double* db, const double* dx, double s_in,
                                    double* s_out) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!dA || !db || !dx || !s_out || rows < 1 || n < 1 || lda < rows)
    return set_err(ctx, ALNNLS_EINVAL, "residual_rowblock: bad argument");
  int st__ = ALNNLS_OK;
  cudaStream_t s = ctx->stream;
  // matvec over the support of x (zero x_j terms are exact no-ops), then the chain
  uint32_t* list = ENSURE(uint32_t, list, n);
  double* vals = ENSURE(double, vals, n + 8);
  int* len = ENSURE(int, mscalar, 4);
  CK(launch_support(dx, (int)n, list, vals, len, s));
  int hlen = 0;
  CK(cudaMemcpyAsync(&hlen, len, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  double* ax = ENSURE(double, ax, rows);
  double* pr = ENSURE(double, bcols, rows + 8);
  double* res = ENSURE(double, resid, 2);
  const double* A = dA;
  uint64_t ld = lda;
  if ((lda & 1) || (reinterpret_cast<uintptr_t>(dA) & 15)) {  // the bulk-copy GEMV's alignment
    double* dst = ENSURE(double, A, round_up(rows, 4) * n);
    CK(launch_copy_pad(dA, lda, dst, round_up(rows, 4), rows, n, s));
    A = dst;
    ld = round_up(rows, 4);
  }
  CK(launch_masked_gemv(A, ld, (int)rows, list, vals, hlen, ax, ctx->sm_count, s));
  CK(launch_residual(ax, db, (int)rows, pr, res, s, s_in));
  return copy_out(ctx, s_out, res, sizeof(double));
}

// ---- Anti+Acc baseline (accelerated.hpp) -------------------------------------------------
namespace {
struct SolverScope {  // routes the wrapped entry to the accelerated loop
  alnnls_ctx* c;
  SolverScope(alnnls_ctx* ctx) : c(ctx) { if (c) c->solver = 1; }
  ~SolverScope() { if (c) c->solver = 0; }
};
}  // namespace

int alnnls_solve_accelerated(alnnls_ctx* ctx, uint64_t m, const double* Q, const double* q,
                             const alnnls_config* cfg, alnnls_summary* out) {
  SolverScope sc(ctx);
  return alnnls_solve_nqp(ctx, m, Q, q, nullptr, cfg, out);
}

int alnnls_solve_accelerated_device(alnnls_ctx* ctx, uint64_t m, const double* dQ, uint64_t ldq,
                                    const double* dq, const alnnls_config* cfg,
                                    alnnls_summary* out) {
  SolverScope sc(ctx);
  return alnnls_solve_nqp_device(ctx, m, dQ, ldq, dq, nullptr, cfg, out);
}

int alnnls_solve_anti_accelerated(alnnls_ctx* ctx, uint64_t d, uint64_t n, const double* A,
                                  const double* b, const alnnls_config* cfg, alnnls_summary* out) {
  SolverScope sc(ctx);
  return alnnls_solve_nnls(ctx, d, n, A, b, cfg, out);
}

int alnnls_solve_anti_accelerated_device(alnnls_ctx* ctx, uint64_t d, uint64_t n, const double* dA,
                                         uint64_t lda, const double* db, const alnnls_config* cfg,
                                         alnnls_summary* out) {
  SolverScope sc(ctx);
  return alnnls_solve_nnls_device(ctx, d, n, dA, lda, db, cfg, out);
}

// ---- packed upper triangle, finish, multi-GPU batched ------------------------------------

int alnnls_pack_upper_device(alnnls_ctx* ctx, uint64_t n, const double* dH, double* dP) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!dH || !dP || n < 1) return set_err(ctx, ALNNLS_EINVAL, "pack_upper: bad argument");
  CK(launch_pack_upper(const_cast<double*>(dH), n, dP, 0, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return ALNNLS_OK;
}

int alnnls_unpack_upper_device(alnnls_ctx* ctx, uint64_t n, const double* dP, double* dH) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!dH || !dP || n < 1) return set_err(ctx, ALNNLS_EINVAL, "unpack_upper: bad argument");
  CK(launch_pack_upper(dH, n, const_cast<double*>(dP), 1, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return ALNNLS_OK;
}

int alnnls_finish(alnnls_ctx* ctx, uint64_t d, uint64_t n, const double* A, const double* b,
                  const double* y, uint64_t m, double* x, double* residual_sq) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!A || !b || !x || !residual_sq || (m && !y) || d < 1 || n < 1)
    return set_err(ctx, ALNNLS_EINVAL, "finish: bad argument");
  if (!ctx->last_nnls || ctx->last_n != n || ctx->last_m != m)
    return set_err(ctx, ALNNLS_EINVAL, "unscale: dimension mismatch");
  if (!all_finite(y, m)) return set_err(ctx, ALNNLS_EINVAL, "Vector: non-finite entry");
  int st__ = ALNNLS_OK;
  cudaStream_t s = ctx->stream;
  uint64_t lda = 0;
  if ((rc = upload_matrix(ctx, ctx->A, d, n, A, &lda))) return rc;
  double* dA = static_cast<double*>(ctx->A.p);
  double* db = ENSURE(double, b, d);
  CK(cudaMemcpyAsync(db, b, sizeof(double) * d, cudaMemcpyHostToDevice, s));
  if ((rc = device_check_finite(ctx, {{dA, d, n, lda, "DenseMatrix: non-finite entry"},
                                      {db, d, 1, d, "Vector: non-finite entry"}})))
    return rc;
  double* dy = ENSURE(double, y_out, m ? m : 1);
  if (m) CK(cudaMemcpyAsync(dy, y, sizeof(double) * m, cudaMemcpyHostToDevice, s));
  double* xn = ENSURE(double, X, n);
  CK(launch_unscale(dy, static_cast<double*>(ctx->scale.p), static_cast<uint32_t*>(ctx->retained.p),
                    (int)m, xn, (int)n, s));
  uint32_t* list = ENSURE(uint32_t, list, n);
  double* vals = ENSURE(double, vals, n + 8);
  int* len = ENSURE(int, mscalar, 4);
  CK(launch_support(xn, (int)n, list, vals, len, s));
  int hlen = 0;
  CK(cudaMemcpyAsync(&hlen, len, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  double* ax = ENSURE(double, ax, d);
  double* pr = ENSURE(double, bcols, d + 8);
  double* res = ENSURE(double, resid, 2);
  CK(launch_masked_gemv(dA, lda, (int)d, list, vals, hlen, ax, ctx->sm_count, s));
  CK(launch_residual(ax, db, (int)d, pr, res, s));
  if ((rc = copy_out(ctx, x, xn, sizeof(double) * n))) return rc;
  return copy_out(ctx, residual_sq, res, sizeof(double));
}

int alnnls_matmat_device(alnnls_ctx* ctx, uint64_t rows, uint64_t inner, uint64_t cols,
                         const double* dA, uint64_t lda, const double* dH, uint64_t ldh,
                         double* dC, uint64_t ldc) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!dA || !dH || !dC || rows < 1 || inner < 1 || cols < 1 || lda < rows || ldh < inner ||
      ldc < rows || rows > 0x7fffffffULL || inner > 0x7fffffffULL || cols > 0x7fffffffULL)
    return set_err(ctx, ALNNLS_EINVAL, "matmat: bad argument");
  CK(launch_matmat(dA, lda, (int)rows, (int)inner, dH, ldh, (int)cols, dC, ldc, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return ALNNLS_OK;
}

int alnnls_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  return c;
}

int alnnls_solve_nnls_batched_multi(alnnls_ctx* const* ctxs, int nctx, uint64_t d, uint64_t n,
                                    const double* A, uint64_t nrhs, const double* B,
                                    const alnnls_config* cfg, double* X,
                                    alnnls_column_result* cols, alnnls_summary* out) {
  if (!ctxs || nctx < 1) return ALNNLS_EINVAL;
  for (int c = 0; c < nctx; ++c)
    if (!ctxs[c]) return ALNNLS_EINVAL;
  if (!cfg || !A || !B || !X || !cols)
    return set_err(ctxs[0], ALNNLS_EINVAL, "solve_nnls_batched: null argument");
  if (d < 1 || n < 1 || nrhs < 1)
    return set_err(ctxs[0], ALNNLS_EINVAL, "DenseMatrix: rows and cols must be >= 1");
  const int used = (uint64_t)nctx > nrhs ? (int)nrhs : nctx;
  std::vector<int> rc(used, ALNNLS_OK);
  std::vector<alnnls_summary> sums(used);
  std::vector<std::thread> th;
  const uint64_t base = nrhs / used, extra = nrhs % used;
  uint64_t col0 = 0;
  for (int c = 0; c < used; ++c) {
    const uint64_t kc = base + ((uint64_t)c < extra ? 1 : 0);
    th.emplace_back([&, c, col0, kc] {
      rc[c] = alnnls_solve_nnls_batched(ctxs[c], d, n, A, kc, B + col0 * d, cfg, X + col0 * n,
                                        cols + col0, &sums[c]);
    });
    col0 += kc;
  }
  for (auto& t : th) t.join();
  alnnls_summary tot{};
  for (int c = 0; c < used; ++c) {
    if (rc[c] != ALNNLS_OK) {
      if (c > 0) ctxs[0]->err = ctxs[c]->err;
      return rc[c];
    }
    const alnnls_summary& s = sums[c];
    tot.t_setup_s = std::max(tot.t_setup_s, s.t_setup_s);
    tot.t_loop_s = std::max(tot.t_loop_s, s.t_loop_s);
    tot.t_finish_s = std::max(tot.t_finish_s, s.t_finish_s);
    tot.t_total_s = std::max(tot.t_total_s, s.t_total_s);
    tot.iterations += s.iterations;
    tot.multiplies_total += s.multiplies_total;
    tot.numeric_failure |= s.numeric_failure;
    tot.n = s.n;
    tot.m = s.m;
    tot.n_dropped = s.n_dropped;
  }
  if (out) *out = tot;
  return ALNNLS_OK;
}

// ---- NMF by alternating NNLS -------------------------------------------------------------

int alnnls_nmf_device(alnnls_ctx* ctx, uint64_t d, uint64_t N, uint64_t k, const double* dV,
                      double* dW, double* dH, uint64_t outer_iters, const alnnls_config* cfg,
                      double* objective) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!cfg || !dV || !dW || !dH) return set_err(ctx, ALNNLS_EINVAL, "nmf: null argument");
  if (d < 1 || N < 1 || k < 1) return set_err(ctx, ALNNLS_EINVAL, "DenseMatrix: rows and cols must be >= 1");
  if (k > 1024) return set_err(ctx, ALNNLS_EINVAL, "nmf: k > 1024 not supported (batched solver bound)");
  int st__ = ALNNLS_OK;
  cudaStream_t s = ctx->stream;
  {  // inputs: finite V, finite nonnegative start W (linalg.hpp:84, like solve_nqp's start)
    int* flag = ENSURE(int, flag, 4);
    CK(cudaMemsetAsync(flag, 0, sizeof(int) * 3, s));
    CK(launch_check_finite(dV, d, N, d, flag, s));
    CK(launch_check_finite(dW, d, k, d, flag + 1, s));
    CK(launch_check_matrix(dW, d, k, d, 1, flag + 2, s));
    int hf[3] = {0, 0, 0};
    if ((rc = copy_out(ctx, hf, flag, sizeof(hf)))) return rc;
    if (hf[0] || hf[1]) return set_err(ctx, ALNNLS_EINVAL, "DenseMatrix: non-finite entry");
    if (hf[2]) return set_err(ctx, ALNNLS_EINVAL, "nmf: W must be nonnegative");
  }
  double* VT = ENSURE(double, nvt, N * d);  // V^T (N x d)
  double* HT = ENSURE(double, nht, N * k);  // H^T (N x k)
  double* WT = ENSURE(double, nwt, k * d);  // W^T (k x d)
  CK(launch_transpose(dV, d, (int)d, (int)N, VT, N, s));
  std::vector<alnnls_column_result> colsH(N), colsW(d);
  for (uint64_t t = 0; t < outer_iters; ++t) {
    // H <- argmin ||W H - V||: columns of V against A = W
    alnnls_summary sum{};
    if ((rc = run_batched(ctx, d, k, dW, d, N, dV, d, cfg, dH, colsH.data(), &sum))) return rc;
    if (objective) {
      double obj = 0.0;
      for (uint64_t j = 0; j < N; ++j) obj += colsH[j].residual_sq;
      objective[t] = obj;
    }
    // W <- argmin ||H^T W^T - V^T||: columns of V^T against A = H^T
    CK(launch_transpose(dH, k, (int)k, (int)N, HT, N, s));
    if ((rc = run_batched(ctx, N, k, HT, N, d, VT, N, cfg, WT, colsW.data(), &sum))) return rc;
    CK(launch_transpose(WT, k, (int)k, (int)d, dW, d, s));
  }
  CK(cudaStreamSynchronize(s));
  return ALNNLS_OK;
}

int alnnls_nmf(alnnls_ctx* ctx, uint64_t d, uint64_t N, uint64_t k, const double* V, double* W,
               double* H, uint64_t outer_iters, const alnnls_config* cfg, double* objective) {
  int rc = check_ctx(ctx);
  if (rc) return rc;
  if (!cfg || !V || !W || !H) return set_err(ctx, ALNNLS_EINVAL, "nmf: null argument");
  if (d < 1 || N < 1 || k < 1) return set_err(ctx, ALNNLS_EINVAL, "DenseMatrix: rows and cols must be >= 1");
  int st__ = ALNNLS_OK;
  cudaStream_t s = ctx->stream;
  double* dV = ENSURE(double, nv, d * N);
  double* dW = ENSURE(double, nw, d * k);
  double* dH = ENSURE(double, nh, k * N);
  CK(cudaMemcpyAsync(dV, V, sizeof(double) * d * N, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dW, W, sizeof(double) * d * k, cudaMemcpyHostToDevice, s));
  if ((rc = alnnls_nmf_device(ctx, d, N, k, dV, dW, dH, outer_iters, cfg, objective))) return rc;
  if ((rc = copy_out(ctx, W, dW, sizeof(double) * d * k))) return rc;
  return copy_out(ctx, H, dH, sizeof(double) * k * N);
}

}  // extern "C"
