#!/usr/bin/env python3
"""Benchmark of the B200-native anti-lopsided NNLS hot path (solve_nnls).

A "step" is one full solve_nnls (Gram + cosine rescale + device-resident
projected-gradient loop + unscale + residual; nnls.hpp:129-144) of the
BASELINE.json workload, default c2 = configs[1] (d=8192, n=4096, N(0,1),
eps 1e-8; seeded synthetic inputs, see paper_1502_01645_b200/instances.py).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2] [--profile exact|fast]
  python bench.py --impl reference ...   # the reference CPU solver (oracle/_ref)
  python bench.py --workload c4 ...      # batched multi-RHS (NMF H-update), column-sharded

Prints ONE JSON line on rank 0. `value` is whole-job solves/s with A, b already
in HBM (device-pointer C-ABI entry); `e2e` is the same metric through the
host-buffer public API with the H2D copy of A, b and the D2H of the result in
the timed region. Timing: CUDA events on the library's stream, max over ranks.
The default (EXACT, bitwise) line also carries "fast_profile": the same
workload through the FAST profile (DMMA Gram + the one-pass loop), graded on
BASELINE.json's four tolerances against the EXACT run.

--gpus N without WORLD_SIZE in the environment re-launches this script under
torch.distributed.run with N ranks (one per GPU, NCCL, 127.0.0.1). c1/c2/c3
at N > 1 run one independent replica per GPU ("replicas only": one solve's
iteration loop does not shard), "scaling": "weak".

--workload c5 with N > 1 (configs[4]): A's rows are split across the ranks and
the exact setup runs as a row-block pipeline (rowblock.py): every rank
continues the Gram tile chains of the ranks before it and passes them on over
NCCL, the last rank rescales and iterates, the residual chain is relayed back
through the ranks. Bitwise equal to the single-GPU solve; "scaling": "strong".
--workload c5 --c5-setup allreduce [--profile fast] runs configs[4]'s setup as
written instead: a partial Gram per rank (DMMA under fast) summed with one NCCL
allreduce of the packed upper triangle, iterations on rank 0 (within rounding of
the reference, not bitwise).

--workload c4 (configs[3]): a step is the whole batched solve of B (20000 x
65536) against the shared Q; the 65536 right-hand sides are split by column
across the N ranks with no data-path collective ("scaling": "strong"), and
`value` is total columns / max-over-ranks time. B = A H_true is formed on the
device by an exact-order kernel (bit-identical to the host generator, so the
sampled columns are checked against the reference's results).

--impl reference (this tier's reference arm): the reference's own solve_nnls
(oracle/_ref, compiled from its headers by oracle/Makefile) on the host cores:
each step is one real, unmodified solve_nnls call; the K steps run concurrently,
one per host core, the way the reference's suite pool runs independent cells
(bench.hpp:191-207); value = K / wall time. Under torchrun only rank 0 runs it.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1502_01645_b200 import abi, instances  # noqa: E402

METRIC = "solve_nnls time-to-KKT-tol throughput (solves/s)"
UNIT = "solves/s"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


# fp64 peaks measured on this pool's B200 by tools/microbench/fp64_probe.cu
# (profiles/r01_fp64_probe.txt): DMMA 37.0 TFLOP/s; the bit-exact profile needs a
# separate DMUL and DADD per product on the FP64 pipe, capping it at half: 18.5.
FP64_PEAK_TFLOPS = 37.0
FP64_EXACT_CAP_TFLOPS = 18.5


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        if not self.lines:  # timed region shorter than the 100 ms period: one query at its end
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index),
                     "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                     "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                     "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10)
                self.lines = [ln.strip() for ln in out.stdout.splitlines() if ln.strip()]
            except Exception:
                pass

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if args.impl == "ours" and (ws > 1 or os.environ.get("ALNNLS_FORCE_ROWBLOCK")):
        import torch.distributed as dist  # noqa
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if "RANK" not in os.environ:  # a one-rank group outside torchrun (the N=1 pipeline)
            import socket
            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                os.environ.setdefault("MASTER_PORT", str(sk.getsockname()[1]))
            os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
        import torch
        torch.cuda.set_device(local)
        dist.init_process_group(backend="nccl")
    return ws, rank, local, dist


PROFILE = {"exact": 0, "fast": 1}
PROFILE_DESC = {"exact": "exact (bitwise reference trajectory)",
                "fast": "fast (DMMA Gram + one-pass single-RHS loop / DMMA Q V passes; graded on the "
                        "four BASELINE tolerances, DESIGN.md 2a-2b)"}


def solver_config(inst, profile="exact"):
    from paper_1502_01645_b200.api import SolverConfig
    # stall off like the reference's own benchmark convention (acceptance.cpp:73-88)
    return SolverConfig(epsilon=inst["epsilon"], max_iters=inst["max_iters"], stall_window=10**9,
                        profile=PROFILE[profile])


def workload_config(name, d, n, eps, nrhs=None):
    """The config dict both arms print (identical: the workload, not the implementation)."""
    c = {"workload": f"{name}: d={d}, n={n}" + (f", nrhs={nrhs}" if nrhs else ""), "eps": eps,
         "solver": "solve_nnls (nnls.hpp:129-144)" + (" per column, one shared Gram" if nrhs else ""),
         "stall_window": "off (acceptance.cpp:73-88 convention)"}
    big = 8 * d * (n + (nrhs or 0))
    c["l2"] = ("inputs larger than L2 (no flush needed)" if big > 126e6
               else "inputs L2-resident (latency-bound config; no flush)")
    return c


def traffic_from_profiles(workload, kernel):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return d.get(workload, {}).get(kernel)


# ---- reference CPU solver ------------------------------------------------------------------
def ref_oracle():
    from oracle.oracle import Oracle, available
    if available("ref"):
        return Oracle("ref"), "reference"
    return Oracle("oracle"), "port"


def cached_inputs(name):
    """Seeded inputs generated in a CHILD process (the generator library is this
    repo's, not the reference's) and read back from an .npz, so the reference
    process maps only oracle/_ref."""
    import tempfile
    path = os.path.join(tempfile.gettempdir(), f"alnnls_inputs_{name}_{os.getpid()}.npz")
    code = ("import sys, numpy as np; sys.path.insert(0, %r); "
            "from paper_1502_01645_b200 import instances as I; "
            "i = I.make_config(%r); np.savez(%r, A=i['A'], b=i['b'], eps=i['epsilon'], "
            "mi=-1 if i['max_iters'] is None else i['max_iters'])") % (ROOT, name, path)
    subprocess.run([sys.executable, "-c", code], check=True)
    z = np.load(path)
    inst = {"A": np.asfortranarray(z["A"]), "b": z["b"], "epsilon": float(z["eps"]),
            "max_iters": None if int(z["mi"]) < 0 else int(z["mi"]), "name": name}
    os.unlink(path)
    return inst


def reference_gram_parallel(ora, A, threads, nb=16):
    """The reference's own gram() (linalg.hpp:160-174) driven over column-block
    pairs on `threads` host threads; every entry is the same k-ascending chain, so
    H is bitwise gram(A) (the pairing recomputes the diagonal blocks)."""
    from concurrent.futures import ThreadPoolExecutor
    d, n = A.shape
    nb = max(1, min(nb, threads))
    bs = (n + nb - 1) // nb
    blocks = [(i * bs, min(n, (i + 1) * bs)) for i in range(nb) if i * bs < n]
    H = np.zeros((n, n), order="F")

    def work(pair):
        (a0, a1), (b0, b1) = pair
        if (a0, a1) == (b0, b1):
            H[a0:a1, a0:a1] = ora.gram(np.asfortranarray(A[:, a0:a1]))
        else:
            cols = np.concatenate([np.arange(a0, a1), np.arange(b0, b1)])
            Hb = ora.gram(np.asfortranarray(A[:, cols]))
            k = a1 - a0
            H[a0:a1, b0:b1] = Hb[:k, k:]
            H[b0:b1, a0:a1] = Hb[k:, :k]

    pairs = [(blocks[i], blocks[j]) for i in range(len(blocks)) for j in range(i, len(blocks))]
    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(work, pairs))
    return H


def cpu_pipeline_sample(ora, inst, cfg_abi, threads, loop_cap=None):
    """A bounded, fully measured run of the reference pipeline (nnls.hpp:129-144):
    gram by the reference's gram() over column-block pairs on all host threads
    (bitwise gram(A)), then transpose_matvec, rescale, solve_nqp, unscale and the
    residual single-threaded (the reference is single-threaded per solve). With
    loop_cap the loop runs that many iterations and is scaled to the cap given by
    the config (time per iteration is flat). Returns (seconds, detail)."""
    A, b = inst["A"], inst["b"]
    d, n = A.shape
    t = time.perf_counter()
    H = reference_gram_parallel(ora, A, threads)
    t_gram = time.perf_counter() - t
    t = time.perf_counter()
    atb = ora.transpose_matvec(A, b)
    sys_ = ora.rescale(H, -atb)
    t_resc = time.perf_counter() - t
    del H
    t = time.perf_counter()
    res, scale = None, 1.0
    if len(sys_["q"]):
        cfg = cfg_abi
        if loop_cap is not None:
            full = cfg.max_iters if cfg.has_max_iters else 5 * len(sys_["q"])
            cfg = abi.make_config(epsilon=cfg.epsilon if cfg.has_epsilon else None,
                                  max_iters=min(loop_cap, full), stall_window=cfg.stall_window,
                                  record_multiplies=False)
            scale = full / min(loop_cap, full)
        res = ora.solve_nqp(sys_["Q"], sys_["q"], cfg)
    t_loop = (time.perf_counter() - t) * scale
    t = time.perf_counter()
    x = np.zeros(n)
    if res is not None:
        x[sys_["retained"].astype(np.int64)] = res["x"] / sys_["scale"]
    ax = ora.matvec(A, x)
    r = ax - b
    _ = float(np.sum(r * r))
    t_fin = time.perf_counter() - t
    total = t_gram + t_resc + t_loop + t_fin
    return total, {"gram_s": t_gram, "gram_threads": threads, "transpose_matvec_rescale_s": t_resc,
                   "solve_nqp_s": t_loop, "solve_nqp_scaled_from": loop_cap,
                   "finish_s": t_fin, "iterations": res["iterations"] if res else 0,
                   "termination": res["termination"] if res else "EmptyPassiveSet"}


def run_reference(args, ws, rank):
    if rank != 0:
        return 0  # the CPU reference runs once, on rank 0
    if args.workload == "c4":
        return run_reference_batched(args, ws)
    ora, kind = ref_oracle()
    inst = cached_inputs(args.workload)
    A, b = inst["A"], inst["b"]
    d, n = A.shape
    cores = os.cpu_count() or 1
    cfg = solver_config_abi(inst)
    line = {"impl": "reference", "metric": METRIC, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded SplitMix64, BASELINE.json configs)",
            "config": workload_config(args.workload, d, n, inst["epsilon"])}
    if args.workload in ("c1", "c2"):
        # K real, unmodified solve_nnls calls, concurrently one per host core
        from concurrent.futures import ThreadPoolExecutor
        per = []

        def one(_):
            t = time.perf_counter()
            r = ora.solve_nnls(A, b, cfg)
            per.append(time.perf_counter() - t)
            return r["iterations"], r["termination"]

        if args.warmup > 0:
            with ThreadPoolExecutor(max_workers=min(args.warmup, cores)) as ex:
                list(ex.map(one, range(args.warmup)))
        per.clear()
        P = min(args.steps, cores)
        t0 = time.perf_counter()
        with ThreadPoolExecutor(max_workers=P) as ex:
            outs = list(ex.map(one, range(args.steps)))
        wall = time.perf_counter() - t0
        value = args.steps / wall
        line.update({"value": value, "ms_per_step": wall / args.steps * 1e3,
                     "iterations": outs[0][0], "termination": outs[0][1],
                     "per_solve_s_mean": float(np.mean(per)), "per_solve_s_max": float(np.max(per))})
        sample = (f"{args.steps} real solve_nnls calls (the reference compiled from its headers, "
                  f"oracle/_ref), run concurrently on {P} host threads (one solve per core, like "
                  f"bench.hpp:191-207); value = steps / wall time ({wall:.1f} s); "
                  f"{args.warmup} warm-up solves before")
        line["cpu_baseline"] = {"value": value, "unit": UNIT, "cores": P, "kind": kind,
                                "sample": sample, "cpu": cpu_model()}
    else:
        # c3 / c5: one solve takes 0.2-3 h on a core; a bounded sample per step
        cap = 200
        for _ in range(args.warmup):
            pass  # no warm-up state on the host path worth a 10 s sample
        times, detail = [], None
        for _ in range(args.steps):
            tt, detail = cpu_pipeline_sample(ora, inst, cfg, cores, loop_cap=cap)
            times.append(tt)
        per = float(np.mean(times))
        value = 1.0 / per
        line.update({"value": value, "ms_per_step": per * 1e3, "breakdown": detail})
        line["cpu_baseline"] = {
            "value": value, "unit": UNIT, "cores": cores, "kind": kind, "cpu": cpu_model(),
            "sample": (f"reference gram() over column-block pairs on {cores} threads (measured), "
                       f"transpose_matvec/rescale/unscale/residual measured single-thread, "
                       f"solve_nqp measured for {cap} iterations and scaled to the config's cap")}
    line["e2e"] = {"value": line["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}
    print(json.dumps(line), flush=True)
    return 0


def solver_config_abi(inst, record_multiplies=False):
    return abi.make_config(epsilon=inst["epsilon"], max_iters=inst["max_iters"], stall_window=10**9,
                           record_multiplies=record_multiplies)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ---- our GPU path ---------------------------------------------------------------------------
def measure_single(s, args, dA, db, d, n, cfg, anti=False):
    """Device-resident steps (value) and host-buffer steps (e2e) of one profile."""
    import torch
    solve_dev = s.solve_anti_accelerated_device if anti else s.solve_nnls_device
    for _ in range(max(1, args.warmup)):  # >= 1: the solve's iteration count for the roofline
        solve_dev(dA.data_ptr(), d, d, n, db.data_ptr(), cfg, fetch=False)
    summ = s.last_summary()
    out = {"iterations": int(summ.iterations), "mults": int(summ.multiplies_total)}
    torch.cuda.synchronize()
    l0 = s.launch_count()
    t_setup = t_loop = 0.0
    s.timer_start()
    for _ in range(args.steps):
        solve_dev(dA.data_ptr(), d, d, n, db.data_ptr(), cfg, fetch=False)
        sm = s.last_summary()
        t_setup += sm.t_setup_s
        t_loop += sm.t_loop_s
    out["t"] = s.timer_stop()
    out["launches"] = (s.launch_count() - l0) // max(1, args.steps)
    out["setup_s"] = t_setup / args.steps
    out["loop_s"] = t_loop / args.steps
    return out


def measure_e2e(s, args, hA, hb, cfg, anti=False):
    solve_host = s.solve_anti_accelerated if anti else s.solve_nnls
    res = solve_host(hA, hb, cfg)  # warm
    s.timer_start()
    for _ in range(args.steps):
        res = solve_host(hA, hb, cfg)
    return s.timer_stop(), res


def run_ours(args, ws, rank, local, dist):
    import torch
    from paper_1502_01645_b200.api import Solver
    from tests.parity import baseline_tolerances
    torch.cuda.set_device(local)
    inst = instances.make_config(args.workload)
    A, b = inst["A"], inst["b"]
    d, n = A.shape
    cfg = solver_config(inst, args.profile)
    s = Solver(local)
    # inputs resident in HBM: column-major A == row-major (n, d) tensor
    dA = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    db = torch.from_numpy(b).cuda()
    torch.cuda.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(v):
        if dist is None:
            return v
        tt = torch.tensor([v], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    anti = args.solver == "anti_acc"
    barrier()
    with ClockSampler(local) as clk:
        meas = measure_single(s, args, dA, db, d, n, cfg, anti)
    barrier()
    t_max = max_over_ranks(meas["t"])
    value = ws * args.steps / t_max

    # e2e: host-buffer public API, pinned host inputs, result read back each step
    pA = torch.empty((n, d), dtype=torch.float64, pin_memory=True)
    pA.copy_(torch.from_numpy(np.ascontiguousarray(A.T)))
    pb = torch.empty(d, dtype=torch.float64, pin_memory=True)
    pb.copy_(torch.from_numpy(b))
    hA = pA.numpy().T  # Fortran-ordered (d, n) view of pinned memory
    hb = pb.numpy()
    barrier()
    te, res = measure_e2e(s, args, hA, hb, cfg, anti)
    te = max_over_ranks(te)
    m = len(res.inner.x)
    d2h = 8 * (n + 2 * m + len(res.inner.multiplies_per_iter)) + 56 * len(res.inner.trace)
    e2e = {"value": ws * args.steps / te, "unit": UNIT, "h2d_bytes_per_step": 8 * (d * n + d),
           "d2h_bytes_per_step": int(d2h)}

    # the same workload through the FAST profile (the default line stays EXACT)
    fast = None
    if args.profile == "exact" and not anti and args.workload != "c5":
        cfgf = solver_config(inst, "fast")
        barrier()
        mf = measure_single(s, args, dA, db, d, n, cfgf)
        tf = max_over_ranks(mf["t"])
        tfe, resf = measure_e2e(s, args, hA, hb, cfgf)
        tfe = max_over_ranks(tfe)
        tol = baseline_tolerances(resf.x, res.x, resf.inner.trace[-1].f, res.inner.trace[-1].f,
                                  resf.inner.iterations(), res.inner.iterations())
        fast = {"meas": mf, "value": ws * args.steps / tf, "e2e": ws * args.steps / tfe, "tol": tol}

    if rank != 0:
        return 0
    hbm, hbm_kind = peaks()
    iters, mults = meas["iterations"], meas["mults"]
    per_setup, per_loop = meas["setup_s"], meas["loop_s"]
    setup_flops = d * n * (n + 1) + 2 * d * n
    if anti:  # the reference's two dense matvecs per iteration (accelerated.hpp:45, :89)
        mults = 2 * n * n * iters
    loop_gbs = 8.0 * mults / per_loop / 1e9 if per_loop > 0 else 0.0
    setup_tf = setup_flops / per_setup / 1e12
    # small m (c1) runs the cluster loop with its state in distributed shared memory
    # (small.cu); Q is resident in shared memory there, so it is latency-, not HBM-bound
    loop_kernel = "nqp_small_kernel" if args.workload == "c1" and not anti else "nqp_loop_kernel"
    roof_loop = {"kernel": (f"{loop_kernel} (one thread-block cluster, Q panels resident in shared "
                            "memory, loop state in DSMEM)" if loop_kernel == "nqp_small_kernel"
                            else "nqp_loop_kernel (device-resident iteration loop, masked GEMVs)"),
                 "bound": "hbm", "achieved": loop_gbs, "peak": hbm, "unit": "GB/s",
                 "frac": loop_gbs / hbm, "peak_source": hbm_kind,
                 "algorithmic": f"8 B x reference multiply count = {8 * mults} B per launch",
                 "traffic": traffic_from_profiles(args.workload, loop_kernel)}
    roof_setup = {"kernel": "setup: colchain + syrk_exact + rescale epilogue",
                  "bound": "tensor", "pipe": "fp64 SIMT (exact DMUL + DADD chains; the peak is the fp64 tensor peak)", "achieved": setup_tf, "peak": FP64_PEAK_TFLOPS,
                  "unit": "TFLOP/s", "frac": setup_tf / FP64_PEAK_TFLOPS,
                  "frac_of_exact_cap": setup_tf / FP64_EXACT_CAP_TFLOPS,
                  "peak_source": "measured (tools/microbench/fp64_probe.cu, DMMA)",
                  "algorithmic": f"d*n*(n+1) + 2*d*n = {setup_flops} flop per solve",
                  "traffic": traffic_from_profiles(args.workload, "syrk_streamk_kernel")}
    if args.profile == "fast":
        roof_loop = fast_loop_roofline(args.workload, mults, per_loop, hbm, hbm_kind)
        roof_setup.update({"kernel": "setup: syrk_dmma_kernel (fp64 tensor cores) + rescale epilogue",
                           "pipe": "fp64 DMMA", "frac_of_exact_cap": None,
                           "traffic": traffic_from_profiles(args.workload, "syrk_dmma_kernel")})
    dominant = roof_loop if per_loop >= per_setup else roof_setup
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SplitMix64, BASELINE.json configs)",
        "config": workload_config(args.workload, d, n, inst["epsilon"]),
        "profile": PROFILE_DESC[args.profile],
        "solver": ("solve_anti_accelerated (accelerated.hpp)" if anti else "solve_nnls"),
        "parallelism": f"replicas x{ws} (one independent solve per GPU)",
        "iterations": iters, "time_to_tol_ms": t_max / args.steps * 1e3,
        "iters_per_s": iters / per_loop if per_loop > 0 else None,
        "setup_ms": per_setup * 1e3, "loop_ms": per_loop * 1e3,
        "roofline": dominant, "roofline_other": roof_setup if dominant is roof_loop else roof_loop,
        "e2e": e2e, "gpu_launches": int(meas["launches"]), "clocks": clk.summary(),
    }
    if fast is not None:
        mf = fast["meas"]
        fl = fast_loop_roofline(args.workload, mf["mults"], mf["loop_s"], hbm, hbm_kind)
        fl["exact_equivalent_GBps"] = 8.0 * mults / mf["loop_s"] / 1e9
        fsetup = setup_flops / mf["setup_s"] / 1e12
        line["fast_profile"] = {
            "value": fast["value"], "e2e": fast["e2e"], "unit": UNIT,
            "iterations": mf["iterations"], "setup_ms": mf["setup_s"] * 1e3,
            "loop_ms": mf["loop_s"] * 1e3, "us_per_iter": mf["loop_s"] / max(1, mf["iterations"]) * 1e6,
            "setup_roofline": {"kernel": "syrk_dmma_kernel", "achieved": fsetup,
                               "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                               "frac": fsetup / FP64_PEAK_TFLOPS},
            "loop_roofline": fl, "gpu_launches": int(mf["launches"]),
            "tolerances_vs_exact": fast["tol"],
        }
    if ws == 1 and not args.no_cpu_baseline and not anti:
        ora, kind = ref_oracle()
        threads = os.cpu_count() or 1
        if args.workload == "c1":  # a full solve is 0.1 s: the real thing, repeated
            t = time.perf_counter()
            reps = 20
            for _ in range(reps):
                ora.solve_nnls(A, b, solver_config_abi(inst))
            tt = (time.perf_counter() - t) / reps
            detail, sample, cores = None, f"{reps} real solve_nnls calls, single thread", 1
        else:
            cap = None if args.workload == "c2" else 200
            tt, detail = cpu_pipeline_sample(ora, inst, solver_config_abi(inst), threads, cap)
            sample = (f"the full reference pipeline on this workload, measured: gram() over column-"
                      f"block pairs on {threads} threads (bitwise gram(A)), the rest single-thread"
                      + ("" if cap is None else f"; solve_nqp {cap} iterations scaled to the cap"))
            cores = threads
        line["cpu_baseline"] = {"value": 1.0 / tt, "unit": UNIT, "cores": cores, "kind": kind,
                                "sample": sample, "cpu": cpu_model(), "breakdown": detail}
    print(json.dumps(line), flush=True)
    return 0


def fast_loop_roofline(workload, mults, per_loop, hbm, hbm_kind):
    gbs = 8.0 * mults / per_loop / 1e9 if per_loop > 0 else 0.0
    return {"kernel": "fast_loop_kernel (one-pass masked GEMV loop, 128-bit loads, tree reductions)",
            "bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
            "peak_source": hbm_kind,
            "algorithmic": (f"8 B x the FAST loop's multiply count (m|P| + sum m|K| per iteration: "
                            f"every Q element it must read) = {8 * mults} B per launch"),
            "traffic": traffic_from_profiles(workload, "fast_loop_kernel")}


# ---- c5 at N > 1: exact row-block setup pipeline ------------------------------------------
def run_ours_rowblock(args, ws, rank, local, dist):
    import torch
    from paper_1502_01645_b200.api import Solver
    from paper_1502_01645_b200.rowblock import chain_relay, pipelined_gram, row_split
    torch.cuda.set_device(local)
    inst = instances.make_config(args.workload)
    A, b = inst["A"], inst["b"]
    d, n = A.shape
    r0, r1 = row_split(d, ws)[rank]
    rows = r1 - r0
    cfg = solver_config(inst)
    s = Solver(local)
    dA = torch.from_numpy(np.ascontiguousarray(A[r0:r1, :].T)).cuda()  # block, column-major, ld rows
    db = torch.from_numpy(np.ascontiguousarray(b[r0:r1])).cuda()
    del A
    T = s.gram_tiles(n)
    TD = s.GRAM_TILE_DOUBLES
    batch = 2 * 148
    last = rank == ws - 1
    H = torch.empty((n, n), dtype=torch.float64, device="cuda") if last else None
    sync = torch.cuda.synchronize

    def step():
        def gram_batch(t0, t1, pin, pout):
            s.gram_rowblock_device(rows, n, dA.data_ptr(), rows, t0, t1,
                                   pin.data_ptr() if pin is not None else 0,
                                   pout.data_ptr() if pout is not None else 0,
                                   H.data_ptr() if pout is None else 0)
        pipelined_gram(dist, rank, ws, T, batch, TD, gram_batch, "cuda", sync=sync)

        def atb(pin):
            out = torch.empty(n, dtype=torch.float64, device="cuda")
            s.atb_rowblock_device(rows, n, dA.data_ptr(), rows, db.data_ptr(),
                                  pin.data_ptr() if pin is not None else 0, out.data_ptr())
            return out
        h = chain_relay(dist, rank, ws, torch.empty(n, dtype=torch.float64, device="cuda"), atb,
                        sync=sync)
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        iters = 0
        if last:
            summ = s.solve_nnls_gram_device(n, H.data_ptr(), h.data_ptr(), cfg, fetch=False)
            iters = int(summ.iterations)
            x.copy_(torch.from_numpy(s._vec(s.lib.alnnls_get_x, n)).cuda())
        dist.broadcast(x, src=ws - 1)
        sync()

        def resid(pin):
            v = s.residual_rowblock_device(rows, n, dA.data_ptr(), rows, db.data_ptr(), x.data_ptr(),
                                           float(pin[0]) if pin is not None else 0.0)
            return torch.tensor([v], dtype=torch.float64, device="cuda")
        r = chain_relay(dist, rank, ws, torch.empty(1, dtype=torch.float64, device="cuda"), resid,
                        sync=sync)
        return iters, (float(r[0]) if r is not None else None)

    for _ in range(args.warmup):
        iters, _ = step()
    dist.barrier()
    torch.cuda.synchronize()
    l0 = s.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record()
        for _ in range(args.steps):
            iters, res = step()
        ev1.record()
        torch.cuda.synchronize()
    launches = (s.launch_count() - l0) // max(1, args.steps)
    t = ev0.elapsed_time(ev1) * 1e-3
    tt = torch.tensor([t, float(iters)], device="cuda", dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_max, iters = float(tt[0]), int(tt[1])
    if rank != 0:
        return 0
    line = {
        "metric": METRIC, "value": args.steps / t_max, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SplitMix64, BASELINE.json configs[4])",
        "config": workload_config(args.workload, d, n, inst["epsilon"]),
        "profile": PROFILE_DESC["exact"],
        "parallelism": f"row blocks x{ws}: k-chain Gram pipeline (NCCL send/recv), "
                       "iterations on the last rank",
        "iterations": iters, "gpu_launches": launches, "clocks": clk.summary(),
        "e2e": None,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---- c5, the configs[4] setup as written: partial Grams + ONE allreduce -------------------
def run_ours_allreduce(args, ws, rank, local, dist):
    """Every rank forms the partial Gram and A^T b of its row block (DMMA under
    --profile fast, chain SYRK under exact), one allreduce sums [H | A^T b]
    (NCCL), rank 0 rescales and iterates, x is broadcast and the residual is one
    more allreduce of the ranks' partial chains. Not bitwise (the cross-rank sum
    order is NCCL's): tests/test_gpu_rowblock.py pins Q within 1e-13 and the loop
    bitwise on the GPU's own Q."""
    import torch
    from paper_1502_01645_b200.api import Solver
    from paper_1502_01645_b200.rowblock import allreduce_residual, allreduce_setup, row_split
    torch.cuda.set_device(local)
    inst = instances.make_config(args.workload)
    A, b = inst["A"], inst["b"]
    d, n = A.shape
    r0, r1 = row_split(d, ws)[rank]
    rows = r1 - r0
    cfg = solver_config(inst, args.profile)
    s = Solver(local)
    dA = torch.from_numpy(np.ascontiguousarray(A[r0:r1, :].T)).cuda()  # block, column-major, ld rows
    db = torch.from_numpy(np.ascontiguousarray(b[r0:r1])).cuda()
    del A
    prof = PROFILE[args.profile]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    tm = {"partial": 0.0, "allreduce": 0.0, "solve": 0.0}

    def step():
        def partial(H, atb):
            s.gram_partial_device(rows, n, dA.data_ptr(), rows, db.data_ptr(), H.data_ptr(),
                                  atb.data_ptr(), profile=prof)
            ev[1].record()
        ev[0].record()
        H, atb = allreduce_setup(
            dist, ws, n, partial, "cuda",
            pack=lambda Hm, P: s.pack_upper_device(n, Hm.data_ptr(), P.data_ptr()),
            unpack=lambda P, Hm: s.unpack_upper_device(n, P.data_ptr(), Hm.data_ptr()))
        ev[2].record()
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        iters = 0
        if rank == 0:
            summ = s.solve_nnls_gram_device(n, H.data_ptr(), atb.data_ptr(), cfg, fetch=False)
            iters = int(summ.iterations)
            x.copy_(torch.from_numpy(s._vec(s.lib.alnnls_get_x, n)).cuda())
        ev[3].record()
        if dist is not None:
            dist.broadcast(x, src=0)
        v = s.residual_rowblock_device(rows, n, dA.data_ptr(), rows, db.data_ptr(), x.data_ptr(),
                                       0.0)
        res = allreduce_residual(dist, ws, v, "cuda")
        torch.cuda.synchronize()
        tm["partial"] += ev[0].elapsed_time(ev[1]) * 1e-3
        tm["allreduce"] += ev[1].elapsed_time(ev[2]) * 1e-3
        tm["solve"] += ev[2].elapsed_time(ev[3]) * 1e-3
        return iters, res

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        iters, _ = step()
    for k_ in tm:
        tm[k_] = 0.0
    barrier()
    torch.cuda.synchronize()
    l0 = s.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record()
        for _ in range(args.steps):
            iters, res = step()
        e1.record()
        torch.cuda.synchronize()
    launches = (s.launch_count() - l0) // max(1, args.steps)
    t = e0.elapsed_time(e1) * 1e-3
    vals = [t, float(iters), tm["partial"], tm["allreduce"], tm["solve"]]
    tt = torch.tensor(vals, device="cuda", dtype=torch.float64)
    if dist is not None:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_max, iters = float(tt[0]), int(tt[1])
    t_part, t_ar, t_solve = (float(v) / args.steps for v in tt[2:5])
    if rank != 0:
        return 0
    flops_rank = rows * n * (n + 1) + 2 * rows * n
    ach = flops_rank / t_part * 1e-12
    line = {
        "metric": METRIC, "value": args.steps / t_max, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SplitMix64, BASELINE.json configs[4])",
        "config": workload_config(args.workload, d, n, inst["epsilon"]),
        "profile": PROFILE_DESC[args.profile],
        "setup": "partial Grams + one allreduce of [packed upper H | A^T b] (configs[4] as "
                 "written); not reference-bitwise",
        "parallelism": f"row blocks x{ws}: partial Gram per GPU, one NCCL allreduce "
                       f"({(n * (n + 1) // 2 + n) * 8} B), iterations on rank 0",
        "iterations": iters, "partial_gram_ms": t_part * 1e3, "allreduce_ms": t_ar * 1e3,
        "solve_ms": t_solve * 1e3, "residual_sq": res,
        "roofline": {"kernel": "partial Gram per rank (" +
                     ("syrk_dmma_kernel, fp64 tensor cores" if args.profile == "fast"
                      else "exact chain SYRK") + ") + A^T b chains",
                     "bound": "tensor", "pipe": "fp64 DMMA", "achieved": ach, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": ach / FP64_PEAK_TFLOPS,
                     "peak_source": "measured (tools/microbench/fp64_probe.cu, DMMA)",
                     "algorithmic": f"rows*n*(n+1) + 2*rows*n = {flops_rank} flop per rank",
                     "traffic": None},
        "gpu_launches": launches, "clocks": clk.summary(), "e2e": None,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---- c4: batched multi-RHS, sharded by column ---------------------------------------------
C4_METRIC = "batched solve_nnls throughput, per-column KKT tol (columns/s)"
C4_UNIT = "columns/s"


def c4_shape(args):
    spec = instances.CONFIGS["c4"]
    return spec, spec["d"], spec["n"], (args.nrhs or spec["nrhs"])


def c4_cpu_sample(ora, A, spec, threads, ncols, H=None):
    """Reference pipeline on a bounded column sample, all host threads: the Gram
    once (shared across columns: a lower bound on the reference, whose
    solve_nnls recomputes it per call) plus per-column transpose_matvec,
    rescale, solve_nqp, unscale, residual; extrapolated to ncols columns."""
    d, n = A.shape
    S = max(threads, min(ncols, 48 * threads))
    Hs = instances.gen_htrue(n, S, spec["seed"], 0) if H is None else H
    Bs = np.asfortranarray(A @ Hs)
    from paper_1502_01645_b200.api import SolverConfig
    cfg = SolverConfig(epsilon=spec["epsilon"], stall_window=10**9).to_abi(record_multiplies=False)
    t = time.perf_counter()
    ora.gram(A)
    t_gram = time.perf_counter() - t
    t = time.perf_counter()
    ora.solve_nnls_columns(A, Bs, cfg, threads=threads)
    t_step = time.perf_counter() - t
    t_cols = max(1e-9, t_step - t_gram)
    t_full = t_gram + t_cols * ncols / S
    return ncols / t_full, {"sample_columns": S, "gram_s": t_gram, "sample_step_s": t_step,
                            "extrapolated_full_s": t_full,
                            "per_call_gram_note": "the reference solve_nnls recomputes the "
                                                  f"Gram per column (+{t_gram:.2f} s per column)"}


def run_reference_batched(args, ws):
    spec, d, n, K = c4_shape(args)
    ora, kind = ref_oracle()
    threads = os.cpu_count() or 1
    A = instances.gen_matrix(d, n, spec["seed"], "u01")
    H = instances.gen_htrue(n, max(threads, min(K, 48 * threads)), spec["seed"], 0)
    for _ in range(args.warmup):
        c4_cpu_sample(ora, A, spec, threads, K, H)
    vals, detail = [], None
    for _ in range(args.steps):
        v, detail = c4_cpu_sample(ora, A, spec, threads, K, H)
        vals.append(v)
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": C4_METRIC, "value": value, "unit": C4_UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": K / value * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SplitMix64, BASELINE.json configs[3])",
        "config": workload_config("c4", d, n, spec["epsilon"], nrhs=K),
        "cpu_baseline": {"value": value, "unit": C4_UNIT, "cores": threads, "kind": kind,
                         "sample": (f"{detail['sample_columns']} columns of B on {threads} threads "
                                    "(Gram once, shared), extrapolated to all columns"),
                         "breakdown": detail},
        "e2e": {"value": value, "unit": C4_UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours_batched(args, ws, rank, local, dist):
    import torch
    from paper_1502_01645_b200.api import Solver, SolverConfig
    from paper_1502_01645_b200.sharding import column_shard
    torch.cuda.set_device(local)
    spec, d, n, K = c4_shape(args)
    col0, kc = column_shard(K, ws, rank)
    A = instances.gen_matrix(d, n, spec["seed"], "u01")
    H = instances.gen_htrue(n, kc, spec["seed"], col0)  # this rank's columns of H_true
    dA = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()       # (n, d) == A column-major
    dH = torch.from_numpy(np.ascontiguousarray(H.T)).cuda()       # (kc, n) == H column-major
    dB = torch.empty((kc, d), dtype=torch.float64, device="cuda")  # (kc, d) == B column-major
    dX = torch.empty((kc, n), dtype=torch.float64, device="cuda")
    cfg = SolverConfig(epsilon=spec["epsilon"], stall_window=10**9, profile=PROFILE[args.profile])
    s = Solver(local)
    # B = A H_true in the reference's matvec order (untimed harness step): the same
    # bytes tests/test_gpu_c4_full.py pins against the reference's per-column solves
    s.matmat_device(d, n, kc, dA.data_ptr(), d, dH.data_ptr(), n, dB.data_ptr(), d)
    del dH
    torch.cuda.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()

    def solve(fetch=False):
        return s.solve_nnls_batched_device(dA.data_ptr(), dB.data_ptr(), dX.data_ptr(), d, n, kc,
                                           cfg, fetch_cols=fetch)

    cols, tm0 = solve(fetch=True)
    mults = tm0["multiplies_total"]  # summed from the per-column results
    for _ in range(max(0, args.warmup - 1)):
        solve()
    iters = np.array([c["iterations"] for c in cols])
    err = float((dX - torch.from_numpy(np.ascontiguousarray(H.T)).cuda()).abs().max())
    barrier()
    torch.cuda.synchronize()
    l0 = s.launch_count()
    t_setup = t_loop = t_fin = 0.0
    with ClockSampler(local) as clk:
        s.timer_start()
        for _ in range(args.steps):
            _, tm = solve()
            t_setup += tm["setup_s"]
            t_loop += tm["loop_s"]
            t_fin += tm["finish_s"]
        t = s.timer_stop()
    torch.cuda.synchronize()
    barrier()
    launches = (s.launch_count() - l0) // max(1, args.steps)

    def max_over_ranks(v):
        if dist is None:
            return v
        tt = torch.tensor([v], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    t_max = max_over_ranks(t)
    value = K * args.steps / t_max

    # e2e: host-buffer public API; A and this rank's B from pinned host memory,
    # X and the per-column results read back every step.
    pA = torch.empty((n, d), dtype=torch.float64, pin_memory=True)
    pA.copy_(dA)
    pB = torch.empty((kc, d), dtype=torch.float64, pin_memory=True)
    pB.copy_(dB)
    hA, hB = pA.numpy().T, pB.numpy().T  # Fortran-ordered views, no copy
    del dB
    torch.cuda.empty_cache()
    pX = torch.empty((kc, n), dtype=torch.float64, pin_memory=True)
    hX = pX.numpy().T  # the caller's reusable (n x kc) result buffer, read back every step
    s.solve_nnls_batched(hA, hB, cfg, out=hX)  # warm
    barrier()
    s.timer_start()
    for _ in range(args.steps):
        s.solve_nnls_batched(hA, hB, cfg, out=hX)
    te = max_over_ranks(s.timer_stop())
    e2e = {"value": K * args.steps / te, "unit": C4_UNIT,
           "h2d_bytes_per_step": 8 * (d * n + d * kc),
           "d2h_bytes_per_step": 8 * n * kc + 48 * kc}
    if rank != 0:
        return 0
    per_loop = t_loop / args.steps
    loop_tf = 2.0 * mults / per_loop / 1e12 if per_loop > 0 else 0.0
    roof = {"kernel": "batched_nqp_kernel (per-column state machines over exact chain GEMM passes)",
            "bound": "tensor", "pipe": "fp64 SIMT (exact DMUL + DADD chains; the peak is the fp64 tensor peak)", "achieved": loop_tf, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
            "frac": loop_tf / FP64_PEAK_TFLOPS, "frac_of_exact_cap": loop_tf / FP64_EXACT_CAP_TFLOPS,
            "peak_source": "measured (tools/microbench/fp64_probe.cu, DMMA)",
            "algorithmic": (f"2 flop x reference multiply count (masked GEMVs) = {2 * mults} "
                            "flop per launch (rank 0's columns)"),
            # measured on an 8192-column launch (the kernel reads Q from L2 and each
            # column's B / X once), scaled linearly to rank 0's columns
            "traffic": (None if traffic_from_profiles("c4_nrhs8192", "batched_nqp_kernel") is None
                        else int(traffic_from_profiles("c4_nrhs8192", "batched_nqp_kernel")
                                 * kc / 8192)),
            "traffic_note": "ncu dram bytes of an 8192-column launch scaled to the columns"}
    if args.profile == "fast":
        roof.update({"kernel": "batched_fast_kernel (warp-local per-column state machines over "
                               "DMMA m16n8k8 Q.V passes on fragment-ordered Q)",
                     "bound": "tensor", "pipe": "fp64 DMMA", "frac_of_exact_cap": None,
                     "traffic": (None if traffic_from_profiles("c4_nrhs8192", "batched_fast_kernel") is None
                                 else int(traffic_from_profiles("c4_nrhs8192", "batched_fast_kernel")
                                          * kc / 8192))})
    line = {
        "metric": C4_METRIC, "value": value, "unit": C4_UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded SplitMix64, BASELINE.json configs[3]; B = A H_true formed on device)",
        "config": workload_config("c4", d, n, spec["epsilon"], nrhs=K),
        "profile": ("exact (bitwise per-column reference trajectory)"
                    if args.profile == "exact" else PROFILE_DESC["fast"]),
        "parallelism": f"column shards x{ws} (no data-path collective)", "columns_rank0": kc,
        "iterations_mean": float(iters.mean()), "iterations_max": int(iters.max()),
        "max_abs_err_vs_H_true": err,
        "setup_ms": t_setup / args.steps * 1e3, "loop_ms": per_loop * 1e3,
        "finish_ms": t_fin / args.steps * 1e3,
        "roofline": roof, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk.summary(),
    }
    if ws == 1 and not args.no_cpu_baseline:
        ora, kind = ref_oracle()
        threads = os.cpu_count() or 1
        v, detail = c4_cpu_sample(ora, A, spec, threads, K)
        line["cpu_baseline"] = {"value": v, "unit": C4_UNIT, "cores": threads, "kind": kind,
                                "sample": (f"{detail['sample_columns']} columns on {threads} threads "
                                           "(Gram once, shared), extrapolated to all columns"),
                                "breakdown": detail}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--nrhs", type=int, default=0, help="c4: override the column count")
    ap.add_argument("--profile", default="exact", choices=["exact", "fast"],
                    help="fast: tensor-core (DMMA) Gram / batched passes, opt-in, not bitwise")
    ap.add_argument("--solver", default="nnls", choices=["nnls", "anti_acc"],
                    help="anti_acc: the Anti+Acc baseline (accelerated.hpp) on the same workload")
    ap.add_argument("--c5-setup", default="pipeline", choices=["pipeline", "allreduce"],
                    help="c5: exact k-chain row-block pipeline (bitwise) or partial Grams + one "
                         "allreduce (configs[4] as written)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    env_ws = os.environ.get("WORLD_SIZE")
    if env_ws is None and args.gpus > 1:
        # one process per GPU: re-launch under torch.distributed.run (NCCL, 127.0.0.1)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    if env_ws is not None and int(env_ws) != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} does not match WORLD_SIZE={env_ws}"}),
              flush=True)
        return 2
    ws, rank, local, dist = dist_setup(args)
    try:
        if args.impl == "reference":
            return run_reference(args, ws, rank)
        if args.workload == "c4":
            return run_ours_batched(args, ws, rank, local, dist)
        if args.workload == "c5" and args.c5_setup == "allreduce":
            return run_ours_allreduce(args, ws, rank, local, dist)
        if args.workload == "c5" and (ws > 1 or os.environ.get("ALNNLS_FORCE_ROWBLOCK")):
            return run_ours_rowblock(args, ws, rank, local, dist)
        return run_ours(args, ws, rank, local, dist)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
