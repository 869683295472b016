"""The reference's own benchmark harness, unmodified, over this repo's GPU facade
(harness integration, instance families, report formats).

oracle/Makefile `harness` compiles tests/cpp/ref_harness_driver.cpp against the
reference's bench.hpp / testgen.hpp / io.hpp / active_set.hpp in place, twice:
over the reference's own solver headers (harness_ref, CPU) and over
include/antilop (harness_gpu: every gram / matvec / solve_nnls /
solve_accelerated / solve_anti_accelerated call goes through libalnnls on the
GPU). Both print the suite's bench-report/1 JSON (bench.hpp:287-369); apart
from wall times they must be identical: same instances (testgen T1-T6), same
objectives, gaps, iteration counts and terminations, bit for bit, for all four
solvers of the reference's lineup (the CPU active-set "fast" baseline included,
its linear algebra now on the GPU)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref", "harness_ref")
GPU = os.path.join(ROOT, "oracle", "_ref", "harness_gpu")
WALL = {"wall_s", "mean_wall_s"}


def _strip(x):
    if isinstance(x, dict):
        return {k: _strip(v) for k, v in x.items() if k not in WALL}
    if isinstance(x, list):
        return [_strip(v) for v in x]
    return x


def _run(exe, args):
    r = subprocess.run([exe] + [str(a) for a in args], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr
    return json.loads(r.stdout)


def _need():
    if not (os.path.exists(REF) and os.path.exists(GPU)):
        pytest.skip("oracle/_ref harness binaries not built (reference sources absent at build)")


@pytest.mark.gpu
@pytest.mark.parametrize("args", [
    # the reference's default desk suite: T1-T6 x 5 sub-tests, n=400, d=600, all solvers
    (400, 600, 5, 1, "T1,T2,T3,T4,T5,T6", "antilop,fast,accer,anti-accer"),
    (37, 53, 3, 11, "T1,T3,T5", "antilop,anti-accer"),
])
def test_reference_harness_over_gpu_facade(args):
    _need()
    ref = _run(REF, args)
    gpu = _run(GPU, args)
    assert ref["schema"] == gpu["schema"] == "bench-report/1"
    assert len(ref["cells"]) == len(gpu["cells"]) > 0
    for a, b in zip(ref["cells"], gpu["cells"]):
        assert _strip(a) == _strip(b), (a, b)
    assert _strip(ref) == _strip(gpu)


def test_reference_harness_cpu_runs():
    """CPU side: the harness compiled over the reference headers runs (no GPU needed)."""
    _need()
    rep = _run(REF, (12, 18, 2, 5, "T2", "antilop"))
    assert rep["schema"] == "bench-report/1" and len(rep["cells"]) == 2


def _trace_wo_time(path):
    rows = [ln.split(",") for ln in open(path).read().strip().splitlines()]
    assert rows[0][1] == "elapsed_ms"
    return [r[:1] + r[2:] for r in rows]


@pytest.mark.gpu
@pytest.mark.parametrize("kind,n,d,sp,seed", [("T5", 30, 45, 0.2, 9), ("T2", 120, 200, 0.3, 4),
                                              ("T6", 64, 64, 0.0, 2)])
@pytest.mark.parametrize("solver", ["antilop", "anti-accer", "accer", "fast"])
def test_reference_cli_bodies_over_gpu_facade(tmp_path, kind, n, d, sp, seed, solver):
    """bench.hpp cmd_generate -> MatrixMarket instance dir (io.hpp, testgen.hpp save/load),
    then cmd_solve through both builds: the result summary JSON (nnls.hpp:146-153) and
    the trace CSV (nqp.hpp:345-357, minus its wall-clock column) agree bit for bit."""
    _need()
    a, b = tmp_path / "ref", tmp_path / "gpu"
    subprocess.run([REF, "gen", kind, str(n), str(d), str(sp), str(seed), str(a)], check=True,
                   capture_output=True)
    subprocess.run([REF, "gen", kind, str(n), str(d), str(sp), str(seed), str(b)], check=True,
                   capture_output=True)
    out_r = subprocess.run([REF, "solve", solver, str(a)], capture_output=True, text=True)
    out_g = subprocess.run([GPU, "solve", solver, str(b)], capture_output=True, text=True)
    assert out_r.returncode == out_g.returncode, (out_r.stdout, out_g.stdout, out_g.stderr)
    assert out_r.stdout == out_g.stdout
    tr = f"trace-{solver}.csv"
    assert _trace_wo_time(a / tr) == _trace_wo_time(b / tr)


ACC_REF = os.path.join(ROOT, "oracle", "_ref", "acceptance_ref")
ACC_GPU = os.path.join(ROOT, "oracle", "_ref", "acceptance_gpu")


@pytest.mark.gpu
def test_reference_acceptance_gate_over_gpu_facade():
    """The reference's acceptance gate (tests/acceptance.cpp: rescaling invariants, the 2^n
    brute-force oracle, KKT certification of the desk suite, the 2-variable contrast, the
    linear-rate envelope, monotone descent, optimality, bit-for-bit replay), compiled over
    the GPU facade: every criterion passes and every reported figure (worst gaps, certified
    counts, iteration counts, ratios) equals the CPU reference build's."""
    if not (os.path.exists(ACC_REF) and os.path.exists(ACC_GPU)):
        pytest.skip("oracle/_ref acceptance binaries not built (reference sources absent at build)")
    ref = subprocess.run([ACC_REF], capture_output=True, text=True, timeout=1500)
    gpu = subprocess.run([ACC_GPU], capture_output=True, text=True, timeout=1500)
    assert gpu.returncode == 0, gpu.stdout + gpu.stderr
    assert "all criteria passed" in gpu.stdout
    assert ref.stdout == gpu.stdout
