"""CPU checks of the drop-in boundary: the C-ABI library loads without a GPU,
exports every symbol include/alnnls.h declares, its POD layouts match the
ctypes mirrors, and the product fails loudly (no CPU fallback) when no GPU is
present. No compute calls are made here."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_1502_01645_b200 import _native, abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "alnnls.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(alnnls_[A-Za-z_0-9]+)\s*\(", src)))


def test_header_symbols_listed():
    assert set(declared_symbols()) == set(_native.EXPORTS)


def test_library_exports_every_symbol():
    lib = C.CDLL(_native.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    for name in declared_symbols():
        assert re.search(rf"\bT {name}\b", out), name


def test_pod_layouts_match_ctypes(tmp_path):
    prog = tmp_path / "sizes.c"
    prog.write_text(f'''#include <stdio.h>
#include <stddef.h>
#include "{HEADER}"
int main(void) {{
  printf("%zu %zu %zu %zu\\n", sizeof(alnnls_config), sizeof(alnnls_iter_record),
         sizeof(alnnls_summary), sizeof(alnnls_column_result));
  printf("%zu %zu %zu\\n", offsetof(alnnls_config, profile), offsetof(alnnls_summary, t_setup_s),
         offsetof(alnnls_iter_record, has_alpha));
  return 0;
}}''')
    exe = tmp_path / "sizes"
    subprocess.run(["gcc", "-std=c11", "-o", str(exe), str(prog)], check=True)
    lines = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    sizes = [int(v) for v in lines[0].split()]
    offs = [int(v) for v in lines[1].split()]
    assert sizes == [C.sizeof(abi.Config), C.sizeof(abi.IterRecord), C.sizeof(abi.Summary),
                     C.sizeof(abi.ColumnResult)]
    assert offs == [abi.Config.profile.offset, abi.Summary.t_setup_s.offset,
                    abi.IterRecord.has_alpha.offset]


def test_config_defaults_match_reference():
    lib = _native.load()
    c = abi.Config()
    lib.alnnls_config_default(C.byref(c))
    # SolverConfig{} (nqp.hpp:71-99): unset epsilon/max_iters/time_cap, stall 50, trace 1
    assert (c.has_epsilon, c.has_max_iters, c.has_time_cap) == (0, 0, 0)
    assert (c.stall_window, c.trace_every, c.profile) == (50, 1, abi.PROFILE_EXACT)
    assert lib.alnnls_abi_version() == 2


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_1502_01645_b200.api import Solver
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        Solver(0)
    lib = _native.load()
    ctx = C.c_void_p()
    assert lib.alnnls_create(C.byref(ctx), 0) == abi.ENODEV


def test_sm100a_code_only():
    """The library carries sm_100a SASS (tcgen05-era target), no PTX fallback for other archs."""
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_solver_config_resolution():
    from paper_1502_01645_b200.api import SolverConfig
    c = SolverConfig()
    assert c.resolve_epsilon(300) == 1e-10 * 300 and c.resolve_max_iters(300) == 1500
    with pytest.raises(ValueError):
        SolverConfig(epsilon=0.0).resolve_epsilon(3)
    with pytest.raises(ValueError):
        SolverConfig(max_iters=0).resolve_max_iters(3)
    assert abi.trace_capacity(SolverConfig(max_iters=10, trace_every=4).to_abi(), 5) == 4
