"""The C-ABI library loads and exports every symbol include/clomp_b200.h
declares; host-side logic that needs no GPU (CPU-only)."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2501_11592_b200 as cl

HEADER = Path(__file__).resolve().parents[1] / "include" / "clomp_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:[\w\*]+\s+\**)+\**(cl_\w+)\s*\(", text, re.M)))


def test_header_declares_what_python_binds():
    syms = declared_symbols()
    assert "cl_solve_batch" in syms and "cl_create" in syms
    for s in syms:
        assert s in cl.EXPORTED, s


def test_library_exports_every_declared_symbol(built_lib):
    h = C.CDLL(str(built_lib))
    for s in declared_symbols() + ["cl_rng_draws", "cl_gen_problem_1d"]:
        assert hasattr(h, s), f"missing export {s}"
    assert h.cl_abi_version() == 1


def test_python_struct_mirrors_match_the_library(built_lib):
    """The ctypes mirrors have the library's struct sizes (a field added on one
    side only would shift every later pointer)."""
    h = C.CDLL(str(built_lib))
    out = (C.c_int64 * 4)()
    h.cl_abi_struct_sizes(out)
    assert list(out) == [C.sizeof(cl.CConfig), C.sizeof(cl.CResult), C.sizeof(cl.CDeviceResult),
                         C.sizeof(cl.CStats)]


def test_default_config_matches_reference(built_lib):
    c = cl.CConfig()
    cl.lib().cl_config_default(C.byref(c))
    d = cl.ClompConfig()
    for f, _ in cl.CConfig._fields_:
        if f == "pad0":
            continue
        assert getattr(c, f) == getattr(d, f), f
    # clomp.hpp:16-33
    assert (d.th, d.max_outer, d.eps, d.inner_steps, d.lr, d.opt) == (0.7, 200, 1e-6, 50, 0.01, cl.ADAM)


def test_no_device_fails_loudly(built_lib):
    if cl.lib().cl_device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(cl.CudaError):
        cl.ClompContext(np.ones((4, 8), np.float32))


def test_baseline_mapping():
    c = cl.ClompConfig.baseline(32)
    assert (c.th, c.max_outer, c.inner_steps, c.lr, c.opt, c.w_tv, c.w_lv) == (1.0, 32, 200, 0.1, cl.PLAIN, 0.0, 0.0)


def test_ragged_rows_view_counts():
    import paper_2501_11592_b200 as cl
    r = cl.Ragged(np.arange(12, dtype=np.int32).reshape(3, 4), np.array([1, 4, 0]))
    assert len(r) == 3
    assert r[0].tolist() == [0] and r[1].tolist() == [4, 5, 6, 7] and r[2].size == 0
    assert [x.tolist() for x in r[0:2]] == [[0], [4, 5, 6, 7]]
    res = cl.BatchSolveResult(None, None, np.zeros(3), np.zeros(3), np.zeros(3, bool),
                              np.zeros(3, np.int32), r, r)
    assert res.support[1].tolist() == [4, 5, 6, 7]


def test_header_is_plain_c_and_links(built_lib, tmp_path):
    """include/clomp_b200.h compiles as C99 (pedantic) and as C++, and a C
    program using it links against the library (no CUDA, torch or C++ types in
    the boundary)."""
    import shutil
    import subprocess

    if not shutil.which("gcc"):
        pytest.skip("no gcc")
    inc = HEADER.parent
    src = tmp_path / "use_abi.c"
    src.write_text(
        '#include <stdio.h>\n#include "clomp_b200.h"\n'
        "int main(void) {\n"
        "  cl_config c; int64_t sz[4]; cl_config_default(&c); cl_abi_struct_sizes(sz);\n"
        "  cl_result r = {0}; (void)r;\n"
        '  printf("%d %d %lld %lld\\n", cl_abi_version(), (int)(c.th * 10), (long long)sz[0], (long long)sizeof(cl_config));\n'
        "  return sz[0] == (int64_t)sizeof(cl_config) && sz[1] == (int64_t)sizeof(cl_result) ? 0 : 1;\n}\n")
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", f"-I{inc}",
                    "-fsyntax-only", str(src)], check=True)
    subprocess.run(["g++", "-std=c++17", "-Wall", "-Werror", f"-I{inc}", "-fsyntax-only", "-x", "c++",
                    str(src)], check=True)
    exe = tmp_path / "use_abi"
    lib = Path(built_lib)
    subprocess.run(["gcc", "-std=c99", f"-I{inc}", str(src), "-o", str(exe), f"-L{lib.parent}",
                    "-lclomp_b200", f"-Wl,-rpath,{lib.parent}"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.split()[:2] == ["1", "7"]
