"""Build libclomp_b200.so in-tree (sm_100a only).

    python -m paper_2501_11592_b200.build        # or __graft_entry__.build()

Every .cu / .cpp under csrc/ (except csrc/shim/, built separately) is compiled
with nvcc for `-gencode arch=compute_100a,code=sm_100a -lineinfo` and linked
into paper_2501_11592_b200/_build/libclomp_b200.so with the CUDA runtime
linked statically, so the library loads on a CPU-only host (for the ABI
tests) and needs only the driver on the GPU box.
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT = PKG / "_build"
INCLUDE = PKG.parent / "include"
LIB = OUT / "libclomp_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
    "-Xcompiler", "-Wall", "--expt-relaxed-constexpr", "-Xptxas", "-v",
    f"-I{INCLUDE}", f"-I{CSRC}",
]


# Experiment hook: extra -D flags (e.g. CL_NVCC_EXTRA="-DCL_SQ_COST=2").
NVCC_FLAGS += os.environ.get("CL_NVCC_EXTRA", "").split()


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _sources() -> list[Path]:
    return sorted(p for p in CSRC.glob("*") if p.suffix in (".cu", ".cpp"))


def _digest(paths: list[Path]) -> str:
    h = hashlib.sha256()
    for p in paths:
        h.update(p.name.encode())
        h.update(p.read_bytes())
    h.update(" ".join(NVCC_FLAGS).encode())
    return h.hexdigest()


def _compile(src: Path) -> tuple[Path, str]:
    obj = OUT / (src.stem + ".o")
    cmd = [nvcc()] + NVCC_FLAGS + ["-c", str(src), "-o", str(obj)]
    if src.suffix == ".cpp":
        cmd = [nvcc(), "-x", "cu"] + NVCC_FLAGS + ["-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src.name}:\n{res.stdout}\n{res.stderr}")
    return obj, res.stderr


def build_debug() -> Path:
    """libclomp_b200_dbg.so: the same sources with -DCL_DEBUG_CHECKS (device-side
    asserts on data-derived indices, clomp_internal.cuh), objects kept apart."""
    dbg = OUT / "dbg"
    dbg.mkdir(parents=True, exist_ok=True)
    lib = OUT / "libclomp_b200_dbg.so"
    srcs = _sources()
    headers = sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))
    stamp = dbg / "build.stamp"
    digest = _digest(srcs + headers)
    if lib.exists() and stamp.exists() and stamp.read_text() == digest:
        return lib

    def comp(src: Path) -> Path:
        obj = dbg / (src.stem + ".o")
        # --split-compile: ptxas works through a translation unit's kernels in
        # parallel (k_solve.cu is ~4 min of single-threaded ptxas).  Debug build
        # only: it measured 3-13 % slower code on the release kernels.
        flags = [f for f in NVCC_FLAGS if f not in ("-Xptxas", "-v")] + [
            "-DCL_DEBUG_CHECKS", "--split-compile", str(min(8, os.cpu_count() or 1))]
        cmd = [nvcc()] + (["-x", "cu"] if src.suffix == ".cpp" else []) + flags + ["-c", str(src), "-o", str(obj)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc (debug) failed on {src.name}:\n{res.stdout}\n{res.stderr}")
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = [str(o) for o in ex.map(comp, srcs)]
    cmd = [nvcc()] + ARCH + ["-shared", "-cudart", "static", "-o", str(lib)] + objs + ["-lpthread", "-ldl", "-lrt"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link (debug) failed:\n{res.stdout}\n{res.stderr}")
    stamp.write_text(digest)
    return lib


def build(verbose: bool = False, force: bool = False) -> Path:
    OUT.mkdir(parents=True, exist_ok=True)
    srcs = _sources()
    headers = sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))
    stamp = OUT / "build.stamp"
    digest = _digest(srcs + headers)
    if LIB.exists() and stamp.exists() and stamp.read_text() == digest and not force:
        return LIB
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        results = list(ex.map(_compile, srcs))
    log = "\n".join(f"== {o.name}\n{err}" for o, err in results)
    (OUT / "ptxas.log").write_text(log)
    if verbose:
        print(log)
    objs = [str(o) for o, _ in results]
    cmd = [nvcc()] + ARCH + ["-shared", "-cudart", "static", "-o", str(LIB)] + objs + ["-lpthread", "-ldl", "-lrt"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    stamp.write_text(digest)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
    if "--debug" in sys.argv:
        print(build_debug())
