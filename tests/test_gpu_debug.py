"""The debug build (-DCL_DEBUG_CHECKS: device-side asserts on every index the
kernels form from data — atoms, support slots, list slots, tiles;
clomp_internal.cuh) runs every kernel family without tripping a check and
returns the same results as the release build.  Stands in for
compute-sanitizer, which this GPU pool does not allow."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
DBG = ROOT / "paper_2501_11592_b200" / "_build" / "libclomp_b200_dbg.so"


def _run(lib):
    env = dict(os.environ)
    if lib:
        env["CLOMP_B200_LIB"] = str(lib)
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "debug_build_probe.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "PROBE OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
    return [ln for ln in r.stdout.splitlines() if ": " in ln]


def test_debug_build_runs_clean_and_agrees(gpu_available):
    if not DBG.exists():
        pytest.fail(f"{DBG} not built (python -m paper_2501_11592_b200.build --debug)")
    assert _run(DBG) == _run(None)
