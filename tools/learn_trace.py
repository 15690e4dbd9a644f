"""Phase timing of k_learn_fast per signal (build with CL_NVCC_EXTRA=-DCL_LEARN_TRACE).

    python tools/learn_trace.py [--max-outer T]   # the last launch is the t = T one
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2501_11592_b200 as cl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--max-outer", type=int, default=32)
a = ap.parse_args()
c = dict(cl.CONFIGS[2])
A, X, Y, _ = cl.gen_problem_1d(c["seed"], c["m"], c["n"], c["k"], c["batch"], snr_db=c["snr_db"])
ctx = cl.ClompContext(A)
cfg = cl.ClompConfig.baseline(c["k"])
cfg.max_outer = a.max_outer
for _ in range(2):
    cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL, dense=False)
B = c["batch"]
buf = np.zeros((B, 8), np.uint64)
n = cl.lib().cl_debug_learn_trace(C.c_void_p(buf.ctypes.data), B)
if n == 0:
    raise SystemExit("library not built with -DCL_LEARN_TRACE")
t = buf.astype(np.int64)
start_ns = t[:, 0] - t[:, 0].min()
names = ["state loads + record merge", "selection", "Gram row + b_k", "wait staged rows",
         "epochs", "residual + control"]
d = np.diff(t[:, 1:], axis=1).astype(np.float64)  # cycles per phase
tot = (t[:, 7] - t[:, 1]).astype(np.float64)
print(f"t = {a.max_outer}: {B} signals; per-warp cycles (median / mean / p95), share of the warp's time")
for i, nm in enumerate(names):
    print(f"  {nm:28s} {np.median(d[:, i]):9.0f} {d[:, i].mean():9.0f} {np.percentile(d[:, i], 95):9.0f}"
          f"   {d[:, i].sum() / tot.sum():6.3f}")
print(f"  {'whole warp':28s} {np.median(tot):9.0f} {tot.mean():9.0f} {np.percentile(tot, 95):9.0f}")
first = start_ns < 2000
print(f"warps starting within 2 us of the first: {first.sum()} ; later starts: median {np.median(start_ns[~first]) / 1e3 if (~first).any() else 0:.1f} us, "
      f"max {start_ns.max() / 1e3:.1f} us")
for lbl, sel in (("first wave", first), ("later", ~first)):
    if sel.any():
        print(f"  {lbl}: whole-warp cycles median {np.median(tot[sel]):.0f} ({np.median(tot[sel]) / 1.965e3:.1f} us at 1965 MHz)")
