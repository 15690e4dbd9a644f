"""Run one config solve (after a warm-up) for ncu / compute-sanitizer captures.

    python tools/prof_solve.py [--config 2] [--batch B] [--path 0|1|2]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2501_11592_b200 as cl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--path", type=int, default=0)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--events", action="store_true", help="profiling mode: plain launches, no graphs")
a = ap.parse_args()
c = dict(cl.CONFIGS[a.config])
B = a.batch or c["batch"]
A, X, Y, _ = cl.gen_problem_1d(c["seed"], c["m"], c["n"], c["k"], B,
                               value_law=c["value_law"], snr_db=c["snr_db"])
ctx = cl.ClompContext(A)
if a.path:
    ctx.set_corr_path(a.path)
if a.events:
    ctx.set_profiling(True)
cfg = cl.ClompConfig.baseline(c["k"])
for _ in range(1 + a.reps):
    r = cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL)
print("ok", ctx.stats(), int(r.status.max()))
