"""Small power-form / cluster / tie problem for compute-sanitizer runs:
    compute-sanitizer --tool memcheck python tools/sanitize_power.py"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2501_11592_b200 as cl  # noqa: E402

m, n, B, K = 512, 1024, 6, 72
A, X, Y, _ = cl.gen_problem_1d(7, m, n, K, B, value_law=1)
cfg = cl.ClompConfig.baseline(K)
cfg.inner_steps = 203  # leftover plain epochs (PH 1) + squarings + PH 2
ctx = cl.ClompContext(A)
ctx.set_fused(False)
r = cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL)
print("status", r.status.tolist(), "iters", r.iterations.tolist(), "supports",
      r.mask.sum(axis=0).tolist())
