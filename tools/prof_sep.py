"""One separable config solve for ncu captures: python tools/prof_sep.py --config 4 --batch 64 --max-outer 740 [--direct K]"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2501_11592_b200 as cl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--max-outer", type=int, default=0)
ap.add_argument("--direct", type=int, default=-1)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
c = dict(cl.CONFIGS[a.config])
B = a.batch or c["batch"]
Ar, Ac, X, Y = cl.gen_problem_2d(c["seed"], c["n_r"], c["n_c"], c["m_r"], c["m_c"], c["k"], B)
ctx = cl.ClompContext.separable(Ar, Ac)
ctx.set_direct_form(a.direct)
cfg = cl.ClompConfig.baseline(c["k"])
if a.max_outer:
    cfg.max_outer = a.max_outer
for _ in range(a.reps):
    t0 = time.time()
    r = cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL, dense=False)
    print(f"solve {time.time() - t0:.3f}s outer {cfg.max_outer} status {int(r.status.max())} stats {ctx.stats()}")
