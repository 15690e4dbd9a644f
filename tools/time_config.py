"""Time a full BASELINE config solve through the C-ABI (events inside the
library), e.g.  python tools/time_config.py --config 3 --batch 256"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2501_11592_b200 as cl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--max-outer", type=int, default=0)
a = ap.parse_args()
c = dict(cl.CONFIGS[a.config])
B = a.batch or c["batch"]
t0 = time.time()
if "n_r" in c:  # separable 2D configs
    Ar, Ac, X, Y = cl.gen_problem_2d(c["seed"], c["n_r"], c["n_c"], c["m_r"], c["m_c"], c["k"], B)
    t1 = time.time()
    ctx = cl.ClompContext.separable(Ar, Ac)
else:
    A, X, Y, _ = cl.gen_problem_1d(c["seed"], c["m"], c["n"], c["k"], B,
                                   value_law=c["value_law"], snr_db=c["snr_db"])
    t1 = time.time()
    ctx = cl.ClompContext(A)
t2 = time.time()
cfg = cl.ClompConfig.baseline(c["k"])
if a.max_outer:
    cfg.max_outer = a.max_outer
for r in range(a.reps):
    t3 = time.time()
    res = cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL)
    t4 = time.time()
    st = ctx.stats()
    print(f"rep {r}: wall {t4 - t3:.3f}s e2e {st['e2e_ms']:.1f} ms, {B / (st['e2e_ms'] / 1e3):.1f} signals/s, "
          f"rescans {st['rescans']}, status max {int(res.status.max())}")
rec = np.mean([set(np.flatnonzero(res.mask[:, b])) <= set(np.flatnonzero(X[:, b])) for b in range(B)])
print(f"gen {t1 - t0:.1f}s ctx {t2 - t1:.2f}s; support recovered for {rec * 100:.1f}% of signals; "
      f"iterations {np.unique(res.iterations)}")
