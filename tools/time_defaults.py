"""Timing of non-headline configurations at config 2's shape: th < 1, Adam,
the reference's default ClompConfig (priors on, per signal), joint mode."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2501_11592_b200 as cl  # noqa: E402

c = dict(cl.CONFIGS[2])
B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
A, X, Y, _ = cl.gen_problem_1d(c["seed"], c["m"], c["n"], c["k"], B, snr_db=c["snr_db"])
ctx = cl.ClompContext(A)
ctx.set_basis(cl.dct_basis(c["n"]))


def run(name, cfg, mode=cl.MODE_PER_SIGNAL, reps=2):
    best = 1e9
    for _ in range(reps):
        t0 = time.perf_counter()
        r = cl.clomp_solve_batch(ctx, Y, cfg, mode=mode, dense=False)
        best = min(best, time.perf_counter() - t0)
    st = ctx.stats()
    print(f"{name:46s} {best * 1e3:9.2f} ms  {B / best:12.0f} signals/s  iters max {int(r.iterations.max()):3d} "
          f"support mean {np.mean([len(s) for s in r.support]):6.1f} launches {st['kernel_launches']} status max {int(r.status.max())}")


base = cl.ClompConfig.baseline(c["k"])
run("baseline (th 1, plain, K = 32)", base)
adam = cl.ClompConfig.baseline(c["k"]); adam.opt = cl.ADAM; adam.lr = 0.02
run("th 1, Adam", adam)
mom = cl.ClompConfig.baseline(c["k"]); mom.opt = cl.MOMENTUM; mom.lr = 0.02
run("th 1, momentum", mom)
th07 = cl.ClompConfig.baseline(c["k"]); th07.th = 0.7; th07.max_outer = 12
run("th 0.7, plain, 12 outer", th07)
joint = cl.ClompConfig.baseline(c["k"])
run("baseline, joint mode (clomp_solve_batch)", joint, mode=cl.MODE_JOINT)
d = cl.ClompConfig(); d.max_outer = 20
run("reference defaults (th 0.7, Adam, TV auto), 20 outer", d)
d0 = cl.ClompConfig(); d0.max_outer = 20; d0.w_tv = 0.0; d0.w_lv = 0.0
run("defaults without priors, 20 outer", d0)
