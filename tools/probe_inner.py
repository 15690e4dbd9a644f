"""Config-2 solve time vs inner_steps (epochs): separates the learning
kernel's epoch cost from selection / extension / residual / K1."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2501_11592_b200 as cl  # noqa: E402

c = dict(cl.CONFIGS[2])
A, X, Y, _ = cl.gen_problem_1d(c["seed"], c["m"], c["n"], c["k"], c["batch"],
                               value_law=c["value_law"], snr_db=c["snr_db"])
ctx = cl.ClompContext(A)
Yd = torch.from_numpy(Y.T.copy()).cuda()
for inner in (200, 100, 16, 1):
    cfg = cl.ClompConfig.baseline(c["k"])
    cfg.inner_steps = inner
    cfg.stall_patience = 1 << 30  # keep every signal to max_outer
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL, dense=False)
        dt = time.perf_counter() - t0
    st = ctx.stats()
    print(f"inner={inner:4d} e2e {dt*1e3:7.3f} ms  lib {st['e2e_ms']:.3f} ms  iters {int(r.iterations.mean())}")
