import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import time, numpy as np, torch
import paper_2501_11592_b200 as cl
c = cl.CONFIGS[2]
A, X, Y, _ = cl.gen_problem_1d(1, c["m"], c["n"], c["k"], c["batch"], snr_db=40.0)
ctx = cl.ClompContext(A)
cfg = cl.ClompConfig.baseline(c["k"])
Yp = torch.empty(Y.shape, dtype=torch.float32, pin_memory=True).numpy(); Yp[...] = Y
for i in range(6):
    t0 = time.perf_counter()
    r = cl.clomp_solve_batch(ctx, Yp, cfg, mode=cl.MODE_PER_SIGNAL, dense=False)
    t1 = time.perf_counter()
    print(i, "wall ms", (t1 - t0) * 1e3, "lib e2e ms", ctx.stats()["e2e_ms"], "total_ms", ctx.stats()["total_ms"])
for i in range(2):
    t0 = time.perf_counter()
    r = cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL, dense=True)
    print("dense pageable wall ms", (time.perf_counter() - t0) * 1e3, "lib", ctx.stats()["e2e_ms"])
