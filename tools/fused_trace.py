"""Phase timing of the fused small solve (config 1), build with -DCL_LEARN_TRACE."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2501_11592_b200 as cl  # noqa: E402

c = dict(cl.CONFIGS[1])
A, X, Y, _ = cl.gen_problem_1d(c["seed"], c["m"], c["n"], c["k"], 1)
ctx = cl.ClompContext(A)
cfg = cl.ClompConfig.baseline(c["k"])
for _ in range(3):
    r = cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL, dense=False)
buf = np.zeros((16, 8), np.uint64)
n = cl.lib().cl_debug_learn_trace(C.c_void_p(buf.ctypes.data), 16)
t = buf.astype(np.int64)
names = ["correlation", "select", "gram + b", "epochs", "sync", "residual", "control"]
print("outer: " + " ".join(f"{nm:>12s}" for nm in names) + "   (cycles)")
for o in range(1, c["k"] + 1):
    d = [t[o, i + 1] - t[o, i] for i in range(6)] + [t[o + 1, 0] - t[o, 6] if o < c["k"] else 0]
    print(f"{o:5d}: " + " ".join(f"{int(v):12d}" for v in d) + f"   total {int(t[o, 6] - t[o, 0])}")
print("stats", ctx.stats())
