"""Epoch-loop cycle split of the cluster learning kernel, CTA 0 of each launch
(build with CL_NVCC_EXTRA=-DCL_CLUSTER_TRACE):  python tools/cluster_trace.py [config]"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2501_11592_b200 as cl  # noqa: E402

c = cl.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 7]
A, X, Y, _ = cl.gen_problem_1d(c["seed"], c["m"], c["n"], c["k"], c["batch"],
                               value_law=c["value_law"], snr_db=c["snr_db"])
ctx = cl.ClompContext(A)
cfg = cl.ClompConfig.baseline(c["k"])
cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL, dense=False)
buf = np.zeros(8, np.uint64)
cl.lib().cl_debug_cluster_trace(buf.ctypes.data_as(C.c_void_p))
E = max(int(buf[4]), 1)
for nm, v in zip(["wait", "fma", "reduce", "step+store"], buf[:4]):
    print(f"{nm:12s} {int(v) / E:8.1f} cycles/epoch")
print("epochs traced", E)
S = max(int(buf[7]), 1)
print(f"per signal: prologue {int(buf[5]) / S:.0f} cycles, after-epochs {int(buf[6]) / S:.0f} cycles, "
      f"epochs {E / S:.1f}, signals traced {S}")
