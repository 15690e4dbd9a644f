"""Phase timeline of the CTA-pair K1 kernel (build with CL_NVCC_EXTRA=-DCL_K1_TRACE):
    python tools/k1_trace.py [--config 2]"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2501_11592_b200 as cl  # noqa: E402

c = cl.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 2]
A, X, Y, _ = cl.gen_problem_1d(c["seed"], c["m"], c["n"], c["k"], c["batch"],
                               value_law=c["value_law"], snr_db=c["snr_db"])
ctx = cl.ClompContext(A)
cfg = cl.ClompConfig.baseline(c["k"])
cfg.max_outer = 3
for _ in range(3):
    cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL, dense=False)
buf = np.zeros((1024, 16), np.uint64)
n = cl.lib().cl_debug_k1_trace(buf.ctypes.data_as(C.c_void_p), 1024)
ntile = (c["n"] + 255) // 256 * ((c["batch"] + 127) // 128)
t = buf[:ntile, :12].astype(np.int64)
t0 = t[:, 0].min()
rel = (t - t0) / 1000.0
names = ["entry", "setup done", "first stage", "last MMA issued", "accum ready", "epilogue done",
         "exit", "tmem loaded (t96)", "scan done (t96)", "scan done (t480)", "merge barrier (t0)",
         "record stored (t0)"]
for i, nm in enumerate(names):
    col = rel[:, i][rel[:, i] >= 0]
    print(f"{nm:16s} min {col.min():7.2f}  median {np.median(col):7.2f}  max {col.max():7.2f} us")
