"""Runs representative solves of every kernel family and prints a digest of the
results.  tests/test_gpu_debug.py runs it twice, against the normal library
and against the debug build (device-side index asserts), and compares."""
import hashlib
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2501_11592_b200 as cl  # noqa: E402


def digest(r):
    h = hashlib.sha256()
    for a in (r.mask, r.iterations, r.status, np.round(r.s, 9)):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


out = []
# batched th = 1 path (tcgen05 pair kernel, fused selection + warp learners), with
# duplicated atoms: exact ties -> rescoring, supports past the bucket, block kernel
A, X, Y, _ = cl.gen_problem_1d(5, 128, 512, 12, 300, snr_db=40.0)
A[:, 17] = A[:, 3]
A[:, 400] = A[:, 3]
ctx = cl.ClompContext(A)
ctx.set_fused(False)
out.append(("batched+ties", digest(cl.clomp_solve_batch(ctx, Y, cl.ClompConfig.baseline(12), mode=cl.MODE_PER_SIGNAL))))
# fused small solve
A, X, Y, _ = cl.gen_problem_1d(0, 128, 256, 10, 3)
out.append(("fused", digest(cl.clomp_solve_batch(cl.ClompContext(A), Y, cl.ClompConfig.baseline(10), mode=cl.MODE_PER_SIGNAL))))
# cluster learners + power form (33..256 atoms), GEMV correlation (B <= 4), column shards
A, X, Y, _ = cl.gen_problem_1d(7, 512, 1024, 72, 6, value_law=1)
cfg = cl.ClompConfig.baseline(72)
cfg.inner_steps = 203
ctx = cl.ClompContext(A)
out.append(("cluster+power", digest(cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL))))
out.append(("gemv", digest(cl.clomp_solve_batch(ctx, Y[:, :2], cfg, mode=cl.MODE_PER_SIGNAL))))
ctx.set_virtual_shards(2)
out.append(("colshard", digest(cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL))))
# th < 1, Adam, joint mode, priors (TV-1D per signal and image mode)
A, X, Y, _ = cl.gen_problem_1d(9, 64, 128, 5, 9)
ctx = cl.ClompContext(A)
ctx.set_basis(cl.dct_basis(128))
d = cl.ClompConfig()
d.max_outer = 8
out.append(("defaults per signal", digest(cl.clomp_solve_batch(ctx, Y, d, mode=cl.MODE_PER_SIGNAL))))
out.append(("defaults joint (image mode)", digest(cl.clomp_solve_batch(ctx, Y, d, mode=cl.MODE_JOINT))))
# separable: tensor-core correlation, Gram form then direct form
Ar, Ac, S, Y = cl.gen_problem_2d(31, 256, 32, 40, 24, 30, 3)
ctx = cl.ClompContext.separable(Ar, Ac)
ctx.set_direct_form(12)
out.append(("separable", digest(cl.clomp_solve_batch(ctx, Y, cl.ClompConfig.baseline(30), mode=cl.MODE_PER_SIGNAL))))
for name, dg in out:
    print(f"{name}: {dg}")
print("PROBE OK")
