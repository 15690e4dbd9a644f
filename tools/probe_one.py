"""One config-2 solve with a given inner_steps (for ncu launch lists)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2501_11592_b200 as cl  # noqa: E402

inner = int(sys.argv[1]) if len(sys.argv) > 1 else 200
c = dict(cl.CONFIGS[2])
A, X, Y, _ = cl.gen_problem_1d(c["seed"], c["m"], c["n"], c["k"], c["batch"],
                               value_law=c["value_law"], snr_db=c["snr_db"])
ctx = cl.ClompContext(A)
cfg = cl.ClompConfig.baseline(c["k"])
cfg.inner_steps = inner
cfg.stall_patience = 1 << 30
for _ in range(3):
    r = cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL, dense=False)
print("ok", ctx.stats()["e2e_ms"])
