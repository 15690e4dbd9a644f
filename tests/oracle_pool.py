"""Parallel oracle solves for the full-size parity tests.

TEST INFRASTRUCTURE ONLY.  Per-signal semantics (clomp_solve on every
column) make the columns of a batch independent, so the oracle
restatement (oracle/clomp_oracle.c) can re-solve any subset of a full-size
batch in parallel worker processes.  Each spawned worker draws the workload
itself with the reference's own cskit::Rng (refbind.ref_gen_problem_1d, bit
for bit the product generator's inputs: tests/test_datagen.py), so only
column indices and results cross the process boundary, and no worker loads
the CUDA library.
"""
from __future__ import annotations

import dataclasses
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
_W: dict = {}


def _init(gen):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import refbind

    seed, m, n, k, batch, law, snr = gen
    A, _, Y = refbind.ref_gen_problem_1d(seed, m, n, k, batch, value_law=law, snr_db=snr,
                                         want_x=False)
    _W["A"] = A.astype(np.float64)
    _W["Y"] = Y.astype(np.float64)
    _W["refbind"] = refbind


def _solve(job):
    cols, cfgd = job
    from paper_2501_11592_b200.configs import ClompConfig

    rb = _W["refbind"]
    r = rb.orc_solve(_W["A"], _W["Y"][:, cols], ClompConfig(**cfgd), mode=rb.MODE_PER_SIGNAL)
    mask = r["mask"]
    out = []
    for q, b in enumerate(cols):
        sup = np.flatnonzero(mask[:, q])
        out.append((b, sup, r["s"][sup, q], int(r["iterations"][q]), bool(r["converged"][q]),
                    int(r["status"][q]), float(r["final_residual_norm"][q])))
    return out


def host_workers() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def solve_columns(c: dict, cols, cfg, workers: int | None = None, per_task: int = 1) -> dict:
    """Oracle per-signal solves of columns `cols` of BASELINE config `c`
    (a CONFIGS entry): {b: (support, coefficients on it, iterations,
    converged, status, final residual norm)}."""
    import multiprocessing as mp

    workers = workers or host_workers()
    cols = list(cols)
    gen = (c["seed"], c["m"], c["n"], c["k"], c["batch"], c["value_law"], c["snr_db"])
    cfgd = dataclasses.asdict(cfg)
    jobs = [(cols[i:i + per_task], cfgd) for i in range(0, len(cols), per_task)]
    ctx = mp.get_context("spawn")
    with ctx.Pool(min(workers, len(jobs)), initializer=_init, initargs=(gen,)) as pool:
        res = pool.map(_solve, jobs, chunksize=1)
    out = {}
    for part in res:
        for b, sup, vals, it, conv, st, rn in part:
            out[b] = (sup, vals, it, conv, st, rn)
    return out


def _solve_sep(job):
    Ar, Ac, Yc, cols, cfgd = job
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import refbind
    from paper_2501_11592_b200.configs import ClompConfig

    r = refbind.orc_solve_sep_gram(Ar, Ac, Yc, ClompConfig(**cfgd))
    out = []
    for q, b in enumerate(cols):
        sup = np.flatnonzero(r["mask"][:, q])
        out.append((b, sup, r["s"][sup, q], int(r["iterations"][q]), bool(r["converged"][q]),
                    int(r["status"][q]), float(r["final_residual_norm"][q])))
    return out


def solve_sep_columns(Ar, Ac, Y, cols, cfg, workers: int | None = None) -> dict:
    """Separable per-signal solves (the Gram-form fp64 checker) of columns
    `cols` of Y, one image per worker."""
    import multiprocessing as mp

    workers = workers or host_workers()
    cfgd = dataclasses.asdict(cfg)
    jobs = [(np.asarray(Ar), np.asarray(Ac), np.ascontiguousarray(Y[:, [b]]), [b], cfgd)
            for b in cols]
    ctx = mp.get_context("spawn")
    with ctx.Pool(min(workers, len(jobs))) as pool:
        res = pool.map(_solve_sep, jobs, chunksize=1)
    return {b: rest for part in res for (b, *rest) in part}
