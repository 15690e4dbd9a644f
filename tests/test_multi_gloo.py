"""Multi-process (world_size 2, gloo, CPU) test of the N > 1 host path.

Signal sharding has no data-path collective, so what N ranks share is the
host logic bench.py runs under torchrun: every rank derives its workload from
(rank, world) — its own seed for weak scaling, its contiguous slice of one
batch for strong scaling (sharding.shard_range, the split cl_create_group uses
too) — times its steps, and the job's number is all ranks' signals over the
slowest rank's time (an all-reduce MAX, NCCL on the GPUs, gloo here).  The
per-rank solves run the oracle restatement here (no GPU); gathered, the
slices must equal the whole batch solved at once (clomp.cpp:294-311).
"""
import argparse
import os
import socket
import sys
from pathlib import Path

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    rng = np.random.default_rng(7)
    m, n, B, k = 24, 60, 7, 3
    A = (rng.standard_normal((m, n)) / np.sqrt(m)).astype(np.float32).astype(np.float64)
    X = np.zeros((n, B))
    for b in range(B):
        X[rng.choice(n, k, replace=False), b] = rng.standard_normal(k)
    Y = (A @ X + 0.01 * rng.standard_normal((m, B))).astype(np.float32).astype(np.float64)
    return A, Y


def _args(scaling):
    return argparse.Namespace(config=2, colshard=False, scaling=scaling, max_outer=0, batch=0)


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        import refbind
        from paper_2501_11592_b200 import ClompConfig
        from paper_2501_11592_b200.sharding import shard_range

        # bench.py's per-rank workloads
        weak = bench.workload(_args("weak"), rank, world)
        strong = bench.workload(_args("strong"), rank, world)
        # the strong-scaling slice of a small batch, solved by the oracle
        A, Y = _problem()
        cfg = ClompConfig.baseline(4)
        lo, hi = shard_range(Y.shape[1], rank, world)
        r = refbind.orc_solve(A, Y[:, lo:hi], cfg, mode=refbind.MODE_PER_SIGNAL)
        parts = [None] * world
        dist.all_gather_object(parts, (lo, hi, r["s"], r["mask"], r["iterations"]))
        # timing reduction: rank r "measured" 2 + r ms device and 3 - r ms e2e
        ms = bench.max_over_ranks([2.0 + rank, 3.0 - rank], "cpu", True)
        v_weak = bench.job_throughput(weak, weak["batch"], world, False, ms[0])
        v_strong = bench.job_throughput(strong, strong["sig_hi"] - strong["sig_lo"], world, True, ms[0])
        info = [None] * world
        dist.all_gather_object(info, (weak["seed"], strong["seed"], strong["sig_lo"], strong["sig_hi"],
                                      ms, v_weak, v_strong))
        if rank == 0:
            q.put(("ok", parts, info, weak["batch"]))
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e)))
    finally:
        dist.destroy_process_group()


def test_signal_sharding_host_path_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert out[0] == "ok", out
    _, parts, info, batch = out
    sys.path.insert(0, str(ROOT / "tests"))
    import refbind
    from paper_2501_11592_b200 import ClompConfig

    # the gathered slices are the whole batch solved at once
    A, Y = _problem()
    full = refbind.orc_solve(A, Y, ClompConfig.baseline(4), mode=refbind.MODE_PER_SIGNAL)
    assert [p[0] for p in parts] == [0, 4] and [p[1] for p in parts] == [4, 7]
    s = np.concatenate([p[2] for p in parts], axis=1)
    mk = np.concatenate([p[3] for p in parts], axis=1)
    it = np.concatenate([p[4] for p in parts])
    assert np.array_equal(s, full["s"]) and np.array_equal(mk, full["mask"])
    assert np.array_equal(it, full["iterations"])
    # weak scaling: distinct seeds, every rank a full batch; strong: one seed,
    # contiguous slices that partition the batch
    assert info[0][0] != info[1][0] and info[0][1] == info[1][1]
    assert (info[0][2], info[0][3], info[1][2], info[1][3]) == (0, batch // 2, batch // 2, batch)
    # every rank sees the slowest rank's time; the job value is total / that
    for r in range(2):
        assert info[r][4] == [3.0, 3.0]
        assert info[r][5] == 2 * batch / 3e-3 and info[r][6] == batch / 3e-3


def test_shard_range():
    from paper_2501_11592_b200.sharding import shard_range

    assert [shard_range(10, r, 3) for r in range(3)] == [(0, 4), (4, 7), (7, 10)]
    assert shard_range(2, 2, 4) == (2, 2)
    for n, w in ((4096, 8), (1024, 3), (5, 8)):
        cuts = [shard_range(n, r, w) for r in range(w)]
        assert cuts[0][0] == 0 and cuts[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(cuts, cuts[1:]))
        assert max(h - l for l, h in cuts) - min(h - l for l, h in cuts) <= 1
