"""Multi-process (world_size 2, gloo, CPU) tests of the partitioning logic.

* Signal sharding: each rank solves its contiguous slice of the batch; the
  gathered result equals the whole batch solved at once (per-signal semantics,
  clomp.cpp:294-311).  The solver here is the oracle restatement (CPU); on the
  GPU box the same slices go through the C-ABI (bench.py under torchrun).
* Column sharding: the per-signal global argmax over atom shards is one
  max all-reduce of packed (|score|, ~index) keys, identical to the argmax over
  all atoms with the lowest-index tie rule.
"""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
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


def _worker(rank, world, port, q):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import refbind
        from paper_2501_11592_b200 import ClompConfig
        from paper_2501_11592_b200.sharding import (argmax_allreduce, local_argmax_keys,
                                                    shard_range, unpack_keys)

        A, Y = _problem()
        cfg = ClompConfig.baseline(4)
        lo, hi = shard_range(Y.shape[1], rank, world)
        r = refbind.orc_solve(A, Y[:, lo:hi], cfg, mode=refbind.MODE_PER_SIGNAL)
        parts = [None] * world
        dist.all_gather_object(parts, (lo, hi, r["s"], r["mask"], r["iterations"]))
        # column sharding of one correlation step: scores = |A^T Y|
        rng = np.random.default_rng(3)
        S = np.abs(rng.standard_normal((5, 50)))
        S[2, 7] = S[2, 31] = S[2].max() + 1.0  # exact tie across shards
        a0, a1 = shard_range(S.shape[1], rank, world)
        keys = argmax_allreduce(local_argmax_keys(S[:, a0:a1], a0))
        val, idx = unpack_keys(keys)
        if rank == 0:
            q.put(("ok", parts, idx.tolist(), val.tolist(), S))
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e)))
    finally:
        dist.destroy_process_group()


def test_signal_and_column_sharding_world2():
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
    _, parts, idx, val, S = out
    sys.path.insert(0, str(ROOT / "tests"))
    import refbind
    from paper_2501_11592_b200 import ClompConfig

    A, Y = _problem()
    full = refbind.orc_solve(A, Y, ClompConfig.baseline(4), mode=refbind.MODE_PER_SIGNAL)
    s = np.concatenate([p[2] for p in parts], axis=1)
    mk = np.concatenate([p[3] for p in parts], axis=1)
    it = np.concatenate([p[4] for p in parts])
    assert np.array_equal(s, full["s"]) and np.array_equal(mk, full["mask"])
    assert np.array_equal(it, full["iterations"])
    assert idx == [int(np.argmax(S[b])) for b in range(S.shape[0])]
    assert idx[2] == 7  # tie -> lowest index
    assert np.allclose(val, S.max(1).astype(np.float32))


def test_shard_range_and_keys():
    from paper_2501_11592_b200.sharding import pack_keys, shard_range, unpack_keys

    assert [shard_range(10, r, 3) for r in range(3)] == [(0, 4), (4, 7), (7, 10)]
    assert shard_range(2, 2, 4) == (2, 2)
    s = np.array([0.5, 2.0, 2.0, 0.0], np.float32)
    k = pack_keys(s, np.array([3, 9, 4, 0]))
    assert np.argmax(k) == 2  # equal scores: lower atom index wins
    v, i = unpack_keys(k)
    assert np.array_equal(v, s) and i.tolist() == [3, 9, 4, 0]
