"""Multi-GPU partitioning of the CLOMP path.

Signal sharding (configs 2, 4, 5): clomp_solve semantics make every column
independent (clomp.cpp:294-311), so a batch splits into contiguous per-rank
slices with no data-path collective; one process per GPU.

Column sharding (config 3, one very large dictionary): each rank owns a
contiguous slice of atoms and computes its local correlation maximum; the
global argmax is a max-reduction of packed 64-bit keys (non-negative fp32
|score| bits in the high word, ~index in the low word, so equal scores prefer
the lowest atom index).  `argmax_allreduce` is that exchange over
torch.distributed (NCCL on B200s, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np


def shard_range(n_items: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) slice of n_items for rank (sizes differ by <= 1)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def pack_keys(scores: np.ndarray, idx: np.ndarray) -> np.ndarray:
    """(|score|, atom index) -> int64 keys ordered by score, then lowest index."""
    s = np.abs(np.asarray(scores, np.float32)).view(np.uint32).astype(np.uint64)
    i = (~np.asarray(idx, np.uint64)) & np.uint64(0xFFFFFFFF)
    return ((s << np.uint64(32)) | i).view(np.int64)


def unpack_keys(keys: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    k = np.asarray(keys, np.int64).view(np.uint64)
    s = (k >> np.uint64(32)).astype(np.uint32).view(np.float32)
    i = ((~k) & np.uint64(0xFFFFFFFF)).astype(np.int64)
    return s, i


def local_argmax_keys(scores_local: np.ndarray, atom0: int) -> np.ndarray:
    """Per-signal packed key of the local maximum; scores_local is B x n_local."""
    a = np.abs(scores_local)
    j = np.argmax(a, axis=1)  # first maximum = lowest local index
    return pack_keys(a[np.arange(a.shape[0]), j], j + atom0)


def argmax_allreduce(keys: np.ndarray) -> np.ndarray:
    """Global per-signal argmax over column shards: one max all-reduce of B keys."""
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(np.ascontiguousarray(keys, np.int64))
    if dist.get_backend() == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.cpu().numpy()


def solve_signal_shard(ctx, y_cols: np.ndarray, cfg, rank: int, world: int):
    """Solve this rank's slice of the columns of y (m x B) with per-signal
    semantics; returns (lo, hi, BatchSolveResult)."""
    from . import MODE_PER_SIGNAL, clomp_solve_batch

    lo, hi = shard_range(y_cols.shape[1], rank, world)
    res = clomp_solve_batch(ctx, np.ascontiguousarray(y_cols[:, lo:hi]), cfg, mode=MODE_PER_SIGNAL)
    return lo, hi, res
