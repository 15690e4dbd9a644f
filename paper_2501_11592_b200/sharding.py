"""Host side of the multi-GPU signal sharding.

clomp_solve semantics make every column independent (clomp.cpp:294-311), so a
batch splits into contiguous per-rank slices with no data-path collective: one
process per GPU (bench.py --scaling strong, the driver's torchrun launch) or
one host thread per GPU inside one process (cl_create_group, csrc/group.cpp,
which uses the same split).  The column-sharded dictionary's exchange
(candidate-record and residual all-gathers, active-count all-reduce over NCCL)
lives in the library (csrc/colshard.cu, clomp_api.cu).
"""
from __future__ import annotations

import numpy as np


def shard_range(n_items: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) slice of n_items for rank (sizes differ by <= 1; the
    split cl_group_solve_batch uses)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def solve_signal_shard(ctx, y_cols: np.ndarray, cfg, rank: int, world: int):
    """Solve this rank's slice of the columns of y (m x B) with per-signal
    semantics; returns (lo, hi, BatchSolveResult)."""
    from . import MODE_PER_SIGNAL, clomp_solve_batch

    lo, hi = shard_range(y_cols.shape[1], rank, world)
    res = clomp_solve_batch(ctx, np.ascontiguousarray(y_cols[:, lo:hi]), cfg, mode=MODE_PER_SIGNAL)
    return lo, hi, res
