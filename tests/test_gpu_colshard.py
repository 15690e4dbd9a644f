"""Column-sharded dictionary on one GPU with virtual shards:
K1 runs per atom shard into a [shards][B][tiles] candidate table that is
exchanged exactly as the NCCL all-gather would deliver it, so supports,
coefficients and iterations must be bit-identical to the unsharded solve."""
import numpy as np
import pytest

import paper_2501_11592_b200 as cl
import refbind

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shards", [2, 4, 8])
@pytest.mark.parametrize("path", [2, 1])
def test_virtual_column_shards_match_unsharded(gpu_available, shards, path):
    A, X, Y, _ = cl.gen_problem_1d(31, 512, 4096, 40, 96, value_law=1)
    cfg = cl.ClompConfig.baseline(40)
    ref_ctx = cl.ClompContext(A)
    ref_ctx.set_corr_path(path)
    ref = cl.clomp_solve_batch(ref_ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL)
    ctx = cl.ClompContext(A)
    ctx.set_corr_path(path)
    ctx.set_virtual_shards(shards)
    got = cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL)
    assert np.array_equal(got.mask, ref.mask)
    assert np.array_equal(got.s, ref.s)
    assert np.array_equal(got.iterations, ref.iterations)
    if shards == 4 and path == 2:
        o = refbind.orc_solve(A.astype(np.float64), Y[:, :3].astype(np.float64), cfg,
                              mode=refbind.MODE_PER_SIGNAL)
        assert np.array_equal(got.mask[:, :3], o["mask"])


def test_colshard_rejects_unsupported(gpu_available):
    A, X, Y, _ = cl.gen_problem_1d(32, 64, 300, 4, 4)
    ctx = cl.ClompContext(A)
    ctx.set_virtual_shards(2)
    with pytest.raises(cl.DimensionError):  # 300 atoms do not split into 2 x 256
        cl.clomp_solve_batch(ctx, Y, cl.ClompConfig.baseline(4), mode=cl.MODE_PER_SIGNAL)
    with pytest.raises(cl.UnsupportedError):
        cl.clomp_solve_batch(ctx, Y, cl.ClompConfig.baseline(4), mode=cl.MODE_JOINT)


def test_virtual_shards_switched_on_a_used_context(gpu_available):
    """cl_set_virtual_shards on a context that already solved (workspace and
    power-form buffers allocated) re-carves both; round 2's debug-build probe
    found the power-form buffer freed but still referenced here."""
    A, X, Y, _ = cl.gen_problem_1d(33, 512, 1024, 72, 6, value_law=1)
    cfg = cl.ClompConfig.baseline(72)
    ctx = cl.ClompContext(A)
    ref = cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL)  # cluster learners + power form
    for shards in (2, 1, 4):
        ctx.set_virtual_shards(shards)
        got = cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL)
        assert np.array_equal(got.mask, ref.mask) and np.array_equal(got.s, ref.s)
