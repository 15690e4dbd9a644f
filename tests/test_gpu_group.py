"""cl_create_group: one process, several contexts.

The box has one GPU, so the signal-shard group lists device 0 several times
(independent contexts and streams, one host thread each): the split, the
per-shard row offsets, the gather of the reference's interleaved y and the
scatter of the dense s / mask must reproduce the single-context solve bit for
bit.  Column-shard groups need distinct devices (one NCCL rank each)."""
import numpy as np
import pytest

import paper_2501_11592_b200 as cl

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ndev,B", [(2, 37), (3, 64), (4, 3)])
@pytest.mark.parametrize("layout", ["ref", "t"])
def test_signal_shard_group_equals_single_context(gpu_available, ndev, B, layout):
    m, n, k = 96, 256, 6
    A, _, Y, _ = cl.gen_problem_1d(21, m, n, k, B, snr_db=40.0)
    cfg = cl.ClompConfig.baseline(k)
    ctx = cl.ClompContext(A)
    ref = cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL)
    grp = cl.ClompGroup(A, [0] * ndev, cl.GROUP_SIGNAL_SHARD)
    assert len(grp) == ndev
    y = Y if layout == "ref" else np.ascontiguousarray(Y.T)
    got = grp.solve_batch(y, cfg, mode=cl.MODE_PER_SIGNAL, layout=layout)
    assert np.array_equal(got.mask, ref.mask)
    assert np.array_equal(got.s, ref.s)
    assert np.array_equal(got.iterations, ref.iterations)
    assert np.array_equal(got.final_residual_norm, ref.final_residual_norm)
    assert np.array_equal(got.converged, ref.converged)
    for b in range(B):
        assert np.array_equal(got.support[b], ref.support[b])
        assert np.array_equal(got.coef[b], ref.coef[b])
    compact = grp.solve_batch(y, cfg, mode=cl.MODE_PER_SIGNAL, layout=layout, dense=False)
    assert compact.s is None
    for b in range(B):
        assert np.array_equal(compact.support[b], ref.support[b])


def test_group_rules(gpu_available):
    A, _, Y, _ = cl.gen_problem_1d(4, 64, 128, 4, 8)
    cfg = cl.ClompConfig.baseline(4)
    grp = cl.ClompGroup(A, [0, 0], cl.GROUP_SIGNAL_SHARD)
    with pytest.raises(cl.UnsupportedError):  # joint batches couple their columns
        grp.solve_batch(Y, cfg, mode=cl.MODE_JOINT)
    bad = cl.ClompConfig.baseline(4)
    bad.th = 1.5
    with pytest.raises(cl.ConfigError):
        grp.solve_batch(Y, bad)
    with pytest.raises(cl.ConfigError):  # NCCL: one rank per distinct device
        cl.ClompGroup(A, [0, 0], cl.GROUP_COLUMN_SHARD)
    with pytest.raises(cl.CudaError):
        cl.ClompGroup(A, [0, 99], cl.GROUP_SIGNAL_SHARD)
    one = cl.ClompGroup(A, [0], cl.GROUP_COLUMN_SHARD)  # a group of one: the plain context
    r = one.solve_batch(Y, cfg, mode=cl.MODE_JOINT)
    ref = cl.clomp_solve_batch(cl.ClompContext(A), Y, cfg, mode=cl.MODE_JOINT)
    assert np.array_equal(r.s, ref.s)
