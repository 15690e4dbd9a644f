"""Host-buffer entry point: pinned vs pageable y, dense vs compact results.

cl_solve_batch stages pageable y through the context's pinned buffer and sends
page-locked y straight to the DMA engine; both must give the same solve, and
dense=False must return the same supports/coefficients without s/mask.
"""
import numpy as np
import pytest
import torch

import paper_2501_11592_b200 as cl

pytestmark = pytest.mark.gpu


def test_pinned_pageable_dense_compact_agree(gpu_available):
    A, X, Y, _ = cl.gen_problem_1d(7, 96, 256, 6, 40, snr_db=40.0)
    ctx = cl.ClompContext(A)
    cfg = cl.ClompConfig.baseline(6)
    ref = cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL)
    st_ref = ctx.stats()
    assert st_ref["e2e_ms"] > 0 and st_ref["h2d_bytes"] == Y.size * 4
    Yp = torch.empty(Y.shape, dtype=torch.float32, pin_memory=True).numpy()
    Yp[...] = Y
    for y in (Yp, np.ascontiguousarray(Y, np.float32)):
        r = cl.clomp_solve_batch(ctx, y, cfg, mode=cl.MODE_PER_SIGNAL, dense=False)
        assert r.s is None and r.mask is None
        assert np.array_equal(r.iterations, ref.iterations)
        assert np.array_equal(r.final_residual_norm, ref.final_residual_norm)
        for b in range(Y.shape[1]):
            assert np.array_equal(r.support[b], ref.support[b])
            assert np.array_equal(r.coef[b], ref.coef[b])
            assert np.array_equal(np.flatnonzero(ref.mask[:, b]), np.sort(ref.support[b]))


def _same(r, ref, B):
    assert np.array_equal(r.iterations, ref.iterations)
    assert np.array_equal(r.final_residual_norm, ref.final_residual_norm)
    assert np.array_equal(r.status, ref.status)
    for b in range(B):
        assert np.array_equal(r.support[b], ref.support[b])
        assert np.array_equal(r.coef[b], ref.coef[b])


@pytest.mark.parametrize("shape", [(96, 256, 6, 40), (512, 1024, 12, 300)])
def test_submit_wait_pipeline_equals_blocking_calls(gpu_available, shape):
    """cl_submit / cl_wait with two batches in flight return, in submission
    order, exactly what blocking cl_solve_batch calls return (pinned and
    pageable y, different batch sizes back to back)."""
    m, n, k, B = shape
    A, _, Y, _ = cl.gen_problem_1d(11, m, n, k, B, snr_db=40.0)
    ctx = cl.ClompContext(A)
    cfg = cl.ClompConfig.baseline(k)
    batches = []
    for i, lo in enumerate((0, B // 3, B // 2, 1)):
        y = np.ascontiguousarray(Y[:, lo:])
        if i % 2 == 0:
            yp = torch.empty(y.shape, dtype=torch.float32, pin_memory=True).numpy()
            yp[...] = y
            y = yp
        batches.append(y)
    refs = [cl.clomp_solve_batch(ctx, y, cfg, mode=cl.MODE_PER_SIGNAL, dense=False) for y in batches]
    got = []
    cl.clomp_submit(ctx, batches[0], cfg, mode=cl.MODE_PER_SIGNAL, dense=False)
    for y in batches[1:]:
        cl.clomp_submit(ctx, y, cfg, mode=cl.MODE_PER_SIGNAL, dense=False)
        got.append(cl.clomp_wait(ctx))
    got.append(cl.clomp_wait(ctx))
    for y, r, ref in zip(batches, got, refs):
        _same(r, ref, y.shape[1])
    st = ctx.stats()
    assert st["h2d_bytes"] == batches[-1].size * 4 and st["e2e_ms"] > 0


def test_submit_limits_and_errors(gpu_available):
    A, _, Y, _ = cl.gen_problem_1d(3, 64, 128, 4, 8)
    ctx = cl.ClompContext(A)
    cfg = cl.ClompConfig.baseline(4)
    with pytest.raises(cl.ConfigError):
        cl.clomp_wait(ctx)  # nothing in flight
    bad = cl.ClompConfig.baseline(4)
    bad.lr = 0.0
    with pytest.raises(cl.ConfigError):
        cl.clomp_submit(ctx, Y, bad, mode=cl.MODE_PER_SIGNAL)  # leaves nothing in flight
    assert not ctx._pending
    cl.clomp_submit(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL)
    cl.clomp_submit(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL)
    with pytest.raises(cl.ConfigError):
        cl.clomp_submit(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL)  # third in flight
    assert len(ctx._pending) == 2
    with pytest.raises(cl.ConfigError):
        cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL)  # blocking call while in flight
    a, b = cl.clomp_wait(ctx), cl.clomp_wait(ctx)
    _same(a, b, Y.shape[1])
    # a diverging joint batch reports through cl_wait
    div = cl.ClompConfig.baseline(4)
    div.lr = 1e6
    cl.clomp_submit(ctx, Y, div, mode=cl.MODE_JOINT)
    with pytest.raises(cl.NumericalError):
        cl.clomp_wait(ctx)


def test_synthesis_x_hat_on_gpu(gpu_available):
    """x_hat = D (s * mask) (clomp.cpp:289) formed on the GPU from the compact
    supports equals the dense host product; it needs a basis and the switch."""
    n, m, k, B = 128, 64, 5, 9
    A, _, Y, _ = cl.gen_problem_1d(5, m, n, k, B)
    D = cl.dct_basis(n)
    ctx = cl.ClompContext(A)
    cfg = cl.ClompConfig.baseline(k)
    ctx.set_synthesis(True)
    with pytest.raises(cl.UnsupportedError):  # no basis yet
        cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL)
    ctx.set_basis(D)
    for mode in (cl.MODE_PER_SIGNAL, cl.MODE_JOINT):
        r = cl.clomp_solve_batch(ctx, Y, cfg, mode=mode)
        want = D @ (r.s * r.mask)
        assert r.x_hat.shape == (n, B)
        assert np.max(np.abs(r.x_hat - want)) <= 1e-12 * max(1.0, np.max(np.abs(want)))
    r1 = cl.clomp_solve_batch(ctx, Y[:, :1], cfg, mode=cl.MODE_JOINT)
    assert np.max(np.abs(r1.x_hat - D @ (r1.s * r1.mask))) <= 1e-12
    ctx.set_synthesis(False)
    assert cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL).x_hat is None
