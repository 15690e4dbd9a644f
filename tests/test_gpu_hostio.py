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
