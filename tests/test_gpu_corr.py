"""K1 correlation kernels on the GPU: the tcgen05 split-fp16 (3 MMA) scores against fp64
scores, and the measured error against the bound the selection step uses to
decide when a near-tie must be re-decided in fp64 (clomp_api.cu delta_for)."""
import numpy as np
import pytest

import paper_2501_11592_b200 as cl

pytestmark = pytest.mark.gpu


def delta_rel(m):
    ldm = (m + 31) // 32 * 32
    return 1e-5 + (ldm // 8) * 1.2e-7


@pytest.mark.parametrize("m,n,B", [(128, 256, 5), (512, 1024, 300), (1000, 700, 129), (4096, 4096, 64)])
def test_tc_scores_within_bound(gpu_available, m, n, B):
    rng = np.random.default_rng(m + n)
    A = (rng.standard_normal((m, n)) / np.sqrt(m)).astype(np.float32)
    A /= np.linalg.norm(A.astype(np.float64), axis=0).astype(np.float32)
    R = rng.standard_normal((B, m)).astype(np.float32)
    ctx = cl.ClompContext(A)
    s64 = ctx.debug_scores(R, 1)                 # |A^T r| fp64
    stc = np.abs(ctx.debug_scores(R, 2))         # split fp16 on tcgen05
    exact = np.abs(R.astype(np.float64) @ A.astype(np.float64))
    assert np.max(np.abs(s64 - exact)) <= 1e-12 * np.max(exact)
    colmax = np.max(np.linalg.norm(A.astype(np.float64), axis=0))
    rn = np.linalg.norm(R.astype(np.float64), axis=1, keepdims=True)
    err = np.abs(stc - exact) / (colmax * rn)
    worst = float(err.max())
    print(f"m={m} n={n} B={B}: max split-fp16 error {worst:.3e} of ||a||*||r||, bound {delta_rel(m):.3e}")
    assert worst <= delta_rel(m) / 4, "split-fp16 error too close to the rescan bound"


def test_tc_argmax_matches_fp64(gpu_available):
    rng = np.random.default_rng(5)
    m, n, B = 512, 1024, 512
    A = (rng.standard_normal((m, n)) / np.sqrt(m)).astype(np.float32)
    R = rng.standard_normal((B, m)).astype(np.float32)
    ctx = cl.ClompContext(A)
    s64 = ctx.debug_scores(R, 1)
    stc = np.abs(ctx.debug_scores(R, 2))
    top = np.sort(s64, axis=1)
    gap = (top[:, -1] - top[:, -2]) / np.linalg.norm(R, axis=1)
    clear = gap > 2 * delta_rel(m)
    assert clear.mean() > 0.9
    assert np.array_equal(np.argmax(stc, 1)[clear], np.argmax(s64, 1)[clear])


@pytest.mark.parametrize("m,n,B", [(128, 256, 1), (512, 1024, 3), (1000, 700, 4), (384, 130, 2),
                                   (4096, 16384, 1)])
def test_gemv_scores_fp64_exact(gpu_available, m, n, B):
    """K1b (the B <= 4 GEMV): fp64 accumulation of fp32 atoms, the same error
    class as the fp64 SIMT kernel (the selection's 1e-12 bound), ragged n
    (partial candidate tiles) and m not a multiple of 128."""
    rng = np.random.default_rng(m * 7 + n + B)
    A = (rng.standard_normal((m, n)) / np.sqrt(m)).astype(np.float32)
    R = rng.standard_normal((B, m)).astype(np.float32)
    ctx = cl.ClompContext(A)
    sg = ctx.debug_scores(R, 3)
    exact = np.abs(R.astype(np.float64) @ A.astype(np.float64))
    rn = np.linalg.norm(R.astype(np.float64), axis=1, keepdims=True)
    err = np.abs(sg - exact) / rn
    assert float(err.max()) <= 1e-13, f"max GEMV error {err.max():.3e} of ||a||*||r||"
    assert np.array_equal(np.argmax(sg, 1), np.argmax(exact, 1))
