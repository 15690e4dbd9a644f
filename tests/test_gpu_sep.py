"""Separable 2D mode on the GPU (Y = A_r S A_c^T, north-star "2D mode").

Semantics are clomp_solve on the explicit Kronecker matrix A = A_c (x) A_r:
the small golden cases were produced by the reference itself on np.kron, and
the full-size BASELINE config 4/5 problems are checked on a truncated prefix
(max_outer = T << K) against the matrix-free oracle.
"""
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2501_11592_b200 as cl
import refbind

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden"
CASES = json.loads((GOLD / "cases.json").read_text())
ARR = np.load(GOLD / "golden.npz")


def rel_err(a, b):
    den = np.max(np.abs(b)) if np.any(b) else 1.0
    return float(np.max(np.abs(a - b)) / den)


@pytest.mark.parametrize("case", [c for c in CASES if c["kind"] == "sep"], ids=lambda c: c["name"])
def test_separable_matches_reference_golden(case, gpu_available):
    name = case["name"]
    ctx = cl.ClompContext.separable(ARR[f"{name}/Ar"], ARR[f"{name}/Ac"])
    mode = cl.MODE_JOINT if case["api"] == "batch" else cl.MODE_PER_SIGNAL
    r = cl.clomp_solve_batch(ctx, ARR[f"{name}/Y"], cl.ClompConfig(**case["cfg"]), mode=mode)
    assert np.array_equal(r.mask, ARR[f"{name}/mask"])
    assert np.array_equal(r.iterations, ARR[f"{name}/iterations"])
    assert rel_err(r.s, ARR[f"{name}/s"]) <= 1e-9
    np.testing.assert_allclose(r.final_residual_norm, ARR[f"{name}/final_residual_norm"], rtol=1e-6)


def _prefix_parity(c, batch, prefix, per_image_check):
    Ar, Ac, S, Y = cl.gen_problem_2d(c["seed"], c["n_r"], c["n_c"], c["m_r"], c["m_c"], c["k"], batch)
    ctx = cl.ClompContext.separable(Ar, Ac)
    cfg = cl.ClompConfig.baseline(c["k"])
    cfg.max_outer = prefix
    r = cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL)
    assert np.all(r.status == 0) and np.all(r.iterations == prefix)
    idx = list(range(per_image_check))
    ref = refbind.orc_solve_sep(Ar, Ac, Y[:, idx], cfg, mode=refbind.MODE_PER_SIGNAL)
    for q, b in enumerate(idx):
        assert np.array_equal(np.flatnonzero(r.mask[:, b]), np.flatnonzero(ref["mask"][:, q]))
        assert rel_err(r.s[:, b], ref["s"][:, q]) <= 1e-6
    # every selected atom of the prefix is a true coefficient
    hits = np.mean([np.all(S[np.flatnonzero(r.mask[:, b]), b] != 0) for b in range(batch)])
    return hits


def test_config4_prefix_full_size(gpu_available):
    """BASELINE config 4 shapes (256x256 coefficients, 128x128 measurements,
    K=1500), 8 images, first 12 outer iterations; 2 images re-solved by the
    matrix-free oracle."""
    hits = _prefix_parity(cl.CONFIGS[4], 8, 10, 1)
    assert hits >= 0.5


def test_separable_reduced_full_solve(gpu_available):
    """Reduced 2D problem solved to K (supports past 32 atoms: block kernel)."""
    Ar, Ac, S, Y = cl.gen_problem_2d(9, 32, 24, 20, 16, 40, 3)
    ctx = cl.ClompContext.separable(Ar, Ac)
    cfg = cl.ClompConfig.baseline(40)
    r = cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL)
    ref = refbind.orc_solve_sep(Ar, Ac, Y, cfg, mode=refbind.MODE_PER_SIGNAL)
    assert np.array_equal(r.mask, ref["mask"])
    assert np.array_equal(r.iterations, ref["iterations"])
    assert rel_err(r.s, ref["s"]) <= 1e-8


def test_config4_full_K_parity(gpu_available):
    """BASELINE config 4 at full size: 64 images of 256 x 256 DCT
    coefficients (K = 1500), 128 x 128 separable Gaussian measurements, the
    whole solve (1500 outer iterations x 200 epochs).  4 images are re-solved
    by the fp64 separable checker in Gram form (oracle/clomp_oracle.c,
    orc_clomp_solve_sep_gram, pinned to the exact restatement by
    tests/test_oracle.py): identical supports and iteration counts,
    coefficients within the north star's 1e-4 and SNR within 0.1 dB."""
    import oracle_pool

    c = cl.CONFIGS[4]
    Ar, Ac, S, Y = cl.gen_problem_2d(c["seed"], c["n_r"], c["n_c"], c["m_r"], c["m_c"], c["k"],
                                     c["batch"])
    ctx = cl.ClompContext.separable(Ar, Ac)
    cfg = cl.ClompConfig.baseline(c["k"])
    r = cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL)
    assert np.all(r.status == 0)
    cols = [0, 21, 42, 63]
    ref = oracle_pool.solve_sep_columns(Ar, Ac, Y, cols, cfg)

    def snr(x, xh):
        return 10 * np.log10(np.sum(x ** 2) / max(np.sum((x - xh) ** 2), 1e-300))

    worst = 0.0
    for b in cols:
        sup, vals, it, conv, st, rn = ref[b]
        assert st == 0
        assert np.array_equal(np.flatnonzero(r.mask[:, b]), sup), f"image {b}: support"
        assert r.iterations[b] == it
        assert bool(r.converged[b]) == conv
        s_ref = np.zeros(r.s.shape[0])
        s_ref[sup] = vals
        err = rel_err(r.s[:, b], s_ref)
        worst = max(worst, err)
        assert err <= 1e-4, f"image {b}: coefficient error {err}"
        assert abs(snr(S[:, b], r.s[:, b]) - snr(S[:, b], s_ref)) < 0.1
    print(f"config 4 full K: 4/4 images identical supports, worst coef err {worst:.2e}")


@pytest.mark.parametrize("shape", [(256, 64, 48, 40, 40, 5), (512, 32, 64, 24, 30, 3)])
def test_separable_tensor_core_correlation_equals_fp64_path(gpu_available, shape):
    """Stage 2 of the separable correlation on tcgen05 (K1 on the rows of
    U = R A_c, candidate records, near-ties re-decided from exact fp64 scores)
    selects exactly what the fp64 score matrix selects; n_r must be a multiple
    of the 256-atom tile, smaller factors keep the fp64 path."""
    n_r, n_c, m_r, m_c, k, batch = shape
    Ar, Ac, S, Y = cl.gen_problem_2d(31, n_r, n_c, m_r, m_c, k, batch)
    cfg = cl.ClompConfig.baseline(k)
    out = {}
    for path in (1, 2):
        ctx = cl.ClompContext.separable(Ar, Ac)
        ctx.set_corr_path(path)
        out[path] = cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL)
        assert ctx.stats()["corr_path"] == (1 if path == 2 else 0)
    a, b = out[1], out[2]
    assert np.array_equal(a.mask, b.mask)
    assert np.array_equal(a.iterations, b.iterations)
    assert rel_err(b.s, a.s) <= 1e-9
    auto = cl.ClompContext.separable(Ar, Ac)
    cl.clomp_solve_batch(auto, Y[:, :1], cfg, mode=cl.MODE_PER_SIGNAL)
    assert auto.stats()["corr_path"] == 1  # auto: tensor cores
    ref = refbind.orc_solve_sep(Ar, Ac, Y[:, :1], cfg, mode=refbind.MODE_PER_SIGNAL)
    assert np.array_equal(np.flatnonzero(b.mask[:, 0]), np.flatnonzero(ref["mask"][:, 0]))
    assert rel_err(b.s[:, 0], ref["s"][:, 0]) <= 1e-8
    small = cl.ClompContext.separable(Ar[:, :96], Ac)
    with pytest.raises(cl.UnsupportedError):
        small.set_corr_path(2)
        cl.clomp_solve_batch(small, Y, cfg, mode=cl.MODE_PER_SIGNAL)


@pytest.mark.parametrize("case", [c for c in CASES if c["kind"] == "sep"], ids=lambda c: c["name"])
def test_separable_direct_form_matches_reference_golden(case, gpu_available):
    """Direct-form learning (the reference's epoch applied through A_r / A_c, no
    support Gram matrix) on the reference's own separable golden cases, from
    the first iteration and switching over from the Gram form mid-solve."""
    name = case["name"]
    mode = cl.MODE_JOINT if case["api"] == "batch" else cl.MODE_PER_SIGNAL
    for start in (1, 3):
        ctx = cl.ClompContext.separable(ARR[f"{name}/Ar"], ARR[f"{name}/Ac"])
        ctx.set_direct_form(start)
        r = cl.clomp_solve_batch(ctx, ARR[f"{name}/Y"], cl.ClompConfig(**case["cfg"]), mode=mode)
        assert np.array_equal(r.mask, ARR[f"{name}/mask"])
        assert np.array_equal(r.iterations, ARR[f"{name}/iterations"])
        assert rel_err(r.s, ARR[f"{name}/s"]) <= 1e-9
        np.testing.assert_allclose(r.final_residual_norm, ARR[f"{name}/final_residual_norm"], rtol=1e-6)


@pytest.mark.parametrize("opt", [cl.PLAIN, cl.ADAM])
def test_separable_direct_form_vs_oracle_and_gram_form(gpu_available, opt):
    Ar, Ac, S, Y = cl.gen_problem_2d(9, 32, 24, 20, 16, 40, 3)
    cfg = cl.ClompConfig.baseline(40)
    cfg.opt = opt
    if opt == cl.ADAM:
        cfg.lr, cfg.inner_steps = 0.02, 60
    ref = refbind.orc_solve_sep(Ar, Ac, Y, cfg, mode=refbind.MODE_PER_SIGNAL)
    for start in (0, 1, 17):
        ctx = cl.ClompContext.separable(Ar, Ac)
        ctx.set_direct_form(start)
        r = cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL)
        assert np.array_equal(r.mask, ref["mask"]), f"direct from {start}"
        assert np.array_equal(r.iterations, ref["iterations"])
        assert rel_err(r.s, ref["s"]) <= 1e-8


def test_separable_capacity_above_gram_limit(gpu_available):
    """max_outer above 2048 atoms per image: no support Gram matrix is ever
    allocated, every iteration learns in direct form (round 1 refused this
    with 'support capacity above 2048 atoms')."""
    Ar, Ac, S, Y = cl.gen_problem_2d(13, 64, 64, 40, 40, 24, 2)
    cfg = cl.ClompConfig.baseline(24)
    cfg.max_outer = 2100          # capacity 2116 > 2048; the noiseless solves stop by eps
    cfg.inner_steps = 120
    ctx = cl.ClompContext.separable(Ar, Ac)
    r = cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL)
    ref = refbind.orc_solve_sep(Ar, Ac, Y, cfg, mode=refbind.MODE_PER_SIGNAL)
    assert np.all(r.status == 0)
    assert np.array_equal(r.mask, ref["mask"])
    assert np.array_equal(r.iterations, ref["iterations"])
    assert np.array_equal(r.converged, ref["converged"].astype(bool))
    assert rel_err(r.s, ref["s"]) <= 1e-8
    off = cl.ClompContext.separable(Ar, Ac)
    off.set_direct_form(0)
    with pytest.raises(cl.UnsupportedError):
        cl.clomp_solve_batch(off, Y, cfg, mode=cl.MODE_PER_SIGNAL)


@pytest.mark.parametrize("cfg_id", [5, 6])
def test_config5_shape_direct_form_prefix(gpu_available, cfg_id):
    """BASELINE config 5 shapes (512 x 512 coefficients, K = 13107; 128 x 128 and
    256 x 256 measurements): the support capacity the full solve needs (13123
    atoms per image) has no Gram form, so every iteration learns in direct
    form behind the tensor-core correlation.  The solver is deterministic, so a
    truncated run must agree with the oracle's (prefix parity):
    3 images, 40 outer iterations, against the fp64 Gram-form checker."""
    c = cl.CONFIGS[cfg_id]
    Ar, Ac, S, Y = cl.gen_problem_2d(c["seed"], c["n_r"], c["n_c"], c["m_r"], c["m_c"], c["k"], 3)
    ctx = cl.ClompContext.separable(Ar, Ac)
    ctx.set_direct_form(1)  # what max_outer = K selects by itself (capacity > 2048)
    cfg = cl.ClompConfig.baseline(c["k"])
    cfg.max_outer = 40
    r = cl.clomp_solve_batch(ctx, Y, cfg, mode=cl.MODE_PER_SIGNAL)
    assert ctx.stats()["corr_path"] == 1
    ref = refbind.orc_solve_sep_gram(Ar, Ac, Y, cfg)
    assert ref["code"] == 0 and np.all(r.status == 0)
    assert np.array_equal(r.mask, ref["mask"])
    assert np.array_equal(r.iterations, ref["iterations"])
    assert rel_err(r.s, ref["s"]) <= 1e-6
    np.testing.assert_allclose(r.final_residual_norm, ref["final_residual_norm"], rtol=1e-6)
