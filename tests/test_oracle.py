"""Pin the oracle restatement (oracle/clomp_oracle.c) to the reference.

CPU-only.  Bit-exact against the golden fixtures produced by the unmodified
reference library (tests/golden/make_golden.py) and, when oracle/_ref is built,
against the live reference on fresh random problems for both kernel ISAs
(kernels_avx2.cpp / kernels_scalar.cpp).
"""
import json
from pathlib import Path

import numpy as np
import pytest

import refbind
from paper_2501_11592_b200 import ClompConfig, ADAM, MOMENTUM, PLAIN

GOLD = Path(__file__).resolve().parent / "golden"
CASES = json.loads((GOLD / "cases.json").read_text())
ARR = np.load(GOLD / "golden.npz")


def _cfg(d):
    return ClompConfig(**d)


@pytest.mark.parametrize("case", [c for c in CASES if c["kind"] == "solve"], ids=lambda c: c["name"])
def test_oracle_matches_reference_golden(case):
    name = case["name"]
    A = ARR[f"{name}/A"].astype(np.float64)
    Y = ARR[f"{name}/Y"].astype(np.float64)
    mode = refbind.MODE_JOINT if case["api"] == "batch" else refbind.MODE_PER_SIGNAL
    D = ARR[f"{name}/D"] if case.get("basis") else None
    r = refbind.orc_solve(A, Y, _cfg(case["cfg"]), mode=mode, basis=D)
    assert r["code"] == case["code"], r["err"]
    if case["code"] != 0:
        return
    assert np.array_equal(r["mask"], ARR[f"{name}/mask"])
    assert np.array_equal(r["s"], ARR[f"{name}/s"])  # bit-exact
    assert np.array_equal(r["iterations"], ARR[f"{name}/iterations"])
    assert np.array_equal(r["final_residual_norm"], ARR[f"{name}/final_residual_norm"])
    assert np.array_equal(r["converged"], ARR[f"{name}/converged"].astype(bool))


@pytest.mark.parametrize("case", [c for c in CASES if c["kind"] == "inject"], ids=lambda c: c["name"])
def test_oracle_inject_matches_golden(case):
    name = case["name"]
    code, mk = refbind.orc_inject(ARR[f"{name}/A"], ARR[f"{name}/R"], case["th"], ARR[f"{name}/mask_in"])
    assert code == 0
    assert np.array_equal(mk, ARR[f"{name}/mask_out"])


def test_orthonormal_exact_recovery_property():
    # test_clomp.cpp:289-297: first injection reads a^T y = s0, so the mask is
    # exactly the support and the coefficients are recovered.
    A = ARR["orthonormal_exact/A"].astype(np.float64)
    Y = ARR["orthonormal_exact/Y"].astype(np.float64)
    r = refbind.orc_solve(A, Y, ClompConfig(w_tv=0.0, w_lv=0.0, lr=0.05, max_outer=100),
                          mode=refbind.MODE_PER_SIGNAL)
    assert list(np.flatnonzero(r["mask"][:, 0])) == [4, 11]
    s = r["s"][:, 0]
    err = (s[4] - 1.0) ** 2 + (s[11] + 0.9) ** 2
    assert err / 16 < 1e-6


def test_wrapper_equals_one_column_batch():
    # test_clomp.cpp:255-273
    A = ARR["small_th1_plain_b3_noisy/A"].astype(np.float64)
    Y = ARR["small_th1_plain_b3_noisy/Y"].astype(np.float64)
    cfg = ClompConfig(max_outer=6, inner_steps=12, w_tv=0.0, w_lv=0.0)
    one = refbind.orc_solve(A, Y[:, :1], cfg, mode=refbind.MODE_PER_SIGNAL)
    bat = refbind.orc_solve(A, Y[:, :1], cfg, mode=refbind.MODE_JOINT)
    for k in ("s", "mask", "iterations", "final_residual_norm"):
        assert np.array_equal(one[k], bat[k])


def test_priors_need_the_basis():
    """Priors chain through the synthesis basis; without one the oracle says
    so instead of running something else."""
    A = ARR["small_th1_plain_b1/A"].astype(np.float64)
    Y = ARR["small_th1_plain_b1/Y"].astype(np.float64)
    r = refbind.orc_solve(A, Y, ClompConfig())  # defaults: auto priors on, no basis
    assert r["code"] == 5


def test_tv_prior_is_a_quadratic_form_on_dct_coefficients():
    """TV-1D of x = D s equals s^T H s with H = D^T Delta^T Delta D / n
    (priors.cpp:11-26); for the DCT basis (sensing.cpp:13-29) H is diagonal
    with entries (2 - 2 cos(pi k / n)) / n.  This is the identity the B200
    learning kernels use to fold the prior into the support Gram matrix."""
    n = 64
    D = ARR["prior_default_single/D"]
    Dl = np.diff(D, axis=0)  # rows x_{j+1} - x_j of Delta D
    H = Dl.T @ Dl / n
    lam = (2 - 2 * np.cos(np.pi * np.arange(n) / n)) / n
    assert np.allclose(H, np.diag(lam), atol=1e-12)


@pytest.mark.skipif(not refbind.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("isa", [refbind.ISA_AVX2, refbind.ISA_SCALAR])
@pytest.mark.parametrize("opt,w_tv", [(ADAM, -1.0), (PLAIN, 0.05), (MOMENTUM, -1.0)])
def test_oracle_priors_match_live_reference(isa, opt, w_tv):
    """TV-1D prior chained through the DCT basis, per-signal and one-column
    joint solves, both kernel ISAs, bit for bit."""
    rng = np.random.default_rng(200 + 10 * isa + opt)
    n, m, B, k = 48, 24, 3, 4
    D = np.zeros((n, n))
    refbind.ref().ref_dct_basis(n, refbind._p(D))
    A = (rng.standard_normal((m, n)) / np.sqrt(m) @ D).astype(np.float32).astype(np.float64)
    X = np.zeros((n, B))
    for b in range(B):
        X[rng.choice(n, k, replace=False), b] = rng.standard_normal(k)
    Y = (A @ X + 0.02 * rng.standard_normal((m, B))).astype(np.float32).astype(np.float64)
    cfg = ClompConfig(th=0.7 if opt == ADAM else 1.0, max_outer=8, inner_steps=30,
                      lr=0.05 if opt != ADAM else 0.02, opt=opt, w_tv=w_tv)
    assert refbind.ref().ref_force_isa(isa) == 0
    try:
        orc = refbind.orc_solve(A, Y, cfg, mode=refbind.MODE_PER_SIGNAL, isa=isa, basis=D)
        for b in range(B):
            ref = refbind.ref_solve_batch(A, Y[:, b:b + 1], cfg, basis=D)
            assert ref["code"] == orc["status"][b] == 0
            assert np.array_equal(ref["s"][:, 0], orc["s"][:, b])
            assert np.array_equal(ref["mask"][:, 0], orc["mask"][:, b])
            assert ref["iterations"] == orc["iterations"][b]
            assert ref["final_residual_norm"] == orc["final_residual_norm"][b]
    finally:
        refbind.ref().ref_force_isa(refbind.ISA_AVX2)


@pytest.mark.skipif(not refbind.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("isa", [refbind.ISA_AVX2, refbind.ISA_SCALAR])
@pytest.mark.parametrize("cfgd", [dict(max_outer=8),  # defaults: TV-2D + LV, Adam, th 0.7
                                  dict(th=1.0, opt=PLAIN, lr=0.05, max_outer=6, w_tv=0.05, w_lv=0.0),
                                  dict(opt=MOMENTUM, lr=0.02, max_outer=6, w_tv=0.0, w_lv=0.1),
                                  dict(max_outer=5, lv_window=4, lv_stride=3),
                                  dict(max_outer=5, lv_stride=3)],  # ConfigError
                         ids=["default", "tv2d_plain", "lv_momentum", "lv_w4s3", "bad_stride"])
def test_oracle_image_mode_priors_match_live_reference(isa, cfgd):
    """The reference's column-batch image mode (clomp_solve_batch on many
    columns, cskit.cpp:620-652): TV-2D (priors.cpp:28-59) and local variance
    (priors.cpp:74-116) on x = D S, joint stopping — bit for bit, both ISAs."""
    rng = np.random.default_rng(300 + isa)
    n, m, B, k = 48, 24, 7, 4
    D = np.zeros((n, n))
    refbind.ref().ref_dct_basis(n, refbind._p(D))
    A = (rng.standard_normal((m, n)) / np.sqrt(m) @ D).astype(np.float32).astype(np.float64)
    X = np.zeros((n, B))
    for b in range(B):
        X[rng.choice(n, k, replace=False), b] = rng.standard_normal(k)
    Y = (A @ X + 0.01 * rng.standard_normal((m, B))).astype(np.float32).astype(np.float64)
    cfg = ClompConfig(**cfgd)
    assert refbind.ref().ref_force_isa(isa) == 0
    try:
        ref = refbind.ref_solve_batch(A, Y, cfg, basis=D)
        orc = refbind.orc_solve(A, Y, cfg, mode=refbind.MODE_JOINT, isa=isa, basis=D)
    finally:
        refbind.ref().ref_force_isa(refbind.ISA_AVX2)
    assert ref["code"] == orc["code"], orc["err"]
    if ref["code"]:
        return
    assert np.array_equal(ref["s"], orc["s"])
    assert np.array_equal(ref["mask"], orc["mask"])
    assert ref["iterations"] == orc["iterations"][0]
    assert ref["final_residual_norm"] == orc["final_residual_norm"][0]


@pytest.mark.skipif(not refbind.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("isa", [refbind.ISA_AVX2, refbind.ISA_SCALAR])
@pytest.mark.parametrize("opt,th", [(PLAIN, 1.0), (PLAIN, 0.7), (MOMENTUM, 1.0), (ADAM, 0.7)])
def test_oracle_matches_live_reference(isa, opt, th):
    rng = np.random.default_rng(100 + 10 * isa + opt)
    m, n, B, k = 37, 90, 9, 6
    A = rng.standard_normal((m, n)).astype(np.float32).astype(np.float64) / 6.0
    X = np.zeros((n, B))
    for b in range(B):
        X[rng.choice(n, k, replace=False), b] = rng.standard_normal(k)
    Y = (A @ X + 0.01 * rng.standard_normal((m, B))).astype(np.float32).astype(np.float64)
    cfg = ClompConfig(th=th, max_outer=k + 2, inner_steps=30, lr=0.05 if opt == PLAIN else 0.02,
                      opt=opt, w_tv=0.0, w_lv=0.0)
    assert refbind.ref().ref_force_isa(isa) == 0
    try:
        ref = refbind.ref_solve_batch(A, Y, cfg)
        orc = refbind.orc_solve(A, Y, cfg, mode=refbind.MODE_JOINT, isa=isa)
    finally:
        refbind.ref().ref_force_isa(refbind.ISA_AVX2)
    assert ref["code"] == orc["code"] == 0
    assert np.array_equal(ref["s"], orc["s"])
    assert np.array_equal(ref["mask"], orc["mask"])
    assert ref["iterations"] == orc["iterations"][0]
    assert ref["final_residual_norm"] == orc["final_residual_norm"][0]


@pytest.mark.parametrize("case", [c for c in CASES if c["kind"] == "sep"], ids=lambda c: c["name"])
def test_oracle_separable_matches_reference_on_explicit_kron(case):
    """The matrix-free separable oracle equals the reference run on the dense
    Kronecker matrix, bit for bit."""
    name = case["name"]
    mode = refbind.MODE_JOINT if case["api"] == "batch" else refbind.MODE_PER_SIGNAL
    r = refbind.orc_solve_sep(ARR[f"{name}/Ar"], ARR[f"{name}/Ac"], ARR[f"{name}/Y"],
                              _cfg(case["cfg"]), mode=mode)
    assert r["code"] == case["code"] == 0, r["err"]
    for k in ("s", "mask", "iterations", "final_residual_norm"):
        assert np.array_equal(r[k], ARR[f"{name}/{k}"]), k


@pytest.mark.parametrize("dims,K,opt", [((24, 20, 12, 16), 12, 0), ((32, 32, 16, 16), 40, 0),
                                        ((16, 24, 10, 12), 10, 2)])
def test_separable_gram_oracle_pinned_to_exact_restatement(dims, K, opt):
    """The Gram-form separable checker (products regrouped; used for the
    full-size config-4 parity where the exact matrix-free restatement is
    infeasible) against the exact restatement, itself bit-exact with the
    reference on the explicit Kronecker matrix (test above): identical
    supports, iterations and converged flags; coefficients to 1e-10."""
    import paper_2501_11592_b200 as cl

    nr, nc, mr, mc = dims
    Ar, Ac, X, Y = cl.gen_problem_2d(100 + K, nr, nc, mr, mc, K // 2, 3)
    cfg = cl.ClompConfig.baseline(K)
    cfg.opt = opt
    if opt == 2:
        cfg.lr = 0.01
    ex = refbind.orc_solve_sep(Ar, Ac, Y, cfg, mode=refbind.MODE_PER_SIGNAL)
    gr = refbind.orc_solve_sep_gram(Ar, Ac, Y, cfg)
    assert ex["code"] == 0 and gr["code"] == 0
    assert np.all(gr["status"] == 0)
    assert np.array_equal(ex["mask"], gr["mask"])
    assert np.array_equal(ex["iterations"], gr["iterations"])
    assert np.array_equal(ex["converged"], gr["converged"])
    den = np.max(np.abs(ex["s"]))
    assert np.max(np.abs(ex["s"] - gr["s"])) / den <= 1e-10
    np.testing.assert_allclose(gr["final_residual_norm"], ex["final_residual_norm"], rtol=1e-9,
                               atol=1e-13)
