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
    r = refbind.orc_solve(A, Y, _cfg(case["cfg"]), mode=mode)
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


def test_priors_are_rejected_not_faked():
    A = ARR["small_th1_plain_b1/A"].astype(np.float64)
    Y = ARR["small_th1_plain_b1/Y"].astype(np.float64)
    r = refbind.orc_solve(A, Y, ClompConfig())  # defaults: auto priors on
    assert r["code"] == 5


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
