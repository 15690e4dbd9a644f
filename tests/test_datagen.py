"""The product's input generator restates cskit::Rng bit-for-bit (CPU-only)."""
from pathlib import Path

import numpy as np
import pytest

import paper_2501_11592_b200 as cl

ARR = np.load(Path(__file__).resolve().parent / "golden" / "golden.npz")


@pytest.mark.parametrize("seed", [0, 1, 12345])
@pytest.mark.parametrize("kind", ["u64", "uniform", "normal", "below"])
def test_rng_matches_reference_stream(built_lib, seed, kind):
    got = cl.rng_draws(seed, kind, 64, bound=1000)
    assert np.array_equal(got, ARR[f"rng/{seed}/{kind}"])


def test_problem_generation_is_deterministic_and_normalised(built_lib):
    a1 = cl.gen_problem_1d(7, 64, 128, 5, 3, snr_db=40.0)
    a2 = cl.gen_problem_1d(7, 64, 128, 5, 3, snr_db=40.0)
    for x, y in zip(a1, a2):
        assert np.array_equal(x, y)
    A, X, Y, S = a1
    norms = np.linalg.norm(A.astype(np.float64), axis=0)
    assert np.allclose(norms, 1.0, atol=1e-6)
    assert all(np.count_nonzero(X[:, b]) == 5 for b in range(3))
    assert all(set(np.flatnonzero(X[:, b])) == set(S[b]) for b in range(3))
    # 40 dB: noise energy is 1e-4 of the clean energy
    clean = A.astype(np.float64) @ X
    snr = 10 * np.log10((clean ** 2).sum(0) / ((Y - clean) ** 2).sum(0))
    assert np.all(np.abs(snr - 40.0) < 3.0)


def test_config1_golden_inputs_regenerate(built_lib):
    c = cl.CONFIGS[1]
    A, X, Y, _ = cl.gen_problem_1d(c["seed"], c["m"], c["n"], c["k"], 1)
    assert np.array_equal(A, ARR["cfg1_full/A"])
    assert np.array_equal(Y, ARR["cfg1_full/Y"])


def test_value_law_pm_uniform(built_lib):
    _, X, _, _ = cl.gen_problem_1d(3, 32, 64, 8, 4, value_law=1)
    v = np.abs(X[X != 0])
    assert np.all((v >= 1.0) & (v < 2.0))


def test_dct_basis_matches_reference_bit_for_bit(built_lib):
    """cl_dct_basis restates dct_basis (sensing.cpp:13-29): equal to the
    reference's own output (tests/golden dct8) and orthonormal."""
    assert np.array_equal(cl.dct_basis(8), ARR["dct8"])
    D = cl.dct_basis(64)
    assert np.allclose(D.T @ D, np.eye(64), atol=1e-13)


@pytest.mark.parametrize("args", [(7, 64, 128, 5, 3, 0, 40.0), (2, 96, 300, 12, 5, 1, -1.0),
                                  (1, 128, 256, 10, 9, 0, 40.0)])
def test_reference_side_generator_matches_product(built_lib, args):
    """bench.py's reference arm draws its inputs with the reference's own
    cskit::Rng (oracle/ref_harness.cpp) instead of the product library; both
    generators must produce the same bits."""
    import refbind

    if not refbind.ref_available():
        pytest.skip("oracle/_ref not built")
    seed, m, n, k, B, law, snr = args
    A, X, Y, _ = cl.gen_problem_1d(seed, m, n, k, B, value_law=law, snr_db=snr)
    A2, X2, Y2 = refbind.ref_gen_problem_1d(seed, m, n, k, B, value_law=law, snr_db=snr)
    assert np.array_equal(A, A2)
    assert np.array_equal(X, X2)
    assert np.array_equal(Y, Y2)
