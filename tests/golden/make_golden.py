"""Generate the golden fixtures from the UNMODIFIED reference library.

    make -C oracle && python tests/golden/make_golden.py

Runs cskit::clomp_solve / clomp_solve_batch / inject_support / Rng / dct_basis
(compiled from /root/reference/proj/src into oracle/_ref/libcskit_ref.so by
oracle/Makefile) on small seeded problems and stores inputs and outputs in
tests/golden/golden.npz + cases.json.  The reference has no CLOMP golden
vectors of its own, so these outputs, produced by the
reference itself in this container, pin the oracle restatement and the GPU
path.  The cases re-express the CLOMP properties of
proj/tests/test_clomp.cpp (exact orthonormal recovery :275-298, divergence
:315-326, config validation :328-343, inject_support :46-69) plus the
BASELINE config-1 problem at full size.

Inputs are rounded to fp32 (the GPU operand precision) before the reference
sees them, so every side solves the same problem.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import refbind  # noqa: E402
from paper_2501_11592_b200 import ClompConfig, PLAIN, MOMENTUM, ADAM  # noqa: E402
import paper_2501_11592_b200 as cl  # noqa: E402


def f32(a):
    return np.asarray(a, np.float64).astype(np.float32).astype(np.float64)


def rand_problem(seed, m, n, k, B, snr_db=None, normalize=True):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, n)) / np.sqrt(m)
    if normalize:
        A /= np.linalg.norm(A, axis=0, keepdims=True)
    A = f32(A)
    X = np.zeros((n, B))
    for b in range(B):
        X[rng.choice(n, k, replace=False), b] = rng.standard_normal(k)
    Y = A @ X
    if snr_db is not None:
        sig = np.sqrt(np.mean(Y ** 2, axis=0, keepdims=True))
        Y = Y + sig * 10 ** (-snr_db / 20) * rng.standard_normal(Y.shape)
    return A, f32(Y)


def main():
    arrays = {}
    cases = []

    def add_solve(name, A, Y, cfg, api, round_a=True, basis=None, gpu_code=None):
        """api: 'batch' (clomp_solve_batch) or 'single' (clomp_solve per column).
        basis: synthesis matrix D (x = D s) handed to the reference, which its
        priors need; gpu_code: the status the B200 library is expected to give
        where it differs from the reference's (unsupported configurations)."""
        A = f32(A) if round_a else np.asarray(A, np.float64)
        Y = f32(Y)
        if Y.ndim == 1:
            Y = Y.reshape(-1, 1)
        m, n = A.shape
        B = Y.shape[1]
        if api == "batch":
            r = refbind.ref_solve_batch(A, Y, cfg, basis=basis)
            out = dict(code=r["code"], s=r["s"], mask=r["mask"],
                       iterations=np.full(B, r["iterations"]),
                       final_residual_norm=np.full(B, r["final_residual_norm"]),
                       converged=np.full(B, r["converged"]))
        else:
            s = np.zeros((n, B))
            mk = np.zeros((n, B), np.uint8)
            its = np.zeros(B, np.int64)
            rns = np.zeros(B)
            cvs = np.zeros(B, bool)
            code = 0
            for b in range(B):
                r = refbind.ref_solve_batch(A, Y[:, b:b + 1], cfg, basis=basis)  # == clomp_solve
                code = code or r["code"]
                s[:, b] = r["s"][:, 0]
                mk[:, b] = r["mask"][:, 0]
                its[b] = r["iterations"]
                rns[b] = r["final_residual_norm"]
                cvs[b] = r["converged"]
            out = dict(code=code, s=s, mask=mk, iterations=its, final_residual_norm=rns,
                       converged=cvs)
        arrays[f"{name}/A"] = A.astype(np.float32)
        arrays[f"{name}/Y"] = Y.astype(np.float32)
        for k in ("s", "mask", "iterations", "final_residual_norm", "converged"):
            arrays[f"{name}/{k}"] = np.asarray(out[k])
        if basis is not None:
            arrays[f"{name}/D"] = np.asarray(basis, np.float64)
        case = dict(name=name, kind="solve", api=api, code=int(out["code"]),
                    cfg={f: getattr(cfg, f) for f in cfg.__dataclass_fields__},
                    basis=basis is not None)
        if gpu_code is not None:
            case["gpu_code"] = gpu_code
        cases.append(case)
        print(f"{name:34s} code={out['code']} iters={np.asarray(out['iterations'])[:4]} "
              f"rn={np.asarray(out['final_residual_norm'])[:2]}")

    base = ClompConfig.baseline

    A, Y = rand_problem(1, 32, 64, 5, 1)
    add_solve("small_th1_plain_b1", A, Y, base(5), "single")
    A, Y = rand_problem(2, 32, 64, 5, 3, snr_db=40)
    add_solve("small_th1_plain_b3_noisy", A, Y, base(5), "batch")
    add_solve("small_th1_plain_b3_noisy_single", A, Y, base(5), "single")
    A, Y = rand_problem(3, 40, 72, 6, 9, snr_db=30)
    add_solve("small_th1_plain_b9_tile", A, Y, base(6), "batch")
    A, Y = rand_problem(4, 24, 48, 4, 2, snr_db=25)
    add_solve("th07_adam_nopriors", A, Y, ClompConfig(max_outer=12, w_tv=0.0, w_lv=0.0), "batch")
    add_solve("th07_adam_nopriors_single", A, Y, ClompConfig(max_outer=12, w_tv=0.0, w_lv=0.0), "single")
    A, Y = rand_problem(5, 24, 48, 4, 2, snr_db=35)
    add_solve("th1_momentum", A, Y, ClompConfig(th=1.0, max_outer=6, inner_steps=40, lr=0.05,
                                                opt=MOMENTUM, w_tv=0.0, w_lv=0.0), "single")
    add_solve("th1_adam", A, Y, ClompConfig(th=1.0, max_outer=6, inner_steps=40, lr=0.02,
                                            opt=ADAM, w_tv=0.0, w_lv=0.0), "single")
    # test_clomp.cpp:275-298 — identity sensing composed with DCT is orthonormal.
    D = np.zeros((16, 16))
    refbind.ref().ref_dct_basis(16, refbind._p(D))
    s0 = np.zeros(16)
    s0[4], s0[11] = 1.0, -0.9
    Ad = f32(D)
    add_solve("orthonormal_exact", Ad, Ad @ s0, ClompConfig(w_tv=0.0, w_lv=0.0, lr=0.05,
                                                           max_outer=100), "single")
    A, Y = rand_problem(6, 32, 64, 5, 3, snr_db=40)
    Y[:, 1] = 0.0
    add_solve("zero_column_joint", A, Y, base(5), "batch")
    add_solve("diverging_lr", A, Y[:, :1], ClompConfig(th=1.0, opt=PLAIN, lr=1e6, w_tv=0.0,
                                                       w_lv=0.0, max_outer=5), "batch")
    add_solve("eps_at_start", A, np.zeros((32, 1)), base(5), "single")
    # Joint early stops: noiseless batch that converges before max_outer (eps
    # break, clomp.cpp:238-242) and a stalled batch (clomp.cpp:264-273).
    A2, Y2 = rand_problem(7, 40, 80, 3, 4)
    add_solve("joint_eps_break", A2, Y2, base(9), "batch")
    add_solve("joint_stall", A2, Y2, ClompConfig(th=1.0, opt=PLAIN, lr=1e-6, inner_steps=1,
                                                max_outer=40, w_tv=0.0, w_lv=0.0), "batch")
    add_solve("stall_small_lr", A, Y[:, :1], ClompConfig(th=1.0, opt=PLAIN, lr=1e-6,
                                                         inner_steps=1, max_outer=50,
                                                         w_tv=0.0, w_lv=0.0), "single")
    # Exact ties under th = 1: every tied atom is injected (clomp.cpp:49-51).
    I4 = np.eye(4)
    add_solve("exact_ties", I4, np.array([1.0, -1.0, 0.5, 0.1]), base(3), "single")
    # BASELINE config 1 at full size (product datagen, seed 0).
    c1 = cl.CONFIGS[1]
    A1, X1, Y1, _ = cl.gen_problem_1d(c1["seed"], c1["m"], c1["n"], c1["k"], 1)
    add_solve("cfg1_full", A1, Y1, base(c1["k"]), "single")
    arrays["cfg1_full/X"] = X1
    # Separable 2D operator (north-star 2D mode): the reference
    # has no separable mode, so its semantics are clomp_solve on the explicit
    # Kronecker matrix A = A_c (x) A_r (column-major vec), built here with
    # np.kron (fp64 products of the fp32 factors).
    for name, (nr, nc, mr, mc, kk, B), cfg, api in [
        ("sep_small_single", (12, 10, 6, 8, 5, 3), base(6), "single"),
        ("sep_small_joint_adam", (10, 8, 6, 5, 4, 2),
         ClompConfig(max_outer=8, lr=0.02, w_tv=0.0, w_lv=0.0), "batch"),
    ]:
        Ar, Ac, S2, Y2 = cl.gen_problem_2d(100 + nr, nr, nc, mr, mc, kk, B)
        Kr = np.kron(Ac.astype(np.float64), Ar.astype(np.float64))
        add_solve(name, Kr, Y2, cfg, api, round_a=False)
        cases[-1]["kind"] = "sep"
        arrays[f"{name}/Ar"] = Ar
        arrays[f"{name}/Ac"] = Ac
        arrays[f"{name}/S"] = S2
        del arrays[f"{name}/A"]
    # Priors (clomp.cpp:93-119): the reference's default configuration (Adam,
    # th = 0.7, auto TV / LV weights) on a make_setup-style problem A = Phi D
    # with the DCT synthesis basis (sensing.cpp:13-29, 60-79).  A column solved
    # alone sees TV-1D only (LV needs batch >= window); a multi-column batch
    # (the image mode) runs TV-2D + local variance.
    nP, mP = 64, 32
    DP = np.zeros((nP, nP))
    refbind.ref().ref_dct_basis(nP, refbind._p(DP))
    rngp = np.random.default_rng(77)
    AP = f32(rngp.standard_normal((mP, nP)) / np.sqrt(mP) @ DP)
    XP = np.zeros((nP, 3))
    for b in range(3):
        XP[rngp.choice(nP, 5, replace=False), b] = rngp.standard_normal(5)
    YP = f32(AP @ XP + 0.01 * rngp.standard_normal((mP, 3)))
    add_solve("prior_default_single", AP, YP, ClompConfig(max_outer=15), "single", basis=DP)
    add_solve("prior_plain_th1_single", AP, YP, ClompConfig(th=1.0, opt=PLAIN, lr=0.1, max_outer=6,
                                                            w_tv=0.05), "single", basis=DP)
    add_solve("prior_momentum_auto_single", AP, YP, ClompConfig(th=1.0, opt=MOMENTUM, lr=0.05,
                                                                max_outer=6, inner_steps=40,
                                                                w_tv=-1.0), "single", basis=DP)
    add_solve("prior_joint_b1", AP, YP[:, :1], ClompConfig(max_outer=12), "batch", basis=DP)
    add_solve("prior_joint_b3_tv2d", AP, YP, ClompConfig(max_outer=8), "batch", basis=DP)
    # identity basis: TV of the coefficients themselves
    Ai, Yi = rand_problem(8, 32, 64, 5, 2, snr_db=30)
    add_solve("prior_identity_basis_single", Ai, Yi, ClompConfig(th=1.0, opt=ADAM, lr=0.02,
                                                               max_outer=8, inner_steps=60,
                                                               w_tv=0.2), "single",
              basis=np.eye(64))

    # config validation (test_clomp.cpp:328-343)
    add_solve("bad_th", A, Y[:, :1], ClompConfig(th=0.0), "batch")
    add_solve("bad_inner", A, Y[:, :1], ClompConfig(inner_steps=0), "batch")

    # inject_support (test_clomp.cpp:46-69): zero third column, pre-set bit kept.
    rng = np.random.default_rng(61)
    A = f32(rng.standard_normal((10, 20)) / np.sqrt(10))
    R = f32(rng.uniform(-1, 1, (10, 3)))
    R[:, 2] = 0.0
    mk = np.zeros((20, 3), np.uint8)
    mk[5, 2] = 1
    for th in (0.7, 1.0):
        out = mk.copy()
        code = refbind.ref().ref_inject_support(refbind._p(A), 10, 20, refbind._p(R), 3, th,
                                                refbind._p(out))
        name = f"inject_th{th}"
        arrays[f"{name}/A"] = A.astype(np.float32)
        arrays[f"{name}/R"] = R
        arrays[f"{name}/mask_in"] = mk
        arrays[f"{name}/mask_out"] = out
        cases.append(dict(name=name, kind="inject", th=th, code=int(code)))

    # cskit::Rng streams (rng.hpp:13-79) and dct_basis (sensing.cpp:13-29).
    for seed in (0, 1, 12345):
        for kind, k in (("u64", 0), ("uniform", 1), ("normal", 2), ("below", 3)):
            out = np.zeros(64)
            out64 = np.zeros(64, np.uint64)
            refbind.ref().ref_rng_draws(seed, k, 1000, 64, refbind._p(out), refbind._p(out64))
            arrays[f"rng/{seed}/{kind}"] = out64 if k in (0, 3) else out
    D8 = np.zeros((8, 8))
    refbind.ref().ref_dct_basis(8, refbind._p(D8))
    arrays["dct8"] = D8

    np.savez_compressed(HERE / "golden.npz", **arrays)
    (HERE / "cases.json").write_text(json.dumps(cases, indent=1))
    print("wrote", HERE / "golden.npz", len(cases), "cases")


if __name__ == "__main__":
    main()
