"""ctypes bindings to the test-side checkers (oracle/ and oracle/_ref/).

TEST INFRASTRUCTURE ONLY: used by tests/, __graft_entry__.smoke() and the CPU
legs of bench.py, never by the product package.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

from paper_2501_11592_b200.configs import CConfig, ClompConfig

ROOT = Path(__file__).resolve().parents[1]
ORACLE_SO = ROOT / "oracle" / "_build" / "libclomp_oracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libcskit_ref.so"

ISA_SCALAR, ISA_AVX2 = 0, 1
MODE_JOINT, MODE_PER_SIGNAL = 0, 1


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def build_oracle() -> None:
    if not ORACLE_SO.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], check=True)


_orc = None
_ref = None


def oracle() -> C.CDLL:
    global _orc
    if _orc is None:
        build_oracle()
        h = C.CDLL(str(ORACLE_SO))
        vp, i64 = C.c_void_p, C.c_int64
        h.orc_clomp_solve_batch.argtypes = [vp, i64, i64, vp, i64, C.POINTER(CConfig), C.c_int,
                                            C.c_int, vp, vp, vp, vp, vp, vp, vp, C.c_char_p, C.c_int]
        h.orc_clomp_solve_batch_basis.argtypes = [vp, i64, i64, vp, vp, i64, C.POINTER(CConfig),
                                                  C.c_int, C.c_int, vp, vp, vp, vp, vp, vp, vp,
                                                  C.c_char_p, C.c_int]
        h.orc_clomp_solve_sep.argtypes = [vp, i64, i64, vp, i64, i64, vp, i64, C.POINTER(CConfig),
                                          C.c_int, C.c_int, vp, vp, vp, vp, vp, vp, vp,
                                          C.c_char_p, C.c_int]
        h.orc_clomp_solve_sep_gram.argtypes = [vp, i64, i64, vp, i64, i64, vp, i64,
                                               C.POINTER(CConfig), vp, vp, vp, vp, vp, vp,
                                               C.c_char_p, C.c_int]
        h.orc_inject_support.argtypes = [vp, i64, i64, vp, i64, C.c_double, C.c_int, vp]
        h.orc_clomp_loss.argtypes = [vp, i64, i64, vp, i64, vp, vp, C.POINTER(CConfig), C.c_int, vp, vp]
        h.orc_gradient_step.argtypes = [vp, vp, vp, vp, vp, vp, i64, C.POINTER(CConfig)]
        _orc = h
    return _orc


def ref_available() -> bool:
    return REF_SO.exists()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        h = C.CDLL(str(REF_SO))
        vp, i64 = C.c_void_p, C.c_int64
        h.ref_clomp_solve_batch.argtypes = [vp, i64, i64, vp, i64, C.POINTER(CConfig), vp, vp, vp,
                                            vp, vp, vp, C.c_char_p, C.c_int]
        h.ref_clomp_solve_batch_b.argtypes = [vp, i64, i64, vp, vp, i64, C.POINTER(CConfig), vp,
                                              vp, vp, vp, vp, vp, vp, C.c_char_p, C.c_int]
        h.ref_clomp_solve.argtypes = [vp, i64, i64, vp, C.POINTER(CConfig), vp, vp, vp, vp, vp, vp,
                                      C.c_char_p, C.c_int]
        h.ref_inject_support.argtypes = [vp, i64, i64, vp, i64, C.c_double, vp]
        h.ref_rng_draws.argtypes = [C.c_uint64, C.c_int, C.c_uint64, i64, vp, vp]
        h.ref_dct_basis.argtypes = [i64, vp]
        h.ref_gen_problem_1d.argtypes = [C.c_uint64, i64, i64, i64, i64, C.c_int, C.c_int,
                                         C.c_double, vp, vp, vp]
        h.ref_force_isa.argtypes = [C.c_int]
        _ref = h
    return _ref


def ref_gen_problem_1d(seed, m, n, k, batch, normalize=True, value_law=0, snr_db=-1.0,
                       want_x=True):
    """The harness's seeded problem drawn with the reference's cskit::Rng
    (oracle/ref_harness.cpp): (A m x n fp32, X n x B fp64 or None, Y m x B fp32)."""
    A = np.zeros((m, n), np.float32)
    X = np.zeros((n, batch)) if want_x else None
    Y = np.zeros((m, batch), np.float32)
    code = ref().ref_gen_problem_1d(seed, m, n, k, batch, int(normalize), int(value_law),
                                    float(snr_db), _p(A), _p(X), _p(Y))
    if code:
        raise ValueError("ref_gen_problem_1d: bad sizes")
    return A, X, Y


def orc_solve(A, Y, cfg: ClompConfig, mode=MODE_JOINT, isa=ISA_AVX2, trace=False, basis=None):
    """Oracle restatement. A m x n, Y m x B (fp64 arrays of fp32 values);
    basis: n x n synthesis matrix for the priors (None: no basis)."""
    A = np.ascontiguousarray(A, np.float64)
    D = None if basis is None else np.ascontiguousarray(basis, np.float64)
    Y = np.ascontiguousarray(Y, np.float64)
    if Y.ndim == 1:
        Y = Y.reshape(-1, 1)
    m, n = A.shape
    B = Y.shape[1]
    s = np.zeros((n, B))
    mk = np.zeros((n, B), np.uint8)
    it = np.zeros(B, np.int64)
    rn = np.zeros(B)
    cv = np.zeros(B, np.uint8)
    st = np.zeros(B, np.int32)
    tr = np.zeros((B, max(1, cfg.max_outer), 4)) if trace else None
    err = C.create_string_buffer(256)
    c = cfg.to_c()
    code = oracle().orc_clomp_solve_batch_basis(_p(A), m, n, _p(D), _p(Y), B, C.byref(c), isa,
                                                mode, _p(s), _p(mk), _p(it), _p(rn), _p(cv),
                                                _p(st), _p(tr), err, 256)
    return dict(code=code, err=err.value.decode(), s=s, mask=mk, iterations=it,
                final_residual_norm=rn, converged=cv.astype(bool), status=st, trace=tr)


def orc_solve_sep(Ar, Ac, Y, cfg: ClompConfig, mode=MODE_JOINT, isa=ISA_AVX2):
    """Oracle restatement with the separable operator A = A_c (x) A_r."""
    Ar = np.ascontiguousarray(Ar, np.float64)
    Ac = np.ascontiguousarray(Ac, np.float64)
    Y = np.ascontiguousarray(Y, np.float64)
    if Y.ndim == 1:
        Y = Y.reshape(-1, 1)
    n = Ar.shape[1] * Ac.shape[1]
    B = Y.shape[1]
    s = np.zeros((n, B))
    mk = np.zeros((n, B), np.uint8)
    it = np.zeros(B, np.int64)
    rn = np.zeros(B)
    cv = np.zeros(B, np.uint8)
    st = np.zeros(B, np.int32)
    err = C.create_string_buffer(256)
    c = cfg.to_c()
    code = oracle().orc_clomp_solve_sep(_p(Ar), Ar.shape[0], Ar.shape[1], _p(Ac), Ac.shape[0],
                                        Ac.shape[1], _p(Y), B, C.byref(c), isa, mode, _p(s), _p(mk),
                                        _p(it), _p(rn), _p(cv), _p(st), None, err, 256)
    return dict(code=code, err=err.value.decode(), s=s, mask=mk, iterations=it,
                final_residual_norm=rn, converged=cv.astype(bool), status=st)


def orc_solve_sep_gram(Ar, Ac, Y, cfg: ClompConfig):
    """Separable per-signal loop in Gram form (fp64, products regrouped): the
    full-size 2D checker (oracle/clomp_oracle.c, orc_clomp_solve_sep_gram)."""
    Ar = np.ascontiguousarray(Ar, np.float64)
    Ac = np.ascontiguousarray(Ac, np.float64)
    Y = np.ascontiguousarray(Y, np.float64)
    if Y.ndim == 1:
        Y = Y.reshape(-1, 1)
    n = Ar.shape[1] * Ac.shape[1]
    B = Y.shape[1]
    s = np.zeros((n, B))
    mk = np.zeros((n, B), np.uint8)
    it = np.zeros(B, np.int64)
    rn = np.zeros(B)
    cv = np.zeros(B, np.uint8)
    st = np.zeros(B, np.int32)
    err = C.create_string_buffer(256)
    c = cfg.to_c()
    code = oracle().orc_clomp_solve_sep_gram(_p(Ar), Ar.shape[0], Ar.shape[1], _p(Ac),
                                             Ac.shape[0], Ac.shape[1], _p(Y), B, C.byref(c),
                                             _p(s), _p(mk), _p(it), _p(rn), _p(cv), _p(st),
                                             err, 256)
    return dict(code=code, err=err.value.decode(), s=s, mask=mk, iterations=it,
                final_residual_norm=rn, converged=cv.astype(bool), status=st)


def ref_solve_batch(A, Y, cfg: ClompConfig, basis=None):
    """The unmodified reference clomp_solve_batch (basis: n x n synthesis
    matrix, needed by the priors; None: the 1 x n dummy of SURVEY.md D8)."""
    A = np.ascontiguousarray(A, np.float64)
    D = None if basis is None else np.ascontiguousarray(basis, np.float64)
    Y = np.ascontiguousarray(Y, np.float64)
    if Y.ndim == 1:
        Y = Y.reshape(-1, 1)
    m, n = A.shape
    B = Y.shape[1]
    s = np.zeros((n, B))
    mk = np.zeros((n, B), np.uint8)
    it = np.zeros(1, np.int64)
    rn = np.zeros(1)
    cv = np.zeros(1, np.uint8)
    wall = np.zeros(1)
    err = C.create_string_buffer(256)
    c = cfg.to_c()
    xh = np.zeros((n, B)) if D is not None else None
    code = ref().ref_clomp_solve_batch_b(_p(A), m, n, _p(D), _p(Y), B, C.byref(c), _p(s), _p(mk),
                                         _p(it), _p(rn), _p(cv), _p(xh), _p(wall), err, 256)
    return dict(code=code, err=err.value.decode(), s=s, mask=mk, iterations=int(it[0]),
                final_residual_norm=float(rn[0]), converged=bool(cv[0]), wall_s=float(wall[0]),
                x_hat=xh)


def orc_inject(A, R, th, mask, isa=ISA_AVX2):
    A = np.ascontiguousarray(A, np.float64)
    R = np.ascontiguousarray(R, np.float64)
    if R.ndim == 1:
        R = R.reshape(-1, 1)
    mk = np.ascontiguousarray(mask, np.uint8).copy()
    code = oracle().orc_inject_support(_p(A), A.shape[0], A.shape[1], _p(R), R.shape[1],
                                       float(th), isa, _p(mk))
    return code, mk


def support_sets(mask):
    return [tuple(np.flatnonzero(mask[:, b])) for b in range(mask.shape[1])]
