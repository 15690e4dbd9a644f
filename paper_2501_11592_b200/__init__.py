"""B200-native CLOMP reconstruction loop (arXiv 2501.11592), host mirror.

A thin ctypes layer over the C-ABI in include/clomp_b200.h
(paper_2501_11592_b200/_build/libclomp_b200.so).  Names, argument meaning and
error behaviour follow the reference library's public API
(/root/reference/proj/include/cskit/clomp.hpp:16-101):

    ClompConfig            <- cskit::ClompConfig          (clomp.hpp:16-33)
    ClompContext           <- cskit::MeasurementSetup     (sensing.hpp:37-45),
                              uploaded once (atom-major fp32 in HBM)
    clomp_solve_batch()    <- cskit::clomp_solve_batch    (clomp.cpp:211-292)
    clomp_solve()          <- cskit::clomp_solve          (clomp.cpp:294-311)
    inject_support()       <- cskit::inject_support       (clomp.cpp:142-154)
    ConfigError / DimensionError / NumericalError  <- errors.hpp:10-37

There is no CPU path: if the CUDA library is missing or no B200 is visible the
calls raise.  Numerics: fp32 operands, fp64 learning, tensor-core correlations
with fp64 re-decision of near-tied selections.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from collections.abc import Sequence
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
# CLOMP_B200_LIB selects another build of the same library (the debug build
# with device-side index checks, _build/libclomp_b200_dbg.so); never a fallback
LIB_PATH = Path(os.environ.get("CLOMP_B200_LIB") or _PKG / "_build" / "libclomp_b200.so")

from .configs import ADAM, CONFIGS, MOMENTUM, PLAIN, CConfig, ClompConfig  # noqa: F401
MODE_JOINT, MODE_PER_SIGNAL = 0, 1
LAYOUT_REF, LAYOUT_T = 0, 1

CL_OK, CL_ERR_INTERNAL, CL_ERR_CONFIG, CL_ERR_DIMENSION = 0, 1, 2, 3
CL_ERR_NUMERICAL, CL_ERR_UNSUPPORTED, CL_ERR_CUDA, CL_ERR_CAPACITY = 4, 5, 6, 7


class Error(RuntimeError):
    """cskit::Error (errors.hpp:10)."""


class DimensionError(Error):
    """cskit::DimensionError (errors.hpp:16)."""


class ConfigError(Error):
    """cskit::ConfigError (errors.hpp:22)."""


class NumericalError(Error):
    """cskit::NumericalError (errors.hpp:28)."""


class UnsupportedError(Error):
    """Priors requested: not implemented on the B200 path (no CPU fallback)."""


class CudaError(Error):
    """No device, wrong architecture, or a CUDA runtime failure."""


class CapacityError(Error):
    """The support outgrew the per-signal capacity."""


_ERRORS = {
    CL_ERR_INTERNAL: Error,
    CL_ERR_CONFIG: ConfigError,
    CL_ERR_DIMENSION: DimensionError,
    CL_ERR_NUMERICAL: NumericalError,
    CL_ERR_UNSUPPORTED: UnsupportedError,
    CL_ERR_CUDA: CudaError,
    CL_ERR_CAPACITY: CapacityError,
}


class CResult(C.Structure):
    _fields_ = [
        ("cap", C.c_int64),
        ("support", C.c_void_p),
        ("coef", C.c_void_p),
        ("count", C.c_void_p),
        ("s", C.c_void_p),
        ("mask", C.c_void_p),
        ("iterations", C.c_void_p),
        ("final_residual_norm", C.c_void_p),
        ("converged", C.c_void_p),
        ("status", C.c_void_p),
        ("x_hat", C.c_void_p),
        ("flags", C.c_int32),
        ("pad0", C.c_int32),
    ]


class CDeviceResult(C.Structure):
    _fields_ = [
        ("cap", C.c_int64),
        ("support", C.c_void_p),
        ("coef", C.c_void_p),
        ("count", C.c_void_p),
        ("iterations", C.c_void_p),
        ("final_residual_norm", C.c_void_p),
        ("converged", C.c_void_p),
        ("status", C.c_void_p),
    ]


class CStats(C.Structure):
    _fields_ = [
        ("kernel_launches", C.c_int64),
        ("rescans", C.c_int64),
        ("outer_iterations", C.c_int64),
        ("corr_ms", C.c_double),
        ("learn_ms", C.c_double),
        ("total_ms", C.c_double),
        ("corr_path", C.c_int32),
        ("pad0", C.c_int32),
        ("e2e_ms", C.c_double),
        ("select_ms", C.c_double),
        ("h2d_bytes", C.c_int64),
        ("d2h_bytes", C.c_int64),
    ]


# Every symbol include/clomp_b200.h declares (tests check the .so exports them).
EXPORTED = [
    "cl_config_default", "cl_create", "cl_destroy", "cl_last_error",
    "cl_solve_batch", "cl_submit", "cl_wait", "cl_solve_batch_device", "cl_synchronize",
    "cl_inject_support", "cl_get_stats", "cl_set_corr_path", "cl_set_profiling",
    "cl_set_stream", "cl_debug_scores", "cl_set_gram_cache", "cl_create_sep", "cl_set_fused", "cl_set_cluster_learn", "cl_set_power_levels", "cl_set_basis", "cl_set_synthesis", "cl_set_direct_form",
    "cl_nccl_unique_id", "cl_create_colshard", "cl_set_virtual_shards",
    "cl_create_group", "cl_destroy_group", "cl_group_size", "cl_group_context",
    "cl_group_last_error", "cl_group_solve_batch",
    "cl_gen_problem_2d", "cl_dct_basis",
    "cl_abi_version", "cl_device_count", "cl_abi_struct_sizes", "cl_rng_draws", "cl_gen_problem_1d",
]

_lib_handle = None


def lib() -> C.CDLL:
    """Load libclomp_b200.so; raises if it was not built (no fallback)."""
    global _lib_handle
    if _lib_handle is None:
        if not LIB_PATH.exists():
            raise CudaError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() "
                "(python -m paper_2501_11592_b200.build)")
        h = C.CDLL(str(LIB_PATH))
        vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int
        h.cl_create.restype = vp
        h.cl_create.argtypes = [i32, vp, i64, i64, i32, C.POINTER(C.c_int)]
        h.cl_destroy.argtypes = [vp]
        h.cl_last_error.restype = C.c_char_p
        h.cl_last_error.argtypes = [vp]
        h.cl_solve_batch.argtypes = [vp, vp, i64, i32, C.POINTER(CConfig), i32, C.POINTER(CResult)]
        h.cl_submit.argtypes = [vp, vp, i64, i32, C.POINTER(CConfig), i32]
        h.cl_wait.argtypes = [vp, C.POINTER(CResult)]
        h.cl_solve_batch_device.argtypes = [vp, vp, i64, C.POINTER(CConfig), i32, C.POINTER(CDeviceResult)]
        h.cl_synchronize.argtypes = [vp]
        h.cl_inject_support.argtypes = [vp, vp, i64, C.c_double, vp]
        h.cl_get_stats.argtypes = [vp, C.POINTER(CStats)]
        h.cl_set_corr_path.argtypes = [vp, i32]
        h.cl_set_profiling.argtypes = [vp, i32]
        h.cl_set_stream.argtypes = [vp, vp]
        h.cl_debug_scores.argtypes = [vp, vp, i64, i32, vp]
        h.cl_set_gram_cache.argtypes = [vp, i32]
        h.cl_set_fused.argtypes = [vp, i32]
        h.cl_set_cluster_learn.argtypes = [vp, i32]
        h.cl_set_power_levels.argtypes = [vp, i32]
        h.cl_set_basis.argtypes = [vp, vp, C.c_int64, i32]
        h.cl_set_synthesis.argtypes = [vp, i32]
        h.cl_set_direct_form.argtypes = [vp, i32]
        h.cl_nccl_unique_id.argtypes = [vp]
        h.cl_create_colshard.restype = vp
        h.cl_create_colshard.argtypes = [i32, vp, i64, i64, i32, i32, i32, vp, C.POINTER(C.c_int)]
        h.cl_set_virtual_shards.argtypes = [vp, i32]
        h.cl_create_group.restype = vp
        h.cl_create_group.argtypes = [vp, i32, vp, i64, i64, i32, i32, C.POINTER(C.c_int)]
        h.cl_destroy_group.argtypes = [vp]
        h.cl_group_size.argtypes = [vp]
        h.cl_group_context.restype = vp
        h.cl_group_context.argtypes = [vp, i32]
        h.cl_group_last_error.restype = C.c_char_p
        h.cl_group_last_error.argtypes = [vp]
        h.cl_group_solve_batch.argtypes = [vp, vp, i64, i32, C.POINTER(CConfig), i32, C.POINTER(CResult)]
        h.cl_create_sep.restype = vp
        h.cl_create_sep.argtypes = [i32, vp, i64, i64, vp, i64, i64, i32, C.POINTER(C.c_int)]
        h.cl_gen_problem_2d.argtypes = [C.c_uint64, i64, i64, i64, i64, i64, i64, vp, vp, vp, vp]
        h.cl_dct_basis.argtypes = [i64, vp]
        h.cl_config_default.argtypes = [C.POINTER(CConfig)]
        h.cl_rng_draws.argtypes = [C.c_uint64, i32, C.c_uint64, i64, vp, vp]
        h.cl_gen_problem_1d.argtypes = [C.c_uint64, i64, i64, i64, i64, i32, i32, C.c_double, vp, vp, vp, vp]
        _lib_handle = h
    return _lib_handle


def _ptr(a):
    # the raw address (half the cost of ctypes.data_as; the array outlives the call)
    return None if a is None else C.c_void_p(a.ctypes.data)


class Ragged(Sequence):
    """Per-signal rows of a [B][cap] array cut at counts[b] (views, built on
    access): the compact support / coefficient lists of a batch."""

    def __init__(self, data: np.ndarray, counts: np.ndarray):
        self.data, self.counts = data, counts

    def __len__(self) -> int:
        return len(self.counts)

    def __getitem__(self, b):
        if isinstance(b, slice):
            return [self[i] for i in range(*b.indices(len(self)))]
        return self.data[b, :self.counts[b]]


@dataclasses.dataclass
class BatchSolveResult:
    """cskit::BatchSolveResult (clomp.hpp:82-90) plus the compact support."""

    s: np.ndarray                 # n x B fp64 (reference layout)
    mask: np.ndarray              # n x B uint8
    iterations: np.ndarray        # [B]
    final_residual_norm: np.ndarray
    converged: np.ndarray
    status: np.ndarray
    support: Ragged               # per signal, ascending atom indices
    coef: Ragged                  # per signal, aligned with support
    x_hat: np.ndarray | None = None   # n x B fp64, basis @ (s * mask) (set_synthesis)


@dataclasses.dataclass
class SolveResult:
    """cskit::SolveResult (solvers.hpp:12-19), without x_hat."""

    values: np.ndarray
    mask: np.ndarray
    iterations: int
    final_residual_norm: float
    converged: bool


def _raise(code: int, handle=None):
    if code == CL_OK:
        return
    msg = lib().cl_last_error(handle)
    msg = msg.decode() if msg else f"status {code}"
    raise _ERRORS.get(code, Error)(msg)


class ClompContext:
    """A dictionary resident on one B200 (replaces MeasurementSetup.a).

    a: m x n (layout='ref', the reference la::Mat layout) or n x m ('t').
    Values are rounded to fp32 (north-star operand precision)."""

    def __init__(self, a, device: int = 0, layout: str = "ref"):
        a = np.ascontiguousarray(a, dtype=np.float32)
        if a.ndim != 2:
            raise DimensionError("dictionary must be 2-D")
        if layout == "ref":
            self.m, self.n = a.shape
            lay = LAYOUT_REF
        else:
            self.n, self.m = a.shape
            lay = LAYOUT_T
        st = C.c_int(0)
        h = lib().cl_create(int(device), _ptr(a), self.m, self.n, lay, C.byref(st))
        if not h:
            _raise(st.value or CL_ERR_CUDA, None)
        self._h = h
        self.device = device

    @classmethod
    def separable(cls, a_r, a_c, device: int = 0) -> "ClompContext":
        """Separable 2D operator A = A_c (x) A_r (Y = A_r S A_c^T), column-major
        vec: atom p = i + n_r*j, measurement q = qr + m_r*qc.  The Kronecker
        matrix is never formed."""
        ar = np.ascontiguousarray(a_r, dtype=np.float32)
        ac = np.ascontiguousarray(a_c, dtype=np.float32)
        self = cls.__new__(cls)
        st = C.c_int(0)
        h = lib().cl_create_sep(int(device), _ptr(ar), ar.shape[0], ar.shape[1], _ptr(ac),
                                ac.shape[0], ac.shape[1], LAYOUT_REF, C.byref(st))
        if not h:
            _raise(st.value or CL_ERR_CUDA, None)
        self._h = h
        self.device = device
        self.m = ar.shape[0] * ac.shape[0]
        self.n = ar.shape[1] * ac.shape[1]
        self.shape2d = (ar.shape, ac.shape)
        return self

    @classmethod
    def colshard(cls, a, rank: int, world: int, nccl_id: bytes | None,
                 device: int = 0) -> "ClompContext":
        """Column-sharded dictionary over `world` GPUs (cl_create_colshard)."""
        a = np.ascontiguousarray(a, dtype=np.float32)
        self = cls.__new__(cls)
        self.m, self.n = a.shape
        st = C.c_int(0)
        idbuf = C.create_string_buffer(bytes(nccl_id), 128) if nccl_id else None
        h = lib().cl_create_colshard(int(device), _ptr(a), self.m, self.n, LAYOUT_REF, int(rank),
                                     int(world), idbuf, C.byref(st))
        if not h:
            _raise(st.value or CL_ERR_CUDA, None)
        self._h = h
        self.device = device
        return self

    def set_virtual_shards(self, shards: int):
        """Emulate `shards` column shards on this GPU (tests the sharded math)."""
        _raise(lib().cl_set_virtual_shards(self._h, int(shards)), self._h)

    @property
    def handle(self):
        return self._h

    @property
    def _pending(self) -> list:
        # result buffers of batches submitted with clomp_submit (oldest first)
        p = self.__dict__.get("_pend_list")
        if p is None:
            p = self.__dict__["_pend_list"] = []
        return p

    def close(self):
        if getattr(self, "_h", None):
            lib().cl_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_corr_path(self, path: int):
        _raise(lib().cl_set_corr_path(self._h, int(path)), self._h)

    def set_direct_form(self, from_outer: int):
        """Separable contexts: learn in direct form (no support Gram matrix) from
        outer iteration `from_outer` on; -1 auto, 0 never."""
        _raise(lib().cl_set_direct_form(self._h, int(from_outer)), self._h)

    def set_gram_cache(self, mode: int):
        """1 build / 0 drop / -1 auto the fp64 A^T A cache."""
        _raise(lib().cl_set_gram_cache(self._h, int(mode)), self._h)

    def set_fused(self, on: bool):
        """Allow (default) or forbid the one-block-per-signal latency path."""
        _raise(lib().cl_set_fused(self._h, int(bool(on))), self._h)

    def set_basis(self, D):
        """Synthesis basis D (n x n, x = D s; MeasurementSetup::basis) for the
        TV prior of single-column solves; None clears it."""
        if D is None:
            _raise(lib().cl_set_basis(self._h, None, 0, 0), self._h)
            return
        D = np.ascontiguousarray(D, np.float64)
        if D.ndim != 2 or D.shape[0] != D.shape[1]:
            raise DimensionError("set_basis: D must be square")
        _raise(lib().cl_set_basis(self._h, _ptr(D), D.shape[0], 0), self._h)

    def set_synthesis(self, on: bool):
        """Also return x_hat = D (s * mask) (BatchSolveResult.x_hat, clomp.cpp:289),
        formed on the GPU from the compact supports; needs set_basis."""
        _raise(lib().cl_set_synthesis(self._h, int(bool(on))), self._h)
        self.__dict__["_synth_on"] = bool(on)

    @property
    def _synthesis(self) -> bool:
        return self.__dict__.get("_synth_on", False)

    def set_cluster_learn(self, on):
        """Learn supports of 33..256 atoms on CTA clusters with register-resident
        Gram blocks (True / 1, default; 2 = eight-CTA variant above 128 atoms) or
        on the block-per-signal kernel (False / 0)."""
        _raise(lib().cl_set_cluster_learn(self._h, int(on)), self._h)

    def set_power_levels(self, levels: int):
        """Power form of plain GD on cluster-learned supports: -1 auto (L = 3),
        0 off (one cluster epoch per reference epoch), L squaring levels."""
        _raise(lib().cl_set_power_levels(self._h, int(levels)), self._h)

    def set_profiling(self, on: bool):
        _raise(lib().cl_set_profiling(self._h, int(bool(on))), self._h)

    def set_stream(self, stream_handle: int | None):
        """Issue work on a caller-owned cudaStream_t (e.g. torch's
        stream.cuda_stream); None restores the context's own stream."""
        _raise(lib().cl_set_stream(self._h, C.c_void_p(stream_handle) if stream_handle else None),
               self._h)

    def debug_scores(self, r_signal_major, path: int) -> np.ndarray:
        """A^T r for B x m fp32 residuals via path 1 (fp64 SIMT, |.|), 2 (tcgen05,
        signed) or 3 (the B <= 4 GEMV, |.|)."""
        r = np.ascontiguousarray(r_signal_major, dtype=np.float32)
        out = np.zeros((r.shape[0], self.n), np.float64)
        _raise(lib().cl_debug_scores(self._h, _ptr(r), r.shape[0], int(path), _ptr(out)), self._h)
        return out

    def stats(self) -> dict:
        s = CStats()
        _raise(lib().cl_get_stats(self._h, C.byref(s)), self._h)
        return {f: getattr(s, f) for f, _ in CStats._fields_ if f != "pad0"}


GROUP_SIGNAL_SHARD, GROUP_COLUMN_SHARD = 0, 1


class ClompGroup:
    """One dictionary on several GPUs of this process (cl_create_group):
    mode GROUP_SIGNAL_SHARD splits a batch's independent signals across the
    devices, GROUP_COLUMN_SHARD splits one large dictionary by atoms (NCCL)."""

    def __init__(self, a, devices, mode: int = GROUP_SIGNAL_SHARD, layout: str = "ref"):
        a = np.ascontiguousarray(a, dtype=np.float32)
        if a.ndim != 2:
            raise DimensionError("dictionary must be 2-D")
        self.m, self.n = a.shape if layout == "ref" else a.shape[::-1]
        devs = (C.c_int * len(devices))(*[int(d) for d in devices])
        st = C.c_int(0)
        h = lib().cl_create_group(devs, len(devices), _ptr(a), self.m, self.n,
                                  LAYOUT_REF if layout == "ref" else LAYOUT_T, int(mode), C.byref(st))
        if not h:
            msg = lib().cl_group_last_error(None)
            raise _ERRORS.get(st.value or CL_ERR_CUDA, Error)(msg.decode() if msg else "cl_create_group")
        self._g = h
        self.devices = list(devices)
        self._synthesis = False

    def close(self):
        if getattr(self, "_g", None):
            lib().cl_destroy_group(self._g)
            self._g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __len__(self) -> int:
        return lib().cl_group_size(self._g)

    def solve_batch(self, y_cols, cfg: ClompConfig | None = None, mode: int = MODE_PER_SIGNAL,
                    layout: str = "ref", dense: bool = True) -> BatchSolveResult:
        cfg = cfg or ClompConfig()
        y, B, lay = _prep_y(self, y_cols, layout)
        pend = _Pending(self, y, B, cfg, dense)
        c = cfg.to_c()
        code = lib().cl_group_solve_batch(self._g, _ptr(y), B, lay, C.byref(c), int(mode),
                                          C.byref(pend.res))
        if code:
            msg = lib().cl_group_last_error(self._g)
            raise _ERRORS.get(code, Error)(msg.decode() if msg else f"status {code}")
        return pend.result()


def nccl_unique_id() -> bytes:
    """ncclUniqueId (128 bytes) for cl_create_colshard, created on rank 0."""
    buf = C.create_string_buffer(128)
    _raise(lib().cl_nccl_unique_id(buf), None)
    return buf.raw


def _prep_y(ctx: ClompContext, y_cols, layout: str):
    y = np.ascontiguousarray(y_cols, dtype=np.float32)
    if y.ndim == 1:
        y = y.reshape(-1, 1) if layout == "ref" else y.reshape(1, -1)
    if layout == "ref":
        if y.shape[0] != ctx.m:
            raise DimensionError(f"clomp: y rows {y.shape[0]} vs m={ctx.m}")
        return y, y.shape[1], LAYOUT_REF
    if y.shape[1] != ctx.m:
        raise DimensionError(f"clomp: y cols {y.shape[1]} vs m={ctx.m}")
    return y, y.shape[0], LAYOUT_T


class _Pending:
    """Result buffers of one submitted batch (filled by cl_wait)."""

    def __init__(self, ctx: ClompContext, y, B: int, cfg: ClompConfig, dense: bool):
        n = ctx.n
        cap = max(1, n if cfg.th < 1.0 else min(n, max(1, int(cfg.max_outer)) + 16))
        self.y, self.B, self.cap, self.dense = y, B, cap, dense  # y kept alive for the DMA
        # uninitialised: cl_wait writes every entry of the compact rows (zeros
        # past each count), which saves zeroing ~2 MB per config-2 call
        self.sup = np.empty((max(B, 1), cap), np.int32)
        self.coef = np.empty((max(B, 1), cap), np.float64)
        if B == 0:
            self.sup.fill(0)
            self.coef.fill(0.0)
        self.cnt = np.zeros(max(B, 1), np.int32)
        self.s = np.zeros((n, max(B, 1)), np.float64) if dense else None
        self.mask = np.zeros((n, max(B, 1)), np.uint8) if dense else None
        self.it = np.zeros(max(B, 1), np.int64)
        self.rn = np.zeros(max(B, 1), np.float64)
        self.cv = np.zeros(max(B, 1), np.uint8)
        self.st = np.zeros(max(B, 1), np.int32)
        self.xh = np.zeros((n, max(B, 1)), np.float64) if ctx._synthesis else None
        self.res = CResult(cap, _ptr(self.sup), _ptr(self.coef), _ptr(self.cnt), _ptr(self.s),
                           _ptr(self.mask), _ptr(self.it), _ptr(self.rn), _ptr(self.cv),
                           _ptr(self.st), _ptr(self.xh), 1, 0)  # s / mask are np.zeros: PREZEROED

    def result(self) -> BatchSolveResult:
        B, cap, dense = self.B, self.cap, self.dense
        counts = np.minimum(self.cnt[:B], cap)
        return BatchSolveResult(self.s[:, :B] if dense else None,
                                self.mask[:, :B] if dense else None, self.it[:B], self.rn[:B],
                                self.cv[:B].astype(bool), self.st[:B], Ragged(self.sup, counts),
                                Ragged(self.coef, counts),
                                self.xh[:, :B] if self.xh is not None else None)


def clomp_submit(ctx: ClompContext, y_cols, cfg: ClompConfig | None = None,
                 mode: int = MODE_JOINT, layout: str = "ref", dense: bool = True) -> None:
    """First half of a pipelined clomp_solve_batch (cl_submit): starts the
    upload of y and queues the solve and the download of its results; returns
    at once.  Up to two batches may be in flight per context; clomp_wait
    returns them in submission order.  Streams of batches overlap batch i + 1's
    upload and batch i's download with the other's solve."""
    cfg = cfg or ClompConfig()
    y, B, lay = _prep_y(ctx, y_cols, layout)
    pend = _Pending(ctx, y, B, cfg, dense)
    c = cfg.to_c()
    _raise(lib().cl_submit(ctx.handle, _ptr(y), B, lay, C.byref(c), int(mode)), ctx.handle)
    ctx._pending.append(pend)


def clomp_wait(ctx: ClompContext) -> BatchSolveResult:
    """Second half (cl_wait): the oldest submitted batch's result."""
    if not ctx._pending:
        raise ConfigError("clomp_wait: nothing in flight")
    pend = ctx._pending.pop(0)
    _raise(lib().cl_wait(ctx.handle, C.byref(pend.res)), ctx.handle)
    return pend.result()


def clomp_solve_batch(ctx: ClompContext, y_cols, cfg: ClompConfig | None = None,
                      mode: int = MODE_JOINT, layout: str = "ref",
                      dense: bool = True) -> BatchSolveResult:
    """Reconstruct a batch; y_cols is m x B (reference layout) or B x m ('t').

    dense=False skips materialising the n x B `s` / `mask` matrices (they are
    None in the result); supports and coefficients are always returned.  A y
    in page-locked memory (e.g. a pinned torch tensor's numpy view) is copied
    to the GPU directly, pageable y through the context's pinned staging."""
    cfg = cfg or ClompConfig()
    y, B, lay = _prep_y(ctx, y_cols, layout)
    pend = _Pending(ctx, y, B, cfg, dense)
    c = cfg.to_c()
    code = lib().cl_solve_batch(ctx.handle, _ptr(y), B, lay, C.byref(c), int(mode),
                                C.byref(pend.res))
    _raise(code, ctx.handle)
    return pend.result()


def clomp_solve(ctx: ClompContext, y, cfg: ClompConfig | None = None) -> SolveResult:
    """Single-signal wrapper: exactly a one-column batch (clomp.cpp:294-311)."""
    y = np.asarray(y, dtype=np.float32).reshape(-1)
    if y.shape[0] != ctx.m:
        raise DimensionError(f"clomp: y has {y.shape[0]} entries, setup expects {ctx.m}")
    r = clomp_solve_batch(ctx, y.reshape(-1, 1), cfg, MODE_JOINT)
    return SolveResult(r.s[:, 0].copy(), r.mask[:, 0].copy(), int(r.iterations[0]),
                       float(r.final_residual_norm[0]), bool(r.converged[0]))


def inject_support(ctx: ClompContext, r_cols, th: float, mask) -> np.ndarray:
    """mask |= thresholded |A^T r| per column (clomp.cpp:142-154); returns mask."""
    r = np.ascontiguousarray(r_cols, dtype=np.float64)
    if r.ndim == 1:
        r = r.reshape(-1, 1)
    if r.shape[0] != ctx.m:
        raise DimensionError(f"inject_support: residual rows {r.shape[0]} vs m={ctx.m}")
    B = r.shape[1]
    mk = np.ascontiguousarray(mask, dtype=np.uint8)
    if mk.size != ctx.n * B:
        raise DimensionError("inject_support: mask size mismatch")
    mk = mk.reshape(ctx.n, B).copy()
    _raise(lib().cl_inject_support(ctx.handle, _ptr(r), B, float(th), _ptr(mk)), ctx.handle)
    return mk


# ------------------------------------------------------------- datagen
def rng_draws(seed: int, kind: str, count: int, bound: int = 0) -> np.ndarray:
    """Draws of the restated cskit::Rng (rng.hpp:13-79)."""
    k = {"u64": 0, "uniform": 1, "normal": 2, "below": 3}[kind]
    out = np.zeros(count, np.float64)
    out64 = np.zeros(count, np.uint64)
    lib().cl_rng_draws(seed, k, bound, count, _ptr(out), _ptr(out64))
    return out64 if k in (0, 3) else out


def gen_problem_1d(seed: int, m: int, n: int, k: int, batch: int,
                   normalize: bool = True, value_law: int = 0,
                   snr_db: float = -1.0):
    """Seeded synthetic problem.  Returns (A m x n fp32,
    X n x B fp64, Y m x B fp32, supports B x k int32)."""
    A = np.zeros((m, n), np.float32)
    X = np.zeros((n, batch), np.float64)
    Y = np.zeros((m, batch), np.float32)
    S = np.zeros((batch, k), np.int32)
    code = lib().cl_gen_problem_1d(seed, m, n, k, batch, int(normalize), int(value_law),
                                   float(snr_db), _ptr(A), _ptr(X), _ptr(Y), _ptr(S))
    if code:
        raise DimensionError("gen_problem_1d: bad sizes")
    return A, X, Y, S


def gen_problem_2d(seed: int, n_r: int, n_c: int, m_r: int, m_c: int, k: int, batch: int):
    """Separable 2D problem.  Returns (A_r m_r x n_r fp32,
    A_c m_c x n_c fp32, S (n_r n_c) x B fp64 vec'd coefficients, Y (m_r m_c) x B
    fp32 vec'd measurements), column-major vec."""
    Ar = np.zeros((m_r, n_r), np.float32)
    Ac = np.zeros((m_c, n_c), np.float32)
    S = np.zeros((n_r * n_c, batch), np.float64)
    Y = np.zeros((m_r * m_c, batch), np.float32)
    code = lib().cl_gen_problem_2d(seed, n_r, n_c, m_r, m_c, k, batch, _ptr(Ar), _ptr(Ac),
                                   _ptr(S), _ptr(Y))
    if code:
        raise DimensionError("gen_problem_2d: bad sizes")
    return Ar, Ac, S, Y


# BASELINE.json configs.  lr / epochs for configs 2-5 are not
# stated there; config 1's are used and recorded.
def dct_basis(n: int) -> np.ndarray:
    """dct_basis (sensing.cpp:13-29): the orthonormal DCT-II synthesis matrix
    D (n x n, x = D s) of make_setup problems, for ClompContext.set_basis."""
    D = np.zeros((n, n), np.float64)
    _raise(lib().cl_dct_basis(int(n), _ptr(D)))
    return D


