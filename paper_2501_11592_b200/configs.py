"""Pure-Python pieces of the host mirror that load no native code: the
cskit::ClompConfig mirror (clomp.hpp:16-33), its C layout (cl_config in
include/clomp_b200.h) and the BASELINE.json workloads.  bench.py's reference
arm and the test-side checkers import only this module, never the CUDA
library."""
from __future__ import annotations

import ctypes as C
import dataclasses

PLAIN, MOMENTUM, ADAM = 0, 1, 2


class CConfig(C.Structure):
    """cl_config (include/clomp_b200.h), same layout as orc_config."""

    _fields_ = [
        ("th", C.c_double),
        ("max_outer", C.c_uint64),
        ("eps", C.c_double),
        ("inner_steps", C.c_uint64),
        ("lr", C.c_double),
        ("opt", C.c_int32),
        ("pad0", C.c_int32),
        ("w_tv", C.c_double),
        ("w_lv", C.c_double),
        ("lv_window", C.c_uint64),
        ("lv_stride", C.c_uint64),
        ("stall_tol", C.c_double),
        ("stall_patience", C.c_uint64),
    ]



@dataclasses.dataclass
class ClompConfig:
    """cskit::ClompConfig with the reference defaults (clomp.hpp:16-33)."""

    th: float = 0.7
    max_outer: int = 200
    eps: float = 1e-6
    inner_steps: int = 50
    lr: float = 0.01
    opt: int = ADAM
    w_tv: float = -1.0
    w_lv: float = -1.0
    lv_window: int = 3
    lv_stride: int = 2
    stall_tol: float = 1e-4
    stall_patience: int = 2

    @classmethod
    def baseline(cls, k: int, lr: float = 0.1, epochs: int = 200) -> "ClompConfig":
        """BASELINE.json mapping: sparsity K -> th=1,
        max_outer=K; plain gradient descent; priors off."""
        return cls(th=1.0, max_outer=k, inner_steps=epochs, lr=lr, opt=PLAIN,
                   w_tv=0.0, w_lv=0.0)

    def to_c(self) -> CConfig:
        def u64(v):
            return max(0, int(v)) if int(v) >= 0 else 0
        return CConfig(float(self.th), u64(self.max_outer), float(self.eps),
                       u64(self.inner_steps), float(self.lr), int(self.opt), 0,
                       float(self.w_tv), float(self.w_lv), u64(self.lv_window),
                       u64(self.lv_stride), float(self.stall_tol),
                       u64(self.stall_patience))


# BASELINE.json configs (DESIGN.md §5 for the seeds and value laws).
CONFIGS = {
    1: dict(name="cfg1_1d_single", m=128, n=256, k=10, batch=1, value_law=0, snr_db=-1.0, seed=0),
    2: dict(name="cfg2_1d_batched", m=512, n=1024, k=32, batch=4096, value_law=0, snr_db=40.0, seed=1),
    3: dict(name="cfg3_1d_long", m=4096, n=16384, k=256, batch=256, value_law=1, snr_db=-1.0, seed=2),
    4: dict(name="cfg4_2d_sep", n_r=256, n_c=256, m_r=128, m_c=128, k=1500, batch=64, seed=3),
    5: dict(name="cfg5_2d_sweep_r025", n_r=512, n_c=512, m_r=128, m_c=128, k=13107, batch=1024, seed=4),
    6: dict(name="cfg5_2d_sweep_r05", n_r=512, n_c=512, m_r=256, m_c=256, k=13107, batch=1024, seed=5),
    # config 3's dictionary solved one signal at a time (the CLI's per-signal
    # clomp_solve loop, cskit.cpp:543-551): the correlation is the B = 1 GEMV
    7: dict(name="cfg3_1d_long_single", m=4096, n=16384, k=256, batch=1, value_law=1, snr_db=-1.0, seed=2),
}
