"""Throughput of S independent contexts solving B/S signals each on S streams
concurrently (host threads), vs one context with all B: is there idle GPU
time that concurrent half-batches would fill?   python tools/probe_streams.py"""
import ctypes as C
import sys
import threading
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2501_11592_b200 as cl  # noqa: E402

c = cl.CONFIGS[2]
A, X, Y, _ = cl.gen_problem_1d(c["seed"], c["m"], c["n"], c["k"], c["batch"], snr_db=40.0)
cfg = cl.ClompConfig.baseline(c["k"])
ccfg = cfg.to_c()
dev = torch.device("cuda", 0)
B = c["batch"]


def make(S):
    jobs = []
    for s in range(S):
        lo, hi = s * B // S, (s + 1) * B // S
        ctx = cl.ClompContext(A)
        st = torch.cuda.Stream(device=dev)
        ctx.set_stream(st.cuda_stream)
        n = hi - lo
        dy = torch.from_numpy(np.ascontiguousarray(Y[:, lo:hi].T)).to(dev)
        cap = min(c["n"], c["k"] + 16)
        outs = [torch.zeros(n * cap, dtype=torch.int32, device=dev),
                torch.zeros(n * cap, dtype=torch.float64, device=dev),
                torch.zeros(n, dtype=torch.int32, device=dev),
                torch.zeros(n, dtype=torch.int32, device=dev),
                torch.zeros(n, dtype=torch.float64, device=dev),
                torch.zeros(n, dtype=torch.uint8, device=dev),
                torch.zeros(n, dtype=torch.int32, device=dev)]
        res = cl.CDeviceResult(cap, *[o.data_ptr() for o in outs])
        jobs.append((ctx, st, dy, n, res, outs))
    return jobs


def run(jobs):
    def one(j):
        ctx, st, dy, n, res, _ = j
        code = cl.lib().cl_solve_batch_device(ctx.handle, C.c_void_p(dy.data_ptr()), n,
                                              C.byref(ccfg), cl.MODE_PER_SIGNAL, C.byref(res))
        assert code == 0, code
    ts = [threading.Thread(target=one, args=(j,)) for j in jobs]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    torch.cuda.synchronize()


for S in (1, 2, 4):
    jobs = make(S)
    for _ in range(3):
        run(jobs)
    t0 = time.perf_counter()
    R = 10
    for _ in range(R):
        run(jobs)
    dt = (time.perf_counter() - t0) / R
    print(f"S={S}: {dt * 1e3:.3f} ms per {B} signals -> {B / dt:.0f} signals/s (wall)")
