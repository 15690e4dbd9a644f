"""Where the e2e time of config 2 goes: public call (pinned y, compact results)
vs the device-resident call vs the raw copies, all without an L2 flush."""
import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import ctypes as C, time, numpy as np, torch
import paper_2501_11592_b200 as cl
c = cl.CONFIGS[2]
A, X, Y, _ = cl.gen_problem_1d(1, c["m"], c["n"], c["k"], c["batch"], snr_db=40.0)
ctx = cl.ClompContext(A)
cfg = cl.ClompConfig.baseline(c["k"])
B = Y.shape[1]
Yp = torch.empty(Y.shape, dtype=torch.float32, pin_memory=True).numpy(); Yp[...] = Y
for i in range(6):
    t0 = time.perf_counter()
    r = cl.clomp_solve_batch(ctx, Yp, cfg, mode=cl.MODE_PER_SIGNAL, dense=False)
    t1 = time.perf_counter()
    print(i, "public wall ms %.3f" % ((t1 - t0) * 1e3), "lib e2e ms %.3f" % ctx.stats()["e2e_ms"])
dev = torch.device("cuda:0")
# (cl_solve_batch_device takes signal-major B x m y only)
for lay, d_y in (("signal-major", torch.from_numpy(np.ascontiguousarray(Y.T)).to(dev)),):
    cap = min(c["n"], c["k"] + 16)
    o = [torch.zeros((B, cap), dtype=torch.int32, device=dev), torch.zeros((B, cap), dtype=torch.float64, device=dev)]
    o += [torch.zeros(B, dtype=t, device=dev) for t in (torch.int32, torch.int32, torch.float64, torch.uint8, torch.int32)]
    dres = cl.CDeviceResult(cap, *[x.data_ptr() for x in o])
    ccfg = cfg.to_c()
    fn = cl.lib().cl_solve_batch_device
    for i in range(4):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter(); e0.record()
        code = fn(ctx.handle, C.c_void_p(d_y.data_ptr()), B, C.byref(ccfg), cl.MODE_PER_SIGNAL, C.byref(dres))
        e1.record(); torch.cuda.synchronize()
        print(lay, "device call: wall ms %.3f events ms %.3f" % ((time.perf_counter() - t0) * 1e3, e0.elapsed_time(e1)), code)
hy = torch.empty(Y.size, dtype=torch.float32, pin_memory=True); dy = torch.empty(Y.size, dtype=torch.float32, device=dev)
ho = torch.empty(2445312, dtype=torch.uint8, pin_memory=True); do = torch.empty(2445312, dtype=torch.uint8, device=dev)
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    dy.copy_(hy, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    ho.copy_(do, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
    print("raw H2D 8MiB ms %.3f  D2H 2.4MB ms %.3f" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3))
