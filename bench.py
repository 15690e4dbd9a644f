#!/usr/bin/env python
"""bench.py — CLOMP reconstruction throughput on B200.

Metric (BASELINE.json): signals reconstructed per second at fixed (N, M, K),
plus the roofline fraction of the correlation kernel.  Default workload is
BASELINE config 2 (configs[1]): N=1024, M=512, K=32, 4096 signals per GPU,
40 dB, lr 0.1, 200 epochs, th=1 / max_outer=K / plain GD / priors off
(SURVEY.md §8d mapping).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 1..7] [--colshard] [--max-outer T]
    torchrun --nproc-per-node N bench.py --gpus N ...

A step = one full CLOMP solve (K outer iterations x 200 epochs) of one batch
already resident in HBM.  Multi-GPU: by default every rank solves its own
batch (per-signal semantics: no data-path collective; scaling "weak");
--colshard (config 3) shards one dictionary by columns over the ranks with
NCCL exchanges and solves one batch together (scaling "strong").  Configs 4-6
(separable 2D) are timed on a truncated prefix (--max-outer, default 64; the
full K = 1500 / 13107 outer iterations take minutes to hours per batch).

--impl reference times the unmodified reference library (oracle/_ref,
compiled from /root/reference/proj/src) on the host cores: P single-threaded
workers (the library has no threads), each solving a contiguous chunk of 8
signals with clomp_solve_batch (its AVX2 4x8 GEMM tile path).  For config 3
the reference needs ~25 min per signal per core, so each worker times 2 outer
iterations and the figure is extrapolated (the reference's cost per outer
iteration does not depend on the support size, clomp.cpp:84-89, 237-245).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "signals reconstructed/sec at fixed (N,M,K)"
UNIT = "signals/s"
CHUNK = 8  # signals per reference worker call (AVX2 tile width)
# the arithmetic the path computes in: fp32 operands (A, y), the batched
# correlation as a split-fp16 tcgen05 GEMM (three f16 MMAs, fp32 TMEM
# accumulation) with fp64 rescoring of near-tied selections, every learning
# product, residual and reduction in fp64
DTYPE = "f32 operands; 3xf16 tcgen05 correlation + f64 rescoring; f64 learning"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--colshard", action="store_true")
    ap.add_argument("--vshards", type=int, default=4,
                    help="--colshard on one GPU: virtual column shards (the NCCL path's kernels "
                         "and exchanges, one device)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: every rank solves its own batch of the config's size; strong: "
                         "the config's batch is split across the ranks")
    ap.add_argument("--max-outer", type=int, default=0,
                    help="outer iterations (0: K for the 1D configs, a 64-iteration prefix for the "
                         "2D ones; -1: the config's full K)")
    ap.add_argument("--batch", type=int, default=0,
                    help="time-box a heavy config on fewer signals / images than it names")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--corr-path", type=int, default=0, help="0 auto, 1 fp64 SIMT, 2 tcgen05, 3 GEMV")
    ap.add_argument("--power-levels", type=int, default=-1,
                    help="plain GD on cluster-sized supports: squaring levels (-1 auto, 0 off)")
    return ap.parse_args()


def workload(args, rank: int, world: int = 1):
    from paper_2501_11592_b200.configs import CONFIGS

    c = dict(CONFIGS[args.config])
    c["sep"] = "n_r" in c
    if args.batch:
        c["batch"] = args.batch
    if c["sep"]:
        c["n"], c["m"] = c["n_r"] * c["n_c"], c["m_r"] * c["m_c"]
        c["max_outer"] = c["k"] if args.max_outer < 0 else (args.max_outer or 64)
    else:
        c["max_outer"] = c["k"] if args.max_outer < 0 else (args.max_outer or c["k"])
    c["sig_lo"], c["sig_hi"] = 0, c["batch"]
    if args.colshard:
        pass  # one batch solved together by all ranks
    elif args.scaling == "strong":
        # strong scaling: the config's batch is the GLOBAL batch (config 5:
        # "batch 1024 sharded by image across 1/2/4/8 GPUs"); every rank draws
        # the same problem and solves its contiguous slice of the signals
        from paper_2501_11592_b200.sharding import shard_range

        c["sig_lo"], c["sig_hi"] = shard_range(c["batch"], rank, world)
    else:
        c["seed"] = c["seed"] + 1000 * rank  # weak scaling: each rank its own batch
    return c


def make_problem(c):
    import paper_2501_11592_b200 as cl

    if c["sep"]:
        Ar, Ac, X, Y = cl.gen_problem_2d(c["seed"], c["n_r"], c["n_c"], c["m_r"], c["m_c"],
                                         c["k"], c["batch"])
        return (Ar, Ac), X, Y
    A, X, Y, _ = cl.gen_problem_1d(c["seed"], c["m"], c["n"], c["k"], c["batch"],
                                   value_law=c["value_law"], snr_db=c["snr_db"])
    return A, X, Y


def solver_config(c):
    from paper_2501_11592_b200.configs import ClompConfig

    cfg = ClompConfig.baseline(c["k"])
    cfg.max_outer = c["max_outer"]
    return cfg


def config_block(c, n_gpus, mode):
    """mode: "weak" (a batch per GPU), "strong" (the batch split by signal),
    "colshard" (one batch, the dictionary split by atoms)."""
    if c["sep"]:
        shape = (f"{c['n_r']}x{c['n_c']} coefficients, {c['m_r']}x{c['m_c']} measurements, "
                 f"K={c['k']} (" + ("full solve" if c["max_outer"] >= c["k"] else
                                   f"prefix: {c['max_outer']} outer iterations") + ")")
    else:
        shape = f"N={c['n']} M={c['m']} K={c['k']}"
    noise = "" if c["sep"] or c["snr_db"] < 0 else f" {c['snr_db']} dB"
    weak = mode == "weak"
    return {
        "workload": f"{c['name']}: {shape} batch={c['batch']}{'/GPU' if weak else ''}{noise}",
        "n": c["n"], "m": c["m"], "k": c["k"],
        "batch_per_gpu": c["batch"] if weak else -(-c["batch"] // n_gpus),
        "global_batch": c["batch"] * (n_gpus if weak else 1), "lr": 0.1, "epochs": 200,
        "th": 1.0, "max_outer": c["max_outer"], "optimizer": "plain", "priors": "off",
        "mode": "per_signal (clomp_solve per column)", "seed": c["seed"],
        "parallelism": {"weak": f"signal-shard x{n_gpus} (a batch per GPU), no collectives",
                        "strong": f"signal-shard x{n_gpus} (one batch split), no collectives",
                        "colshard": f"column-shard x{n_gpus} (NCCL all-gathers)"}[mode],
        "l2": "flushed between timed steps (256 MiB write)",
    }


# ----------------------------------------------------------- reference arm
# The reference arm and the cpu_baseline leg run the UNMODIFIED reference
# library (oracle/_ref/libcskit_ref.so) in P spawned single-threaded worker
# processes, one pinned per host core.  Each worker draws the workload itself
# with the reference's own cskit::Rng (refbind.ref_gen_problem_1d, the same
# bits as the product's generator: tests/test_datagen.py), so no process of
# this arm loads the B200 library.
_W = {}


def _ref_init(core_counter, gen_args):
    import multiprocessing as mp  # noqa: F401

    with core_counter.get_lock():
        idx = core_counter.value
        core_counter.value += 1
    try:
        cores = sorted(os.sched_getaffinity(0))
        os.sched_setaffinity(0, {cores[idx % len(cores)]})
    except Exception:
        pass
    sys.path.insert(0, str(ROOT / "tests"))
    import refbind

    seed, m, n, k, batch, law, snr = gen_args
    A, _, Y = refbind.ref_gen_problem_1d(seed, m, n, k, batch, value_law=law, snr_db=snr,
                                         want_x=False)
    _W["A"] = A.astype(np.float64)
    _W["Y"] = Y.astype(np.float64)
    _W["refbind"] = refbind


def _ref_task(job):
    lo, cfgd = job
    from paper_2501_11592_b200.configs import ClompConfig

    refbind = _W["refbind"]
    Y = _W["Y"]
    B = Y.shape[1]
    chunk = np.ascontiguousarray(Y[:, lo % B:lo % B + CHUNK])
    t0 = time.perf_counter()
    r = refbind.ref_solve_batch(_W["A"], chunk, ClompConfig(**cfgd))
    return time.perf_counter() - t0, r["code"], chunk.shape[1]


class ReferencePool:
    """P spawned reference workers holding the workload (generated once)."""

    def __init__(self, c, workers: int):
        import multiprocessing as mp

        ctx = mp.get_context("spawn")
        self.workers = workers
        counter = ctx.Value("i", 0)
        gen = (c["seed"], c["m"], c["n"], c["k"], c["batch"], c["value_law"], c["snr_db"])
        self.pool = ctx.Pool(workers, initializer=_ref_init, initargs=(counter, gen))
        # every worker has generated its inputs before the first timed round
        self.pool.map(_ref_noop, range(4 * workers), chunksize=1)

    def round(self, cfg, workers: int, scale: float = 0.0):
        """One bounded sample: `workers` tasks x CHUNK signals in parallel.
        With scale, the sample is a truncated solve (reference_plan) and its
        wall time is multiplied by scale to extrapolate to the full one."""
        import dataclasses

        cfgd = dataclasses.asdict(cfg)
        jobs = [(w * CHUNK, cfgd) for w in range(workers)]
        t0 = time.perf_counter()
        res = self.pool.map(_ref_task, jobs, chunksize=1)
        wall = time.perf_counter() - t0
        if any(code != 0 for _, code, _ in res):
            raise RuntimeError("reference solve failed")
        sig = sum(n for _, _, n in res)
        if scale:
            wall = wall * scale
        return sig / wall, wall, sig

    def close(self):
        self.pool.close()
        self.pool.join()


def _ref_noop(_):
    return os.getpid()


def cpu_info():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def host_workers():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def reference_plan(c):
    """(config for the timed sample, wall-time scale factor or 0, note).

    The reference's cost per outer iteration does not depend on the support
    (every product is dense over N: clomp.cpp:84, 89, 237, 245) and is
    2*inner_steps + 3 dense products (residual, correlation, inner_steps x
    (forward, transposed), final loss), so truncated samples extrapolate
    linearly."""
    cfg = solver_config(c)
    if c["n"] * c["m"] > 4_000_000 and c["batch"] == 1:
        # one signal per worker: ~100 s per full outer iteration per core, so
        # time one outer iteration with 8 inner steps
        full_outer, full_inner = cfg.max_outer, cfg.inner_steps
        cfg.max_outer, cfg.inner_steps = 1, 8
        scale = full_outer * (2 * full_inner + 3) / (2 * cfg.inner_steps + 3)
        return cfg, scale, (f"1 outer iteration with 8 inner steps timed, extrapolated "
                            f"x{scale:.0f} (cost per outer iteration = 2*inner+3 dense products)")
    if c["n"] * c["m"] > 4_000_000:  # config 3: time 2 outer iterations per worker
        full = cfg.max_outer
        cfg.max_outer = 2
        return cfg, full / 2, f"2 outer iterations timed, extrapolated x{full / 2:.0f}"
    return cfg, 0, "full solves"


def run_reference(args, rank, world):
    if rank != 0:
        return  # torchrun: rank 0 alone times the host cores
    sys.path.insert(0, str(ROOT / "tests"))
    import refbind

    c = workload(args, 0)
    if c["sep"]:
        print(json.dumps({"impl": "reference", "unavailable":
                          "the reference has no separable mode; its explicit Kronecker matrix "
                          "(8.6-137 GB fp64) does not fit the workers"}))
        return
    if not refbind.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libcskit_ref.so not built"}))
        return
    cfg, extra, note = reference_plan(c)
    P = host_workers()
    pool = ReferencePool(c, P)
    for _ in range(args.warmup):
        pool.round(cfg, min(P, 2), extra)
    vals, walls = [], []
    sig = 0
    for _ in range(args.steps):
        v, wall, sig = pool.round(cfg, P, extra)
        vals.append(v)
        walls.append(wall)
    pool.close()
    value = statistics.mean(vals)
    sample = (f"{P} workers x {CHUNK} signals per step (clomp_solve_batch, AVX2), {sig} "
              f"signals/step, {note}")
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * statistics.mean(walls), "higher_is_better": True,
        "scaling": "strong" if args.colshard or args.scaling == "strong" else "weak",
        "vs_baseline": None, "dtype": "f64 (the reference computes in double)",
        "data": "synthetic (seeded cskit::Rng, BASELINE config laws)",
        "config": config_block(c, world, "colshard" if args.colshard else args.scaling),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": P, "kind": "reference",
                         "sample": sample, "cpu": cpu_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))


# ------------------------------------------------------------------ clocks
class NvmlClockSampler:
    """Polls SM clocks and clock-event reasons through NVML from a thread for
    the duration of the timed region (a config-2 step is ~2 ms, far shorter than
    nvidia-smi's sampling period, so the subprocess sampler saw nothing)."""

    NAMES = [("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
             ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
             ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
             ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
             ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown")]

    def __init__(self, device: int):
        import threading
        import pynvml as nv
        import torch

        self.nv = nv
        nv.nvmlInit()
        pr = torch.cuda.get_device_properties(device)
        try:
            bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
            self.h = nv.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            self.h = nv.nvmlDeviceGetHandleByIndex(device)
        self.smax = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        self.samples = []  # (t, sm_mhz, reasons bitmask)
        self.stop_flag = False
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        nv = self.nv
        while not self.stop_flag:
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((time.perf_counter(), sm, rs))
            except Exception:
                pass
            time.sleep(0.0005)

    def stop(self, t0: float, t1: float):
        self.stop_flag = True
        self.t.join()
        inside = [s for s in self.samples if t0 <= s[0] <= t1]
        used = inside or self.samples
        reasons = set()
        for _, _, rs in used:
            for name, attr in self.NAMES:
                if rs & getattr(self.nv, attr, 0):
                    reasons.add(name)
        sm = [s[1] for s in used]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.smax,
                "reasons": sorted(reasons), "samples": len(inside),
                "source": "NVML polled every ~0.5 ms during the timed region"
                          + ("" if inside else " (no sample inside it: whole-run samples)")}


def clock_sampler(device: int):
    try:
        return NvmlClockSampler(device)
    except Exception:
        return ClockSampler(device)


class ClockSampler:
    def __init__(self, index: int):
        self.path = Path(f"/tmp/bench_clocks_{os.getpid()}.csv")
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self, t0: float = 0.0, t1: float = 0.0):
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.path.read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def max_over_ranks(values, device, dist_on: bool):
    """Element-wise maximum of per-rank timings (ms) over the process group
    (NCCL on the GPUs, gloo in the CPU tests): the job is as slow as its
    slowest rank."""
    import torch

    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist_on:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return [float(v) for v in t.cpu()]


def job_throughput(c, batch_local: int, world: int, strong: bool, ms_max: float) -> float:
    """Whole-job signals/s: all ranks' signals over the slowest rank's time."""
    total = c["batch"] if strong else batch_local * world
    return total / (ms_max / 1000.0)


# ---------------------------------------------------------------- our arm
def run_ours(args, rank, world, local_rank):
    import ctypes as C
    import torch
    import paper_2501_11592_b200 as cl

    dist = world > 1
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    c = workload(args, rank, world)
    A, X, Y = make_problem(c)
    if (c["sig_lo"], c["sig_hi"]) != (0, c["batch"]):
        Y = np.ascontiguousarray(Y[:, c["sig_lo"]:c["sig_hi"]])
    B, m, n = Y.shape[1], c["m"], c["n"]
    if B == 0:
        raise SystemExit("strong scaling: more ranks than signals")
    cfg = solver_config(c)
    if c["sep"]:
        ctx = cl.ClompContext.separable(A[0], A[1], device=local_rank)
    elif args.colshard and dist:
        nid = [cl.nccl_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(nid, src=0)
        ctx = cl.ClompContext.colshard(A, rank, world, nid[0], device=local_rank)
    else:
        ctx = cl.ClompContext(A, device=local_rank)
        if args.colshard:  # one GPU: the column-shard code path with virtual shards
            ctx.set_virtual_shards(args.vshards)
    if args.corr_path:
        ctx.set_corr_path(args.corr_path)
    if args.power_levels != -1 and not c["sep"]:
        ctx.set_power_levels(args.power_levels)
    stream = torch.cuda.Stream(device=dev)
    ctx.set_stream(stream.cuda_stream)
    d_y = torch.from_numpy(np.ascontiguousarray(Y.T)).to(dev)  # signal-major B x m
    cap = min(n, c["max_outer"] + 16)
    o_sup = torch.zeros((B, cap), dtype=torch.int32, device=dev)
    o_coef = torch.zeros((B, cap), dtype=torch.float64, device=dev)
    o_cnt = torch.zeros(B, dtype=torch.int32, device=dev)
    o_it = torch.zeros(B, dtype=torch.int32, device=dev)
    o_rn = torch.zeros(B, dtype=torch.float64, device=dev)
    o_cv = torch.zeros(B, dtype=torch.uint8, device=dev)
    o_st = torch.zeros(B, dtype=torch.int32, device=dev)
    dres = cl.CDeviceResult(cap, o_sup.data_ptr(), o_coef.data_ptr(), o_cnt.data_ptr(),
                            o_it.data_ptr(), o_rn.data_ptr(), o_cv.data_ptr(), o_st.data_ptr())
    ccfg = cfg.to_c()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def step():
        code = cl.lib().cl_solve_batch_device(ctx.handle, C.c_void_p(d_y.data_ptr()), B,
                                              C.byref(ccfg), cl.MODE_PER_SIGNAL, C.byref(dres))
        if code:
            cl._raise(code, ctx.handle)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    assert int(o_st.max()) == 0, "solve reported a failing signal"
    launches_per_step = ctx.stats()["kernel_launches"]

    if dist:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    sampler = clock_sampler(local_rank)
    time.sleep(0.01)
    evs = []
    t_region0 = time.perf_counter()
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    t_region1 = time.perf_counter()
    if dist:
        torch.distributed.barrier()
    clocks = sampler.stop(t_region0, t_region1)
    times = [a.elapsed_time(b) for a, b in evs]
    ms = statistics.mean(times)
    ms_max = max_over_ranks([ms], dev, dist)[0]
    strong = args.colshard or args.scaling == "strong"
    total_signals = c["batch"] if strong else B * world
    value = job_throughput(c, B, world, strong, ms_max)

    # Per-phase breakdown of one solve (profiling events, outside the timed region).
    prof = None
    if not args.colshard:
        ctx.set_profiling(True)
        with torch.cuda.stream(stream):
            flush.fill_(2)
        step()
        torch.cuda.synchronize()
        prof = ctx.stats()
        ctx.set_profiling(False)

    # End to end through the public API: every step's y comes from pinned host
    # memory and its compact per-signal results (supports, coefficients, norms,
    # flags) land back in host memory.  Pipelined (clomp_submit / clomp_wait,
    # two batches in flight): step i + 1's upload and step i's download run on
    # copy streams under the other step's solve; the L2 flush is queued on the
    # solve stream before every step, inside the timed region.  Host wall clock
    # over the whole K-step region / K.  The blocking single call is reported
    # beside it (e2e.blocking_call).
    n_rot = 3
    Y_pins = []
    for i in range(n_rot):
        yp = torch.empty(Y.shape, dtype=torch.float32, pin_memory=True).numpy()
        yp[...] = Y
        Y_pins.append(yp)
    for _ in range(max(args.warmup, 3)):  # warm-up (graphs, pinned staging, host pages)
        cl.clomp_solve_batch(ctx, Y_pins[0], cfg, mode=cl.MODE_PER_SIGNAL, dense=False)
    e2e_ms = []
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(3)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = cl.clomp_solve_batch(ctx, Y_pins[0], cfg, mode=cl.MODE_PER_SIGNAL, dense=False)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        st = ctx.stats()
    assert np.all(r.status == 0)
    blocking_ms = statistics.mean(e2e_ms)

    def flush_step(i):
        with torch.cuda.stream(stream):
            flush.fill_(3)
        cl.clomp_submit(ctx, Y_pins[i % n_rot], cfg, mode=cl.MODE_PER_SIGNAL, dense=False)

    for rep in range(2):  # rep 0: warm-up of the pipelined loop
        if dist:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        flush_step(0)
        for i in range(1, args.steps):
            flush_step(i)
            r = cl.clomp_wait(ctx)
            assert r.status.max() == 0
        r = cl.clomp_wait(ctx)
        assert r.status.max() == 0
        pipe_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    te = max_over_ranks([pipe_ms, blocking_ms], dev, dist)
    e2e_val = total_signals / (te[0] / 1000.0)
    e2e_blocking = total_signals / (te[1] / 1000.0)

    # One-off context cost (dictionary transpose + upload, fp16 split, A^T A).
    t0 = time.perf_counter()
    if c["sep"]:
        ctx2 = cl.ClompContext.separable(A[0], A[1], device=local_rank)
    else:
        ctx2 = cl.ClompContext(A, device=local_rank)
    create_ms = (time.perf_counter() - t0) * 1e3
    ctx2.close()

    if rank != 0:
        return
    peaks = {}
    pk = ROOT / "MEASURED_PEAKS.json"
    if pk.exists():
        peaks = json.loads(pk.read_text())
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max,
        "higher_is_better": True, "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": DTYPE,
        "data": "synthetic (seeded cskit::Rng restatement, BASELINE config laws)",
        "config": config_block(c, world, "colshard" if args.colshard else args.scaling),
    }
    if prof and prof["corr_path"] == 3 and not c["sep"]:
        # K1b GEMV: HBM-bound; algorithmic bytes per launch = the fp32
        # dictionary (n x ldm) + the fp64 residuals read + 32-byte candidate
        # records written.
        outers = max(prof["outer_iterations"], 1)
        ldm = (m + 127) // 128 * 128
        gemv_bytes = 4.0 * n * ldm + 8.0 * B * ldm + 32.0 * B * ((n + 63) // 64)
        t_launch = prof["corr_ms"] / outers
        achieved = gemv_bytes / (t_launch / 1000.0) / 1e9
        peak = peaks.get("hbm_gbs", 7700.0)
        out["roofline"] = {
            "kernel": "K1b correlation GEMV A^T r + top-2 epilogue (k_corr_gemv)",
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": None,
            "peak_source": ("MEASURED_PEAKS.json hbm_gbs (copy bandwidth)" if "hbm_gbs" in peaks
                            else "fallback 7700 GB/s (B200_PROFILING.md)"),
            "algorithmic_per_launch": f"4*n*ldm + 8*B*ldm + 32*B*tiles = {gemv_bytes:.4e} B",
            "avg_launch_ms": t_launch,
            "phase_ms_per_step": {"corr": prof["corr_ms"], "select_rescan": prof["select_ms"],
                                  "learn_residual": prof["learn_ms"], "total": prof["total_ms"]},
            "note": "phase times come from a separately profiled solve (per-iteration sync)",
        }
    if prof and prof["corr_path"] in (0, 1) and not c["sep"]:
        outers = max(prof["outer_iterations"], 1)
        corr_flops = 2.0 * n * m * B  # one launch: A^T R over the batch
        corr_ms_launch = prof["corr_ms"] / outers
        if prof["corr_path"] == 1:
            # split fp16 (3 f16 MMAs per product, fp32 accumulation): the useful
            # rate is compared with the measured dense bf16/f16 peak / 3.
            # A K1 launch is ~20 us inside a ~2 ms step (config 2), far too
            # short to heat the part: the burst figure applies.
            dense = peaks.get("bf16_tflops", 1590.0)
            peak = dense / 3.0
            bound, punit = "tensor", "TFLOP/s (fp32-equivalent, 3 x f16 MMA)"
            peak_src = ("MEASURED_PEAKS.json bf16_tflops (burst dense bf16 = f16 rate) / 3, derived"
                        if "bf16_tflops" in peaks else "fallback 1590 TFLOP/s / 3")
        else:
            clk = (clocks.get("sm_mhz") or 1965.0) * 1e6
            peak = 148 * 64 * 2 * clk / 1e12
            bound, punit = "fp64", "TFLOP/s"
            peak_src = "derived fp64 pipe: 148 SM x 64 DFMA/clk x 2 x measured SM clock"
        achieved = corr_flops / (corr_ms_launch / 1000.0) / 1e12
        out["roofline"] = {
            "kernel": "K1 correlation A^T R + top-2 epilogue (k_corr_tc)",
            "bound": bound, "achieved": achieved, "peak": peak, "unit": punit,
            "frac": achieved / peak,
            "traffic": 10.57e6 if prof["corr_path"] == 1 and args.config == 2 else None,
            "traffic_note": ("ncu dram__bytes_read+write per launch (10.57 MB read, 0 written; "
                             "algorithmic 10.49 MB), profiles/r2/final/k1.summary.txt"
                             if prof["corr_path"] == 1 and args.config == 2 else None),
            "peak_source": peak_src,
            "algorithmic_per_launch": f"2*N*M*B = {corr_flops:.3e} FLOP",
            "avg_launch_ms": corr_ms_launch,
            "phase_ms_per_step": {"corr": prof["corr_ms"], "select_rescan": prof["select_ms"],
                                  "learn_residual": prof["learn_ms"], "total": prof["total_ms"]},
            "rescans_per_step": prof["rescans"],
            "note": ("phase times come from a separately profiled solve (per-iteration sync); "
                     "the learning kernels (fp64 pipe / shared-memory bound) are the largest share, "
                     "see DESIGN.md §4"),
        }
    # The learning phase (selection, Gram extension, epochs, residual, stopping
    # rules) is the larger share of a 1D step: report it as the dominant
    # kernel's roofline when it is, the correlation kernel's beside it.
    if prof and "roofline" in out and not c["sep"]:
        outers = max(prof["outer_iterations"], 1)
        E = cfg.inner_steps
        # algorithmic work of the learning phase, Gram form:
        # per signal and outer iteration t, E epochs of the t x t system
        # (2 E t^2) and the residual A_S c - y (2 m t); th = 1 adds one atom per
        # iteration, so t = 1 .. outers.
        ts = np.arange(1, outers + 1, dtype=np.float64)
        learn_flops = B * float(np.sum(2.0 * E * ts ** 2 + 2.0 * m * ts))
        learn_ms = prof["learn_ms"] + prof["select_ms"]
        clk = (clocks.get("sm_mhz") or 1965.0) * 1e6
        fp64_peak = 148 * 64 * 2 * clk / 1e12
        learn_roof = {
            "kernel": "learning phase (k_learn_fast / k_learn_warp / k_learn_cluster + residual)",
            "bound": "fp64", "achieved": learn_flops / (learn_ms / 1e3) / 1e12,
            "peak": fp64_peak, "unit": "TFLOP/s",
            "frac": learn_flops / (learn_ms / 1e3) / 1e12 / fp64_peak,
            "traffic": 52.82e6 if args.config == 2 and prof["corr_path"] == 1 else None,
            "traffic_note": ("ncu dram__bytes_read+write per launch of k_learn_fast<32,0,1> at t = 30 "
                             "(the largest learning launches, t = 17..32: 51.5 MB read, 1.4 MB "
                             "written: the support Gram rows, per-signal state and y; the atom "
                             "gathers of the residual are L2 hits), profiles/r2/final/learn32.summary.txt"),
            "peak_source": "derived fp64 pipe: 148 SM x 64 DFMA/clk x 2 x SM clock under load",
            "algorithmic_per_step": (f"B * sum_t (2 E t^2 + 2 m t), t = 1..{outers}, E = {E} "
                                     f"= {learn_flops:.4e} FLOP"),
            "ms_per_step": learn_ms,
            "share_of_profiled_step": learn_ms / max(prof["total_ms"], 1e-9),
            "note": ("Gram-form work (what the reference's dense epochs reduce to); the kernels "
                     "run the power form, which executes about half of these FLOPs at t = 32 "
                     "(4 DMMA squarings + 21 matvecs), so the executed-FLOP pipe use is lower"),
        }
        corr_ms = prof["corr_ms"]
        if learn_ms > corr_ms:
            out["roofline_corr"] = out["roofline"]
            out["roofline"] = learn_roof
        else:
            out["roofline_learn"] = learn_roof
    out["e2e"] = {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": st["h2d_bytes"],
                  "d2h_bytes_per_step": st["d2h_bytes"],
                  "path": ("clomp_submit / clomp_wait (dense=False), two batches in flight: every "
                           "step's y from pinned host memory, compact results (supports, "
                           "coefficients, norms, flags) to host, L2 flush queued before every "
                           "step; host wall clock over the K-step region / K"),
                  "blocking_call": {"value": e2e_blocking, "unit": UNIT,
                                    "path": "one clomp_solve_batch call at a time, host wall clock around it"}}
    out["setup"] = {"cl_create_ms": create_ms,
                    "note": "one-off per dictionary (host transpose, upload, fp16 split, A^T A); outside every timed region"}
    # The drop-in boundary itself: cskit::clomp_solve_batch (the reference's C++
    # signature, joint semantics, fp64 host buffers, dense s / mask / x_hat back)
    # served by the C++ shim, timed by a prebuilt binary at this config's shape.
    shim_bin = ROOT / "paper_2501_11592_b200" / "_build" / "shim_bench"
    if world == 1 and shim_bin.exists() and args.config in (1, 2) and not args.colshard:
        try:
            ctx.close()  # free this process's copy before the binary runs on the same GPU
            lines = []
            for ident in (0, 1):
                rr = subprocess.run([str(shim_bin), str(n), str(c["batch"]), str(c["k"]), "5", str(ident)],
                                    capture_output=True, text=True, timeout=300)
                lines.append(json.loads(rr.stdout.strip().splitlines()[-1]))
            out["shim"] = lines
        except Exception as exc:  # the boundary timing is supplementary
            out["shim"] = {"unavailable": repr(exc)[:200]}
    out["gpu_launches"] = int(launches_per_step * args.steps)
    out["clocks"] = clocks
    if world == 1 and not args.no_cpu_baseline and not c["sep"]:
        sys.path.insert(0, str(ROOT / "tests"))
        import refbind
        if refbind.ref_available():
            P = host_workers()
            rcfg, extra, note = reference_plan(c)
            pool = ReferencePool(c, P)
            v, wall, sig = pool.round(rcfg, P, extra)
            pool.close()
            out["cpu_baseline"] = {
                "value": v, "unit": UNIT, "cores": P, "kind": "reference",
                "sample": f"{P} workers x {CHUNK} signals of this workload, one round ({note})",
                "cpu": cpu_info()}
    print(json.dumps(out))


def self_launch(args) -> bool:
    """`bench.py --gpus N` outside torchrun: start the N ranks ourselves (one
    process per GPU, the same torchrun command line the driver uses)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve())] + sys.argv[1:]
    raise SystemExit(subprocess.call(cmd))


def main():
    args = parse()
    self_launch(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.colshard and args.config != 3:
        raise SystemExit("--colshard applies to config 3 (one large dictionary)")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl")
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
