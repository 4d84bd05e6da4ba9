"""Benchmark: shifted-system solves/s + Jacobian builds/s (FP64) on BASELINE configs[4]
(3-D THT Jacobian, 128^3 cells, 16 sources x 64 receivers, Talbot N=32, 4 times) on one B200.

One step = one full Jacobian build (ThtForwardModel::jacobian, jacobian.cpp:189-247):
device assembly of the pencil from the log fields, forward + adjoint FGMRES-Sh solves of
all 80 right-hand sides at each of the 4 times (5120 shifted-system solves), and the
kappa + storativity Jacobian slices (4096 x 2*2,097,152, left on the device per time
slice as SURVEY.md §8d defines a build), plus the 4096 predictions.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 4]

N > 1 (torchrun): every rank builds the Jacobian of its own field realisation (replicas of
the per-GPU workload, no data-path collective; scaling "weak"); value = all ranks' solves
/ max-over-ranks time.  --impl reference times the CPU oracle port (SciPy/SuperLU
restatement of the reference path; the C++ reference needs Eigen, absent) on a bounded
sample with all host cores.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "shifted-system solves/sec + Jacobian builds/sec (FP64), % HBM roofline"
PROFILE_EVERY = 8
UNIT = "shifted-system solves/s"


# FP64 mma.sync m8n8k4 throughput measured on this pool's B200 (scripts/micro/fp64_peak.cu)
FP64_DMMA_TFLOPS = 37.0


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled during the timed region through
    NVML (the library nvidia-smi uses), once every 4 s.  The solver issues many short host
    synchronisations; polling NVML every 200 ms (nvidia-smi -lms 200) stretched the step by
    ~50% and even 1 Hz by ~18%, so the period is 4 s (several samples per timed region)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, index: int, period: float = 4.0):
        self.index = index
        self.period = period
        self.samples = []
        self.stop_flag = threading.Event()
        self.thread = None
        self.error = None

    def start(self):
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _run(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while not self.stop_flag.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, mx, rs))
                self.stop_flag.wait(self.period)
            pynvml.nvmlShutdown()
        except Exception as exc:  # NVML unavailable
            self.error = str(exc)

    def stop(self):
        if self.thread is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["not sampled"]}
        self.stop_flag.set()
        self.thread.join(timeout=5)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [f"nvml unavailable: {self.error}"]}
        sm = [s[0] for s in self.samples]
        reasons = sorted({name for s in self.samples for name, bit in self.REASONS.items() if s[2] & bit})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": reasons, "samples": len(self.samples), "period_s": self.period}


def experiment_for(cfg, L):
    g = L.Grid(tuple(cfg.shape), cfg.h)
    return L.ThtExperiment(g, cfg.sources, cfg.rates, cfg.receivers, cfg.times, cfg.n_quad,
                           solver=L.SolverConfig(kind=cfg.solver_kind), include_storativity=True)


# ---------------------------------------------------------------------------------------
# CPU oracle sample (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------------------
def _oracle_sample_cfg(config_index: int):
    from paper_1409_2556_b200 import inputs
    cfg = inputs.config(config_index)
    if cfg.dim == 3:
        return cfg.scaled((24, 24, 24 if cfg.shape[2] == cfg.shape[0] else 12), n_src=4, n_rec=4, n_times=1)
    return cfg.scaled((128, 128), n_src=4, n_rec=4, n_times=1)


def _oracle_worker(args):
    """Forward/adjoint shifted-family solves of one RHS (own pencil + SuperLU cache)."""
    cfg_index, which, idx = args
    import numpy as np  # noqa
    from oracle import fd as ofd
    from oracle import forward as ofw
    from oracle import jacobian as ojac
    from oracle import shifted_solver as oss
    from oracle import talbot as otal
    cfg = _oracle_sample_cfg(cfg_index)
    lk, ls = cfg.fields()
    grid = ofd.Grid(tuple(cfg.shape), cfg.h)
    ops = ofd.assemble_fd(grid, np.exp(lk), np.exp(ls))
    pencil = oss.ShiftedPencil(ops.stiffness, ops.mass)
    contour = otal.build_contour(cfg.n_quad, cfg.times[0])
    solver = ofw.SolverConfig(kind=cfg.solver_kind)
    if which == "src":
        b = ofd.point_weights(grid, cfg.sources[idx]).astype(np.complex128)
        x = ojac._solve_family_or_throw(pencil, b, list(contour.nodes), solver, "forward solve")
        for k in range(contour.n_half()):
            x[:, k] *= otal.qhat_step(cfg.rates[idx], contour.nodes[k])
    else:
        e = ofd.point_weights(grid, cfg.receivers[idx])
        x = ojac.solve_adjoint_fields(pencil, e, contour, solver)
    return which, idx, x


def oracle_sample(config_index: int, workers: int):
    """Runs the sample once; returns (solves, seconds, description)."""
    from multiprocessing import get_context
    from oracle import fd as ofd
    from oracle import talbot as otal
    cfg = _oracle_sample_cfg(config_index)
    tasks = [(config_index, "src", s) for s in range(len(cfg.sources))] + \
            [(config_index, "rec", r) for r in range(len(cfg.receivers))]
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"  # one core per worker process (spawned children inherit this)
    t0 = time.perf_counter()
    with get_context("spawn").Pool(workers) as pool:
        out = pool.map(_oracle_worker, tasks)
    fwd = {i: x for w, i, x in out if w == "src"}
    adj = {i: x for w, i, x in out if w == "rec"}
    lk, ls = cfg.fields()
    grid = ofd.Grid(tuple(cfg.shape), cfg.h)
    ops = ofd.assemble_fd(grid, np.exp(lk), np.exp(ls))
    contour = otal.build_contour(cfg.n_quad, cfg.times[0])
    for s in fwd:
        for r in adj:
            ofd.sensitivity_rows_fd(ops, fwd[s], adj[r], contour.weights, contour.nodes, True)
    dt = time.perf_counter() - t0
    solves = len(tasks) * (cfg.n_quad // 2)
    desc = (f"oracle (SciPy SuperLU restatement) on configs[{config_index}] statistics at "
            f"{'x'.join(map(str, cfg.shape))}: {len(cfg.sources)} sources + {len(cfg.receivers)} receivers, "
            f"1 time, N={cfg.n_quad}: {solves} shifted solves + {len(fwd) * len(adj)} Jacobian rows, "
            f"{workers} worker processes")
    return solves, dt, desc


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    workers = min(os.cpu_count() or 1, 8)
    vals, dts = [], []
    desc = ""
    for i in range(args.warmup + args.steps):
        solves, dt, desc = oracle_sample(args.config, workers)
        if i >= args.warmup:
            vals.append(solves / dt)
            dts.append(dt)
    v = float(np.mean(vals))
    from paper_1409_2556_b200 import inputs
    cfg = inputs.config(args.config)
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(dts)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": cfg.name, "sample": desc},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": workers, "kind": "port", "sample": desc},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _sample_solves(config_index):
    cfg = _oracle_sample_cfg(config_index)
    return (len(cfg.sources) + len(cfg.receivers)) * (cfg.n_quad // 2)


# ---------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    from paper_1409_2556_b200 import capi, inputs
    from paper_1409_2556_b200 import laptomo as L

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)

    from paper_1409_2556_b200.replicas import max_over_ranks, replica_config
    cfg = replica_config(inputs.config(args.config), rank)  # rank > 0: own realisation
    lk, ls = cfg.fields()
    n = cfg.n_cells
    n_src, n_rec, n_t = len(cfg.sources), len(cfg.receivers), len(cfg.times)
    nh = cfg.n_quad // 2
    solves_per_build = (n_src + n_rec) * n_t * nh
    pairs = n_src * n_rec
    n_param = 2 * n

    ctx = L.Context(local)
    lib = capi.lib()
    ex = experiment_for(cfg, L)
    exc, keep = ex.c()
    grid_c = ex.grid.c()
    stream = torch.cuda.ExternalStream(ctx.stream(), device=torch.device("cuda", local))

    # inputs resident in HBM; J slice buffer on the device
    lk_d = torch.from_numpy(lk).cuda()
    ls_d = torch.from_numpy(ls).cuda()
    J = torch.empty((pairs, n_param), dtype=torch.float64, device="cuda")
    pred = np.zeros(pairs)
    preds = np.zeros((n_t, pairs))
    lk_pin = torch.from_numpy(lk).pin_memory()
    ls_pin = torch.from_numpy(ls).pin_memory()
    row_pin = torch.empty((n_t, n_param), dtype=torch.float64).pin_memory()
    torch.cuda.synchronize()

    def build(mem_host: bool):
        h = C.c_void_p()
        if mem_host:
            capi.check(lib.lt_pencil_create_grid(ctx.handle, C.byref(grid_c),
                                                 C.cast(lk_pin.data_ptr(), capi.PD),
                                                 C.cast(ls_pin.data_ptr(), capi.PD), capi.LT_MEM_HOST, C.byref(h)))
        else:
            capi.check(lib.lt_pencil_create_grid(ctx.handle, C.byref(grid_c),
                                                 C.cast(lk_d.data_ptr(), capi.PD),
                                                 C.cast(ls_d.data_ptr(), capi.PD), capi.LT_MEM_DEVICE, C.byref(h)))
        for t in range(n_t):
            capi.check(lib.lt_jacobian_slice(h, C.byref(exc), t, capi.LT_MEM_DEVICE,
                                             C.cast(J.data_ptr(), capi.PD), capi.dptr(pred)))
            preds[t] = pred
            if mem_host:
                # the step's result read back: the first sensitivity row of every slice
                # (lt_jacobian_slice has synchronised its stream; a blocking copy)
                row_pin[t].copy_(J[0])
        capi.check(lib.lt_pencil_destroy(h))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        build(False)
    # ---- device-resident timed region ----
    sampler = ClockSampler(local)
    if not os.environ.get("LT_BENCH_NOSMI"):
        sampler.start()
    ctx.reset_profile()
    ctx.set_profile_sampling(PROFILE_EVERY)  # events on 1 in 8 launches per kernel class
    ctx.set_profiling(not os.environ.get("LT_BENCH_NOPROF"))
    launches0 = ctx.launch_count()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        build(False)
    e1.record(stream)
    barrier()
    ms = e0.elapsed_time(e1)
    launches = ctx.launch_count() - launches0
    ctx.set_profiling(False)
    clocks = sampler.stop()
    prof = ctx.profile()
    # ---- end-to-end through the public API with host inputs ----
    barrier()
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        build(True)
    f1.record(stream)
    barrier()
    ms_e2e = f0.elapsed_time(f1)

    t_max, t_e2e = max_over_ranks([ms, ms_e2e], device=torch.device("cuda", local))
    per_step = t_max / args.steps
    value = world * solves_per_build * args.steps / (t_max * 1e-3)
    e2e_value = world * solves_per_build * args.steps / (t_e2e * 1e-3)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_kind = peaks()
    # dominant kernel class by device time
    dom = max(prof.items(), key=lambda kv: kv[1][0]) if prof else ("none", (0.0, 1, 0.0))
    dname, (dms, dcnt, dbytes) = dom
    achieved = (dbytes / dcnt) / (dms / dcnt * 1e-3) / 1e9 if dms > 0 else 0.0
    # the dominant HBM-bound class (the stencil / FGMRES kernels of the north star), reported
    # whatever the dominant class is
    hbm_classes = {k: v for k, v in prof.items() if k not in ("jacobian",) and v[2] > 0}
    hname, (hms, hcnt, hbytes) = max(hbm_classes.items(), key=lambda kv: kv[1][0]) if hbm_classes else \
        ("none", (0.0, 1, 0.0))
    h_achieved = (hbytes / hcnt) / (hms / hcnt * 1e-3) / 1e9 if hms > 0 else 0.0
    # per class over the timed region (1 in PROFILE_EVERY launches timed, scaled by the library
    # to the class's launch count)
    breakdown = {k: {"ms_est": round(v[0], 3), "launches": v[1],
                     "avg_us": round(v[0] / v[1] * 1e3, 2) if v[1] else None,
                     "GBps_alg": round(v[2] / (v[0] * 1e-3) / 1e9, 1) if v[0] > 0 and v[2] > 0 else None}
                 for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])}
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(dname)
        except Exception:
            traffic = None
    if dname == "jacobian":
        # FP64 tensor-core GEMM: flops per launch (one time slice) = 2 n_src n_rec K n, with
        # K = n_h shifts x (2d faces x (re, im) + (re, im) for the S block)  (faces-only K,
        # drivers.cu: jacobian_mma4_kernel)
        d = len(cfg.shape)
        flops = 2.0 * n_src * n_rec * (cfg.n_quad // 2) * (2 * (2 * d) + 2) * n
        ach_tf = flops / (dms / dcnt * 1e-3) / 1e12 if dms > 0 else 0.0
        roofline = {"bound": "tensor", "kernel": dname, "achieved": ach_tf, "peak": FP64_DMMA_TFLOPS,
                    "unit": "TFLOP/s", "frac": ach_tf / FP64_DMMA_TFLOPS, "traffic": traffic,
                    "peak_kind": "measured FP64 DMMA (scripts/micro/fp64_peak.cu; MEASURED_PEAKS.json has no FP64 "
                                 "figure)"}
    else:
        roofline = {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        workers = min(os.cpu_count() or 1, 8)
        solves, dt, desc = oracle_sample(args.config, workers)
        cpu = {"value": solves / dt, "unit": UNIT, "cores": workers, "kind": "port", "sample": desc}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "jacobian_builds_per_s": world * args.steps / (t_max * 1e-3),
        "config": {"workload": cfg.name, "grid": list(cfg.shape), "sources": n_src, "receivers": n_rec,
                   "times": n_t, "n_quad": cfg.n_quad, "shifted_solves_per_build": solves_per_build,
                   "jacobian": f"{pairs * n_t} x {n_param} FP64, per-time slices left on device",
                   "l2": "inputs larger than L2 (one 128^3 complex vector = 33.5 MB; a basis/field set "
                         "per time = tens of GB)",
                   "parallelism": "replicas" if world > 1 else "single-gpu"},
        "roofline": roofline,
        "roofline_hbm": {"bound": "hbm", "kernel": hname, "achieved": h_achieved, "peak": peak, "unit": "GB/s",
                         "frac": h_achieved / peak, "peak_kind": peak_kind},
        "kernel_breakdown": breakdown,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 2 * 8 * n,
                "d2h_bytes_per_step": 8 * n_t * (pairs + n_param)},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
