"""Benchmark: shifted-system solves/s + Jacobian builds/s (FP64) on the BASELINE configs, one B200.

Default workload = BASELINE configs[4] (3-D THT Jacobian, 128^3 cells, 16 sources x 64
receivers, Talbot N=32, 4 times).  One step = one full Jacobian build (ThtForwardModel::
jacobian, jacobian.cpp:189-247): device assembly of the pencil from the log fields, forward +
adjoint FGMRES-Sh solves of all 80 right-hand sides at each of the 4 times (5120 shifted-system
solves), the kappa + storativity Jacobian slices (4096 x 2*2,097,152, left on the device per
time slice as SURVEY.md §8d defines a build) and the 4096 predictions.
--config 2 is the 2-D Jacobian build (256^2); --config 0 / 1 / 3 are forward configs, where a
step is solve_forward of every source at every time (forward.cpp:75-118, the sources batched
in lockstep) with the drawdown at the receivers.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 4]

Timing: W untimed warm-up steps, then K steps in each of three device-timed regions
(CUDA events on the library's stream, barrier + synchronize on both sides, max over ranks):
  1. `value`: inputs resident in HBM, no instrumentation (the production path: device-resident
     COCG loop, the iteration body one CUDA-graph launch);
  2. the kernel profile: the same K steps with CUDA events around 1 in 8 launches of every
     kernel (per-kernel time and algorithmic bytes -> `roofline`, `kernel_breakdown`);
  3. `e2e`: through the C ABI with HOST inputs (pinned log fields copied in every step) and the
     step's results read back (predictions / drawdown, the first Jacobian row of every slice).
The full Jacobian's host copy is timed separately (`jacobian_host_copy`).

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
JACOBIAN_CONFIGS = (2, 4)

# FP64 throughputs measured on this pool's B200 (scripts/micro/fp64_peak.cu): mma.sync m8n8k4
# (DMMA) and the DFMA pipe; MEASURED_PEAKS.json has no FP64 figure
FP64_DMMA_TFLOPS = 37.0
FP64_DFMA_TFLOPS = 34.0


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled during the timed region through
    NVML (the library nvidia-smi uses), once every 2 s."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, index: int, period: float = 2.0):
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
# CPU oracle samples (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------------------
def _oracle_sample_cfg(config_index: int):
    """The bounded CPU sample of each config (same statistics, one time)."""
    from paper_1409_2556_b200 import inputs
    if config_index == 0:
        return inputs.config(0).scaled((100, 100), n_times=1)
    if config_index == 1:
        return inputs.config(1).scaled((512, 512), n_src=2, n_times=1)
    if config_index == 2:
        return inputs.config(2).scaled((256, 256), n_src=2, n_rec=2, n_times=1)
    if config_index == 3:
        return inputs.reduced(3, (32, 32, 16), n_src=2, receivers=[0, 1], n_times=1)
    return inputs.config(4).scaled((32, 32, 32), n_src=2, n_rec=2, n_times=1)


def _oracle_rhs(cfg):
    return [("src", s) for s in range(len(cfg.sources))] + \
           ([("rec", r) for r in range(len(cfg.receivers))] if cfg.jacobian else [])


def _oracle_solve(cfg, pencil, grid, which, idx):
    from oracle import fd as ofd
    from oracle import forward as ofw
    from oracle import jacobian as ojac
    from oracle import talbot as otal
    contour = otal.build_contour(cfg.n_quad, cfg.times[0])
    solver = ofw.SolverConfig(kind=cfg.solver_kind)
    if which == "src":
        b = ofd.point_weights(grid, cfg.sources[idx]).astype(np.complex128)
        x = ojac._solve_family_or_throw(pencil, b, list(contour.nodes), solver, "forward solve")
        for k in range(contour.n_half()):
            x[:, k] *= otal.qhat_step(cfg.rates[idx], contour.nodes[k])
    else:
        x = ojac.solve_adjoint_fields(pencil, ofd.point_weights(grid, cfg.receivers[idx]), contour, solver)
    return x


def _oracle_setup(cfg):
    from oracle import fd as ofd
    from oracle import shifted_solver as oss
    lk, ls = cfg.fields()
    grid = ofd.Grid(tuple(cfg.shape), cfg.h)
    ops = ofd.assemble_fd(grid, np.exp(lk), np.exp(ls))
    return grid, ops, oss.ShiftedPencil(ops.stiffness, ops.mass)


def _oracle_finish(cfg, grid, ops, fwd, adj):
    from oracle import fd as ofd
    from oracle import talbot as otal
    contour = otal.build_contour(cfg.n_quad, cfg.times[0])
    for s in fwd:
        if cfg.jacobian:
            for r in adj:
                ofd.sensitivity_rows_fd(ops, fwd[s], adj[r], contour.weights, contour.nodes, True)
        else:
            for q in cfg.receivers:
                otal.inverse_laplace_sum(contour, fwd[s].T @ ofd.point_weights(grid, q))


def _oracle_worker(args):
    """One RHS on its own pencil (own SuperLU factorisations), one core."""
    config_index, which, idx = args
    cfg = _oracle_sample_cfg(config_index)
    grid, ops, pencil = _oracle_setup(cfg)
    return which, idx, _oracle_solve(cfg, pencil, grid, which, idx)


def _single_thread_env():
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"


def oracle_sample_1core(config_index: int):
    """The sample sequentially on one core with one shared pencil (the reference's own
    single-threaded structure, jacobian.cpp:189-247): (solves, seconds, description)."""
    cfg = _oracle_sample_cfg(config_index)
    t0 = time.perf_counter()
    grid, ops, pencil = _oracle_setup(cfg)
    fwd, adj = {}, {}
    for which, idx in _oracle_rhs(cfg):
        (fwd if which == "src" else adj)[idx] = _oracle_solve(cfg, pencil, grid, which, idx)
    _oracle_finish(cfg, grid, ops, fwd, adj)
    dt = time.perf_counter() - t0
    rhs = _oracle_rhs(cfg)
    solves = len(rhs) * (cfg.n_quad // 2)
    return solves, dt, _describe(cfg, config_index, rhs, 1)


def _describe(cfg, config_index, rhs, workers):
    nsrc = sum(1 for w, _ in rhs if w == "src")
    nrec = len(rhs) - nsrc
    what = f"{nsrc} sources + {nrec} receivers" if cfg.jacobian else f"{nsrc} sources, drawdown at {len(cfg.receivers)} receivers"
    return (f"oracle (SciPy SuperLU restatement) on configs[{config_index}] statistics at "
            f"{'x'.join(map(str, cfg.shape))}: {what}, 1 time, N={cfg.n_quad}: "
            f"{len(rhs) * (cfg.n_quad // 2)} shifted solves, {workers} process(es), one core each")


def _workers_for(cfg, cap=None):
    """Host cores usable for independent RHS, bounded by memory (each worker holds its own LU)."""
    n = int(np.prod(cfg.shape))
    per_worker = (120 if len(cfg.shape) == 2 else 1200) * n * 16 * 2 + 200e6  # ~fill x 2 factorisations
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError):
        avail = 16e9
    w = max(1, min(os.cpu_count() or 1, int(0.6 * avail / per_worker)))
    return min(w, cap) if cap else w


def oracle_sample_ncore(config_index: int, workers: int):
    """`workers` RHS in parallel processes (one core each, own pencil): aggregate throughput
    of the host's cores on the sample's first RHS kinds, repeated to fill the workers."""
    from multiprocessing import get_context
    cfg = _oracle_sample_cfg(config_index)
    base = _oracle_rhs(cfg)
    tasks = [(config_index,) + base[i % len(base)] for i in range(max(workers, len(base)))]
    _single_thread_env()
    t0 = time.perf_counter()
    with get_context("spawn").Pool(workers) as pool:
        pool.map(_oracle_worker, tasks)
    dt = time.perf_counter() - t0
    solves = len(tasks) * (cfg.n_quad // 2)
    return solves, dt, _describe(cfg, config_index, [(t[1], t[2]) for t in tasks], workers)


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    _single_thread_env()
    cfg_s = _oracle_sample_cfg(args.config)
    workers = _workers_for(cfg_s)
    vals, dts = [], []
    desc = ""
    for i in range(args.warmup + args.steps):
        solves, dt, desc = oracle_sample_ncore(args.config, workers)
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
            "config": {"workload": cfg.name, "sample": desc, "nproc": os.cpu_count(), "cpu_model": cpu_model()},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": workers, "kind": "port", "sample": desc},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------
def kernel_class(name: str) -> str:
    return name.split(":", 1)[0]


HBM_CLASSES = ("cocg_vec", "cocg_apply", "mg_smooth", "mg_smooth_coarse", "mg_residual", "mg_restrict",
               "mg_prolong", "fgmres_orth", "fgmres_vec", "fgmres_verify", "expand", "recombine")


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
    jac = args.config in JACOBIAN_CONFIGS
    lk, ls = cfg.fields()
    n = cfg.n_cells
    n_src, n_rec, n_t = len(cfg.sources), len(cfg.receivers), len(cfg.times)
    nh = cfg.n_quad // 2
    solves_per_build = ((n_src + n_rec) if jac else n_src) * n_t * nh
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
    J = torch.empty((pairs, n_param), dtype=torch.float64, device="cuda") if jac else None
    pred = np.zeros(pairs)
    preds = np.zeros((n_t, pairs))
    lk_pin = torch.from_numpy(lk).pin_memory()
    ls_pin = torch.from_numpy(ls).pin_memory()
    row_pin = torch.empty((n_t, n_param), dtype=torch.float64).pin_memory() if jac else None
    torch.cuda.synchronize()
    # forward configs: source weights (lt_pencil_point_weights, host arithmetic) and lt_forward
    src_w = rates = times = rec = dd = diag = None
    if not jac:
        probe = L.ShiftedPencil(ex.grid, lk, ls, ctx)
        src_w = np.ascontiguousarray(np.stack([probe.point_weights(q) for q in cfg.sources]))
        probe.close()
        rates = np.ascontiguousarray(np.asarray(cfg.rates, dtype=np.float64))
        times = np.ascontiguousarray(np.asarray(cfg.times, dtype=np.float64))
        rec = np.ascontiguousarray(np.asarray(cfg.receivers, dtype=np.float64))
        dd = np.zeros(n_src * n_rec * n_t)
        diag = (capi.LtTimeDiag * n_t)()
        tp = L.TalbotParams().c()
        sc = L.SolverConfig(kind=cfg.solver_kind).c()

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
        if jac:
            for t in range(n_t):
                capi.check(lib.lt_jacobian_slice(h, C.byref(exc), t, capi.LT_MEM_DEVICE,
                                                 C.cast(J.data_ptr(), capi.PD), capi.dptr(pred)))
                preds[t] = pred
                if mem_host:
                    # the step's result read back: the first sensitivity row of every slice
                    # (lt_jacobian_slice has synchronised its stream; a blocking copy)
                    row_pin[t].copy_(J[0])
        else:
            capi.check(lib.lt_forward(h, capi.dptr(src_w), capi.dptr(rates), n_src, None, capi.dptr(times), n_t,
                                      cfg.n_quad, C.byref(tp), C.byref(sc), 0, capi.LT_MEM_HOST, None,
                                      capi.dptr(rec), n_rec, capi.dptr(dd), diag, None))
        capi.check(lib.lt_pencil_destroy(h))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def timed(mem_host: bool):
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            build(mem_host)
        e1.record(stream)
        barrier()
        return e0.elapsed_time(e1)

    for _ in range(args.warmup):
        build(False)
    # ---- 1. device-resident timed region (production path, no instrumentation) ----
    sampler = ClockSampler(local)
    if not os.environ.get("LT_BENCH_NOSMI"):
        sampler.start()
    ctx.reset_profile()
    launches0 = ctx.launch_count()
    ms = timed(False)
    launches = ctx.launch_count() - launches0
    clocks = sampler.stop()
    # host gaps of the production pass: wall time from the return of a stream synchronisation
    # (stream empty) to the next kernel launch, accumulated by the library
    gap = ctx.profile().get("host_gap", (0.0, 0, 0.0))
    # ---- 2. kernel profile: the same steps, CUDA events on 1 in 8 launches per kernel ----
    ctx.reset_profile()
    ctx.set_profile_sampling(PROFILE_EVERY)
    ctx.set_profiling(True)
    ms_prof = timed(False)
    ctx.set_profiling(False)
    prof = ctx.profile()
    prof.pop("host_gap", None)
    # ---- 3. end-to-end through the public API with host inputs ----
    ms_e2e = timed(True)
    # ---- the full Jacobian's host copy (one time slice, chunked through pinned staging) ----
    host_copy = None
    if jac:
        chunk_rows = max(1, min(pairs, int(2e9 // (8 * n_param))))
        stage = torch.empty((chunk_rows, n_param), dtype=torch.float64).pin_memory()
        torch.cuda.synchronize()
        c0 = time.perf_counter()
        for r0 in range(0, pairs, chunk_rows):
            r1 = min(pairs, r0 + chunk_rows)
            stage[: r1 - r0].copy_(J[r0:r1])
        torch.cuda.synchronize()
        dt = time.perf_counter() - c0
        slice_bytes = 8.0 * pairs * n_param
        host_copy = {"bytes_per_slice": slice_bytes, "bytes_per_build": slice_bytes * n_t, "seconds_per_slice": dt,
                     "GBps": slice_bytes / dt / 1e9, "seconds_per_build": dt * n_t,
                     "how": f"D2H of one slice in {chunk_rows}-row chunks into pinned memory, wall clock"}
        del stage

    t_max, t_e2e, t_prof = max_over_ranks([ms, ms_e2e, ms_prof], device=torch.device("cuda", local))
    per_step = t_max / args.steps
    value = world * solves_per_build * args.steps / (t_max * 1e-3)
    e2e_value = world * solves_per_build * args.steps / (t_e2e * 1e-3)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_kind = peaks()
    # per kernel over the profiled region (1 in PROFILE_EVERY launches timed, scaled by the
    # library to the kernel's launch count)
    breakdown = {k: {"ms_est": round(v[0], 3), "launches": v[1],
                     "avg_us": round(v[0] / v[1] * 1e3, 2) if v[1] else None,
                     "GBps_alg": round(v[2] / (v[0] * 1e-3) / 1e9, 1) if v[0] > 0 and v[2] > 0 else None}
                 for k, v in sorted(prof.items(), key=lambda kv: -kv[1][0])}
    classes = {}
    for k, v in prof.items():
        c = classes.setdefault(kernel_class(k), [0.0, 0, 0.0])
        c[0] += v[0]
        c[1] += v[1]
        c[2] += v[2]
    class_breakdown = {k: {"ms_est": round(v[0], 3), "share": round(v[0] / max(sum(x[0] for x in classes.values()), 1e-9), 4),
                           "GBps_alg": round(v[2] / (v[0] * 1e-3) / 1e9, 1) if v[0] > 0 and v[2] > 0 else None}
                       for k, v in sorted(classes.items(), key=lambda kv: -kv[1][0])}
    traffic_all = {}
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath) and args.config == 4:  # the ncu captures are of configs[4] launches
        try:
            traffic_all = json.load(open(tpath))
        except Exception:
            traffic_all = {}
    # the dominant single kernel by device time
    dname, (dms, dcnt, dbytes) = max(prof.items(), key=lambda kv: kv[1][0]) if prof else ("none", (0.0, 1, 0.0))
    if kernel_class(dname) == "jacobian":
        # FP64 tensor-core GEMM: flops per launch (one time slice) = 2 n_src n_rec K n, with
        # K = n_h shifts x (2d faces x (re, im) + (re, im) for the S block)  (faces-only K,
        # drivers.cu: jacobian_mma4_kernel)
        d = len(cfg.shape)
        flops = 2.0 * n_src * n_rec * nh * (2 * (2 * d) + 2) * n
        ach_tf = flops / (dms / dcnt * 1e-3) / 1e12 if dms > 0 else 0.0
        roofline = {"bound": "tensor", "kernel": dname, "achieved": ach_tf, "peak": FP64_DMMA_TFLOPS,
                    "unit": "TFLOP/s", "frac": ach_tf / FP64_DMMA_TFLOPS, "traffic": traffic_all.get(dname),
                    "peak_kind": "measured FP64 DMMA (scripts/micro/fp64_peak.cu; MEASURED_PEAKS.json has no FP64 "
                                 "figure)"}
    else:
        achieved = (dbytes / dcnt) / (dms / dcnt * 1e-3) / 1e9 if dms > 0 else 0.0
        roofline = {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": traffic_all.get(dname), "peak_kind": peak_kind,
                    "algorithmic_bytes_per_launch": dbytes / dcnt if dcnt else None,
                    "avg_launch_us": dms / dcnt * 1e3 if dcnt else None,
                    "traffic_how": "dram__bytes_read.sum + dram__bytes_write.sum of one launch with every item of "
                                   "the batch active (ncu --set full, profiles/traffic.json via scripts/make_traffic.py); "
                                   "algorithmic_bytes_per_launch averages over the launches of the run, where items "
                                   "that have converged are skipped"}
    # the dominant HBM-bound kernel and the time-weighted HBM fraction over every HBM-bound kernel
    hbm = {k: v for k, v in prof.items() if kernel_class(k) in HBM_CLASSES and v[2] > 0 and v[0] > 0}
    hname, (hms, hcnt, hbytes) = max(hbm.items(), key=lambda kv: kv[1][0]) if hbm else ("none", (0.0, 1, 0.0))
    h_ach = (hbytes / hcnt) / (hms / hcnt * 1e-3) / 1e9 if hms > 0 else 0.0
    agg_ms = sum(v[0] for v in hbm.values())
    agg_gbps = sum(v[2] for v in hbm.values()) / (agg_ms * 1e-3) / 1e9 if agg_ms > 0 else 0.0
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        _single_thread_env()
        s1, d1, desc1 = oracle_sample_1core(args.config)
        cfg_s = _oracle_sample_cfg(args.config)
        wk = _workers_for(cfg_s, cap=16)
        sn, dn, descn = oracle_sample_ncore(args.config, wk)
        cpu = {"value": sn / dn, "unit": UNIT, "cores": wk, "kind": "port", "sample": descn,
               "one_core": {"value": s1 / d1, "unit": UNIT, "cores": 1, "sample": desc1, "seconds": d1},
               "seconds": dn, "nproc": os.cpu_count(), "cpu_model": cpu_model()}
    d2h = 8 * n_t * (pairs + n_param) if jac else 8 * n_src * n_rec * n_t
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "grid": list(cfg.shape), "sources": n_src, "receivers": n_rec,
                   "times": n_t, "n_quad": cfg.n_quad, "shifted_solves_per_step": solves_per_build,
                   "step": ("one Jacobian build: " + f"{pairs * n_t} x {n_param} FP64, per-time slices left on device")
                   if jac else "solve_forward of every source at every time, drawdown at the receivers",
                   "l2": "inputs larger than L2 (basis / field sets per time are GBs)" if n >= 262144 else
                         "working set partly L2-resident (small grid)",
                   "parallelism": "replicas" if world > 1 else "single-gpu"},
        "roofline": roofline,
        "roofline_hbm": {"bound": "hbm", "kernel": hname, "achieved": h_ach, "peak": peak, "unit": "GB/s",
                         "frac": h_ach / peak if peak else None, "peak_kind": peak_kind,
                         "traffic": traffic_all.get(hname)},
        "hbm_aggregate": {"achieved": agg_gbps, "peak": peak, "unit": "GB/s", "frac": agg_gbps / peak if peak else None,
                          "kernels": len(hbm), "share_of_device_time": agg_ms / max(sum(v[0] for v in prof.values()), 1e-9),
                          "how": "sum of algorithmic bytes / sum of device time over every HBM-bound kernel"},
        "profiled_pass_ms_per_step": t_prof / args.steps,
        "class_breakdown": class_breakdown,
        "kernel_breakdown": breakdown,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 2 * 8 * n, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches),
        "host_gap": {"ms_per_step": gap[0] / args.steps, "gaps_per_step": gap[1] / args.steps,
                     "how": "wall time between the return of a stream synchronisation and the next kernel launch "
                            "(the GPU is idle at least that long), production pass"},
        "clocks": clocks,
    }
    if jac:
        line["jacobian_builds_per_s"] = world * args.steps / (t_max * 1e-3)
        line["jacobian_host_copy"] = host_copy
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
