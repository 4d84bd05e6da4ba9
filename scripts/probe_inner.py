"""Perf probe (GPU): inner shift-and-invert solves and one FGMRES-Sh family solve on a
BASELINE-sized grid, with the per-kernel-class CUDA-event profile."""
from __future__ import annotations

import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1409_2556_b200 import inputs  # noqa: E402
from paper_1409_2556_b200 import laptomo as L  # noqa: E402


def main(index=4, B=16):
    cfg = inputs.config(index)
    t0 = time.time()
    lk, ls = cfg.fields()
    print(f"fields {time.time() - t0:.1f}s", flush=True)
    ctx = L.Context(0)
    g = L.Grid(tuple(cfg.shape), cfg.h)
    t0 = time.time()
    p = L.ShiftedPencil(g, lk, ls, ctx)
    print(f"pencil {time.time() - t0:.2f}s levels={p.levels()}", flush=True)
    contour = L.build_contour(cfg.n_quad, cfg.times[0])
    sched = L.select_preconditioner_shifts(contour.nodes)
    rng = np.random.default_rng(0)
    n = g.n_cells
    v = rng.standard_normal((B, n)) + 1j * rng.standard_normal((B, n))
    p.prepare(sched.taus)
    for rep in range(2):
        ctx.reset_profile()
        ctx.set_profiling(True)
        t0 = time.time()
        u = p.factorization(sched.taus[0]).solve(v)
        dt = time.time() - t0
        ctx.set_profiling(False)
        r = p.apply(sched.taus[0], u) - v
        print(f"inner solve B={B}: {dt * 1e3:.1f} ms wall, rel res {np.linalg.norm(r) / np.linalg.norm(v):.2e}",
              flush=True)
    prof = ctx.profile()
    tot = sum(v[0] for v in prof.values())
    for k, (ms, cnt, by) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
        gbs = by / (ms * 1e-3) / 1e9 if ms > 0 else 0.0
        print(f"  {k:18s} {ms:9.2f} ms {cnt:6d} launches  {ms / tot * 100:5.1f}%  {gbs:8.0f} GB/s(alg)")
    # one forward family batch: sources of the config at one time
    from oracle import fd as ofd  # host weights only
    grid_o = ofd.Grid(tuple(cfg.shape), cfg.h)
    bs = np.stack([ofd.point_weights(grid_o, q) for q in cfg.sources]).astype(np.complex128)
    ctx.reset_profile()
    ctx.set_profiling(True)
    t0 = time.time()
    res = L.solve_shifted_flexible(p, bs, contour.nodes, sched, L.ShiftedSolveOptions(record_history=False))
    dt = time.time() - t0
    ctx.set_profiling(False)
    print(f"flexible family solve {len(bs)} RHS x {len(contour.nodes)} shifts: {dt:.2f}s wall, "
          f"iterations {[r.iterations for r in res]}, all_conv {all(r.all_converged for r in res)}", flush=True)
    prof = ctx.profile()
    tot = sum(v[0] for v in prof.values())
    for k, (ms, cnt, by) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
        gbs = by / (ms * 1e-3) / 1e9 if ms > 0 else 0.0
        print(f"  {k:18s} {ms:9.2f} ms {cnt:6d} launches  {ms / tot * 100:5.1f}%  {gbs:8.0f} GB/s(alg)")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 4, int(sys.argv[2]) if len(sys.argv) > 2 else 16)
