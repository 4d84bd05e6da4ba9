"""Diagnose the P1 inner solve in the paper regime (100 m domain, var 1.6).

Run with LT_INNER_TRACE=1 to see each inner COCG's final relative residual.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import scipy.sparse.linalg as spla

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import fem  # noqa: E402
from oracle import shifted_solver as oss  # noqa: E402
from oracle import talbot as otal  # noqa: E402
from paper_1409_2556_b200 import laptomo as L  # noqa: E402


def main(n=101, side=100.0, var=1.6, seed=11):
    rng = np.random.default_rng(seed)
    mesh = fem.build_mesh(n, side)
    lk = np.log(1e-4) + np.sqrt(var) * rng.standard_normal(mesh.n_elements())
    ls = np.log(1e-5) + 0.2 * rng.standard_normal(mesh.n_elements())
    ops = fem.assemble(mesh, np.exp(lk), np.exp(ls))
    p = L.ShiftedPencil(L.build_mesh(n, side), lk, ls)
    print("levels", p.levels() if hasattr(p, "levels") else "?", flush=True)
    b = ops.restrict_to_free(fem.point_source(mesh, 50.0, 50.0)).astype(complex)
    for t in [60.0, 300.0, 1200.0]:
        c = otal.build_contour(40, t)
        sched = oss.select_preconditioner_shifts(list(c.nodes))
        for tau in sched.taus:
            u = p.factorization(tau).solve(b)
            ref = spla.splu((ops.stiffness + tau * ops.mass).tocsc(), permc_spec="COLAMD").solve(b)
            print(f"t={t} tau={tau:.4g} rel={np.linalg.norm(u - ref) / np.linalg.norm(ref):.3e}", flush=True)
        opencil = oss.ShiftedPencil(ops.stiffness, ops.mass)
        ref = oss.solve_shifted_flexible(opencil, b, list(c.nodes), sched)
        try:
            got = L.solve_shifted_flexible(p, b, list(c.nodes), L.PreconditionerSchedule(sched.taus, sched.pattern))
            print(f"t={t} iters dev={got.iterations} ref={ref.iterations} conv={got.all_converged}", flush=True)
        except Exception as e:  # noqa: BLE001
            print(f"t={t} ref iters={ref.iterations} device failed: {e}", flush=True)


if __name__ == "__main__":
    main()
