"""Probe: the inner shift-and-invert solve (MG-COCG) at every preconditioner shift of the
paper-regime cases (scripts/paper_regime.py): final relative residual per tau."""
import sys
sys.path.insert(0, '.'); sys.path.insert(0, 'scripts')
import numpy as np
import paper_regime as PR
from paper_1409_2556_b200 import capi
from paper_1409_2556_b200 import laptomo as L

cases = [(f, t, 101) for f in ("random", "franke") for t in (60.0, 300.0, 1200.0, 3000.0)]
cases += [("franke", 300.0, 41), ("franke", 300.0, 201)]
for field, t, n in cases:
    mesh, lk, ls, b, ops = PR.case(field, n)
    p = L.ShiftedPencil(L.build_mesh(n, PR.SIDE), lk, ls)
    bb = p.point_weights((50.0, 50.0)).astype(np.complex128)
    c = L.build_contour(PR.NZ, t)
    sched = L.select_preconditioner_shifts(c.nodes)
    for tau in sched.taus:
        try:
            p.factorization(tau).solve(bb)
            print(field, t, n, f"tau={tau:.4g}", "ok", flush=True)
        except capi.ConvergenceError as e:
            print(field, t, n, f"tau={tau:.4g}", "FAIL", str(e)[:80], flush=True)
