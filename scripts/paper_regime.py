"""Oracle iteration counts in the paper regime (§4.1-4.2; SPEC.md acceptance 3-6),
written to tests/golden/paper_regime.json for tests/test_paper_regime.py (CPU, the oracle) and
tests/test_gpu_paper_regime.py (the device).

The reference's experiment: 100 m square, P1 on build_mesh(101, 100),
mean transmissivity 1e-4, S = 1e-5, one source at (50, 50), N_z = 40, tol 1e-10.  Fields
(oracle/fields.py, restating fields.cpp): the Franke field (deterministic) and an
exponential-covariance random field (sample_field_on_mesh; the paper gives no correlation
length: 20 m here, seed 7), both at variance 1.6.

    python scripts/paper_regime.py
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import fem, fields  # noqa: E402
from oracle import forward as ofw  # noqa: E402
from oracle import shifted_solver as oss  # noqa: E402
from oracle import talbot as otal  # noqa: E402

SIDE, KAPPA, S, RATE, NZ = 100.0, 1e-4, 1e-5, 8.5e-4, 40
RANDOM_CORR, RANDOM_SEED, VAR = 20.0, 7, 1.6


def case(field: str, n: int = 101):
    """(mesh, log_kappa, log_S, source weights on the free dofs, assembled operators)."""
    mesh = fem.build_mesh(n, SIDE)
    if field == "franke":
        lk = fields.franke_field(mesh, VAR, np.log(KAPPA))
    else:
        lk = fields.sample_field_on_mesh(mesh, VAR, RANDOM_CORR, np.log(KAPPA), RANDOM_SEED)
    ls = np.full(mesh.n_elements(), np.log(S))
    ops = fem.assemble(mesh, np.exp(lk), np.exp(ls))
    b = ops.restrict_to_free(fem.point_source(mesh, 50.0, 50.0))
    return mesh, lk, ls, b, ops


def counts(field: str, t: float, n: int = 101):
    """(single, flexible) outer iterations of one time's shifted family."""
    mesh, lk, ls, b, ops = case(field, n)
    pencil = oss.ShiftedPencil(ops.stiffness, ops.mass)
    shifts = list(otal.build_contour(NZ, t).nodes)
    sched = oss.select_preconditioner_shifts(shifts)
    bc = b.astype(np.complex128)
    single = oss.solve_shifted_single(pencil, bc, shifts, sched.taus[0])
    flexible = oss.solve_shifted_flexible(pencil, bc, shifts, sched)
    assert single.all_converged and flexible.all_converged
    return single.iterations, flexible.iterations


def pooled_times():
    return list(np.linspace(2400.0, 3600.0, 40))


def pooled_count(field: str = "random"):
    mesh, lk, ls, b, ops = case(field)
    sol = ofw.solve_forward_batch(ofw.ForwardProblem(ops.stiffness, ops.mass, b, RATE, None, pooled_times(), NZ))
    return sol.diagnostics[0].iterations


if __name__ == "__main__":
    out = {"fields": {"random_corr_m": RANDOM_CORR, "random_seed": RANDOM_SEED, "variance": VAR}}
    t0 = time.time()
    for field in ("random", "franke"):
        for t in (60.0, 300.0, 1200.0, 3000.0):
            out[f"{field}_n101_t{int(t)}"] = counts(field, t)
            print(field, t, out[f"{field}_n101_t{int(t)}"], f"{time.time() - t0:.0f}s", flush=True)
    for n in (41, 201):
        out[f"franke_n{n}_t300"] = counts("franke", 300.0, n)
        print("franke", n, out[f"franke_n{n}_t300"], flush=True)
    out["random_pooled40"] = pooled_count("random")
    print("pooled", out["random_pooled40"], flush=True)
    (ROOT / "tests" / "golden" / "paper_regime.json").write_text(json.dumps(out, indent=1))
