"""GPU perf probe: Jacobian slices (time 0) of BASELINE configs[4] statistics on a reduced grid,
with the per-kernel-class CUDA-event profile.  Usage: perf_jac.py [n_side=64] [reps=2]"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1409_2556_b200 import capi, inputs  # noqa: E402
from paper_1409_2556_b200 import laptomo as L  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 64
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = inputs.config(4).scaled((side, side, side))
lk, ls = cfg.fields()
ctx = L.Context(0)
g = L.Grid(tuple(cfg.shape), cfg.h)
ex = L.ThtExperiment(g, cfg.sources, cfg.rates, cfg.receivers, cfg.times, cfg.n_quad,
                     solver=L.SolverConfig(kind=cfg.solver_kind), include_storativity=True)
exc, keep = ex.c()
p = L.ShiftedPencil(g, lk, ls, ctx)
pairs = len(cfg.sources) * len(cfg.receivers)
J = np.zeros((pairs, 2 * g.n_cells))
pred = np.zeros(pairs)
lib = capi.lib()
for r in range(reps):
    ctx.reset_profile()
    ctx.set_profiling(True)
    capi.check(lib.lt_jacobian_slice(p._h, C.byref(exc), 0, capi.LT_MEM_HOST, capi.dptr(J), capi.dptr(pred)))
    ctx.set_profiling(False)
prof = ctx.profile()
for k, (ms, cnt, by) in sorted(prof.items(), key=lambda kv: -kv[1][0])[:14]:
    print(f"  {k:16s} {ms:9.2f} ms {cnt:6d}")
print("J row0 norm", float(np.linalg.norm(J[0])))
