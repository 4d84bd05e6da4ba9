"""Small cases that run every warp-specialised TMA / mbarrier kernel once, for
compute-sanitizer (memcheck, racecheck, synccheck): the colour-split red-black sweeps and
residual, the TMA restriction / prolongation, the two-item TMA operator, the natural-layout TMA
z-march, the 4-cell tensor-core Jacobian and the 2-cell fallback, the banded LU."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1409_2556_b200 import inputs  # noqa: E402
from paper_1409_2556_b200 import laptomo as L  # noqa: E402

# colour-split levels (64 x 32 x 16: nx % 4 == 0, nx >= 64), TMA operator (nx >= 32)
cfg = inputs.reduced(4, (64, 32, 16), n_src=4, receivers=[0, 9, 18, 27, 36], n_times=1)
lk, ls = cfg.fields()
g = L.Grid(tuple(cfg.shape), cfg.h)
ex = L.ThtExperiment(g, cfg.sources, cfg.rates, cfg.receivers, cfg.times, cfg.n_quad,
                     solver=L.SolverConfig(kind="flexible"), include_storativity=True)
jr = L.ThtForwardModel(ex, ls).jacobian(lk)
print("3-D colour-split + 4-cell Jacobian:", jr.jacobian.shape, float(np.abs(jr.predictions).max()))
# 2-cell Jacobian fallback (nx % 4 != 0) and natural-layout TMA 2-D levels
cfg2 = inputs.config(2).scaled((66, 64), n_src=2, n_rec=3, n_times=1)
lk2, ls2 = cfg2.fields()
g2 = L.Grid(tuple(cfg2.shape), cfg2.h)
ex2 = L.ThtExperiment(g2, cfg2.sources, cfg2.rates, cfg2.receivers, cfg2.times, cfg2.n_quad,
                      solver=L.SolverConfig(kind="flexible"), include_storativity=True)
jr2 = L.ThtForwardModel(ex2, ls2).jacobian(lk2)
print("2-D natural TMA + 2-cell Jacobian:", jr2.jacobian.shape, float(np.abs(jr2.predictions).max()))
# banded LU (2-D, forced by an inner solve that cannot converge)
p = L.ShiftedPencil(g2, lk2, ls2)
p.set_inner_tolerance(1e-12, 1)
v = np.random.default_rng(0).standard_normal((2, g2.n_cells)) + 0j
u = p.factorization(-0.3 + 0.2j).solve(v)
print("banded LU:", float(np.linalg.norm(u)))
