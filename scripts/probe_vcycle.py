"""Debug probe: one preconditioned COCG iteration (u = alpha B r) of the inner solve, saved to
gpurun_out/<tag>.npy, to compare smoother variants (e.g. LT_MG_HALF=1 vs the fused sweep)."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1409_2556_b200 import capi, inputs  # noqa: E402
from paper_1409_2556_b200 import laptomo as L  # noqa: E402

tag = sys.argv[1]
side = int(sys.argv[2]) if len(sys.argv) > 2 else 64
its = int(sys.argv[3]) if len(sys.argv) > 3 else 1
cfg = inputs.config(4).scaled((side, side, side))
lk, ls = cfg.fields()
g = L.Grid(tuple(cfg.shape), cfg.h)
p = L.ShiftedPencil(g, lk, ls)
capi.check(capi.lib().lt_pencil_set_inner_tolerance(p.handle, C.c_double(1e-12), its))
rng = np.random.default_rng(0)
v = rng.standard_normal((4, g.n_cells)) + 1j * rng.standard_normal((4, g.n_cells))
u = p.factorization(-0.3 + 0.2j).solve(v)
np.save(f"gpurun_out/{tag}.npy", u)
print(tag, np.linalg.norm(u))
