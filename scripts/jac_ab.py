"""A/B of the Jacobian kernel: one configs[4] time slice (128^3, 16 x 64 items) into a device
buffer, kernel time from the library's CUDA-event profile (LT_LIB selects the build, e.g. the
-DLT_JAC_DFMA variant that runs the same m8n8k4 GEMM formulation on the DFMA pipe)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1409_2556_b200 import capi, inputs  # noqa: E402
from paper_1409_2556_b200 import laptomo as L  # noqa: E402

cfg = inputs.config(4)
lk, ls = cfg.fields()
ctx = L.Context(0)
g = L.Grid(tuple(cfg.shape), cfg.h)
ex = L.ThtExperiment(g, cfg.sources, cfg.rates, cfg.receivers, cfg.times, cfg.n_quad,
                     solver=L.SolverConfig(kind=cfg.solver_kind), include_storativity=True)
exc, keep = ex.c()
p = L.ShiftedPencil(g, lk, ls, ctx)
pairs = len(cfg.sources) * len(cfg.receivers)
J = torch.empty((pairs, 2 * g.n_cells), dtype=torch.float64, device="cuda")
pred = np.zeros(pairs)
lib = capi.lib()
for r in range(2):
    ctx.reset_profile()
    ctx.set_profiling(True)
    capi.check(lib.lt_jacobian_slice(p.handle, C.byref(exc), 0, capi.LT_MEM_DEVICE, C.cast(J.data_ptr(), capi.PD),
                                     capi.dptr(pred)))
    ctx.set_profiling(False)
prof = ctx.profile()
ms = prof["jacobian"][0]
d = 3
flops = 2.0 * 16 * 64 * 16 * (2 * (2 * d) + 2) * g.n_cells
print(f"lib={os.environ.get('LT_LIB', 'default')} jacobian {ms:.2f} ms per slice, {flops / (ms * 1e-3) / 1e12:.1f} TF/s "
      f"(faces-only GEMM flops), row0 norm {float(torch.linalg.norm(J[0])):.10e}")
