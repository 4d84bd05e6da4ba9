"""GPU perf probe: one batched inner shift-and-invert solve (B items) on a BASELINE grid,
with the per-kernel-class CUDA-event profile (LT_LIB selects a library variant)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1409_2556_b200 import inputs  # noqa: E402
from paper_1409_2556_b200 import laptomo as L  # noqa: E402

index = int(sys.argv[1]) if len(sys.argv) > 1 else 4
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
cfg = inputs.config(index)
lk, ls = cfg.fields()
ctx = L.Context(0)
g = L.Grid(tuple(cfg.shape), cfg.h)
p = L.ShiftedPencil(g, lk, ls, ctx)
c = L.build_contour(cfg.n_quad, cfg.times[0])
tau = L.select_preconditioner_shifts(c.nodes).taus[0]
rng = np.random.default_rng(0)
v = rng.standard_normal((B, g.n_cells)) + 1j * rng.standard_normal((B, g.n_cells))
f = p.factorization(tau)
if not os.environ.get('NOWARM'):
    f.solve(v[:2])
ctx.reset_profile()
ctx.set_profiling(True)
u = f.solve(v)
ctx.set_profiling(False)
prof = ctx.profile()
prof.pop("host_gap", None)
tot = sum(x[0] for x in prof.values())
its = prof.get("cocg_apply:operator", (0, 0, 0))[1]
print(f"lib={os.environ.get('LT_LIB', 'default')} config={index} B={B} iterations={its} "
      f"kernel_ms={tot:.1f} per_item_iter_us={tot * 1e3 / max(its, 1) / B:.1f}")
for k, (ms, cnt, by) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:16s} {ms:9.2f} ms {cnt:6d}  {ms / tot * 100:5.1f}%  {by / (ms * 1e-3) / 1e9 if ms else 0:7.0f} GB/s")
