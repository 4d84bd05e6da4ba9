LT_INNER_TRACE=1 timeout 300 python scripts/perf_inner.py 4 80 2>&1 | grep -E "inner\]|lib=" | tail -4
cat > /tmp/tr.py <<'P'
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_1409_2556_b200 import inputs
from paper_1409_2556_b200 import laptomo as L
cfg = inputs.config(4)
lk, ls = cfg.fields()
ex = L.ThtExperiment.from_config(cfg) if hasattr(L.ThtExperiment, "from_config") else None
print("ok")
P
