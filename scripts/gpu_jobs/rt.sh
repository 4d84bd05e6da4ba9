for s in 64 96 128; do
  LT_PAIR_PROLONG=1 timeout 300 python scripts/probe_vcycle.py a_$s $s 1 2>&1 | tail -1
  LT_DEBUG_SYNC=1 timeout 300 python scripts/probe_vcycle.py c_$s $s 1 2>&1 | tail -1
done
python - <<'P'
import numpy as np
for s in (64,96,128):
    a=np.load(f"gpurun_out/a_{s}.npy"); b=np.load(f"gpurun_out/c_{s}.npy")
    print(s, "rel diff one step", np.linalg.norm(a-b)/np.linalg.norm(a))
P
rm -f gpurun_out/*.npy
timeout 300 python scripts/perf_inner.py 4 80 | head -9
