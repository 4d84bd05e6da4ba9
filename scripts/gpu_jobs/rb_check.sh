# V-cycle variants: one preconditioned COCG step must agree to FP32 rounding
for s in 64 96 128; do
  LT_NO_RB=1 LT_ZM_TRANSFER=1 timeout 300 python scripts/probe_vcycle.py a_$s $s 1 2>&1 | tail -1
  LT_NO_RB=1 LT_DEBUG_SYNC=1 timeout 300 python scripts/probe_vcycle.py b_$s $s 1 2>&1 | tail -1
  LT_DEBUG_SYNC=1 timeout 300 python scripts/probe_vcycle.py c_$s $s 1 2>&1 | tail -1
done
python - <<'P'
import numpy as np
for s in (64,96,128):
    try:
        a=np.load(f"gpurun_out/a_{s}.npy")
        for t in "bc":
            b=np.load(f"gpurun_out/{t}_{s}.npy")
            print(s, t, "rel diff one step", np.linalg.norm(a-b)/np.linalg.norm(a))
    except Exception as e: print(s, e)
P
rm -f gpurun_out/*.npy
LT_NO_RB=1 timeout 300 python scripts/perf_inner.py 4 80
timeout 300 python scripts/perf_inner.py 4 80
