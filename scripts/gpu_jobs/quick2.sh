timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
timeout 300 python scripts/perf_inner.py 4 80 | grep -E "lib=|cocg_apply"
LT_APPLY_TMA_COEF=1 timeout 300 python scripts/perf_inner.py 4 80 | grep -E "lib=|cocg_apply"
