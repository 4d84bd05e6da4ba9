timeout 300 python scripts/perf_inner.py 4 80 | head -4
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "preconditioner or shifted_solve" 2>&1 | tail -2
