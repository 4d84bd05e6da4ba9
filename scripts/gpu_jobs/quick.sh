timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python scripts/perf_inner.py 4 80
