timeout 300 python scripts/perf_inner.py 4 80 > gpurun_out/pi.txt; head -4 gpurun_out/pi.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
