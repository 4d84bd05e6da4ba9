for nu in 1 3 4; do LT_MG_NU=$nu timeout 300 python scripts/perf_inner.py 4 80 2>&1 | head -1; done
