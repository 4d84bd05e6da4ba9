for v in d8 d8w8 d7; do
  LT_LIB=paper_1409_2556_b200/_lib/liblaptomo_gpu_$v.so timeout 300 python scripts/perf_inner.py 4 80 2>&1 | head -3
done
