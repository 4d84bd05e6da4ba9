# COCG vector-kernel grid size A/B (inner solve, configs[4], 80 items)
for L in liblaptomo_gpu liblaptomo_gpu_vb32 liblaptomo_gpu_vb64 liblaptomo_gpu_vb1000; do
  LT_LIB=paper_1409_2556_b200/_lib/$L.so python scripts/perf_inner.py 4 80 2>&1 | head -6
done
