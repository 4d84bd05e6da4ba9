for v in default h16d4 h16d5 h16d6; do
  if [ $v = default ]; then export LT_LIB=; else export LT_LIB=paper_1409_2556_b200/_lib/liblaptomo_gpu_$v.so; fi
  echo "== $v"; timeout 300 python scripts/perf_inner.py 4 80 | grep -E "lib=|cocg_apply"
done
