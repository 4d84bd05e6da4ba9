for v in nof noc pos; do
  export LT_LIB=paper_1409_2556_b200/_lib/liblaptomo_gpu_$v.so
  for s in 64 128; do
  echo "== $v $s"
  LT_DEBUG_SYNC=1 LT_SWEEP_MASK=1 timeout 120 python scripts/probe_vcycle.py v_$v $s 1 2>&1 | tail -1
  done
done
