# A/B of the colour-split half sweep: persistent ring and bf16 coefficient tiles (inner solve, configs[4], 80 items)
for V in "" base nopersist fp32c; do
  if [ -z "$V" ]; then unset LT_LIB; else export LT_LIB=$PWD/paper_1409_2556_b200/_lib/liblaptomo_gpu_$V.so; fi
  timeout 300 python scripts/perf_inner.py 4 80 > gpurun_out/rb_ab_${V:-default}.log 2>&1
  head -8 gpurun_out/rb_ab_${V:-default}.log
done
unset LT_LIB
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x 2>&1 | tail -3
