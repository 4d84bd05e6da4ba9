# A/B of the colour-split half sweep variants (inner solve, configs[4], 80 items): default library
# first, then any liblaptomo_gpu_<variant>.so present; then the parity tests on the default.
for L in "" $(ls paper_1409_2556_b200/_lib/liblaptomo_gpu_*.so 2>/dev/null); do
  if [ -z "$L" ]; then unset LT_LIB; V=default; else export LT_LIB=$PWD/$L; V=$(basename $L .so | sed 's/liblaptomo_gpu_//'); fi
  timeout 300 python scripts/perf_inner.py 4 80 > gpurun_out/rb_ab_$V.log 2>&1
  head -9 gpurun_out/rb_ab_$V.log
done
unset LT_LIB
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_split.py -q -x 2>&1 | tail -3
