# perf_inner (configs[4], 80 items) on the default library and on every liblaptomo_gpu_<variant>.so present
for L in "" $(ls paper_1409_2556_b200/_lib/liblaptomo_gpu_*.so 2>/dev/null); do
  if [ -z "$L" ]; then unset LT_LIB; V=default; else export LT_LIB=$PWD/$L; V=$(basename $L .so | sed 's/liblaptomo_gpu_//'); fi
  timeout 300 python scripts/perf_inner.py ${CFG:-4} ${NB:-80} > gpurun_out/var_$V.log 2>&1
  head -${NL:-9} gpurun_out/var_$V.log
done
