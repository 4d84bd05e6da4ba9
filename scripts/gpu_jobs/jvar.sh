# timing of experiment builds (liblaptomo_gpu_<variant>.so) of the Jacobian slice
for v in ${VARIANTS:-base}; do
  if [ "$v" = base ]; then LIB=""; else LIB=paper_1409_2556_b200/_lib/liblaptomo_gpu_$v.so; fi
  LT_LIB=$LIB timeout 600 python scripts/perf_jac.py 128 2 > gpurun_out/jvar_$v.log 2>&1
  echo "$v $(grep ' jacobian \|row0' gpurun_out/jvar_$v.log | tr '\n' ' ')"
done
