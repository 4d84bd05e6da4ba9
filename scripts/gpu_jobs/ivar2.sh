# inner-solve timing of experiment builds, with the coarse-level class shown
for v in ${VARIANTS:-base}; do
  if [ "$v" = base ]; then LIB=""; else LIB=paper_1409_2556_b200/_lib/liblaptomo_gpu_$v.so; fi
  LT_LIB=$LIB timeout 600 python scripts/perf_inner.py 4 80 > gpurun_out/ivar_$v.log 2>&1
  echo "== $v"; grep "iterations\|mg_smooth\|mg_residual" gpurun_out/ivar_$v.log
done
