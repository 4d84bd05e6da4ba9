# smoothing counts by level (LT_MG_NU1 on the second level, LT_MG_NU on the coarser ones)
for n1 in 2 3 4 6; do for nc in 4 6 8 12; do
  LT_MG_NU1=$n1 LT_MG_NU=$nc timeout 300 python scripts/perf_inner.py 4 80 > gpurun_out/nu_${n1}_${nc}.log 2>&1
  echo "nu1=$n1 nuc=$nc $(head -1 gpurun_out/nu_${n1}_${nc}.log | awk '{print $4, $5, $6}')"
done; done
