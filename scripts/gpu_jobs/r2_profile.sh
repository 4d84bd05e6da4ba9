# One ncu call per round state: launch list of a bench step, then --set full captures of the
# inner-solve kernels (one inner solve, 80 items, configs[4]) and of the outer / Jacobian kernels
# (one Jacobian slice at 128^3).  Outputs under gpurun_out/$TAG*.
TAG=${1:-r2}
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $OUT/${TAG}_plain_bench.json 2> $OUT/${TAG}_plain_bench.err &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip ${SKIP:-12000} -c ${COUNT:-14000} --csv \
  --log-file $OUT/${TAG}_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
  > $OUT/${TAG}_ncu_launch.log 2>&1 || echo "launch list failed"
NOWARM=1 timeout 300 python scripts/perf_inner.py 4 80 > $OUT/${TAG}_inner_plain.log 2>&1 &&
NOWARM=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"${KIN:-mg_rb_kernel|rbpair_zm|residual_pair|apply_tma2|prolong|restrict|bottom_vcycle|pupdate|axpy_norm}" \
  --launch-skip ${SKIN:-130} -c ${CIN:-70} -o $OUT/${TAG}_full_inner -f python scripts/perf_inner.py 4 80 \
  > $OUT/${TAG}_ncu_inner.log 2>&1 || echo "inner capture failed"
tail -3 $OUT/${TAG}_inner_plain.log
timeout 600 python scripts/perf_jac.py 128 1 > $OUT/${TAG}_jac_plain.log 2>&1 &&
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"${KOUT:-jacobian_mma4|verify_residual|mass_multidot|gs_update|multidot|expand_cm2}" \
  -c ${COUT:-14} -o $OUT/${TAG}_full_outer -f python scripts/perf_jac.py 128 1 \
  > $OUT/${TAG}_ncu_outer.log 2>&1 || echo "outer capture failed"
tail -3 $OUT/${TAG}_jac_plain.log
ls -la $OUT | tail -12
