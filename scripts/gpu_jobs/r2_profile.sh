# One ncu job per round state: launch list of a bench step, then --set full captures of the
# inner-solve kernels (one inner solve, 80 items, configs[4]) and of the outer / Jacobian kernels
# (one Jacobian slice at 128^3).  The .ncu-rep files stay in /tmp on the box (gpurun_out is
# capped at 64 MiB); their per-kernel summaries (scripts/ncu_summary.py) and the source-page
# CSV of the finest half sweep come back under gpurun_out/$TAG*.
TAG=${1:-r2}
OUT=gpurun_out
REP=/tmp/ncu_$TAG
mkdir -p $OUT $REP
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $OUT/${TAG}_plain_bench.json 2> $OUT/${TAG}_plain_bench.err &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip ${SKIP:-12000} -c ${COUNT:-14000} --csv \
  --log-file $REP/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
  > $OUT/${TAG}_ncu_launch.log 2>&1 || echo "launch list failed"
python scripts/launch_shares.py $REP/launches.csv $OUT/${TAG}_launch_shares.json > $OUT/${TAG}_launch_shares.txt 2>&1
gzip -c $REP/launches.csv > $OUT/${TAG}_launches.csv.gz
NOWARM=1 timeout 300 python scripts/perf_inner.py 4 80 > $OUT/${TAG}_inner_plain.log 2>&1 &&
NOWARM=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"${KIN:-mg_rb_kernel|mid_sweeps|rbpair_zm|residual_pair|apply_tma2|prolong|restrict|bottom_vcycle|pupdate|axpy_norm}" \
  --launch-skip ${SKIN:-130} -c ${CIN:-70} -o $REP/full_inner -f python scripts/perf_inner.py 4 80 \
  > $OUT/${TAG}_ncu_inner.log 2>&1 || echo "inner capture failed"
tail -3 $OUT/${TAG}_inner_plain.log
python scripts/ncu_summary.py $REP/full_inner.ncu-rep --json $OUT/${TAG}_ncu_inner.json > $OUT/${TAG}_ncu_inner.txt 2>&1
ncu -i $REP/full_inner.ncu-rep --page source --csv -k regex:mg_rb_kernel -c 1 2>/dev/null | gzip -c > $OUT/${TAG}_src_mg_rb.csv.gz
timeout 600 python scripts/perf_jac.py 128 1 > $OUT/${TAG}_jac_plain.log 2>&1 &&
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"${KOUT:-jacobian_mma4|verify_residual|mass_multidot|gs_update|multidot|expand_cm2}" \
  -c ${COUT:-14} -o $REP/full_outer -f python scripts/perf_jac.py 128 1 \
  > $OUT/${TAG}_ncu_outer.log 2>&1 || echo "outer capture failed"
tail -3 $OUT/${TAG}_jac_plain.log
python scripts/ncu_summary.py $REP/full_outer.ncu-rep --json $OUT/${TAG}_ncu_outer.json > $OUT/${TAG}_ncu_outer.txt 2>&1
du -sh $OUT; ls -la $OUT | tail -16
