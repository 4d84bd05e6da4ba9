# ncu --set full of the Jacobian and expansion kernels of one 128^3 slice (summaries and the
# Jacobian's source page come back; the .ncu-rep stays on the box)
TAG=${1:-r2}
REP=/tmp/ncu_$TAG
mkdir -p gpurun_out $REP
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"jacobian_mma4|expand_cm2" -c 2 \
  -o $REP/full_jac -f python scripts/perf_jac.py 128 1 > gpurun_out/${TAG}_ncu_jac.log 2>&1 || echo "capture failed"
python scripts/ncu_summary.py $REP/full_jac.ncu-rep --json gpurun_out/${TAG}_ncu_jac.json > gpurun_out/${TAG}_ncu_jac.txt 2>&1
ncu -i $REP/full_jac.ncu-rep --page source --csv -k regex:jacobian_mma4 -c 1 2>/dev/null | gzip -c > gpurun_out/${TAG}_src_jac.csv.gz
cat gpurun_out/${TAG}_ncu_jac.txt | cut -c1-900
