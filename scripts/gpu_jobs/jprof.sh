# Jacobian kernel: per-part timings (LT_JW_DBG bits disable consumer mma / producer transform /
# J stores / weights) and one ncu --set full capture with source of the tensor-core kernel.
TAG=${1:-jp}
for d in 0 1 2 3 4 7; do
  LT_JW_DBG=$d LT_PROFILE=1 timeout 600 python scripts/perf_jac.py 128 2 > gpurun_out/${TAG}_d$d.log 2>&1
  echo "dbg=$d $(grep ' jacobian ' gpurun_out/${TAG}_d$d.log | head -1)"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jacobian_mma -c 1 \
  -o gpurun_out/${TAG}_full_jac -f python scripts/perf_jac.py 128 1 > gpurun_out/${TAG}_ncu.log 2>&1 || echo "ncu failed"
tail -3 gpurun_out/${TAG}_ncu.log
