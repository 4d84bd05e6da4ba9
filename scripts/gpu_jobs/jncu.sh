TAG=${1:-jn}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-jacobian_mma4} -c 1 \
  -o gpurun_out/${TAG}_full_jac -f python scripts/perf_jac.py 128 1 > gpurun_out/${TAG}_ncu.log 2>&1 || echo "ncu failed"
tail -2 gpurun_out/${TAG}_ncu.log
