TAG=${1:-jd}
for d in ${DBGS:-1 2 3 4}; do
  LT_JW_DBG=$d timeout 600 python scripts/perf_jac.py 128 2 > gpurun_out/${TAG}_d$d.log 2>&1
  echo "dbg=$d $(grep ' jacobian ' gpurun_out/${TAG}_d$d.log | tr '\n' ' ')"
done
