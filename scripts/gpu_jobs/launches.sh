NOWARM=1 timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/inner_launches.csv python scripts/perf_inner.py 4 80 > /dev/null 2>&1
ls -la gpurun_out/inner_launches.csv
