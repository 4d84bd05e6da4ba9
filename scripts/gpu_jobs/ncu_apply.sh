NOWARM=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"apply_tma|axpy_norm|pupdate" --launch-skip 3 -c 3 -o gpurun_out/apply_full -f python scripts/perf_inner.py 4 80 > gpurun_out/apply_ncu.log 2>&1
tail -1 gpurun_out/apply_ncu.log
