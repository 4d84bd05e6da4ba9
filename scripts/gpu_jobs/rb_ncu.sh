NOWARM=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mg_rb_kernel" --launch-skip 0 -c 5 -o gpurun_out/rb0_full -f python scripts/perf_inner.py 4 80 > gpurun_out/rb_ncu.log 2>&1
tail -2 gpurun_out/rb_ncu.log
