NOWARM=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mg_rb_kernel|restrict_zm|prolong_zm" --launch-skip 60 -c 14 -o gpurun_out/rb_full -f python scripts/perf_inner.py 4 80 > gpurun_out/rb_ncu.log 2>&1
tail -2 gpurun_out/rb_ncu.log
