for d in 0 1 2 4 3 7; do
  LT_JW_DBG=$d LT_TRACE=1 timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline 2> gpurun_out/trace.err > /dev/null
  echo "dbg=$d $(grep '\[lt\]   jacobian' gpurun_out/trace.err | tail -3 | awk '{print $4}' | tr '\n' ' ')"
done
