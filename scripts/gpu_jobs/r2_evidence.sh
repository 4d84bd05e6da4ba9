# round-2 evidence: bench lines of configs 0-3, compute-sanitizer on the TMA / mbarrier kernels
mkdir -p gpurun_out
timeout 600 python bench.py --config 0 --steps 20 --warmup 3 > gpurun_out/r2_bench_c0.json 2> gpurun_out/r2_bench_c0.err; tail -1 gpurun_out/r2_bench_c0.err
timeout 900 python bench.py --config 1 --steps 3 --warmup 3 > gpurun_out/r2_bench_c1.json 2> gpurun_out/r2_bench_c1.err; tail -1 gpurun_out/r2_bench_c1.err
timeout 900 python bench.py --config 2 --steps 3 --warmup 3 > gpurun_out/r2_bench_c2.json 2> gpurun_out/r2_bench_c2.err; tail -1 gpurun_out/r2_bench_c2.err
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 > gpurun_out/r2_bench_c3.json 2> gpurun_out/r2_bench_c3.err; tail -1 gpurun_out/r2_bench_c3.err
for T in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $T --print-limit 20 python scripts/sanitize_probe.py > gpurun_out/r2_sanitize_$T.log 2>&1
  echo "$T rc=$?"; tail -3 gpurun_out/r2_sanitize_$T.log
done
