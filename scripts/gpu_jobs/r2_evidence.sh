# round-2 evidence: bench lines of every config (c4 = the driver's default), then compute-sanitizer
# (memcheck, racecheck, synccheck) on the warp-specialised TMA / mbarrier kernels
TAG=${1:-r2}
mkdir -p gpurun_out
for C in 4 0 1 2 3; do
  S=3; [ $C = 0 ] && S=30; [ $C = 1 ] && S=10; [ $C = 2 ] && S=10; [ $C = 3 ] && S=5
  timeout 1200 python bench.py --config $C --steps $S --warmup 3 > gpurun_out/${TAG}_bench_c$C.json 2> gpurun_out/${TAG}_bench_c$C.err
  python3 -c "
import json;d=json.load(open('gpurun_out/${TAG}_bench_c$C.json'))
r=d['roofline']
print('c$C', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'ms/step', round(d['ms_per_step'],2), 'prof', round(d['profiled_pass_ms_per_step'],2), r['kernel'], round(r['frac'],3), 'agg', round(d['hbm_aggregate']['frac'],3), 'cpu', d['cpu_baseline'] and round(d['cpu_baseline']['value'],2), d['clocks']['reasons'])"
done
for T in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $T --print-limit 20 python scripts/sanitize_probe.py > gpurun_out/${TAG}_sanitize_$T.log 2>&1
  echo "$T rc=$?"; tail -3 gpurun_out/${TAG}_sanitize_$T.log
done
