# the fused bottom sub-cycle vs the level-by-level kernels: inner solve A/B, parity, bench lines
for L in liblaptomo_gpu liblaptomo_gpu_nobottom; do
  LT_LIB=paper_1409_2556_b200/_lib/$L.so python scripts/perf_inner.py 4 80 2>&1 | head -3
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_boundary.py -q -x 2>&1 | tail -2
for C in 4 3 1 2; do
  for L in liblaptomo_gpu liblaptomo_gpu_nobottom; do
    S=3; [ $C = 1 ] && S=10; [ $C = 2 ] && S=10
    LT_LIB=paper_1409_2556_b200/_lib/$L.so timeout 900 python bench.py --config $C --steps $S --warmup 3 --no-cpu-baseline > gpurun_out/bot_${C}_$L.json 2>/dev/null
    python3 -c "
import json;d=json.load(open('gpurun_out/bot_${C}_$L.json'))
print('c$C $L', round(d['value'],1), round(d['e2e']['value'],1), round(d['ms_per_step'],2), 'prof', round(d['profiled_pass_ms_per_step'],2), 'agg', round(d['hbm_aggregate']['frac'],3), [(k, v['ms_est']) for k,v in list(d['class_breakdown'].items())[:4]])"
  done
done
