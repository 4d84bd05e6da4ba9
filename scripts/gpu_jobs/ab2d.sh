# 2-D levels: register z-march kernels (default) vs the TMA z-march kernels (LT_TMA_2D); c0 with the cuSOLVER coarse factor
for C in 0 1 2; do
  for L in liblaptomo_gpu liblaptomo_gpu_tma2d; do
    S=3; [ $C = 0 ] && S=20
    LT_LIB=paper_1409_2556_b200/_lib/$L.so timeout 600 python bench.py --config $C --steps $S --warmup 3 --no-cpu-baseline > gpurun_out/ab2d_${C}_$L.json 2>/dev/null
    python3 -c "
import json;d=json.load(open('gpurun_out/ab2d_${C}_$L.json'))
print('c$C $L', round(d['value'],1), round(d['e2e']['value'],1), round(d['ms_per_step'],2), [(k, v['ms_est']) for k,v in list(d['class_breakdown'].items())[:3]])"
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x 2>&1 | tail -2
