# 2-D smoothing schedules (finest, next, coarser sweeps): c1 and c2, 5 steps
for C in 1 2; do
  for L in liblaptomo_gpu liblaptomo_gpu_nu222 liblaptomo_gpu_nu224 liblaptomo_gpu_nu244 liblaptomo_gpu_nu124; do
    LT_LIB=paper_1409_2556_b200/_lib/$L.so timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/nu_${C}_$L.json 2>/dev/null
    python3 -c "
import json;d=json.load(open('gpurun_out/nu_${C}_$L.json'))
print('c$C $L', round(d['value'],1), round(d['e2e']['value'],1), round(d['ms_per_step'],2), [(k, v['ms_est']) for k,v in list(d['class_breakdown'].items())[:3]])"
  done
done
